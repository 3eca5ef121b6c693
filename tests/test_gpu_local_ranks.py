"""The library's multi-rank code, run for real on ONE B200: g ranks as contexts of this
process joined by the in-process communicator (ipt_ctx_init_local_comm; one host thread
per rank; collectives are event-ordered, no kernel waits on another). Everything the
sharded paths do between ranks executes: the sliced upload + in-place all-gather of
Delta, the per-iteration all-reduce of the stop scalars, the fused peer-store all-gather
of the single-pair iterate (and its collective fallback), the Z / eigenvalue gathers.

Column j of F needs only column j of Z (proj/src/solver.cpp:220; column independence
pinned by proj/tests/test_solver.cpp:188-201), so the column-sharded solve must
reproduce the single-rank Z and eigenvalues BIT FOR BIT with the same iteration count;
only the globally reduced scalars (step, residual) differ, by summation order. The
row-sharded single pair likewise reproduces the single-rank iterate bit for bit when the
row chunk is a multiple of the CSR row group (4); otherwise to rounding."""
import os
import time

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import dist, synth

pytestmark = pytest.mark.gpu


def _solve_full(p, g, product="dmma", warm=None, cfg=None):
    cfg = cfg or ipt.IterationConfig(tolerance=1e-12)
    gaps = ipt.build_gaps(p)
    one = ipt.solve_full(p, gaps, cfg, warm_start=warm, product=product)
    ctxs = dist.local_contexts(g)
    assert all(c.comm_kind == "local" for c in ctxs)
    outs = dist.run_ranks(lambda c: ipt.solve_full(p, gaps, cfg, warm_start=warm, ctx=c, product=product), ctxs)
    for c in ctxs:
        c.close()
    return one, outs


def _check_full(one, outs, exact=True):
    r0 = outs[0]
    assert all(o.iterations == one.iterations for o in outs)
    assert all(o.status == one.status for o in outs)
    if exact:
        assert np.array_equal(r0.Z, one.Z), np.max(np.abs(r0.Z - one.Z))
        assert np.array_equal(r0.eigenvalues, one.eigenvalues)
    else:
        assert np.max(np.abs(r0.Z - one.Z)) <= 1e-14
        assert np.max(np.abs(r0.eigenvalues - one.eigenvalues) / np.abs(one.eigenvalues)) <= 1e-14
    # globally reduced scalars: the same on every rank, equal to the single rank to rounding
    for o in outs:
        assert o.final_step == outs[0].final_step and o.residual_frobenius == outs[0].residual_frobenius
    assert r0.final_step == pytest.approx(one.final_step, rel=1e-10, abs=1e-300)
    assert r0.residual_frobenius == pytest.approx(one.residual_frobenius, rel=1e-6, abs=1e-13)
    assert r0.min_singular_value_estimate == pytest.approx(one.min_singular_value_estimate, rel=1e-12)
    assert r0.matmul_count == one.matmul_count


@pytest.mark.parametrize("g", [2, 3, 4])
def test_column_sharded_dense_solve_is_bitwise_the_single_rank_solve(g):
    p = synth.dense_uniform(1000, 0.02, 42)  # 1000 columns: uneven shards for g = 3
    one, outs = _solve_full(p, g)
    _check_full(one, outs)


def test_column_sharded_solve_at_config2_size():
    p = synth.config2()
    one, outs = _solve_full(p, 4)
    _check_full(one, outs)
    assert one.iterations == 5


@pytest.mark.parametrize("g", [2, 4])
def test_column_sharded_ozaki_solve_is_bitwise(g):
    p = synth.dense_uniform(1536, 0.3 / np.sqrt(1536), 7)
    one, outs = _solve_full(p, g, product="ozaki")
    _check_full(one, outs)


def test_column_sharded_max_abs_rule_and_trace():
    p = synth.dense_uniform(777, 0.02, 5)
    cfg = ipt.IterationConfig(tolerance=1e-12, stop_rule="max_abs", record_trace=True)
    one, outs = _solve_full(p, 3, cfg=cfg)
    _check_full(one, outs)
    # max |F - Z| is a max over ranks: exact
    assert outs[0].trace_max_abs == one.trace_max_abs


def test_column_sharded_warm_start():
    p = synth.dense_uniform(640, 0.02, 9)
    rng = np.random.default_rng(3)
    warm = np.eye(640) + 1e-3 * rng.standard_normal((640, 640))
    one, outs = _solve_full(p, 2, warm=warm)
    _check_full(one, outs)


def test_column_sharded_complex_solve():
    rng = np.random.default_rng(11)
    n = 300
    d = np.arange(1, n + 1) + 0.3j * rng.random(n)
    a = 0.01 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    np.fill_diagonal(a, 0)
    one, outs = _solve_full(ipt.Partition(d, a), 2)
    _check_full(one, outs)


def test_column_sharded_sparse_delta_solve():
    p = synth.csr_ci(2048, 16, 0.01, 3)
    one, outs = _solve_full(p, 4, cfg=ipt.IterationConfig(tolerance=1e-12))
    _check_full(one, outs)


def _solve_single(p, g, anchor=0, cfg=None, p2p=True):
    cfg = cfg or ipt.IterationConfig(tolerance=1e-10)
    gaps = ipt.build_gaps(p, 0.0)
    one = ipt.solve_single(p, gaps, anchor, cfg)
    old = os.environ.get("IPT_P2P")
    os.environ["IPT_P2P"] = "1" if p2p else "0"
    try:
        ctxs = dist.local_contexts(g)
        outs = dist.run_ranks(lambda c: ipt.solve_single(p, gaps, anchor, cfg, ctx=c), ctxs)
        for c in ctxs:
            c.close()
    finally:
        if old is None:
            del os.environ["IPT_P2P"]
        else:
            os.environ["IPT_P2P"] = old
    return one, outs


@pytest.mark.parametrize("g,p2p", [(2, True), (4, True), (4, False), (8, True)])
def test_row_sharded_csr_single_pair_is_bitwise(g, p2p):
    p = synth.csr_ci(1 << 15, 32, 0.01, 42)  # chunk = 2^15 / g, a multiple of the row group
    one, outs = _solve_single(p, g, p2p=p2p)
    for o in outs:
        assert o.iterations == one.iterations and o.status == one.status
        assert np.array_equal(o.z, one.z)
        assert o.eigenvalue == one.eigenvalue
    assert outs[0].residual == pytest.approx(one.residual, rel=1e-8, abs=1e-16)


def test_row_sharded_csr_uneven_chunks_and_interior_anchor():
    p = synth.csr_ci(10007, 24, 0.01, 5)  # chunk 3336: row groups shift, sums agree to rounding
    one, outs = _solve_single(p, 3, anchor=4321)
    for o in outs:
        assert o.iterations == one.iterations
        assert np.max(np.abs(o.z - one.z)) <= 1e-14
        assert abs(o.eigenvalue - one.eigenvalue) <= 1e-13 * abs(one.eigenvalue)


def test_row_sharded_dense_single_pair_and_continuation():
    p = synth.dense_normal(4096)
    one, outs = _solve_single(p, 4, cfg=ipt.IterationConfig(tolerance=1e-12))
    assert all(np.array_equal(o.z, one.z) and o.iterations == one.iterations for o in outs)
    gaps = ipt.build_gaps(p)
    one_c = ipt.solve_single_continuation(p, gaps, 0, ipt.IterationConfig(tolerance=1e-12), shrink_alpha=0.5)
    ctxs = dist.local_contexts(2)
    outs_c = dist.run_ranks(
        lambda c: ipt.solve_single_continuation(p, gaps, 0, ipt.IterationConfig(tolerance=1e-12), shrink_alpha=0.5, ctx=c),
        ctxs)
    assert all(np.array_equal(o.z, one_c.z) and o.iterations == one_c.iterations for o in outs_c)


def test_row_sharded_complex_single_pair():
    rng = np.random.default_rng(4)
    n = 512
    d = np.arange(n) + 0.2j * rng.random(n)
    a = 0.01 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    np.fill_diagonal(a, 0)
    p = ipt.Partition(d, a)
    one, outs = _solve_single(p, 2, cfg=ipt.IterationConfig(tolerance=1e-12))
    for o in outs:
        assert o.iterations == one.iterations
        assert np.max(np.abs(o.z - one.z)) <= 1e-14


def test_a_rank_that_never_joins_fails_the_others_instead_of_hanging():
    os.environ["IPT_LOCAL_COMM_TIMEOUT_S"] = "3"
    try:
        ctxs = dist.local_contexts(2)
    finally:
        del os.environ["IPT_LOCAL_COMM_TIMEOUT_S"]
    p = synth.dense_uniform(256, 0.02, 1)
    t0 = time.time()
    with pytest.raises(RuntimeError, match="local comm"):
        ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12), ctx=ctxs[0])
    assert time.time() - t0 < 60


def test_iteration_batch_is_the_same_on_every_rank():
    """N = 5793 on 8 ranks: shards of 724 and 725 columns fall on either side of the
    per-rank work threshold that sets how many maps are enqueued per host check. The
    batch must follow the global shard width (ipt_full.cu full_iterate), or the ranks'
    collective sequences diverge after convergence (wrong residual, then a hang)."""
    n = 5793
    assert n * 724 < 2048 * 2048 <= n * 725
    p = synth.dense_uniform(n, 0.32 / np.sqrt(n), 11)
    os.environ["IPT_LOCAL_COMM_TIMEOUT_S"] = "120"
    try:
        one, outs = _solve_full(p, 8)
    finally:
        del os.environ["IPT_LOCAL_COMM_TIMEOUT_S"]
    _check_full(one, outs)


@pytest.mark.parametrize("g", [2, 3])
def test_local_column_output_writes_every_block_without_a_gather(g):
    """IPT_OUTPUT_LOCAL_COLUMNS: every rank downloads its own columns of Z and its
    eigenvalues into one shared host array (here: the same numpy arrays across the rank
    threads; across processes a shared mapping) -- no gather to rank 0 -- and sigma_min is
    computed on the shards (y = Z p all-reduced per CG step)."""
    p = synth.dense_uniform(900, 0.02, 17)
    gaps = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-12)
    one = ipt.solve_full(p, gaps, cfg)
    zr = np.full((900, 900), np.nan)
    lr = np.full(900, np.nan)
    ctxs = dist.local_contexts(g)
    outs = dist.run_ranks(lambda c: ipt.solve_full(p, gaps, cfg, ctx=c, output="local", out=(zr, None, lr, None)),
                          ctxs)
    assert np.array_equal(zr, one.Z) and np.array_equal(lr, one.eigenvalues)
    for o in outs:
        assert o.iterations == one.iterations
        assert o.min_singular_value_estimate == outs[0].min_singular_value_estimate  # the same on every rank
    assert outs[0].min_singular_value_estimate == pytest.approx(one.min_singular_value_estimate, rel=1e-12)


def test_local_column_output_complex():
    rng = np.random.default_rng(21)
    n = 260
    d = np.arange(1, n + 1) + 0.2j * rng.random(n)
    a = 0.01 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    np.fill_diagonal(a, 0)
    p = ipt.Partition(d, a)
    gaps = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-12)
    one = ipt.solve_full(p, gaps, cfg)
    zr, zi = np.full((n, n), np.nan), np.full((n, n), np.nan)
    lr, li = np.full(n, np.nan), np.full(n, np.nan)
    ctxs = dist.local_contexts(2)
    outs = dist.run_ranks(lambda c: ipt.solve_full(p, gaps, cfg, ctx=c, output="local", out=(zr, zi, lr, li)), ctxs)
    assert np.array_equal(zr + 1j * zi, one.Z) and np.array_equal(lr + 1j * li, one.eigenvalues)
    assert outs[1].min_singular_value_estimate == pytest.approx(one.min_singular_value_estimate, rel=1e-12)


@pytest.mark.parametrize("n", [1, 5, 9])
def test_more_ranks_than_columns(n):
    """g = 8 ranks on N = 1, 5, 9: some ranks own no column (full spectrum) / no row
    (single pair); they still take part in every collective with zero contributions."""
    p = synth.dense_uniform(n, 0.05, 3)
    one, outs = _solve_full(p, 8)
    _check_full(one, outs)
    q = synth.dense_normal(max(n, 2))
    one_s, outs_s = _solve_single(q, 8, cfg=ipt.IterationConfig(tolerance=1e-12))
    for o in outs_s:
        assert o.iterations == one_s.iterations
        assert np.max(np.abs(o.z - one_s.z)) <= 1e-14
    c = synth.csr_ci(max(n, 4) * 2, 2, 0.01, 1)
    one_c, outs_c = _solve_single(c, 8)
    for o in outs_c:
        assert o.iterations == one_c.iterations
        assert np.max(np.abs(o.z - one_c.z)) <= 1e-14


@pytest.mark.parametrize("devices", [(0, 0), (0, 0, 0)])
def test_devices_argument_is_bitwise_one_gpu(devices):
    """solve_full / solve_single(devices=[...]): ranks of this process on those GPUs (here one
    B200 listed several times), bitwise the one-GPU result; a failed call reopens the group."""
    p = synth.dense_uniform(1000, 0.3 / np.sqrt(1000), 21)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-12)
    one = ipt.solve_full(p, g, cfg)
    r = ipt.solve_full(p, g, cfg, devices=list(devices))
    assert r.iterations == one.iterations
    assert np.array_equal(r.Z, one.Z) and np.array_equal(r.eigenvalues, one.eigenvalues)
    q = synth.csr_ci(1 << 14, 16, 0.01, 3)
    gq = ipt.build_gaps(q, 0.0)
    s1 = ipt.solve_single(q, gq, 0, ipt.IterationConfig(tolerance=1e-10))
    s = ipt.solve_single(q, gq, 0, ipt.IterationConfig(tolerance=1e-10), devices=list(devices))
    assert s.iterations == s1.iterations
    assert np.max(np.abs(s.z - s1.z)) <= 1e-14
    bad = np.eye(1000)
    bad[5, 5] = 0.0
    with pytest.raises(Exception):
        ipt.solve_full(p, g, cfg, warm_start=bad, devices=list(devices))
    r2 = ipt.solve_full(p, g, cfg, devices=list(devices))
    assert np.array_equal(r2.Z, one.Z)
