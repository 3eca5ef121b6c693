"""Row blocks of the single-pair map (the rows one rank maps under the row sharding of
SURVEY §8e, ipt_single.cu): a block [b, e) on one GPU must reproduce rows b..e-1 of the
whole map BIT FOR BIT (dense GEMV rows for any block; CSR row groups of 4 for blocks
starting at a multiple of 4, as the equal row chunks of the sharding do for chunk
sizes divisible by 4). Several steps are emulated by assembling the blocks' rows on
the host between steps -- the all-gather a multi-GPU run does over NCCL -- and must
match the whole run exactly."""
import ctypes as C

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import _lib, synth
from paper_2012_14702_b200._lib import Stats, check, dptr, i32ptr, i64ptr
from paper_2012_14702_b200.ipt import _params


pytestmark = pytest.mark.gpu


def _steps(upload, n, warm, steps):
    lib = _lib.load()
    ctx = ipt.default_context()
    h = C.c_void_p()
    check(upload(ctx, C.byref(h)))
    try:
        check(lib.ipt_single_reset(ctx.handle, h, 0, dptr(warm), None))
        prm = _params(ipt.IterationConfig(max_iterations=steps), ignore_convergence=1, divergence_threshold=1e300)
        st = Stats()
        check(lib.ipt_single_iterate(ctx.handle, h, C.byref(prm), C.byref(st)))
        z = np.empty(n)
        check(lib.ipt_single_download(ctx.handle, h, dptr(z), None))
        return z
    finally:
        lib.ipt_single_free(h)


def _dense(p):
    lib = _lib.load()
    n = p.size()
    delta = np.ascontiguousarray(p.delta)

    def whole(ctx, out):
        return lib.ipt_single_upload_dense(ctx.handle, n, dptr(p.d), None, dptr(delta), None, out)

    def block(b, e):
        return lambda ctx, out: lib.ipt_single_upload_dense_rows(ctx.handle, n, dptr(p.d), None, dptr(delta), None,
                                                                b, e, out)
    return whole, block, delta


def _csr(p):
    lib = _lib.load()
    n = p.size()
    rp, ci, va = p.delta.row_offsets, p.delta.col_indices, p.delta.values

    def whole(ctx, out):
        return lib.ipt_single_upload_csr(ctx.handle, n, dptr(p.d), None, i64ptr(rp), i32ptr(ci), dptr(va), None, out)

    def block(b, e):
        return lambda ctx, out: lib.ipt_single_upload_csr_rows(ctx.handle, n, dptr(p.d), None, i64ptr(rp),
                                                              i32ptr(ci), dptr(va), None, b, e, out)
    return whole, block, None


def _warm(n, seed):
    z = 1e-3 * np.random.default_rng(seed).standard_normal(n)
    z[0] = 1.0
    return z


@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_one_step_blocks_equal_whole_rows(kind):
    if kind == "dense":
        p = synth.dense_normal(3000)
        whole, block, keep = _dense(p)
        blocks = [(0, 1000), (1000, 3000), (777, 2222), (2999, 3000)]
    else:
        p = synth.csr_ci(8192, 32, 0.01, 42)
        whole, block, keep = _csr(p)
        blocks = [(0, 4096), (4096, 8192), (1024, 5000), (8188, 8192)]
    n = p.size()
    warm = _warm(n, 1)
    f = _steps(whole, n, warm, 1)
    for b, e in blocks:
        fb = _steps(block(b, e), n, warm, 1)
        assert np.array_equal(fb[b:e], f[b:e]), (kind, b, e)


@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_emulated_row_sharded_steps_equal_whole_run(kind):
    if kind == "dense":
        p = synth.dense_normal(2048)
        whole, block, keep = _dense(p)
        blocks = [(0, 1024), (1024, 2048)]
    else:
        p = synth.csr_ci(8192, 32, 0.01, 42)
        whole, block, keep = _csr(p)
        blocks = [(0, 2048), (2048, 4096), (4096, 6144), (6144, 8192)]
    n = p.size()
    z = _warm(n, 2)
    want = _steps(whole, n, z, 4)
    for _ in range(4):  # each "rank" maps its rows; the host stands in for the all-gather
        nz = np.empty(n)
        for b, e in blocks:
            nz[b:e] = _steps(block(b, e), n, z, 1)[b:e]
        z = nz
    assert np.array_equal(z, want)


def test_bad_row_blocks_rejected():
    lib = _lib.load()
    ctx = ipt.default_context()
    n = 8
    d = np.arange(n, dtype=float)
    delta = np.zeros((n, n))
    h = C.c_void_p()
    for b, e in [(4, 4), (2, 9), (-1, 3)]:
        with pytest.raises(ValueError):
            check(lib.ipt_single_upload_dense_rows(ctx.handle, n, dptr(d), None, dptr(delta), None, b, e, C.byref(h)))


def _steps_with_peers(upload, n, warm, steps, npeers):
    """As _steps, with npeers local buffers standing in for the peers' z: the map kernel
    stores its rows of every new iterate into them (the fused all-gather of a
    multi-GPU run, ipt_single.cu setup_peer_gather)."""
    lib = _lib.load()
    ctx = ipt.default_context()
    h = C.c_void_p()
    check(upload(ctx, C.byref(h)))
    try:
        check(lib.ipt_single_debug_peers(h, npeers))
        check(lib.ipt_single_reset(ctx.handle, h, 0, dptr(warm), None))
        prm = _params(ipt.IterationConfig(max_iterations=steps), ignore_convergence=1, divergence_threshold=1e300)
        st = Stats()
        check(lib.ipt_single_iterate(ctx.handle, h, C.byref(prm), C.byref(st)))
        z = np.empty(n)
        check(lib.ipt_single_download(ctx.handle, h, dptr(z), None))
        peers = []
        for q in range(npeers):
            pz = np.empty(n)
            check(lib.ipt_single_debug_peer_z(h, q, steps & 1, dptr(pz)))
            peers.append(pz)
        return z, peers
    finally:
        lib.ipt_single_free(h)


@pytest.mark.parametrize("kind", ["dense", "csr"])
@pytest.mark.parametrize("steps", [1, 2, 3])
def test_fused_allgather_stores_reach_every_peer(kind, steps):
    """Each rank's map kernel writes its rows of the new iterate into all peers' z: with
    3 stand-in peers every one holds exactly the block's rows of the current iterate, and
    the run itself is unchanged (bit for bit)."""
    if kind == "dense":
        p = synth.dense_normal(2048)
        whole, block, keep = _dense(p)
        b, e = 512, 1536
    else:
        p = synth.csr_ci(8192, 32, 0.01, 42)
        whole, block, keep = _csr(p)
        b, e = 2048, 6144
    n = p.size()
    warm = _warm(n, 3)
    plain = _steps(block(b, e), n, warm, steps)
    z, peers = _steps_with_peers(block(b, e), n, warm, steps, 3)
    assert np.array_equal(z, plain)
    for pz in peers:
        assert np.array_equal(pz[b:e], z[b:e])


def test_debug_peers_rejected_on_complex_or_too_many():
    lib = _lib.load()
    ctx = ipt.default_context()
    n = 64
    p = synth.dense_normal(n)
    h = C.c_void_p()
    check(lib.ipt_single_upload_dense(ctx.handle, n, dptr(p.d), None, dptr(np.ascontiguousarray(p.delta)), None,
                                      C.byref(h)))
    try:
        with pytest.raises(ValueError):
            check(lib.ipt_single_debug_peers(h, 8))
    finally:
        lib.ipt_single_free(h)
