"""K16 (ipt_closing.cu): the closing residual |MZ - Z Lambda|_F of a converged real dense
solve from the last map's product plus an INT8 tensor-core correction Delta (Z_new - Z_old),
instead of a second FP64 product (solver.cpp:252-270). Z and the eigenvalues do not
depend on it (bit for bit); the residual agrees with the full FP64 closing product to the
noise level of that product's own cancellation."""
import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import dist, synth

pytestmark = pytest.mark.gpu


def _both(p, monkeypatch, product="dmma", cfg=None):
    cfg = cfg or ipt.IterationConfig(tolerance=1e-12)
    g = ipt.build_gaps(p)
    fast = ipt.solve_full(p, g, cfg, product=product)
    monkeypatch.setenv("IPT_CLOSING", "exact")
    exact = ipt.solve_full(p, g, cfg, product=product)
    monkeypatch.delenv("IPT_CLOSING")
    return fast, exact


@pytest.mark.parametrize("n", [512, 1000, 2048, 4096])
def test_closing_residual_matches_the_fp64_closing_product(n, monkeypatch):
    p = synth.dense_uniform(n, 0.32 / np.sqrt(n), 5 + n)
    fast, exact = _both(p, monkeypatch)
    assert np.array_equal(fast.Z, exact.Z) and np.array_equal(fast.eigenvalues, exact.eigenvalues)
    assert fast.iterations == exact.iterations
    assert fast.residual_frobenius == pytest.approx(exact.residual_frobenius, rel=2e-2)
    fro = np.sqrt(np.sum(p.delta ** 2) + np.sum(p.d ** 2))
    assert fast.residual_frobenius <= 1e-10 * fro


def test_closing_residual_with_the_ozaki_product(monkeypatch):
    p = synth.dense_uniform(1536, 0.3 / np.sqrt(1536), 8)
    fast, exact = _both(p, monkeypatch, product="ozaki")
    assert np.array_equal(fast.Z, exact.Z)
    assert fast.residual_frobenius == pytest.approx(exact.residual_frobenius, rel=2e-2)


def test_closing_residual_on_a_nonsymmetric_wide_delta(monkeypatch):
    rng = np.random.default_rng(4)
    n = 1200
    d = np.arange(1.0, n + 1.0)
    delta = 0.2 / np.sqrt(n) * rng.standard_normal((n, n)) * 10.0 ** (-6 * rng.random((n, n)))
    np.fill_diagonal(delta, 0.0)
    p = ipt.Partition(d, delta)
    fast, exact = _both(p, monkeypatch)
    assert fast.residual_frobenius == pytest.approx(exact.residual_frobenius, rel=2e-2)


def test_loose_tolerance_keeps_the_exact_closing_product(monkeypatch):
    """A last step above 1e-6 (a loose tolerance) is not small enough for the INT8
    correction: the full FP64 product runs, so both settings agree bit for bit."""
    p = synth.dense_uniform(1024, 0.01, 3)
    fast, exact = _both(p, monkeypatch, cfg=ipt.IterationConfig(tolerance=1e-4))
    assert fast.final_step > 1e-6
    assert fast.residual_frobenius == exact.residual_frobenius


def test_closing_residual_on_column_shards(monkeypatch):
    p = synth.dense_uniform(1500, 0.32 / np.sqrt(1500), 12)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-12)
    one = ipt.solve_full(p, g, cfg)
    ctxs = dist.local_contexts(3)
    outs = dist.run_ranks(lambda c: ipt.solve_full(p, g, cfg, ctx=c), ctxs)
    assert np.array_equal(outs[0].Z, one.Z)
    assert outs[0].residual_frobenius == pytest.approx(one.residual_frobenius, rel=1e-6)
