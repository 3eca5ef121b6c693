"""FP64-accurate products on the tcgen05 INT8 datapath (Ozaki scheme II, ozaki.cu): the
INT8 GEMM is exact, and the full-spectrum solve with product='ozaki' matches the DMMA
solve (and therefore the reference) far inside the north_star tolerances."""
import ctypes as C

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import _lib, synth
from paper_2012_14702_b200._lib import check

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(128, 256, 128), (256, 512, 1024), (384, 768, 2176)])
def test_i8_gemm_is_exact(shape):
    M, N, K = shape
    rng = np.random.default_rng(M + N + K)
    a = rng.integers(-128, 128, (M, K), dtype=np.int8)
    b = rng.integers(-128, 128, (N, K), dtype=np.int8)
    c = np.empty((M, N), np.int32)
    ms = C.c_double()
    ctx = ipt.default_context()
    check(_lib.load().ipt_i8_gemm(ctx.handle, M, N, K, a.ctypes.data, b.ctypes.data, c.ctypes.data, 0, C.byref(ms)))
    assert np.array_equal(c, a.astype(np.int64) @ b.astype(np.int64).T)


@pytest.mark.parametrize("n", [64, 300, 1000, 2048])
def test_ozaki_solve_matches_dmma(n):
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 11)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-13)
    a = ipt.solve_full(p, g, cfg, product="dmma")
    b = ipt.solve_full(p, g, cfg, product="ozaki")
    assert a.iterations == b.iterations and a.status == b.status
    assert np.max(np.abs(a.eigenvalues - b.eigenvalues) / np.abs(a.eigenvalues)) <= 1e-14
    assert np.max(np.abs(a.Z - b.Z)) <= 1e-13
    assert b.residual_frobenius <= 10 * max(a.residual_frobenius, 1e-14)


def test_ozaki_one_map_from_a_dense_warm_start():
    """A map of a general Z (not the converged basis): entries over many binades."""
    n = 700
    rng = np.random.default_rng(5)
    p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 12)
    g = ipt.build_gaps(p)
    z = np.eye(n) + rng.standard_normal((n, n)) * np.exp(rng.uniform(-20, 2, (n, n)))
    np.fill_diagonal(z, 1.0)
    cfg = ipt.IterationConfig(max_iterations=1, divergence_threshold=1e300)
    a = ipt.solve_full(p, g, cfg, warm_start=z, want_sigma_min=False, product="dmma")
    b = ipt.solve_full(p, g, cfg, warm_start=z, want_sigma_min=False, product="ozaki")
    scale = np.max(np.abs(a.Z), axis=0)
    assert np.max(np.abs(a.Z - b.Z) / scale) <= 1e-14


def test_ozaki_is_bitwise_deterministic():
    p = synth.dense_uniform(512, 0.01, 3)
    g = ipt.build_gaps(p)
    a = ipt.solve_full(p, g, product="ozaki")
    b = ipt.solve_full(p, g, product="ozaki")
    assert np.array_equal(a.Z, b.Z) and np.array_equal(a.eigenvalues, b.eigenvalues)


def test_ozaki_nonfinite_delta_falls_back():
    n = 64
    d = np.arange(n, dtype=float)
    delta = np.zeros((n, n))
    delta[3, 7] = np.inf
    p = ipt.Partition(d, delta)
    r = ipt.solve_full(p, ipt.build_gaps(p), product="ozaki")
    assert r.status == ipt.SolveStatus.Diverged and r.iterations == 1
