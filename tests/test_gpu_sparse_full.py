"""Sparse-Delta full spectrum: solve_full / apply_map_full on a CSR
partition run the fused SpMM map on the device (Z row-major during the loop,
ipt_full.cu spmm_full_kernel) instead of densifying Delta.

Parity anchors: golden vectors from the reference's own sparse path
(solve_full on a CSR Partition -> matmul_sparse_parallel, kernels.cpp:88-108) made by
tests/golden/make_golden.py (sparse_full), plus the dense device path on the same
matrices. Tolerances as in test_gpu_full.py (BASELINE north_star): eigenvalues 1e-10
relative, eigenvectors 1e-9 absolute; the SpMM keeps the reference's CSR summation
order with one rounding per term, so in practice the iterates agree to the last bit
or within a few ulps (asserted at 1e-13).
"""
import math

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from conftest import golden
from paper_2012_14702_b200 import synth

pytestmark = pytest.mark.gpu

LAM_REL = 1e-10
VEC_ABS = 1e-9


def load_case(g, name):
    n = len(g[name + "_d"])
    delta = ipt.CsrMatrix(n, n, g[name + "_rowptr"], g[name + "_cols"].astype(np.int32), g[name + "_vals"])
    return ipt.Partition(g[name + "_d"].copy(), delta)


def random_sparse(n, per_row, seed, scale=0.05, gap=1.0):
    """Seeded sparse symmetric Delta with well separated d (test-local construction)."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n), per_row)
    cols = rng.integers(0, n, n * per_row)
    keep = rows != cols
    rows, cols = rows[keep], cols[keep]
    key = np.unique(np.minimum(rows, cols).astype(np.int64) * n + np.maximum(rows, cols))
    r, c = key // n, key % n
    v = scale * rng.standard_normal(key.size)
    rr = np.concatenate([r, c])
    cc = np.concatenate([c, r])
    vv = np.concatenate([v, v])
    d = gap * np.arange(n, dtype=float) + 0.1 * rng.random(n)
    return ipt.Partition(d, ipt.CsrMatrix.from_triplets(n, n, rr, cc, vv))


def test_sparse_full_matches_reference_golden_256():
    g = golden("sparse_full.npz")
    p = load_case(g, "f256")
    it, status, step, resid, sig, mm = g["f256_meta"]
    r = ipt.solve_full(p, ipt.build_gaps(p, 0.0))
    assert r.iterations == int(it)
    assert int(r.status) == int(status)
    assert r.matmul_count == int(mm)
    assert np.max(np.abs(r.Z - g["f256_Z"])) <= 1e-13
    np.testing.assert_allclose(r.eigenvalues, g["f256_lam"], rtol=1e-13, atol=0)
    assert r.final_step == pytest.approx(step, rel=1e-6, abs=1e-18)
    assert r.residual_frobenius == pytest.approx(resid, rel=1e-3, abs=1e-14)
    assert r.min_singular_value_estimate == pytest.approx(sig, rel=1e-6)


def test_sparse_apply_map_full_matches_reference_golden():
    g = golden("sparse_full.npz")
    p = load_case(g, "f256")
    f = ipt.apply_map_full(p, ipt.build_gaps(p, 0.0), g["f256_map_in"])
    want = g["f256_map_out"]
    assert np.max(np.abs(f - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))
    assert np.all(np.diag(f) == 1.0)


def test_sparse_full_matches_reference_golden_1024():
    g = golden("sparse_full.npz")
    p = load_case(g, "f1024")
    it, status, step, resid, sig, mm = g["f1024_meta"]
    r = ipt.solve_full(p, ipt.build_gaps(p, 0.0))
    assert r.iterations == int(it) and int(r.status) == int(status)
    np.testing.assert_allclose(r.eigenvalues, g["f1024_lam"], rtol=LAM_REL, atol=0)
    cols = g["f1024_zcols_idx"]
    assert np.max(np.abs(r.Z[:, cols] - g["f1024_zcols"])) <= VEC_ABS
    assert r.residual_frobenius == pytest.approx(resid, rel=1e-3, abs=1e-14)
    assert r.min_singular_value_estimate == pytest.approx(sig, rel=1e-6)


def test_sparse_full_config5_construction_diverges_like_reference():
    """Config 5's CI-like operator has near-degenerate d: the full map diverges
    (reference: 3 iterations, Diverged); the sparse device path must report the same."""
    g = golden("sparse_full.npz")
    it, status, nnz = g["ci4096_meta"]
    p = synth.csr_ci(4096)
    assert p.delta.nnz == int(nnz)
    r = ipt.solve_full(p, ipt.build_gaps(p, 0.0), ipt.IterationConfig(tolerance=1e-10), want_sigma_min=False)
    assert r.iterations == int(it)
    assert int(r.status) == int(status) == int(ipt.SolveStatus.Diverged)


@pytest.mark.parametrize("n,per_row", [(300, 5), (1000, 9), (4099, 16)])
def test_sparse_path_agrees_with_dense_path(n, per_row):
    """Same Delta through the SpMM path and the densified DMMA path (ragged n)."""
    p = random_sparse(n, per_row, seed=n)
    gaps = ipt.build_gaps(p, 0.0)
    cfg = ipt.IterationConfig(tolerance=1e-13, record_trace=True)
    rs = ipt.solve_full(p, gaps, cfg, want_sigma_min=False)
    rd = ipt.solve_full(ipt.Partition(p.d, p.delta.to_dense()), gaps, cfg, want_sigma_min=False)
    assert rs.status == ipt.SolveStatus.Converged
    assert abs(rs.iterations - rd.iterations) <= 1
    np.testing.assert_allclose(rs.eigenvalues, rd.eigenvalues, rtol=LAM_REL, atol=0)
    assert np.max(np.abs(rs.Z - rd.Z)) <= VEC_ABS
    m_fro = math.sqrt(np.sum(p.d ** 2) + np.sum(p.delta.values ** 2))
    assert rs.residual_frobenius <= 1e-10 * m_fro


def test_sparse_warm_start_and_determinism():
    p = random_sparse(700, 7, seed=3)
    gaps = ipt.build_gaps(p, 0.0)
    a = ipt.solve_full(p, gaps, want_sigma_min=False)
    b = ipt.solve_full(p, gaps, want_sigma_min=False)
    assert np.array_equal(a.Z, b.Z) and np.array_equal(a.eigenvalues, b.eigenvalues)
    # warm start from the converged basis scaled per column: renormalised, converges at once
    w = a.Z * (1.0 + np.arange(700))[None, :]
    c = ipt.solve_full(p, gaps, warm_start=w, want_sigma_min=False)
    assert c.iterations <= 2
    np.testing.assert_allclose(c.eigenvalues, a.eigenvalues, rtol=LAM_REL, atol=0)


def test_sparse_empty_delta_is_identity():
    n = 130
    p = ipt.Partition(np.arange(n, dtype=float), ipt.CsrMatrix(n, n, np.zeros(n + 1, np.int64),
                                                                np.zeros(0, np.int32), np.zeros(0)))
    r = ipt.solve_full(p, ipt.build_gaps(p, 0.0))
    assert r.iterations == 1 and r.status == ipt.SolveStatus.Converged
    assert np.array_equal(r.Z, np.eye(n))
    assert np.array_equal(r.eigenvalues, p.d)


def test_sparse_complex_delta_takes_dense_complex_path():
    n = 96
    rng = np.random.default_rng(5)
    rows = rng.integers(0, n, 400)
    cols = rng.integers(0, n, 400)
    key = np.unique(rows * n + cols)
    key = key[key // n != key % n]
    vals = 0.01 * (rng.standard_normal(key.size) + 1j * rng.standard_normal(key.size))
    delta = ipt.CsrMatrix.from_triplets(n, n, key // n, key % n, vals)
    p = ipt.Partition(np.arange(n, dtype=float), delta)
    gaps = ipt.build_gaps(p, 0.0)
    rs = ipt.solve_full(p, gaps)
    rd = ipt.solve_full(ipt.Partition(p.d, delta.to_dense()), gaps)
    assert rs.iterations == rd.iterations
    assert np.array_equal(rs.Z, rd.Z) and np.array_equal(rs.eigenvalues, rd.eigenvalues)


def test_sparse_rejects_bad_column_index():
    n = 8
    delta = ipt.CsrMatrix(n, n, np.array([0, 1] + [1] * (n - 1), np.int64), np.array([9], np.int32),
                          np.array([0.5]))
    p = ipt.Partition(np.arange(n, dtype=float), delta)
    with pytest.raises(ValueError):
        ipt.solve_full(p, ipt.build_gaps(p, 0.0))


@pytest.mark.slow
def test_sparse_full_large_residual():
    """N = 16384, ~32 nonzeros per row: converged basis with a small true residual."""
    n = 16384
    p = random_sparse(n, 16, seed=9, scale=0.02)
    r = ipt.solve_full(p, ipt.build_gaps(p, 0.0), ipt.IterationConfig(tolerance=1e-12), want_sigma_min=False)
    assert r.status == ipt.SolveStatus.Converged
    m_fro = math.sqrt(np.sum(p.d ** 2) + np.sum(p.delta.values ** 2))
    assert r.residual_frobenius <= 1e-10 * m_fro
    assert np.all(np.diag(r.Z) == 1.0)
