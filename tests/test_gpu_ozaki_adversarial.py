"""The Ozaki product on adversarial operands: rows of Delta and columns of Z spanning 12+
decades, non-symmetric Delta. What holds, and what does not:

* normwise, the reference's own tolerance (proj/tests/test_kernels.cpp:40-50: max
  |C - C_ref| <= 1e-13 |A|_F |B|_F) holds, and so does the error model of DESIGN.md §8b:
  |C - AB|_ij <= 2^-53 (max_k|A_ik| |B_.j|_1 + max_k|B_kj| |A_i.|_1) + one rounding;
* componentwise it is NOT the FP64 GEMM's bound: an entry far below its row maximum is
  truncated to the row's 53-bit grid, so a product fed only by such entries can lose many
  digits (test_ozaki_is_not_componentwise_stable pins a concrete case). The DMMA product
  keeps the componentwise bound k eps |A||B| on the same operands;
* the IPT solve on a wide-range non-symmetric Delta still matches the reference's
  eigenvalues: the map's products are dominated by the row / column maxima.
The product therefore stays opt-in (product="ozaki"); DMMA is the default."""
import numpy as np
import pytest

import paper_2012_14702_b200 as ipt

pytestmark = pytest.mark.gpu

EPS = np.finfo(float).eps


def _wide(rng, m, k, decades):
    """Entries with magnitudes log-uniform over `decades` inside every row, random signs."""
    mag = 10.0 ** (-decades * rng.random((m, k)))
    return mag * rng.choice([-1.0, 1.0], (m, k))


def _exact(a, b):
    """A B in extended precision (np.longdouble dot products): rounding error ~1e-19 relative."""
    return (a.astype(np.longdouble) @ b.astype(np.longdouble)).astype(np.float64)


@pytest.mark.parametrize("decades", [6, 12, 15])
def test_ozaki_wide_rows_and_columns_meet_the_normwise_bounds(decades):
    rng = np.random.default_rng(decades)
    m, k, n = 96, 700, 80
    a = _wide(rng, m, k, decades)
    b = _wide(rng, n, k, decades).T.copy()  # columns of B span the same range
    c = ipt.kernels.matmul_ozaki(a, b)
    ref = _exact(a, b)
    err = np.abs(c - ref)
    # the reference's tolerance (test_kernels.cpp:40-50)
    assert err.max() <= 1e-13 * np.linalg.norm(a) * np.linalg.norm(b)
    # DESIGN.md §8b error model, entry by entry
    rowmax = np.abs(a).max(axis=1)[:, None]
    colmax = np.abs(b).max(axis=0)[None, :]
    model = 2.0 ** -53 * (rowmax * np.abs(b).sum(axis=0)[None, :] + colmax * np.abs(a).sum(axis=1)[:, None])
    assert np.all(err <= model + 2 * EPS * np.abs(ref))


def test_dmma_keeps_the_componentwise_bound_on_the_same_operands():
    rng = np.random.default_rng(3)
    m, k, n = 64, 500, 64
    a = _wide(rng, m, k, 12)
    b = _wide(rng, n, k, 12).T.copy()
    c = ipt.kernels.matmul(a, b)
    ref = _exact(a, b)
    assert np.all(np.abs(c - ref) <= k * EPS * (np.abs(a) @ np.abs(b)))


def test_ozaki_is_not_componentwise_stable():
    """Row [1, 1.2345e-12 ...] against a column that only meets the small entry: the small
    entry sits ~40 binades below its row maximum and keeps ~13 significant bits."""
    k = 64
    a = np.zeros((1, k))
    a[0, 0] = 1.0
    a[0, 1] = 1.2345e-12
    b = np.zeros((k, 1))
    b[1, 0] = 1.0
    b[0, 0] = 1e-300  # keeps column 0 live without contributing
    c = ipt.kernels.matmul_ozaki(a, b)[0, 0]
    exact = 1.2345e-12
    rel = abs(c - exact) / exact
    assert rel > 1e-8            # far outside FP64's componentwise accuracy ...
    assert abs(c - exact) <= 2.0 ** -53 * 1.0 * 1.0 + 2 * EPS * exact  # ... inside the normwise model
    d = ipt.kernels.matmul(a, b)[0, 0]
    assert abs(d - exact) <= 2 * EPS * exact  # the DMMA product is exact here


@pytest.mark.parametrize("n", [200, 513])
def test_ozaki_solve_on_a_wide_range_nonsymmetric_delta(n, ref_arm):
    rng = np.random.default_rng(n)
    d = np.arange(1.0, n + 1.0)
    delta = 0.2 / np.sqrt(n) * _wide(rng, n, n, 12)  # non-symmetric, 12 decades per row
    np.fill_diagonal(delta, 0.0)
    p = ipt.Partition(d, delta)
    g = ipt.build_gaps(p)
    cfg = ipt.IterationConfig(tolerance=1e-12)
    oz = ipt.solve_full(p, g, cfg, product="ozaki")
    dm = ipt.solve_full(p, g, cfg, product="dmma")
    ref = ref_arm.solve_full(d, delta, tol=1e-12)
    assert oz.status == ipt.SolveStatus.Converged and dm.status == ipt.SolveStatus.Converged
    assert abs(oz.iterations - ref["iterations"]) <= 1 and abs(dm.iterations - ref["iterations"]) <= 1
    lam = ref["eigenvalues"].real
    assert np.max(np.abs(oz.eigenvalues - lam) / np.abs(lam)) <= 1e-10
    assert np.max(np.abs(dm.eigenvalues - lam) / np.abs(lam)) <= 1e-13
    assert np.max(np.abs(oz.Z - ref["Z"].real)) <= 1e-9
    fro = np.sqrt(np.sum(delta ** 2) + np.sum(d ** 2))
    assert oz.residual_frobenius <= 1e-10 * fro
