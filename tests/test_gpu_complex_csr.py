"""Complex CSR single pair (the same entry points with imag != 0) on the
grouped complex SpMV (cspmv_group_kernel: warp-contiguous row groups, z gathered from an
interleaved copy, one 16-byte load per entry) against the reference build itself, and
against the thread-per-row kernel it replaced (IPT_CSPMV_SIMPLE=1)."""
import os

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import synth

pytestmark = pytest.mark.gpu


def _hermitian_csr(n, per_row, seed, imag=0.003, complex_d=False):
    p = synth.csr_ci(n, per_row, 0.01, seed)
    rp, ci, va = p.delta.row_offsets, p.delta.col_indices, p.delta.values
    rows = np.repeat(np.arange(n), np.diff(rp))
    vals = va + 1j * imag * np.sign(ci - rows) * np.abs(va)  # antisymmetric imaginary part: Hermitian
    d = p.d + (0.05j * np.sin(np.arange(n)) if complex_d else 0.0)
    return ipt.Partition(np.asarray(d), ipt.CsrMatrix(n, n, rp.copy(), ci.copy(), vals))


@pytest.mark.parametrize("anchor", [0, 17])
def test_complex_csr_single_pair_matches_the_reference(ref_arm, anchor):
    p = _hermitian_csr(3000, 12, 5)
    g = ipt.build_gaps(p, 0.0)
    cfg = ipt.IterationConfig(tolerance=1e-12)
    r = ipt.solve_single(p, g, anchor, cfg)
    o = ref_arm.solve_single(p.d, p.delta, anchor, tol=1e-12)
    assert r.status == ipt.SolveStatus.Converged
    assert abs(r.iterations - o["iterations"]) <= 1
    assert abs(r.eigenvalue - o["eigenvalue"]) <= 1e-10 * abs(o["eigenvalue"])
    assert np.max(np.abs(r.z - o["z"])) <= 1e-9
    assert np.iscomplexobj(r.z) and np.max(np.abs(r.z.imag)) > 1e-8  # genuinely complex


def test_complex_d_real_delta_and_continuation(ref_arm):
    p = _hermitian_csr(2000, 10, 7, imag=0.0, complex_d=True)  # real Delta, complex d (VI = false)
    g = ipt.build_gaps(p, 0.0)
    cfg = ipt.IterationConfig(tolerance=1e-12)
    r = ipt.solve_single(p, g, 3, cfg)
    o = ref_arm.solve_single(p.d, p.delta, 3, tol=1e-12)
    assert abs(r.eigenvalue - o["eigenvalue"]) <= 1e-10 * abs(o["eigenvalue"])
    assert np.max(np.abs(r.z - o["z"])) <= 1e-9
    rc = ipt.solve_single_continuation(p, g, 3, cfg, 0.5)
    oc = ref_arm.solve_single(p.d, p.delta, 3, tol=1e-12, mode="continuation", alpha=0.5)
    assert abs(rc.iterations - oc["iterations"]) <= 1
    assert np.max(np.abs(rc.z - oc["z"])) <= 1e-9


def test_grouped_and_thread_per_row_kernels_agree(monkeypatch):
    p = _hermitian_csr(1 << 15, 16, 9)
    g = ipt.build_gaps(p, 0.0)
    cfg = ipt.IterationConfig(tolerance=1e-12)
    fast = ipt.solve_single(p, g, 0, cfg)
    monkeypatch.setenv("IPT_CSPMV_SIMPLE", "1")
    slow = ipt.solve_single(p, g, 0, cfg)
    assert fast.iterations == slow.iterations
    assert np.max(np.abs(fast.z - slow.z)) <= 1e-13
    assert abs(fast.eigenvalue - slow.eigenvalue) <= 1e-14 * abs(slow.eigenvalue)
    x = np.random.default_rng(1).standard_normal(1 << 15) + 1j * np.random.default_rng(2).standard_normal(1 << 15)
    monkeypatch.delenv("IPT_CSPMV_SIMPLE")
    y = ipt.kernels.matvec(p.delta, x)
    dense = p.delta
    ref = np.zeros(1 << 15, complex)
    rows = np.repeat(np.arange(1 << 15), np.diff(dense.row_offsets))
    np.add.at(ref, rows, dense.values * x[dense.col_indices])
    assert np.max(np.abs(y - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("n", [1, 2, 37])
def test_real_csr_times_complex_vector(n):
    """kernels::matvec with a real (possibly empty) CSR and a complex x takes the complex
    path on a real problem: the interleaved gather copy is allocated there too."""
    rng = np.random.default_rng(n)
    mask = rng.random((n, n)) < 0.2
    np.fill_diagonal(mask, False)
    a = np.where(mask, rng.standard_normal((n, n)), 0.0)
    r, c = np.nonzero(a)
    csr = ipt.CsrMatrix.from_triplets(n, n, r, c, a[r, c])
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = ipt.kernels.matvec(csr, x)
    assert np.max(np.abs(y - a @ x), initial=0.0) <= 1e-14
