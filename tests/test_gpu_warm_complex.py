"""A complex warm start on a real problem runs in complex arithmetic, as the reference's
solve_full / solve_single do (proj/src/solver.cpp:188-201 renormalises the warm columns
by their complex diagonal; :32-45 for the single pair). The C ABI opens such a problem on
the complex path instead of dropping the imaginary part."""
import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import synth

pytestmark = pytest.mark.gpu


def test_full_complex_warm_start_on_real_delta(ref_arm):
    p = synth.dense_uniform(96, 0.02, 13)
    rng = np.random.default_rng(2)
    warm = np.eye(96) + 1e-3 * (rng.standard_normal((96, 96)) + 1j * rng.standard_normal((96, 96)))
    warm[np.arange(96), np.arange(96)] = 1.0 + 0.5j  # Z_jj complex: renormalisation divides by it
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12), warm_start=warm)
    o = ref_arm.solve_full(p.d, p.delta, tol=1e-12, warm=warm)
    assert np.iscomplexobj(r.Z)
    assert abs(r.iterations - o["iterations"]) <= 1
    assert np.max(np.abs(r.Z - o["Z"])) <= 1e-12
    assert np.max(np.abs(r.eigenvalues - o["eigenvalues"]) / np.abs(o["eigenvalues"])) <= 1e-12


def test_full_purely_imaginary_diagonal_warm_start(ref_arm):
    p = synth.dense_uniform(64, 0.02, 3)
    warm = 1j * np.eye(64)  # Re(Z_jj) = 0: renormalised by i, not by its real part
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12), warm_start=warm)
    o = ref_arm.solve_full(p.d, p.delta, tol=1e-12, warm=warm)
    assert np.all(np.isfinite(r.Z))
    assert np.max(np.abs(r.Z - o["Z"])) <= 1e-12
    assert r.iterations == o["iterations"]


def test_single_complex_warm_start_on_real_delta(ref_arm):
    p = synth.dense_normal(512)
    rng = np.random.default_rng(5)
    warm = np.zeros(512, complex)
    warm[0] = 2.0 - 1.0j
    warm[1:] = 1e-4 * (rng.standard_normal(511) + 1j * rng.standard_normal(511))
    r = ipt.solve_single(p, ipt.build_gaps(p), 0, ipt.IterationConfig(tolerance=1e-12), warm_start=warm)
    o = ref_arm.solve_single(p.d, p.delta, 0, tol=1e-12, warm=warm)
    assert abs(r.iterations - o["iterations"]) <= 1
    assert np.max(np.abs(r.z - o["z"])) <= 1e-12
    assert abs(r.eigenvalue - o["eigenvalue"]) <= 1e-12 * abs(o["eigenvalue"])
