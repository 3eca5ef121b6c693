"""sigma_min (smallest_singular_value_estimate, solver.cpp:275-297) on the device:
the matrix-free CG inverse iteration against the Cholesky-factor path (forced with
IPT_SIGMA=factor) and the CPU oracle (plain-C restatement with the reference's LU).
The CG path must agree with the factor path to 1e-12 relative; both with the oracle
to 1e-8 (the tolerance of test_gpu_full.py's sigma tests)."""
import os

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt

pytestmark = pytest.mark.gpu


def near_identity(n, scale, seed, cplx=False):
    rng = np.random.default_rng(seed)
    z = np.eye(n) + (scale / np.sqrt(n)) * rng.standard_normal((n, n))
    if cplx:
        z = z + 1j * (scale / np.sqrt(n)) * rng.standard_normal((n, n))
    return z


def sigma(z, mode=None):
    old = os.environ.get("IPT_SIGMA")
    try:
        if mode is None:
            os.environ.pop("IPT_SIGMA", None)
        else:
            os.environ["IPT_SIGMA"] = mode
        return ipt.smallest_singular_value_estimate(z)
    finally:
        if old is None:
            os.environ.pop("IPT_SIGMA", None)
        else:
            os.environ["IPT_SIGMA"] = old


@pytest.mark.parametrize("n,scale", [(1, 0.1), (31, 0.05), (257, 0.1), (1024, 0.3), (3001, 0.05)])
def test_cg_path_matches_factor_path(n, scale, port_arm):
    z = near_identity(n, scale, seed=n)
    a = sigma(z)
    b = sigma(z, "factor")
    assert a == pytest.approx(b, rel=1e-12)
    if n <= 1024:
        assert a == pytest.approx(port_arm.sigma_min(z), rel=1e-8)


def test_cg_path_complex(port_arm):
    z = near_identity(300, 0.2, seed=3, cplx=True)
    a = sigma(z)
    assert a == pytest.approx(sigma(z, "factor"), rel=1e-12)
    assert a == pytest.approx(port_arm.sigma_min(z), rel=1e-8)


def test_ill_conditioned_falls_back_and_matches_oracle(port_arm):
    """A Gaussian matrix (condition ~ n): CG cannot reach 1e-15 in 64 steps, so the
    factor path runs; the result is the same as forcing it."""
    rng = np.random.default_rng(11)
    z = rng.standard_normal((400, 400))
    a = sigma(z)
    assert a == sigma(z, "factor")
    assert a == pytest.approx(port_arm.sigma_min(z), rel=1e-8)


def test_singular_input_reports_zero():
    z = np.eye(64)
    z[:, 5] = 0.0
    assert sigma(z) == 0.0
