"""Configs 2 and 3 (N = 8192, 32768) on the B200 against the reference's
solve_single(j) columns (golden, the column route of SURVEY §8c) and the
SURVEY §8(d) anchors, plus size-independent properties at full size."""
import math

import numpy as np
import pytest

import paper_2012_14702_b200 as ipt
from conftest import golden
from paper_2012_14702_b200 import synth

pytestmark = pytest.mark.gpu


def _check_columns(r, g, n):
    cols = g[f"n{n}_cols"]
    lam = g[f"n{n}_lam"]
    assert np.max(np.abs(r.eigenvalues[cols] - lam) / np.abs(lam)) <= 1e-10
    assert np.max(np.abs(r.Z[:, cols] - g[f"n{n}_z"])) <= 1e-9


def _frob(p):
    return math.sqrt(np.sum(p.delta ** 2) + np.sum(p.d ** 2))


def test_config2_n8192():
    p = synth.config2()
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12, record_trace=True))
    assert r.status == ipt.SolveStatus.Converged
    assert abs(r.iterations - 5) <= 1  # 5 iterations for rel-Fro <= 1e-12
    assert r.eigenvalues[0] == pytest.approx(0.999960499073907, abs=1e-13)
    assert r.eigenvalues[-1] == pytest.approx(8192.000031943360227, abs=1e-9)
    assert r.residual_frobenius <= 1e-10 * _frob(p)
    assert np.all(np.diag(r.Z) == 1.0)
    assert r.min_singular_value_estimate == pytest.approx(1.000007, abs=5e-6)
    _check_columns(r, golden("full_columns.npz"), 8192)


@pytest.mark.slow
def test_config3_max_abs_rule_iterations():
    """configs[2] under BASELINE's stop rule max|A_new - A_old| < 1e-12, pinned like above."""
    p = synth.config3()
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12, stop_rule="max_abs",
                                                                 record_trace=True), want_sigma_min=False)
    pin = golden("config3_trace.npz")
    assert r.status == ipt.SolveStatus.Converged and r.final_max_abs < 1e-12
    assert r.iterations == int(pin["iterations_max_abs"])
    mx = np.asarray(pin["max_abs"])
    assert np.allclose(r.trace_max_abs[:3], mx[:3], rtol=1e-6, atol=0)


def test_config2_max_abs_rule():
    p = synth.config2()
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12, stop_rule="max_abs"),
                       want_sigma_min=False)
    assert r.status == ipt.SolveStatus.Converged and r.final_max_abs < 1e-12
    assert 5 <= r.iterations <= 7


@pytest.mark.slow
@pytest.mark.parametrize("product", ["dmma", "ozaki"])
def test_config3_n32768(product):
    """configs[2] at full size against 16 columns of the reference's own solve_single(j)
    (tests/golden/full_columns.npz), with either FP64 product (DMMA / Ozaki on tcgen05)."""
    p = synth.config3()
    r = ipt.solve_full(p, ipt.build_gaps(p), ipt.IterationConfig(tolerance=1e-12, record_trace=True),
                       product=product)
    assert r.status == ipt.SolveStatus.Converged
    # iteration count pinned against the reference loop (solver.cpp:208-250) run to convergence
    # on the same inputs (tests/golden/config3_trace.npz, make_config3_trace.py): north_star +-1,
    # and the step trace agrees iteration by iteration
    pin = golden("config3_trace.npz")
    assert abs(r.iterations - int(pin["iterations_rel_fro"])) <= 1
    assert r.iterations == int(pin["iterations_rel_fro"])
    steps = np.asarray(pin["steps"])
    m = min(len(steps), r.iterations)
    assert np.allclose(r.trace[:m - 1], steps[:m - 1], rtol=1e-6, atol=0)
    assert 0.5 < r.trace[m - 1] / steps[m - 1] < 2.0  # last step ~1e-14: rounding-level differences
    assert r.residual_frobenius <= 1e-10 * _frob(p)
    assert np.all(np.diag(r.Z) == 1.0)
    assert 0.9 < r.min_singular_value_estimate <= 1.0 + 1e-4
    g = golden("full_columns.npz")
    if "n32768_cols" in g.files:
        _check_columns(r, g, 32768)
    else:  # column route on the device itself (test_solver.cpp:188-201)
        for j in (0, 16384, 32767):
            one = ipt.solve_single(p, ipt.build_gaps(p), j, ipt.IterationConfig(tolerance=1e-12))
            assert np.max(np.abs(r.Z[:, j] - one.z)) <= 1e-9
