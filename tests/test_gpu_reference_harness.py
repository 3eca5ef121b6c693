"""The reference's own tests, compiled unmodified from /root/reference/proj/tests
against libipt_b200.so (oracle/Makefile target `harness`), run on the B200.

Doctest files: test_solver.cpp, test_kernels.cpp, test_testgen.cpp, test_matcore.cpp
(hot path) and test_anderson.cpp, test_refine.cpp, test_rspt.cpp (the callers of §8 f1/f4
running on our solvers and device LU), through the doctest-compatible shim
tests/cpp/doctest.h. Acceptance
criteria 1, 2, 5, 9 are the hot-path ones; the others exercise the
reference's off-path modules calling into our solvers."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")

pytestmark = pytest.mark.gpu


def _run(exe, timeout, product="dmma"):
    path = os.path.join(REF, exe)
    if not os.path.exists(path):
        pytest.skip(f"{exe} not built (make -C oracle harness needs /root/reference)")
    env = dict(os.environ)
    env.pop("IPT_PRODUCT", None)
    if product == "ozaki":  # the drop-in ipt::solve_full on the tcgen05 product (solver.cpp)
        env["IPT_PRODUCT"] = "ozaki"
    return subprocess.run([path], capture_output=True, text=True, timeout=timeout, env=env)


@pytest.mark.parametrize("product", ["dmma", "ozaki"])
def test_reference_unit_tests_against_b200_library(product):
    r = _run("unit_b200", 900, product)
    print(r.stdout[-4000:])
    assert "test cases:" in r.stdout
    assert r.returncode == 0, r.stdout[-4000:]


def test_reference_acceptance_hot_path_criteria():
    """Criteria 1, 2, 5, 9 (hot path) and 4, 6, 7, 8 (off-path modules calling our solvers)
    must pass. Criterion 3 (explorer, off-path, run on the reference's own CPU kernels)
    fails identically on the reference build (flip 0.8634, cardioid 30/32).
    Criterion 9 is the reference's cost model T_eig/T_mm per product in [0.5, 2]; with the
    left factor of kernels::matmul kept on the device across the bench repetitions it
    measures 0.83 per product (was 0.53 when every matmul re-uploaded Delta)."""
    r = _run("acceptance_b200", 1800)
    _check_acceptance(r)


def test_reference_acceptance_with_the_ozaki_product():
    """The same criteria with every solve_full on the FP64-accurate tcgen05 product."""
    _check_acceptance(_run("acceptance_b200", 1800, "ozaki"))


def _check_acceptance(r):
    print(r.stdout)
    status = {int(m.group(2)): m.group(1) for m in re.finditer(r"\[(PASS|FAIL)\] criterion (\d+)", r.stdout)}
    for crit in (1, 2, 4, 5, 6, 7, 8, 9):
        assert status.get(crit) == "PASS", (crit, r.stdout)
    assert "flip 0.8634" in r.stdout  # criterion 3: same numbers as the reference build
