"""Memory-safety check standing in for compute-sanitizer memcheck (closed on this GPU pool):
the smoke-size workload over every kernel family (tools/sanitize_smoke.py: DMMA map /
closing / identity map, tcgen05 INT8 GEMM + Ozaki reconstruction, CG and Cholesky
sigma_min, cooperative LU, GEMV / grouped-CSR maps with the fused tail and stand-in peer
stores, Anderson, sparse-Delta SpMM, the in-process communicator at 2 ranks) with
IPT_GUARD=1, which brackets every device buffer with 4 KB byte-pattern guard zones and
checks them when the buffer is released. Any out-of-bounds write next to a buffer fails."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_guard_zones_stay_intact_over_every_kernel_family():
    env = dict(os.environ, IPT_GUARD="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_smoke.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert "guard violations 0 (IPT_GUARD=1)" in p.stdout, p.stdout[-2000:]
    assert "guard violation:" not in p.stderr, p.stderr[-4000:]
    checked = int(p.stdout.split("guard zones checked on ")[1].split()[0])
    assert checked >= 100, p.stdout[-2000:]


def test_guard_zones_catch_a_write_past_the_end():
    code = ("import paper_2012_14702_b200 as ipt; lib = ipt.load_library(); "
            "print('selftest', lib.ipt_guard_selftest(), lib.ipt_guard_violations())")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, IPT_GUARD="1"),
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "selftest 1 1" in p.stdout, p.stdout + p.stderr[-2000:]
    assert "guard violation: trailing guard of a 100-double buffer, byte 0" in p.stderr
