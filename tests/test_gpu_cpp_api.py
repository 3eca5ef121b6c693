"""The ipt::b200 additions to the C++ drop-in API (Ozaki/tcgen05 product, max-abs stop
rule) through the C++ entry points: tests/cpp/test_b200_api.cpp, built by
paper_2012_14702_b200/Makefile and run on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2012_14702_b200", "_build", "test_b200_api")

pytestmark = pytest.mark.gpu


def test_b200_cpp_api():
    assert os.path.exists(EXE), "build() compiles it (make -C paper_2012_14702_b200)"
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "test cases:" in r.stdout
