"""One 8192^3 INT8 tcgen05 GEMM launch (ncu target)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib  # noqa: E402
from paper_2012_14702_b200._lib import check  # noqa: E402

args = [int(x) for x in sys.argv[1:]] or [8192]
M, N, K = (args * 3)[:3] if len(args) < 3 else args[:3]
rng = np.random.default_rng(0)
a = rng.integers(-128, 128, (M, K), dtype=np.int8)
b = rng.integers(-128, 128, (N, K), dtype=np.int8)
ms = C.c_double()
check(_lib.load().ipt_i8_gemm(ipt.default_context().handle, M, N, K, a.ctypes.data, b.ctypes.data, None, 3,
                              C.byref(ms)))
print("M N K", M, N, K, "ms", ms.value, "TOPS", 2.0 * M * N * K / (ms.value * 1e-3) / 1e12)
