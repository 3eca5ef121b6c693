"""tcgen05 INT8 GEMM (ipt_i8_gemm): exactness against numpy and throughput.

    python tools/probes/i8_probe.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib  # noqa: E402
from paper_2012_14702_b200._lib import check  # noqa: E402

lib = _lib.load()
ctx = ipt.default_context()


def gemm(a, b, iters=0):
    M, K = a.shape
    N = b.shape[0]
    c = np.empty((M, N), np.int32)
    ms = C.c_double()
    check(lib.ipt_i8_gemm(ctx.handle, M, N, K, a.ctypes.data, b.ctypes.data, c.ctypes.data, iters, C.byref(ms)))
    return c, ms.value


rng = np.random.default_rng(0)
for (M, N, K) in [(128, 256, 128), (256, 512, 1024), (1024, 1024, 4096)]:
    a = rng.integers(-128, 128, (M, K), dtype=np.int8)
    b = rng.integers(-128, 128, (N, K), dtype=np.int8)
    c, _ = gemm(a, b)
    want = a.astype(np.int64) @ b.astype(np.int64).T
    print(json.dumps(dict(M=M, N=N, K=K, exact=bool(np.array_equal(c, want)),
                          max_err=int(np.max(np.abs(c - want))))), flush=True)
for n in [4096, 8192]:
    a = rng.integers(-128, 128, (n, n), dtype=np.int8)
    b = rng.integers(-128, 128, (n, n), dtype=np.int8)
    _, ms = gemm(a, b, iters=10)
    print(json.dumps(dict(n=n, ms=ms, tops=2.0 * n ** 3 / (ms * 1e-3) / 1e12)), flush=True)
