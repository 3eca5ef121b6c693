"""Complex dense single pair: per-step time and algorithmic GB/s vs the real GEMV map."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
lib = ipt.load_library()
ctx = ipt.default_context()
p = synth.dense_normal(n)
rng = np.random.default_rng(3)
ai = 0.3 / np.sqrt(n) * rng.standard_normal((n, n))
ai = np.ascontiguousarray((ai - ai.T) / np.sqrt(2.0))  # antisymmetric: Hermitian Delta
for name, im in (("real", None), ("complex", ai)):
    h = C.c_void_p()
    check(lib.ipt_single_upload_dense(ctx.handle, n, dptr(p.d), None, dptr(p.delta),
                                      dptr(im) if im is not None else None, C.byref(h)))
    check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
    tot, dom = C.c_double(), C.c_double()
    check(lib.ipt_single_run_steps(ctx.handle, h, 3, C.byref(tot), C.byref(dom)))
    check(lib.ipt_single_run_steps(ctx.handle, h, 10, C.byref(tot), C.byref(dom)))
    lib.ipt_single_free(h)
    b = 8.0 * n * n * (2 if im is not None else 1)
    print(f"{name}: step {tot.value / 10:.3f} ms, {b / (tot.value / 10 * 1e-3) / 1e9:.0f} GB/s algorithmic", flush=True)
