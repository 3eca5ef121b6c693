"""Teardown cost of a full-spectrum problem after an Ozaki / DMMA solve (N from argv)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402
from paper_2012_14702_b200._lib import Params, Stats, check, dptr  # noqa: E402
from paper_2012_14702_b200.ipt import _params  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
lib = ipt.load_library()
ctx = ipt.default_context()
p = synth.dense_uniform(n, 0.32 / n ** 0.5, 42)
for product in (0, 1, 1, 0):
    h = C.c_void_p()
    check(lib.ipt_full_upload(ctx.handle, n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
    check(lib.ipt_full_set_product(h, product))
    check(lib.ipt_full_reset(ctx.handle, h, None, None))
    prm = _params(ipt.IterationConfig(tolerance=1e-12))
    prm.want_sigma_min = 0
    st = Stats()
    check(lib.ipt_full_iterate(ctx.handle, h, C.byref(prm), C.byref(st)))
    check(lib.ipt_full_finalize(ctx.handle, h, C.byref(prm), C.byref(st)))
    ctx.synchronize()
    t0 = time.perf_counter()
    lib.ipt_full_free(h)
    t1 = time.perf_counter()
    print(f"product {'ozaki' if product else 'dmma'}: free {1e3 * (t1 - t0):.1f} ms", flush=True)
