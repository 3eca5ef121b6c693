"""Complex full-spectrum map rate (3M: three real DMMA GEMMs, the complex map fused
into the third GEMM's epilogue) against the real map at the same N. The complex rate
is quoted as 4M-equivalent real flops (8N^3 per map, what the reference's four real
GEMMs perform) and as executed flops (6N^3). Each map with the DMMA product and with the
Ozaki product (tcgen05 INT8) for the real GEMMs.

    python tools/complex_probe.py [n]
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
lib = _lib.load()
ctx = ipt.default_context()
rng = np.random.default_rng(1)
d = np.arange(1.0, n + 1.0)
dr = (0.3 / np.sqrt(n)) * rng.standard_normal((n, n))
di = (0.3 / np.sqrt(n)) * rng.standard_normal((n, n))
np.fill_diagonal(dr, 0.0)
np.fill_diagonal(di, 0.0)
out = {}
for name, im, prod in (("real", None, 0), ("complex", di, 0), ("real_ozaki", None, 1), ("complex_ozaki", di, 1)):
    h = C.c_void_p()
    check(lib.ipt_full_upload(ctx.handle, n, dptr(d), None, dptr(dr), dptr(im), C.byref(h)))
    check(lib.ipt_full_reset(ctx.handle, h, None, None))
    check(lib.ipt_full_set_product(h, prod))
    tot, dom = C.c_double(), C.c_double()
    check(lib.ipt_full_run_maps(ctx.handle, h, 2, C.byref(tot), C.byref(dom)))
    check(lib.ipt_full_run_maps(ctx.handle, h, 4, C.byref(tot), C.byref(dom)))
    lib.ipt_full_free(h)
    ms = tot.value / 4
    flops = (8.0 if im is not None else 2.0) * n ** 3
    out[name] = {"ms_per_map": ms, "TFs_4M_equivalent" if im is not None else "TFs": flops / (ms * 1e-3) / 1e12}
    if im is not None:
        out[name]["TFs_executed_3M"] = 6.0 * n ** 3 / (ms * 1e-3) / 1e12
print(json.dumps({"n": n, **out}))
