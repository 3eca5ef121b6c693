"""Full-spectrum map with W = Delta Z by DMMA (FP64 tensor cores) vs Ozaki scheme II
(tcgen05 INT8 datapath), configs 2/3 construction.

    python tools/probes/ozaki_probe.py 8192 16384 32768
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib, synth  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr  # noqa: E402

lib = _lib.load()
ctx = ipt.default_context()
for n in [int(a) for a in sys.argv[1:]] or [8192]:
    p = synth.config3(n=n)
    out = {"n": n}
    for name, prod in (("dmma", 0), ("ozaki", 1)):
        h = C.c_void_p()
        check(lib.ipt_full_upload(ctx.handle, n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
        check(lib.ipt_full_reset(ctx.handle, h, None, None))
        check(lib.ipt_full_set_product(h, prod))
        tot, ker = C.c_double(), C.c_double()
        check(lib.ipt_full_run_maps(ctx.handle, h, 2, C.byref(tot), C.byref(ker)))
        steps = 3
        check(lib.ipt_full_run_maps(ctx.handle, h, steps, C.byref(tot), C.byref(ker)))
        lib.ipt_full_free(h)
        ms = tot.value / steps
        out[name] = {"ms_per_map": ms, "fp64_equiv_TFs": 2.0 * n ** 3 / (ms * 1e-3) / 1e12,
                     "product_ms": ker.value / steps}
    out["speedup"] = out["dmma"]["ms_per_map"] / out["ozaki"]["ms_per_map"]
    print(json.dumps(out), flush=True)
    del p
