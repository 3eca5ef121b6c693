"""Ozaki-product map sequence: 2 untimed maps (the first from Z = I needs no product),
then `steps` timed maps (also usable under ncu for launch lists).

    python tools/probes/ozaki_only.py N [steps]
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = synth.config3(n=n)
h = C.c_void_p()
check(lib.ipt_full_upload(ctx.handle, n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
check(lib.ipt_full_reset(ctx.handle, h, None, None))
check(lib.ipt_full_set_product(h, 1))
tot, ker = C.c_double(), C.c_double()
check(lib.ipt_full_run_maps(ctx.handle, h, 2, C.byref(tot), C.byref(ker)))
check(lib.ipt_full_run_maps(ctx.handle, h, steps, C.byref(tot), C.byref(ker)))
print(json.dumps({"n": n, "group": os.environ.get("IPT_I8_GROUP", "default"),
                  "kernel": os.environ.get("IPT_I8_KERNEL", "default"),
                  "ms_per_map": tot.value / steps, "fp64_equiv_TFs": 2.0 * n ** 3 / (tot.value / steps * 1e-3) / 1e12}),
      flush=True)
