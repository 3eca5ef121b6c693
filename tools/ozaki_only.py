"""One Ozaki-product map sequence (for ncu launch lists)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib, synth  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr  # noqa: E402

lib = _lib.load()
ctx = ipt.default_context()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
p = synth.config3(n=n)
h = C.c_void_p()
check(lib.ipt_full_upload(ctx.handle, n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
check(lib.ipt_full_reset(ctx.handle, h, None, None))
check(lib.ipt_full_set_product(h, 1))
tot, ker = C.c_double(), C.c_double()
check(lib.ipt_full_run_maps(ctx.handle, h, 3, C.byref(tot), C.byref(ker)))
print("ms per map", tot.value / 3)
