"""Config 5 single-pair CSR step timing for the K8 variant in IPT_SPMV_VARIANT.

    for v in 3 5 6 7 8; do IPT_SPMV_VARIANT=$v python tools/spmv_probe.py; done
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib, synth  # noqa: E402
from paper_2012_14702_b200._lib import Stats, check, dptr, i32ptr, i64ptr  # noqa: E402
from paper_2012_14702_b200.ipt import _params  # noqa: E402

lib = _lib.load()
ctx = ipt.default_context()
p = synth.config5()
n = p.size()
h = C.c_void_p()
check(lib.ipt_single_upload_csr(ctx.handle, n, dptr(p.d), None, i64ptr(p.delta.row_offsets),
                                i32ptr(p.delta.col_indices), dptr(p.delta.values), None, C.byref(h)))
check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
prm = _params(ipt.IterationConfig(tolerance=1e-10))
st = Stats()
check(lib.ipt_single_iterate(ctx.handle, h, C.byref(prm), C.byref(st)))
check(lib.ipt_single_finalize(ctx.handle, h, C.byref(st)))
solve = dict(iterations=st.iterations, eigenvalue=repr(st.eigenvalue_re), residual=st.residual)
check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
tot, dom = C.c_double(), C.c_double()
check(lib.ipt_single_run_steps(ctx.handle, h, 5, C.byref(tot), C.byref(dom)))
check(lib.ipt_single_run_steps(ctx.handle, h, 20, C.byref(tot), C.byref(dom)))
print(json.dumps(dict(variant=os.environ.get("IPT_SPMV_VARIANT", "default"),
                      ms_step=tot.value / 20,
                      ms_kernel=dom.value / 20, **solve)), flush=True)
