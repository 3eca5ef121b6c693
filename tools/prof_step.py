"""Small driver for ncu captures: one workload, a few resident steps, nothing else.

    python tools/prof_step.py full  --n 8192  --steps 2
    python tools/prof_step.py gemv  --n 16384 --steps 2
    python tools/prof_step.py spmv  --n 2097152 --steps 2
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr, i32ptr, i64ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("what", choices=["full", "gemv", "spmv"])
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
a = ap.parse_args()
lib = ipt.load_library()
ctx = ipt.default_context(0)
h = C.c_void_p()
tot, dom = C.c_double(), C.c_double()
if a.what == "full":
    p = synth.config3(n=a.n)
    check(lib.ipt_full_upload(ctx.handle, a.n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
    check(lib.ipt_full_reset(ctx.handle, h, None, None))
    check(lib.ipt_full_run_maps(ctx.handle, h, a.warmup, C.byref(tot), C.byref(dom)))
    check(lib.ipt_full_run_maps(ctx.handle, h, a.steps, C.byref(tot), C.byref(dom)))
    flops = 2.0 * a.n ** 3
    print(f"full n={a.n}: step {tot.value / a.steps:.3f} ms, gemm {dom.value / a.steps:.3f} ms, "
          f"{flops / (dom.value / a.steps * 1e-3) / 1e12:.2f} TF/s")
else:
    if a.what == "gemv":
        p = synth.dense_normal(a.n)
        check(lib.ipt_single_upload_dense(ctx.handle, a.n, dptr(p.d), None, dptr(p.delta), None, C.byref(h)))
        nbytes = 8.0 * a.n * a.n
    else:
        p = synth.csr_ci(a.n)
        check(lib.ipt_single_upload_csr(ctx.handle, a.n, dptr(p.d), None, i64ptr(p.delta.row_offsets),
                                        i32ptr(p.delta.col_indices), dptr(p.delta.values), None, C.byref(h)))
        nbytes = 12.0 * p.delta.nnz + 8.0 * (a.n + 1)
    check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
    check(lib.ipt_single_run_steps(ctx.handle, h, a.warmup, C.byref(tot), C.byref(dom)))
    check(lib.ipt_single_run_steps(ctx.handle, h, a.steps, C.byref(tot), C.byref(dom)))
    ms = dom.value / a.steps
    print(f"{a.what} n={a.n}: step {tot.value / a.steps:.4f} ms, map kernel {ms:.4f} ms, "
          f"{(nbytes + 16.0 * a.n) / (ms * 1e-3) / 1e9:.0f} GB/s")
