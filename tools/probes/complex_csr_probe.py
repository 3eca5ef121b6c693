"""Complex CSR single pair at config-5 size: per-step time of the complex path (Hermitian
Delta: real part of config 5 plus an antisymmetric imaginary part) vs the real fused map."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr, i32ptr, i64ptr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 21)
lib = ipt.load_library()
ctx = ipt.default_context()
p = synth.csr_ci(n, 32, 0.01, 42)
rp, ci, va = p.delta.row_offsets, p.delta.col_indices, p.delta.values
rows = np.repeat(np.arange(n), np.diff(rp))
vi = 0.003 * np.sign(ci - rows) * np.abs(va)  # antisymmetric imaginary part -> Hermitian
for name, im in (("real", None), ("complex", vi)):
    h = C.c_void_p()
    check(lib.ipt_single_upload_csr(ctx.handle, n, dptr(p.d), None, i64ptr(rp), i32ptr(ci), dptr(va),
                                    dptr(im) if im is not None else None, C.byref(h)))
    check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
    tot, dom = C.c_double(), C.c_double()
    check(lib.ipt_single_run_steps(ctx.handle, h, 3, C.byref(tot), C.byref(dom)))
    check(lib.ipt_single_run_steps(ctx.handle, h, 10, C.byref(tot), C.byref(dom)))
    lib.ipt_single_free(h)
    nnz = int(rp[-1])
    bytes_step = nnz * (4 + 8 * (2 if im is not None else 1)) + 8 * (n + 1)
    print(f"{name}: step {tot.value / 10:.3f} ms, {bytes_step / (tot.value / 10 * 1e-3) / 1e9:.0f} GB/s algorithmic",
          flush=True)
