"""CSR single-pair step on skewed row lengths (CI-like Hamiltonians have a few very dense
rows): per-nonzero time vs the uniform config-5 pattern at the same nnz."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr, i32ptr, i64ptr  # noqa: E402

lib = ipt.load_library()
ctx = ipt.default_context()
n = 1 << 21
rng = np.random.default_rng(7)


def step_ms(d, rp, ci, va):
    h = C.c_void_p()
    check(lib.ipt_single_upload_csr(ctx.handle, n, dptr(d), None, i64ptr(rp), i32ptr(ci), dptr(va), None, C.byref(h)))
    check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
    tot, dom = C.c_double(), C.c_double()
    check(lib.ipt_single_run_steps(ctx.handle, h, 3, C.byref(tot), C.byref(dom)))
    check(lib.ipt_single_run_steps(ctx.handle, h, 10, C.byref(tot), C.byref(dom)))
    lib.ipt_single_free(h)
    return tot.value / 10


p = synth.config5()
nnz = int(p.delta.row_offsets[-1])
t = step_ms(p.d, p.delta.row_offsets, p.delta.col_indices, p.delta.values)
print(f"uniform (config 5): nnz {nnz}, step {t:.3f} ms, {t / nnz * 1e9:.3f} ps/nnz", flush=True)
for label, lengths in (
    ("lognormal", np.minimum(np.maximum(rng.lognormal(3.4, 1.0, n).astype(np.int64), 1), 20000)),
    ("heavy rows", np.where(rng.random(n) < 0.002, 8000, 48).astype(np.int64)),
    ("clustered heavy", np.where((np.arange(n) // 4096) % 64 == 0, 900, 36).astype(np.int64)),
):
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(lengths)
    m = int(rp[-1])
    ci = rng.integers(0, n, m, dtype=np.int64).astype(np.int32)
    # sorted columns per row are not needed for the timing; values small (no divergence matter)
    va = rng.standard_normal(m) * 1e-4
    t = step_ms(p.d, rp, ci, va)
    print(f"{label}: nnz {m}, max row {int(lengths.max())}, step {t:.3f} ms, {t / m * 1e9:.3f} ps/nnz", flush=True)
