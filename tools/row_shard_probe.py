"""Per-rank step of the row-sharded CSR single pair (config 5, N = 2^21), measured on one
B200: rank r of g maps rows [r c, (r+1) c), c = ceil(N/g) (ipt_single_upload_csr_rows: the
same kernels a rank launches, the fused peer stores aside). Per step a rank also sends its
c rows (8c bytes) to each peer over NVLink inside the map kernel and joins a four-scalar
all-reduce; those are not in this number.

    python tools/row_shard_probe.py
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib, synth  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr, i32ptr, i64ptr  # noqa: E402

lib = _lib.load()
ctx = ipt.default_context()
p = synth.config5()
n = p.size()
rp, ci, va = p.delta.row_offsets, p.delta.col_indices, p.delta.values
base = None
for g in (1, 2, 4, 8):
    chunk = -(-n // g)
    worst = 0.0
    for r in ((0, g - 1) if g > 1 else (0,)):
        b, e = r * chunk, min(n, (r + 1) * chunk)
        h = C.c_void_p()
        check(lib.ipt_single_upload_csr_rows(ctx.handle, n, dptr(p.d), None, i64ptr(rp), i32ptr(ci), dptr(va), None,
                                             b, e, C.byref(h)))
        check(lib.ipt_single_reset(ctx.handle, h, 0, None, None))
        tot, dom = C.c_double(), C.c_double()
        check(lib.ipt_single_run_steps(ctx.handle, h, 5, C.byref(tot), C.byref(dom)))
        check(lib.ipt_single_run_steps(ctx.handle, h, 20, C.byref(tot), C.byref(dom)))
        lib.ipt_single_free(h)
        worst = max(worst, tot.value / 20)
        kern = dom.value / 20
    base = base or worst
    print(json.dumps({"n": n, "gpus": g, "rank_step_ms": worst, "map_kernel_ms": kern,
                      "peer_store_bytes_per_rank": 8 * chunk * (g - 1),
                      "strong_scaling_efficiency_excl_exchange": base / (g * worst)}), flush=True)
