"""Per-rank step time of the column-sharded full spectrum, measured on one B200: rank r of
g iterates columns [N r/g, N (r+1)/g) with Delta replicated, so its map step is exactly the
column-block map run here (ipt_full_upload_columns: the same kernels a rank launches).
The only cross-rank exchange per step is an all-reduce of four scalars, so this block time
is the multi-GPU step time up to that all-reduce (~tens of microseconds over NVLink).

    python tools/shard_probe.py [N] [product]     (product: dmma | ozaki)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib, synth  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
product = sys.argv[2] if len(sys.argv) > 2 else "dmma"
lib = _lib.load()
ctx = ipt.default_context()
p = synth.config3(n=n)
base = None
for g in (1, 2, 4, 8):
    worst = 0.0
    for r in ((0, g - 1) if g > 1 else (0,)):  # first and last block (the extremes of the split)
        c0, c1 = n * r // g, n * (r + 1) // g
        h = C.c_void_p()
        check(lib.ipt_full_upload_columns(ctx.handle, n, dptr(p.d), None, dptr(p.delta), None, c0, c1, C.byref(h)))
        check(lib.ipt_full_reset(ctx.handle, h, None, None))
        check(lib.ipt_full_set_product(h, 1 if product == "ozaki" else 0))
        tot, ker = C.c_double(), C.c_double()
        check(lib.ipt_full_run_maps(ctx.handle, h, 2, C.byref(tot), C.byref(ker)))
        steps = 3 if g <= 2 else 5
        check(lib.ipt_full_run_maps(ctx.handle, h, steps, C.byref(tot), C.byref(ker)))
        lib.ipt_full_free(h)
        worst = max(worst, tot.value / steps)
    base = base or worst
    print(json.dumps({"n": n, "product": product, "gpus": g, "rank_step_ms": worst,
                      "projected_TFs": 2.0 * n ** 3 / (worst * 1e-3) / 1e12,
                      "strong_scaling_efficiency_excl_allreduce": base / (g * worst)}), flush=True)
