"""Closing residual of the column-sharded solve vs one rank, K16 and exact closing, per product."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import dist, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1536
p = synth.dense_uniform(n, 0.3 / np.sqrt(n), 7)
gaps = ipt.build_gaps(p)
cfg = ipt.IterationConfig(tolerance=1e-12)
for closing in ["k16", "exact"]:
    if closing == "exact":
        os.environ["IPT_CLOSING"] = "exact"
    for product in ["dmma", "ozaki"]:
        res = [ipt.solve_full(p, gaps, cfg, product=product).residual_frobenius]
        for g in (2, 3, 4, 8):
            ctxs = dist.local_contexts(g)
            outs = dist.run_ranks(lambda c: ipt.solve_full(p, gaps, cfg, ctx=c, product=product), ctxs)
            for c in ctxs:
                c.close()
            res.append(outs[0].residual_frobenius)
        print(f"n {n} closing {closing:5s} {product:5s} residual g=1,2,3,4,8: " + " ".join(f"{r:.6e}" for r in res),
              flush=True)
