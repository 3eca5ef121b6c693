"""Full spectrum beyond BASELINE's sizes on one B200: N = 65536 (Delta 34 GB, Z ping-pong
69 GB; the reference would need ~270 GB of host memory and days), DMMA and Ozaki products."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
products = sys.argv[2].split(",") if len(sys.argv) > 2 else ["dmma", "ozaki"]
t0 = time.time()
p = synth.dense_uniform(n, 0.32 / np.sqrt(n), 42)
print(f"generate {time.time() - t0:.1f} s", flush=True)
g = ipt.build_gaps(p)
for product in products:
    t0 = time.time()
    r = ipt.solve_full(p, g, ipt.IterationConfig(tolerance=1e-12), product=product)
    ms = float(np.sqrt(np.sum(p.delta ** 2) + np.sum(p.d ** 2)))
    print(f"n {n} {product}: {time.time() - t0:.1f} s, {r.iterations} it, {r.status.name}, residual/|M|_F "
          f"{r.residual_frobenius / ms:.3e}, sigma_min {r.min_singular_value_estimate:.9f}, lambda0 "
          f"{r.eigenvalues[0]:.15f}, timings {r.timings_ms}", flush=True)
    del r
