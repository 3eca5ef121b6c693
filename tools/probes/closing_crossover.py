"""Closing step time, K16 (last map + INT8 correction) vs the FP64 closing product, by N."""
import os
import subprocess
import sys

code = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import synth
for n in (1024, 1536, 2048, 3072, 4096, 6144, 8192):
    p = synth.dense_uniform(n, 0.32 / np.sqrt(n), 42)
    g = ipt.build_gaps(p)
    best = 1e9
    for rep in range(4):
        r = ipt.solve_full(p, g, ipt.IterationConfig(tolerance=1e-12))
        best = min(best, r.timings_ms["final"])
    print(n, round(best, 3), flush=True)
'''
for mode in ("k16", "exact"):
    env = dict(os.environ)
    if mode == "exact":
        env["IPT_CLOSING"] = "exact"
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stdout
    print(mode, out.replace("\n", " | "), flush=True)
