import time, sys, os
sys.path.insert(0, os.getcwd())
import paper_2012_14702_b200 as ipt
from paper_2012_14702_b200 import synth
p = synth.dense_uniform(1024, 0.01, 42)
g = ipt.build_gaps(p)
for rep in range(4):
    t0 = time.perf_counter(); r = ipt.solve_full(p, g, ipt.IterationConfig(tolerance=1e-12)); t1 = time.perf_counter()
    print(rep, f"{1e3*(t1-t0):.2f} ms", r.iterations, r.timings_ms, flush=True)
