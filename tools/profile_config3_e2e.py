"""Where config 3's drop-in solve time goes (IPT_PROFILE phase marks on stderr): the N = 32768
full-spectrum solve through ipt.solve_full with host buffers, twice (the second is warm)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
product = sys.argv[2] if len(sys.argv) > 2 else "dmma"
p = synth.config3(n=n)
g = ipt.build_gaps(p)
cfg = ipt.IterationConfig(tolerance=1e-12)
for rep in range(2):
    t0 = time.perf_counter()
    r = ipt.solve_full(p, g, cfg, product=product)
    print(f"rep {rep}: {time.perf_counter() - t0:.3f} s, {r.iterations} it, residual {r.residual_frobenius:.4e}, "
          f"timings {r.timings_ms}", flush=True)
