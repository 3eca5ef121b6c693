"""Where config 5's drop-in solve time goes (IPT_PROFILE phase marks of the C ABI on
stderr): the CSR single pair through ipt.solve_single with host buffers, three calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402

p = synth.config5()
g = ipt.build_gaps(p, 0.0)
cfg = ipt.IterationConfig(tolerance=1e-10)
for rep in range(3):
    t0 = time.perf_counter()
    r = ipt.solve_single(p, g, 0, cfg)
    print(f"rep {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms, {r.iterations} it, "
          f"loop {r.timings_ms.get('loop', 0):.2f} ms", flush=True)
