"""The BASELINE configurations under IPT_GUARD=1 (guard zones around every device buffer,
checked at release): config 2 and 3 full spectrum (DMMA and Ozaki, K16 closing, CG
sigma_min), config 4 dense single pair (N = 65536), config 5 CSR single pair (N = 2^21)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402

assert os.environ.get("IPT_GUARD") == "1"
lib = ipt.load_library()
cfg = ipt.IterationConfig(tolerance=1e-12)
for n in (8192, 32768):
    p = synth.config3(n=n) if n == 32768 else synth.dense_uniform(n, 0.32 / np.sqrt(n), 42)
    g = ipt.build_gaps(p)
    for product in ("dmma", "ozaki"):
        t0 = time.time()
        r = ipt.solve_full(p, g, cfg, product=product)
        print(f"full n={n} {product}: {r.iterations} it, residual {r.residual_frobenius:.3e}, {time.time() - t0:.1f} s,"
              f" violations so far {lib.ipt_guard_violations()}", flush=True)
    del p, g
q = synth.config4()
s = ipt.solve_single(q, ipt.build_gaps(q), 0, cfg)
print(f"config 4 dense single n={q.size()}: {s.iterations} it, violations so far {lib.ipt_guard_violations()}", flush=True)
del q
q = synth.config5()
s = ipt.solve_single(q, ipt.build_gaps(q, 0.0), 0, ipt.IterationConfig(tolerance=1e-10))
print(f"config 5 csr single n={q.size()}: {s.iterations} it, violations so far {lib.ipt_guard_violations()}", flush=True)
import gc  # noqa: E402

gc.collect()
print(f"guard zones checked on {lib.ipt_guard_checked()} buffers, {lib.ipt_guard_violations()} violations")
