"""Config 2 (N = 8192) full spectrum: the reference build's own solve_full (OpenMP, the box's
host cores) against the device solve on the same inputs -- every eigenpair, not a column
sample. One-off evidence run (~25 min of CPU), not a test:
    python tools/ref_full_config2.py [n]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
p = synth.dense_uniform(n, 0.32 / np.sqrt(n), 42)
g = ipt.build_gaps(p)
t0 = time.time()
r = ipt.solve_full(p, g, ipt.IterationConfig(tolerance=1e-12))
t_dev = time.time() - t0
print(f"device: {t_dev:.3f} s, {r.iterations} it, residual {r.residual_frobenius:.4e}, "
      f"sigma_min {r.min_singular_value_estimate:.12f}", flush=True)
ref = oracle.ref()
t0 = time.time()
o = ref.solve_full(p.d, p.delta, tol=1e-12)
t_ref = time.time() - t0
print(f"reference (proj/src/solver.cpp, {os.cpu_count()} host cores): {t_ref:.1f} s, {o['iterations']} it, "
      f"residual {o['residual_frobenius']:.4e}, sigma_min {o['sigma_min']:.12f}", flush=True)
dz = float(np.max(np.abs(r.Z - o["Z"])))
lam = o["eigenvalues"]
dl = float(np.max(np.abs(r.eigenvalues - lam) / np.abs(lam)))
ms = float(np.sqrt(np.sum(p.delta ** 2) + np.sum(p.d ** 2)))
print(f"n {n}: iterations {r.iterations} vs {o['iterations']}; max |Z - Z_ref| {dz:.3e} (tol 1e-9); "
      f"max rel |Lambda - Lambda_ref| {dl:.3e} (tol 1e-10); residual / |M|_F {r.residual_frobenius / ms:.3e} "
      f"(ref {o['residual_frobenius'] / ms:.3e}, tol 1e-10); sigma_min rel diff "
      f"{abs(r.min_singular_value_estimate - o['sigma_min']) / o['sigma_min']:.3e}; speed-up {t_ref / t_dev:.0f}x",
      flush=True)
