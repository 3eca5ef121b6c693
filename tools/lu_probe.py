"""Device LU (factor + n-RHS solve) vs the reference's serial lu.cpp, complex n x n.

    python tools/lu_probe.py 1024 2048 4096
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402

ns = [int(a) for a in sys.argv[1:]] or [1024, 2048]
ipt.lu_factor(np.eye(8) * 2.0)  # context + module load
for n in ns:
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    t0 = time.perf_counter()
    f = ipt.lu_factor(a)
    t1 = time.perf_counter()
    x = ipt.lu_solve_matrix(f, b)
    t2 = time.perf_counter()
    res = float(np.max(np.abs(a @ x - b)) / np.max(np.abs(b)))
    out = dict(n=n, factor_s=t1 - t0, solve_matrix_s=t2 - t1, rel_residual=res)
    if n <= 1024 and os.environ.get("LU_REF"):
        import oracle

        R = oracle.ref()
        t0 = time.perf_counter()
        R.lu_factor(a)
        t1 = time.perf_counter()
        R.lu_solve(a, b)  # factor + solve
        t2 = time.perf_counter()
        out.update(ref_factor_s=t1 - t0, ref_factor_plus_solve_s=t2 - t1)
    print(json.dumps(out), flush=True)
