"""Time sigma_min (SYRK + blocked Cholesky + inverse iteration) on a near-identity Z.

    IPT_PROFILE=1 python tools/probes/sigma_probe.py 8192 32768
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [8192]:
    rng = np.random.default_rng(n)
    z = np.eye(n) + (1e-3 / np.sqrt(n)) * rng.standard_normal((n, n))
    ipt.smallest_singular_value_estimate(z)
    t = time.perf_counter()
    s = ipt.smallest_singular_value_estimate(z)
    print(f"n={n} sigma_min={s!r} wall {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
