"""Ozaki solve result for A/B comparison of two library builds (IPT_B200_LIB selects one).

    IPT_B200_LIB=... python tools/probes/oz_bitwise.py out.npz [n]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402

n = int(sys.argv[2]) if len(sys.argv) > 2 else 3001
p = synth.config3(n=n)
g = ipt.build_gaps(p)
r = ipt.solve_full(p, g, want_sigma_min=False, product="ozaki")
if sys.argv[1] != "-":
    np.savez(sys.argv[1], Z=r.Z, lam=r.eigenvalues, it=r.iterations, res=r.residual_frobenius)
print(n, r.iterations, r.residual_frobenius, r.status)
import hashlib  # noqa: E402
print("sha Z", hashlib.sha256(np.ascontiguousarray(r.Z).tobytes()).hexdigest()[:16],
      "sha lam", hashlib.sha256(np.ascontiguousarray(r.eigenvalues).tobytes()).hexdigest()[:16])
