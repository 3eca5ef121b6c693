"""Soak: repeated solves in one process -- results bitwise stable, device memory flat
(the stream-ordered pool keeps freed blocks mapped, so 'used' must plateau, not grow)."""
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import synth  # noqa: E402


def used_mib():
    out = subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout
    return int(out.split()[0])


cfg = ipt.IterationConfig(tolerance=1e-12)
p2 = synth.dense_uniform(8192, 0.32 / np.sqrt(8192), 42)
g2 = ipt.build_gaps(p2)
q5 = synth.config5()
g5 = ipt.build_gaps(q5, 0.0)
ref2 = ref5 = None
mem = []
t0 = time.time()
for rep in range(40):
    r = ipt.solve_full(p2, g2, cfg, product="ozaki" if rep % 4 == 3 else "dmma")
    s = ipt.solve_single(q5, g5, rep % 7, ipt.IterationConfig(tolerance=1e-10))
    z = ipt.kernels.matvec(q5.delta, np.ones(q5.size()))
    if rep % 4 != 3:
        if ref2 is None:
            ref2 = r.Z.copy()
        assert np.array_equal(r.Z, ref2), rep
    if rep % 7 == 0:
        if ref5 is None:
            ref5 = s.z.copy()
        assert np.array_equal(s.z, ref5), rep
    mem.append(used_mib())
print(f"40 rounds of (config-2 solve, config-5 solve, config-5 matvec) in {time.time() - t0:.1f} s; "
      f"device memory used (MiB) after rounds 1, 10, 20, 30, 40: {mem[0]}, {mem[9]}, {mem[19]}, {mem[29]}, {mem[39]}; "
      f"results bitwise stable", flush=True)
assert mem[39] <= mem[9] + 512, "device memory grows across rounds"
