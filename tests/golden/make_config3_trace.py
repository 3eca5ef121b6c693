"""Pin config 3's iteration count (N = 32768): the reference's solve_full loop body
(proj/src/solver.cpp:208-250) restated in numpy float64, run to convergence on the
full problem, recording the per-iteration relative-Frobenius step (solver.cpp:236) and
max |F - Z| (the BASELINE stop rule). TEST INFRASTRUCTURE ONLY (runs here, never on the
GPU box; the GPU test reads the committed tests/golden/config3_trace.npz).

Why a restatement and not the reference build: solve_full at N = 32768 needs ~120 GB
(complex carriers) and ~3.5 h per iteration on this host. The real-valued
restatement needs Delta + two Z buffers (26 GB) and OpenBLAS DGEMM (column blocks of
W = Delta Z), ~4 min per iteration on 8 cores. Its summation order differs from the
reference's k-ascending loop (kernels.cpp:23-47) by rounding only (~1e-16 relative in
each step value), so the iteration count is the reference's unless a step lands within
that distance of tol; the script records the margin |log10(step / tol)| at the decisive
iteration so the test can state it.

Inputs are drawn with the REFERENCE's own Rng (oracle/_ref, ref_rng_draws), in the draw
order of SURVEY §8(d): one stream Rng(stream_seed(42, 0)); upper triangle row-major;
Delta_ij = Delta_ji = eps (2u - 1), eps = 0.32 / sqrt(N); d_i = i + 1.

    nice python tests/golden/make_config3_trace.py            # N = 32768 (~30 min)
    python tests/golden/make_config3_trace.py --n 2048        # quick self-check
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def config_delta(n: int, seed: int = 42) -> np.ndarray:
    eps = 0.32 / math.sqrt(n)
    u = oracle.ref().rng_draws(seed, 1, n * (n - 1) // 2, stream=0)
    u *= 2.0
    u -= 1.0
    u *= eps
    delta = np.zeros((n, n))
    off = 0
    for i in range(n - 1):
        m = n - 1 - i
        delta[i, i + 1:] = u[off:off + m]
        off += m
    del u
    # mirror the upper triangle in row blocks (Delta_ji = Delta_ij)
    bs = 1024
    lower = np.tril_indices(bs, -1)
    for r0 in range(0, n, bs):
        r1 = min(n, r0 + bs)
        # off-diagonal blocks: rows r0:r1, columns < r0
        if r0 > 0:
            delta[r0:r1, :r0] = delta[:r0, r0:r1].T
        # diagonal block: strictly lower part from the strictly upper part
        blk = delta[r0:r1, r0:r1]
        li = lower if r1 - r0 == bs else np.tril_indices(r1 - r0, -1)
        blk[li] = blk.T[li]
    return delta


def run(n: int, tol: float, max_iter: int, block: int):
    d = np.arange(1, n + 1, dtype=np.float64)
    t0 = time.time()
    delta = config_delta(n)
    assert np.array_equal(delta, delta.T)
    print(f"n={n}: Delta generated in {time.time() - t0:.1f} s", flush=True)
    # ZT[j, :] = column j of Z (C-contiguous column blocks)
    zt = np.eye(n)
    ft = np.empty((n, n))
    steps, maxabs, new_norms = [], [], []
    for k in range(max_iter):
        t1 = time.time()
        diff2 = cur2 = new2 = 0.0
        mx = 0.0
        for c0 in range(0, n, block):
            c1 = min(n, c0 + block)
            zb = zt[c0:c1]                       # (nb, n): columns c0..c1 of Z
            wt = zb @ delta                      # (nb, n): W[:, j]^T = (Delta Z)[:, j]^T (Delta symmetric)
            js = np.arange(c0, c1)
            wd = wt[js - c0, js]                 # (Delta Z)_jj  (solver.cpp:211)
            gap = d[None, :] - d[js, None]       # d_i - d_j
            gap[js - c0, js] = 1.0
            fb = (zb * wd[:, None] - wt) / gap   # solver.cpp:220
            fb[js - c0, js] = 1.0
            dz = fb - zb
            diff2 += float(np.sum(dz * dz))
            cur2 += float(np.sum(zb * zb))
            new2 += float(np.sum(fb * fb))
            mx = max(mx, float(np.max(np.abs(dz))))
            ft[c0:c1] = fb
        step = math.sqrt(diff2) / math.sqrt(cur2)
        steps.append(step)
        maxabs.append(mx)
        new_norms.append(math.sqrt(new2))
        zt, ft = ft, zt
        print(f"iter {k + 1}: step {step:.6e} max_abs {mx:.6e} ({time.time() - t1:.1f} s)", flush=True)
        if step <= tol and mx < tol:
            break
    steps, maxabs = np.array(steps), np.array(maxabs)
    it_fro = int(np.argmax(steps <= tol)) + 1
    it_max = int(np.argmax(maxabs < tol)) + 1
    return dict(n=n, tol=tol, steps=steps, max_abs=maxabs, new_norm=np.array(new_norms),
                iterations_rel_fro=it_fro, iterations_max_abs=it_max,
                margin_rel_fro=np.array([math.log10(steps[it_fro - 1] / tol)] +
                                        ([math.log10(steps[it_fro - 2] / tol)] if it_fro > 1 else [])),
                margin_max_abs=np.array([math.log10(maxabs[it_max - 1] / tol)] +
                                        ([math.log10(maxabs[it_max - 2] / tol)] if it_max > 1 else [])),
                source=np.array("solver.cpp:208-250 restated in numpy float64 (OpenBLAS DGEMM), reference Rng inputs"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--tol", type=float, default=1e-12)
    ap.add_argument("--max-iter", type=int, default=12)
    ap.add_argument("--block", type=int, default=2048)
    a = ap.parse_args()
    res = run(a.n, a.tol, a.max_iter, a.block)
    print({k: v for k, v in res.items() if k not in ("steps", "max_abs", "new_norm")}, flush=True)
    if a.n == 32768:
        path = os.path.join(OUT, "config3_trace.npz")
        np.savez_compressed(path, **res)
        print(f"wrote {path}", flush=True)


if __name__ == "__main__":
    main()
