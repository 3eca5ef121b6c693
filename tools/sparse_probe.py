"""Time the sparse-Delta full map (SpMM + fused epilogue) against the dense DMMA map.

    python tools/sparse_probe.py [--n 32768] [--per-row 64] [--steps 5]

Prints one JSON line per variant: ms per map (whole sequence / SpMM kernel alone),
the algorithmic L2->SM gather bytes per map (nnz * ncols * 8) and Z's HBM bytes.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_14702_b200 as ipt  # noqa: E402
from paper_2012_14702_b200 import _lib  # noqa: E402
from paper_2012_14702_b200._lib import check, dptr, i32ptr, i64ptr  # noqa: E402


def build(n, per_row, seed=1):
    rng = np.random.default_rng(seed)
    cols = np.sort(rng.integers(0, n, (n, per_row)), axis=1).astype(np.int32)
    vals = 0.01 * rng.standard_normal((n, per_row))
    vals[cols == np.arange(n)[:, None]] = 0.0  # no diagonal entries (values only; pattern kept)
    rowptr = np.arange(0, n * per_row + 1, per_row, dtype=np.int64)
    d = np.arange(n, dtype=float)
    return d, rowptr, cols.ravel(), vals.ravel()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--per-row", type=int, default=64)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--dense", action="store_true", help="also time the dense map on the densified Delta")
    a = ap.parse_args()
    lib = _lib.load()
    ctx = ipt.default_context()
    d, rp, ci, va = build(a.n, a.per_row)
    h = C.c_void_p()
    check(lib.ipt_full_upload_csr(ctx.handle, a.n, dptr(d), None, i64ptr(rp), i32ptr(ci), dptr(va), None,
                                  C.byref(h)))
    check(lib.ipt_full_reset(ctx.handle, h, None, None))
    tot, ker = C.c_double(), C.c_double()
    check(lib.ipt_full_run_maps(ctx.handle, h, 2, C.byref(tot), C.byref(ker)))
    check(lib.ipt_full_run_maps(ctx.handle, h, a.steps, C.byref(tot), C.byref(ker)))
    nnz = int(rp[-1])
    gather = nnz * a.n * 8.0
    zbytes = 2.0 * a.n * a.n * 8.0  # read Z once + write F once
    ms_k = ker.value / a.steps
    print(json.dumps(dict(variant="sparse", n=a.n, nnz=nnz, ms_per_map=tot.value / a.steps, ms_spmm=ms_k,
                          gather_TBps=gather / (ms_k * 1e-3) / 1e12, z_hbm_TBps=zbytes / (ms_k * 1e-3) / 1e12,
                          vec=os.environ.get("IPT_SPMM_VEC", "4"))), flush=True)
    lib.ipt_full_free(h)
    if a.dense:
        dense = np.zeros((a.n, a.n))
        rows = np.repeat(np.arange(a.n), np.diff(rp))
        np.add.at(dense, (rows, ci), va)
        h2 = C.c_void_p()
        check(lib.ipt_full_upload(ctx.handle, a.n, dptr(d), None, dptr(dense), None, C.byref(h2)))
        check(lib.ipt_full_reset(ctx.handle, h2, None, None))
        check(lib.ipt_full_run_maps(ctx.handle, h2, 1, C.byref(tot), C.byref(ker)))
        check(lib.ipt_full_run_maps(ctx.handle, h2, 2, C.byref(tot), C.byref(ker)))
        print(json.dumps(dict(variant="dense", n=a.n, ms_per_map=tot.value / 2, ms_gemm=ker.value / 2)), flush=True)
        lib.ipt_full_free(h2)


if __name__ == "__main__":
    main()
