"""Seeded synthetic inputs of BASELINE.json's configurations (include/ipt_synth.h).

Draw orders are fixed by SURVEY.md §8(d) so the device path, the CPU oracle and
the reference build see bit-identical inputs (the generator is the reference's
xoshiro256++ / splitmix64 / Box-Muller stream, proj/include/ipt/rng.hpp).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from ._lib import dptr, i32ptr, i64ptr
from .ipt import CsrMatrix, Partition

SEED = 42


def dense_uniform(n: int, eps: float, seed: int = SEED) -> Partition:
    """Configs 1-3: d = 1..n; Delta symmetric zero-diagonal, eps*uniform[-1,1]."""
    d = np.empty(n)
    delta = np.empty((n, n))
    rc = _lib.load().ipt_synth_dense_uniform(n, float(eps), seed, dptr(d), dptr(delta))
    if rc != 0:
        raise RuntimeError(f"ipt_synth_dense_uniform failed ({rc})")
    return Partition(d, delta)


def config1(seed: int = SEED) -> Partition:
    return dense_uniform(1024, 0.01, seed)


def eps_for(n: int) -> float:
    """eps = 0.32/sqrt(N) keeps |eps Delta|_2 ~ 0.37 below the unit gap (configs 2-3)."""
    return 0.32 / math.sqrt(n)


def config2(seed: int = SEED) -> Partition:
    return dense_uniform(8192, eps_for(8192), seed)


def config3(seed: int = SEED, n: int = 32768) -> Partition:
    return dense_uniform(n, eps_for(n), seed)


def dense_normal(n: int, sigma: float | None = None, seed: int = SEED, threads: int = 0) -> Partition:
    """Config 4: d = sort(n u) + i, Delta symmetric zero-diagonal N(0, sigma^2), sigma = 0.3/sqrt(n)."""
    sigma = 0.3 / math.sqrt(n) if sigma is None else sigma
    d = np.empty(n)
    delta = np.empty((n, n))
    rc = _lib.load().ipt_synth_dense_normal(n, float(sigma), seed, int(threads), dptr(d), dptr(delta))
    if rc != 0:
        raise RuntimeError(f"ipt_synth_dense_normal failed ({rc})")
    return Partition(d, delta)


def config4(seed: int = SEED, n: int = 65536) -> Partition:
    return dense_normal(n, None, seed)


def csr_ci(n: int = 1 << 21, per_row: int = 32, sigma: float = 0.01, seed: int = SEED) -> Partition:
    """Config 5: CI-like symmetric CSR, ~2*per_row nonzeros per row, no diagonal."""
    lib = _lib.load()
    h = C.c_void_p()
    nnz = C.c_int64()
    rc = lib.ipt_synth_csr_ci_plan(n, int(per_row), seed, C.byref(h), C.byref(nnz))
    if rc != 0:
        raise RuntimeError(f"ipt_synth_csr_ci_plan failed ({rc})")
    d = np.empty(n)
    rowptr = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(nnz.value, dtype=np.int32)
    vals = np.empty(nnz.value)
    rc = lib.ipt_synth_csr_ci_fill(h, float(sigma), dptr(d), i64ptr(rowptr), i32ptr(cols), dptr(vals))
    if rc != 0:
        raise RuntimeError(f"ipt_synth_csr_ci_fill failed ({rc})")
    return Partition(d, CsrMatrix(n, n, rowptr, cols, vals))


def config5(seed: int = SEED, n: int = 1 << 21) -> Partition:
    return csr_ci(n, 32, 0.01, seed)


def rng_draws(seed: int, kind: int, count: int, stream: int | None = None, bound: int = 0) -> np.ndarray:
    """Raw generator draws (kind 0 next, 1 uniform, 2 normal, 3 below(bound))."""
    out = np.empty(count, dtype=np.uint64 if kind in (0, 3) else np.float64)
    _lib.load().ipt_synth_rng_draws(seed, 0 if stream is None else stream, 0 if stream is None else 1,
                                    kind, bound, count, out.ctypes.data_as(C.c_void_p))
    return out
