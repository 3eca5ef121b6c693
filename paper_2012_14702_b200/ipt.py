"""Python host mirror of the reference's solver API (proj/include/ipt/*.hpp).

Same names, argument meaning and error behaviour as the C++ library, backed by
the B200 kernels through the C ABI (include/ipt_cuda.h). Matrices are numpy
arrays (dense, row-major as ComplexMatrix stores them, complex_matrix.hpp:48) or
`CsrMatrix`. Real inputs run the real fp64 fast path and return real arrays;
complex inputs return complex128.

Reference map:
  IterationConfig / SolveStatus / results ... solver.hpp:10-52
  partition / InverseGaps / build_gaps ...... partition.hpp:15-52, partition.cpp:16-94
  apply_map_single / solve_single ........... solver.cpp:122-136 (run_single :49-93)
  apply_map_full / solve_full ............... solver.cpp:156-273
  solve_single_continuation ................. solver.cpp:138-154
  smallest_singular_value_estimate .......... solver.cpp:275-297
  kernels.matmul / kernels.matvec ........... kernels.cpp:112-181
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import sys
import threading
import time
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _lib
from ._lib import check, dptr, i32ptr, i64ptr

EPS = sys.float_info.epsilon


class SolveStatus(enum.IntEnum):
    Converged = 0
    MaxIterations = 1
    Diverged = 2


def to_string(s: SolveStatus) -> str:
    return {0: "converged", 1: "max_iterations", 2: "diverged"}.get(int(s), "unknown")


@dataclass
class IterationConfig:
    tolerance: float = 100.0 * EPS
    max_iterations: int = 1000
    divergence_threshold: float = 1e8
    record_trace: bool = False
    residual_tolerance: float = 1e-8
    # B200 extension: "rel_fro" (reference, solver.cpp:236) or "max_abs" (BASELINE.json configs)
    stop_rule: str = "rel_fro"


def _validate(cfg: IterationConfig) -> None:  # solver.cpp:18-23
    if not (cfg.tolerance > 0.0):
        raise ValueError("config: tolerance must be positive")
    if cfg.max_iterations <= 0:
        raise ValueError("config: max_iterations must be positive")
    if not (cfg.divergence_threshold > 1.0):
        raise ValueError("config: divergence_threshold must exceed 1")


def _params(cfg: IterationConfig, **kw) -> _lib.Params:
    p = _lib.default_params()
    p.tolerance = cfg.tolerance
    p.max_iterations = cfg.max_iterations
    p.divergence_threshold = cfg.divergence_threshold
    p.record_trace = 1 if cfg.record_trace else 0
    p.stop_rule = _lib.STOP_MAX_ABS if cfg.stop_rule == "max_abs" else _lib.STOP_REL_FRO
    for k, v in kw.items():
        setattr(p, k, v)
    return p


# ----------------------------------------------------------------- matrices


class CsrMatrix:
    """Compressed sparse rows (complex_matrix.hpp:23-76): sorted columns, no
    explicit zeros, duplicates rejected. Indices are int64 offsets / int32 columns
    (the device layout); values float64 or complex128."""

    def __init__(self, n_rows: int, n_cols: int, row_offsets, col_indices, values):
        self.shape = (int(n_rows), int(n_cols))
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.int32)
        self.values = np.ascontiguousarray(values)
        if self.row_offsets.shape != (n_rows + 1,):
            raise ValueError("csr: row_offsets must have n_rows + 1 entries")
        if self.col_indices.shape != self.values.shape:
            raise ValueError("csr: column and value counts differ")

    @staticmethod
    def from_triplets(n_rows: int, n_cols: int, rows, cols, values) -> "CsrMatrix":
        """sparse_from_triplets (complex_matrix.cpp:39-69)."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        values = np.asarray(values)
        if rows.size and (rows.min() < 0 or rows.max() >= n_rows or cols.min() < 0 or cols.max() >= n_cols):
            raise ValueError("sparse_from_triplets: index out of bounds")
        order = np.lexsort((cols, rows))
        rows, cols, values = rows[order], cols[order], values[order]
        if rows.size > 1 and np.any((rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])):
            raise ValueError("sparse_from_triplets: duplicate entry")
        keep = values != 0
        rows, cols, values = rows[keep], cols[keep], values[keep]
        off = np.zeros(n_rows + 1, dtype=np.int64)
        np.add.at(off, rows + 1, 1)
        return CsrMatrix(n_rows, n_cols, np.cumsum(off), cols.astype(np.int32), values)

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.shape, dtype=self.values.dtype)
        r = np.repeat(np.arange(self.shape[0]), np.diff(self.row_offsets))
        out[r, self.col_indices] = self.values
        return out

    def is_complex(self) -> bool:
        return np.iscomplexobj(self.values) and bool(np.any(self.values.imag != 0))


Matrix = Union[np.ndarray, CsrMatrix]


@dataclass
class Partition:
    """M = diag(d) + delta (partition.hpp:15-20)."""

    d: np.ndarray
    delta: Matrix

    def size(self) -> int:
        return int(np.asarray(self.d).shape[0])


class DegenerateDiagonal(RuntimeError):
    """partition.hpp:22-26: two diagonal entries closer than the tolerance."""

    def __init__(self, i: int, j: int, gap: float, tol: float):
        super().__init__(f"degenerate diagonal: |d[{i}] - d[{j}]| = {gap:.6f} <= tolerance {tol:.6f}")
        self.i, self.j, self.gap, self.tol = i, j, gap, tol


class InverseGaps:
    """G_jk = 1/(d_j - d_k), zero diagonal, generated on demand (partition.hpp:33-52).
    Construction sweeps the real-part-sorted diagonal for pairs within the
    tolerance (partition.cpp:54-75); on the device G is never stored."""

    def __init__(self, d, degeneracy_tol: float):
        self._d = np.asarray(d)
        self._tol = float(degeneracy_tol)
        dc = self._d.astype(np.complex128)
        order = np.lexsort((dc.imag, dc.real))
        re = dc.real[order]
        n = dc.shape[0]
        for a in range(n):
            b = a + 1
            while b < n and re[b] - re[a] <= self._tol:
                gap = abs(dc[order[a]] - dc[order[b]])
                if gap <= self._tol:
                    i, j = sorted((int(order[a]), int(order[b])))
                    raise DegenerateDiagonal(i, j, gap, self._tol)
                b += 1

    def size(self) -> int:
        return int(self._d.shape[0])

    def diagonal(self) -> np.ndarray:
        return self._d

    def degeneracy_tolerance(self) -> float:
        return self._tol

    def entry(self, j: int, k: int):
        return 0.0 if j == k else 1.0 / (self._d[j] - self._d[k])

    def column(self, i: int) -> np.ndarray:
        with np.errstate(divide="ignore"):
            g = 1.0 / (self._d - self._d[i])
        g[i] = 0.0
        return g

    def to_matrix(self) -> np.ndarray:
        d = self._d
        with np.errstate(divide="ignore"):
            g = 1.0 / (d[:, None] - d[None, :])
        np.fill_diagonal(g, 0.0)
        return g


def partition(m: Matrix) -> Partition:
    """partition.cpp:16-46."""
    if isinstance(m, CsrMatrix):
        n = m.shape[0]
        if m.shape[0] != m.shape[1]:
            raise ValueError("partition: matrix must be square")
        rows = np.repeat(np.arange(n), np.diff(m.row_offsets))
        diag = rows == m.col_indices
        d = np.zeros(n, dtype=m.values.dtype)
        d[rows[diag]] = m.values[diag]
        off = ~diag
        return Partition(d, CsrMatrix.from_triplets(n, n, rows[off], m.col_indices[off], m.values[off]))
    m = np.asarray(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ValueError("partition: matrix must be square")
    delta = np.array(m, copy=True)
    d = np.diag(m).copy()
    np.fill_diagonal(delta, 0)
    return Partition(d, delta)


def reconstruct(p: Partition) -> np.ndarray:
    m = p.delta.to_dense() if isinstance(p.delta, CsrMatrix) else np.array(p.delta, copy=True)
    m = m.astype(np.result_type(m.dtype, np.asarray(p.d).dtype))
    m[np.diag_indices(p.size())] += p.d
    return m


def build_gaps(p: Partition, degeneracy_tol: float = -1.0) -> InverseGaps:
    """partition.cpp:91-94: a negative tolerance selects 1e-12 * max|d|."""
    if degeneracy_tol < 0.0:
        degeneracy_tol = 1e-12 * (float(np.max(np.abs(p.d))) if p.size() else 0.0)
    return InverseGaps(p.d, degeneracy_tol)


# ----------------------------------------------------------------- results


@dataclass
class EigenpairResult:
    z: np.ndarray = None
    eigenvalue: complex = 0.0
    anchor: int = 0
    iterations: int = 0
    final_step: float = 0.0
    residual: float = 0.0
    status: SolveStatus = SolveStatus.MaxIterations
    trace: list = field(default_factory=list)
    matvec_count: int = 0
    timings_ms: dict = field(default_factory=dict)


@dataclass
class SpectrumResult:
    Z: np.ndarray = None
    eigenvalues: np.ndarray = None
    iterations: int = 0
    final_step: float = 0.0
    residual_frobenius: float = 0.0
    min_singular_value_estimate: float = 0.0
    status: SolveStatus = SolveStatus.MaxIterations
    trace: list = field(default_factory=list)
    matmul_count: int = 0
    final_max_abs: float = 0.0
    trace_max_abs: list = field(default_factory=list)
    timings_ms: dict = field(default_factory=dict)


# ----------------------------------------------------------------- device context


class Context:
    """One CUDA device + stream (+ optional NCCL communicator) of the C ABI."""

    def __init__(self, device: int = 0):
        lib = _lib.load()
        h = C.c_void_p()
        check(lib.ipt_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device
        self.rank, self.nranks = 0, 1

    def init_comm(self, unique_id: bytes, rank: int, nranks: int) -> None:
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(_lib.load().ipt_ctx_init_comm(self.handle, buf, int(rank), int(nranks)))
        self.rank, self.nranks = rank, nranks

    def init_local_comm(self, group: "LocalGroup", rank: int) -> None:
        """Join an in-process group as `rank` (ipt_ctx_init_local_comm)."""
        check(_lib.load().ipt_ctx_init_local_comm(self.handle, group.handle, int(rank)))
        self.rank, self.nranks = rank, group.nranks
        self._group = group  # the group outlives its member contexts

    @property
    def comm_kind(self) -> str:
        return _lib.load().ipt_ctx_comm_kind(self.handle).decode()

    def synchronize(self) -> None:
        check(_lib.load().ipt_ctx_synchronize(self.handle))

    def close(self) -> None:
        if self.handle:
            _lib.load().ipt_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalGroup:
    """In-process communicator group (ipt_local_group_create): nranks contexts of this
    process, one host thread per rank, on one GPU or several (include/ipt_cuda.h)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        check(_lib.load().ipt_local_group_create(int(nranks), C.byref(h)))
        self.handle = h
        self.nranks = nranks

    def __del__(self):
        try:
            if self.handle:
                _lib.load().ipt_local_group_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(_lib.load().ipt_nccl_get_unique_id(buf))
    return buf.raw


# ----------------------------------------------------------------- helpers


def _planar(a, n_expected=None):
    """(re, im|None) contiguous float64 planes of a real or complex array."""
    a = np.asarray(a)
    if np.iscomplexobj(a):
        re = np.ascontiguousarray(a.real, dtype=np.float64)
        im = np.ascontiguousarray(a.imag, dtype=np.float64)
        return re, (im if np.any(im != 0) else None)
    return np.ascontiguousarray(a, dtype=np.float64), None


def _combine(re, im, cplx: bool):
    return re + 1j * im if cplx else re


def _check_sizes(p: Partition, g: InverseGaps, anchor: int = 0) -> None:  # solver.cpp:25-30
    n = p.size()
    if n != g.size():
        raise ValueError("solver: partition/gaps size mismatch")
    shape = p.delta.shape
    if shape != (n, n):
        raise ValueError("solver: residual must be square of matching size")
    if anchor < 0 or anchor >= n:
        raise ValueError("solver: anchor out of range")


def _is_complex_problem(p: Partition, extra=None) -> bool:
    cx = np.iscomplexobj(p.d) and bool(np.any(np.asarray(p.d).imag != 0))
    if isinstance(p.delta, CsrMatrix):
        cx = cx or p.delta.is_complex()
    else:
        cx = cx or (np.iscomplexobj(p.delta) and bool(np.any(np.asarray(p.delta).imag != 0)))
    if extra is not None:
        cx = cx or (np.iscomplexobj(extra) and bool(np.any(np.asarray(extra).imag != 0)))
    return cx


def _out_complex(p: Partition, extra=None) -> bool:
    """Complex result if any input carries a complex dtype (as the reference always does)."""
    return (np.iscomplexobj(p.d) or np.iscomplexobj(getattr(p.delta, "values", p.delta))
            or (extra is not None and np.iscomplexobj(extra)))


# ----------------------------------------------------------------- full spectrum


def apply_map_full(p: Partition, g: InverseGaps, Z, ctx: Optional[Context] = None) -> np.ndarray:
    """F(Z) = I + G o (Z D(Delta Z) - Delta Z), one product (solver.cpp:156-178)."""
    _check_sizes(p, g, 0)
    n = p.size()
    Z = np.asarray(Z)
    if Z.shape != (n, n):
        raise ValueError("apply_map_full: size mismatch")
    ctx = ctx or default_context()
    dr, di = _planar(p.d)
    zr, zi = _planar(Z)
    cx = _out_complex(p, Z)
    fr = np.empty((n, n))
    fi = np.empty((n, n)) if cx else None
    lib = _lib.load()
    if isinstance(p.delta, CsrMatrix):  # kernels.cpp:88-108 (SpMM) on the device
        vr, vi = _planar(p.delta.values)
        check(lib.ipt_apply_map_full_csr(ctx.handle, n, dptr(dr), dptr(di), i64ptr(p.delta.row_offsets),
                                         i32ptr(p.delta.col_indices), dptr(vr), dptr(vi), dptr(zr), dptr(zi),
                                         dptr(fr), dptr(fi)))
    else:
        ar, ai = _planar(p.delta)
        check(lib.ipt_apply_map_full(ctx.handle, n, dptr(dr), dptr(di), dptr(ar), dptr(ai),
                                     dptr(zr), dptr(zi), dptr(fr), dptr(fi)))
    return _combine(fr, fi, cx)


_DEVICE_GROUPS: dict = {}


def _device_group(devices) -> list:
    """Contexts of this process on `devices`, joined by the in-process communicator
    (kept for later calls with the same device list)."""
    key = tuple(int(d) for d in devices)
    if key not in _DEVICE_GROUPS:
        from . import dist

        _DEVICE_GROUPS[key] = dist.local_contexts(len(key), key)
    return _DEVICE_GROUPS[key]


def _run_on_devices(devices, fn):
    """fn(ctx) on one host thread per device of the group; rank 0's result. A failed
    call drops the group (its communicator is aborted) so the next call opens a new one."""
    from . import dist

    ctxs = _device_group(devices)
    try:
        return dist.run_ranks(fn, ctxs)[0]
    except Exception:
        for c in _DEVICE_GROUPS.pop(tuple(int(d) for d in devices), []):
            c.close()
        raise


def solve_full(p: Partition, g: InverseGaps, config: IterationConfig = None, warm_start=None,
               ctx: Optional[Context] = None, want_sigma_min: bool = True, product: str = "dmma",
               output: str = "root", out=None, devices=None) -> SpectrumResult:
    """Fixed-point iteration of F from I (or a renormalised warm start), then the
    closing product, |MZ - Z Lambda|_F and sigma_min (solver.cpp:180-273).

    devices=[0, 1, ...] (two or more; a device may repeat): the columns are sharded over
    ranks of this process on those GPUs (in-process communicator, one host thread per
    rank), each writing its own columns of the result -- bitwise the one-GPU result.

    With a communicator (column shards): output="root" gathers Z and the eigenvalues to
    rank 0; output="local" has every rank write only its own columns into full-size
    outputs -- pass out=(z_re, z_im|None, lam_re, lam_im|None), float64 C-contiguous arrays
    that all ranks share (e.g. np.memmap on /dev/shm, or the same arrays across threads),
    and no gather runs (IPT_OUTPUT_LOCAL_COLUMNS)."""
    config = config or IterationConfig()
    _validate(config)
    _check_sizes(p, g, 0)
    n = p.size()
    if devices is not None and len(devices) > 1:
        if ctx is not None or out is not None:
            raise ValueError("solve_full: devices= runs its own ranks (no ctx / out)")
        cxd = _out_complex(p, warm_start)
        shared = (np.empty((n, n)), np.empty((n, n)) if cxd else None, np.empty(n), np.empty(n) if cxd else None)
        r = _run_on_devices(devices, lambda c: solve_full(p, g, config, warm_start, ctx=c,
                                                          want_sigma_min=want_sigma_min, product=product,
                                                          output="local", out=shared))
        r.Z = _combine(shared[0], shared[1], cxd)
        r.eigenvalues = _combine(shared[2], shared[3], cxd)
        return r
    ctx = ctx or default_context()
    dr, di = _planar(p.d)
    wr = wi = None
    if warm_start is not None:
        warm_start = np.asarray(warm_start)
        if warm_start.shape != (n, n):
            raise ValueError("solve_full: warm start size mismatch")
        wr, wi = _planar(warm_start)
    cx = _out_complex(p, warm_start)
    if output not in ("root", "local"):
        raise ValueError("solve_full: output must be 'root' or 'local'")
    local = output == "local"
    root = ctx.rank == 0 or local
    if out is not None:
        zr, zi, lr, li = out
        for a, shape in ((zr, (n, n)), (zi, (n, n)), (lr, (n,)), (li, (n,))):
            if a is not None and (a.shape != shape or a.dtype != np.float64 or not a.flags.c_contiguous):
                raise ValueError("solve_full: out arrays must be float64, C-contiguous, (n, n) / (n,)")
        if cx and (zi is None or li is None):
            raise ValueError("solve_full: complex results need the imaginary out arrays")
    else:
        zr = np.empty((n, n)) if root else None
        zi = np.empty((n, n)) if (root and cx) else None
        lr = np.empty(n) if root else None
        li = np.empty(n) if (root and cx) else None
    if product not in ("dmma", "ozaki"):
        raise ValueError("solve_full: product must be 'dmma' or 'ozaki'")
    prm = _params(config, want_sigma_min=1 if want_sigma_min else 0,
                  product=_lib.PRODUCT_OZAKI if product == "ozaki" else _lib.PRODUCT_DMMA,
                  output_mode=_lib.OUTPUT_LOCAL_COLUMNS if local else _lib.OUTPUT_ROOT)
    st = _lib.Stats()
    tr = np.zeros(config.max_iterations) if config.record_trace else None
    tm = np.zeros(config.max_iterations) if config.record_trace else None
    st.trace = dptr(tr)
    st.trace_max_abs = dptr(tm)
    lib = _lib.load()
    t_call = time.perf_counter()
    if isinstance(p.delta, CsrMatrix):  # sparse Delta: fused SpMM map (real) on the device
        vr, vi = _planar(p.delta.values)
        check(lib.ipt_full_solve_csr(ctx.handle, n, dptr(dr), dptr(di), i64ptr(p.delta.row_offsets),
                                     i32ptr(p.delta.col_indices), dptr(vr), dptr(vi), dptr(wr), dptr(wi),
                                     C.byref(prm), dptr(zr), dptr(zi), dptr(lr), dptr(li), C.byref(st)))
    else:
        ar, ai = _planar(p.delta)
        check(lib.ipt_full_solve(ctx.handle, n, dptr(dr), dptr(di), dptr(ar), dptr(ai), dptr(wr),
                                 dptr(wi), C.byref(prm), dptr(zr), dptr(zi), dptr(lr), dptr(li),
                                 C.byref(st)))
    if os.environ.get("IPT_PROFILE"):
        print(f"[ipt.py] solve_full C call {1e3 * (time.perf_counter() - t_call):.1f} ms", file=sys.stderr)
    res = SpectrumResult()
    if root:
        res.Z = _combine(zr, zi, cx)
        res.eigenvalues = _combine(lr, li, cx)
    res.iterations = st.iterations
    res.final_step = st.final_step
    res.final_max_abs = st.final_max_abs
    res.residual_frobenius = st.residual
    res.min_singular_value_estimate = st.min_singular_value_estimate
    res.status = SolveStatus(st.status)
    res.matmul_count = st.product_count
    if config.record_trace:
        res.trace = list(tr[: st.iterations])
        res.trace_max_abs = list(tm[: st.iterations])
    res.timings_ms = dict(upload=st.ms_upload, loop=st.ms_loop, final=st.ms_final, sigma=st.ms_sigma,
                          download=st.ms_download)
    return res


def smallest_singular_value_estimate(z, max_iters: int = 50, tol: float = 1e-4,
                                     ctx: Optional[Context] = None) -> float:
    """solver.cpp:275-297 (Cholesky of Z^H Z on the device, same inverse iteration)."""
    z = np.asarray(z)
    n = z.shape[0]
    if n == 0 or z.ndim != 2 or z.shape[1] != n:
        raise ValueError("smallest_singular_value_estimate: square input required")
    ctx = ctx or default_context()
    zr, zi = _planar(z)
    out = C.c_double()
    check(_lib.load().ipt_sigma_min(ctx.handle, n, dptr(zr), dptr(zi), int(max_iters), float(tol),
                                    C.byref(out)))
    return out.value


# ----------------------------------------------------------------- dense LU (lu.hpp)


class LuFactors:
    """PA = LU with unit lower L (lu.hpp): packed `lu` (n x n), `perm[i]` = source row of
    pivoted row i, `singular`; the factors also stay on the device for the solves."""

    def __init__(self, n, lu, perm, singular, handle, ctx):
        self.n, self.lu, self.perm, self.singular = n, lu, perm, singular
        self._h, self._ctx = handle, ctx

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().ipt_lu_free(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None


def lu_factor(a, ctx: Optional[Context] = None) -> LuFactors:
    """lu_factor (lu.cpp:10-49) on the device: partial pivoting by the largest |a_ik|."""
    a = np.asarray(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("lu_factor: matrix must be square")
    n = a.shape[0]
    ctx = ctx or default_context()
    lib = _lib.load()
    ar, ai = _planar(a)
    h = C.c_void_p()
    check(lib.ipt_lu_factor(ctx.handle, n, dptr(ar), dptr(ai), C.byref(h)))
    sing = C.c_int()
    check(lib.ipt_lu_info(h, None, C.byref(sing)))
    lr, li = np.empty((n, n)), np.empty((n, n))
    perm = np.empty(n, np.int64)
    check(lib.ipt_lu_download(ctx.handle, h, dptr(lr), dptr(li), i64ptr(perm)))
    return LuFactors(n, lr + 1j * li, perm, bool(sing.value), h, ctx)


def _lu_solve(f: LuFactors, b, adjoint: bool):
    b = np.asarray(b)
    if b.shape[0] != f.n:
        raise ValueError("lu_solve: size mismatch")
    b2 = b.reshape(f.n, -1)
    br, bi = _planar(b2)
    xr, xi = np.empty(b2.shape), np.empty(b2.shape)
    fn = _lib.load().ipt_lu_solve_adjoint if adjoint else _lib.load().ipt_lu_solve
    check(fn(f._ctx.handle, f._h, b2.shape[1], dptr(br), dptr(bi), dptr(xr), dptr(xi)))
    return (xr + 1j * xi).reshape(b.shape)


def lu_solve(f: LuFactors, b):
    """x = A^{-1} b (lu.cpp:51-66)."""
    return _lu_solve(f, b, False)


def lu_solve_adjoint(f: LuFactors, b):
    """x = A^{-H} b (lu.cpp:68-86)."""
    return _lu_solve(f, b, True)


def lu_solve_matrix(f: LuFactors, b):
    """A X = B for all columns of B at once (lu.cpp:88-103)."""
    b = np.asarray(b)
    if b.ndim != 2:
        raise ValueError("lu_solve_matrix: matrix right-hand side required")
    return _lu_solve(f, b, False)


# ----------------------------------------------------------------- single pair


def _single_call(p, g, anchor, config, warm, schedule, alpha, ctx):
    config = config or IterationConfig()
    _validate(config)
    _check_sizes(p, g, anchor)
    n = p.size()
    ctx = ctx or default_context()
    lib = _lib.load()
    dr, di = _planar(p.d)
    wr = wi = None
    if warm is not None:
        warm = np.asarray(warm)
        if warm.shape != (n,):
            raise ValueError("solver: warm start size mismatch")
        if warm[anchor] == 0:
            raise ValueError("solver: warm start has zero anchor coordinate")
        wr, wi = _planar(warm)
    cx = _out_complex(p, warm)
    zr = np.empty(n)
    zi = np.empty(n) if cx else None
    prm = _params(config, schedule=schedule, shrink_alpha=alpha)
    st = _lib.Stats()
    tr = np.zeros(config.max_iterations) if config.record_trace else None
    st.trace = dptr(tr)
    if isinstance(p.delta, CsrMatrix):
        vr, vi = _planar(p.delta.values)
        check(lib.ipt_single_solve_csr(ctx.handle, n, dptr(dr), dptr(di), i64ptr(p.delta.row_offsets),
                                       i32ptr(p.delta.col_indices), dptr(vr), dptr(vi), int(anchor),
                                       dptr(wr), dptr(wi), C.byref(prm), dptr(zr), dptr(zi), C.byref(st)))
    else:
        ar, ai = _planar(p.delta)
        check(lib.ipt_single_solve_dense(ctx.handle, n, dptr(dr), dptr(di), dptr(ar), dptr(ai), int(anchor),
                                         dptr(wr), dptr(wi), C.byref(prm), dptr(zr), dptr(zi), C.byref(st)))
    res = EigenpairResult()
    res.z = _combine(zr, zi, cx)
    res.eigenvalue = complex(st.eigenvalue_re, st.eigenvalue_im) if cx else st.eigenvalue_re
    res.anchor = int(anchor)
    res.iterations = st.iterations
    res.final_step = st.final_step
    res.residual = st.residual
    res.status = SolveStatus(st.status)
    res.matvec_count = st.product_count
    if config.record_trace:
        res.trace = list(tr[: st.iterations])
    res.timings_ms = dict(loop=st.ms_loop, final=st.ms_final)
    return res


def solve_single(p: Partition, g: InverseGaps, anchor: int, config: IterationConfig = None,
                 warm_start=None, ctx: Optional[Context] = None, devices=None) -> EigenpairResult:
    """solver.cpp:132-136. devices=[0, 1, ...] (two or more): the rows are sharded over ranks
    of this process on those GPUs (the iterate all-gathered every step by peer stores)."""
    if devices is not None and len(devices) > 1:
        if ctx is not None:
            raise ValueError("solve_single: devices= runs its own ranks (no ctx)")
        return _run_on_devices(devices, lambda c: _single_call(p, g, anchor, config, warm_start,
                                                               _lib.SCHEDULE_PLAIN, 0.9, c))
    return _single_call(p, g, anchor, config, warm_start, _lib.SCHEDULE_PLAIN, 0.9, ctx)


def solve_single_continuation(p: Partition, g: InverseGaps, anchor: int, config: IterationConfig = None,
                              shrink_alpha: float = 0.9, ctx: Optional[Context] = None) -> EigenpairResult:
    """solver.cpp:138-154."""
    if not (0.0 <= shrink_alpha < 1.0):
        raise ValueError("continuation: shrink factor must lie in [0, 1)")
    return _single_call(p, g, anchor, config, None, _lib.SCHEDULE_CONTINUATION, shrink_alpha, ctx)


def solve_single_accelerated(p: Partition, g: InverseGaps, anchor: int, config: IterationConfig = None,
                             memory: int = 5, ctx: Optional[Context] = None) -> EigenpairResult:
    """Memory-m Anderson-mixed single pair on the device (anderson.cpp:184-247): stops on the
    true residual |Mz - lambda z|_2 <= config.residual_tolerance. Real inputs, one GPU."""
    config = config or IterationConfig()
    _check_sizes(p, g, anchor)
    if not (config.tolerance > 0.0):
        raise ValueError("config: tolerance must be positive")
    if config.max_iterations <= 0:
        raise ValueError("config: max_iterations must be positive")
    if memory < 0:
        raise ValueError("anderson: memory must be non-negative")
    if _is_complex_problem(p):
        raise ValueError("solve_single_accelerated (device): real inputs only")
    n = p.size()
    ctx = ctx or default_context()
    lib = _lib.load()
    d = np.ascontiguousarray(np.real(p.d), dtype=np.float64)
    z = np.empty(n)
    prm = _params(config)
    st = _lib.Stats()
    tr = np.zeros(config.max_iterations) if config.record_trace else None
    st.trace = dptr(tr)
    if isinstance(p.delta, CsrMatrix):
        vals = np.ascontiguousarray(np.real(p.delta.values), dtype=np.float64)
        check(lib.ipt_single_solve_accelerated_csr(ctx.handle, n, dptr(d), i64ptr(p.delta.row_offsets),
                                                   i32ptr(p.delta.col_indices), dptr(vals), int(anchor), C.byref(prm),
                                                   int(memory), float(config.residual_tolerance), dptr(z),
                                                   C.byref(st)))
    else:
        a = np.ascontiguousarray(np.real(p.delta), dtype=np.float64)
        check(lib.ipt_single_solve_accelerated_dense(ctx.handle, n, dptr(d), dptr(a), int(anchor), C.byref(prm),
                                                     int(memory), float(config.residual_tolerance), dptr(z),
                                                     C.byref(st)))
    res = EigenpairResult()
    res.z = z
    res.eigenvalue = st.eigenvalue_re
    res.anchor = int(anchor)
    res.iterations = st.iterations
    res.final_step = st.final_step
    res.residual = st.residual
    res.status = SolveStatus(st.status)
    res.matvec_count = st.product_count
    if config.record_trace:
        res.trace = list(tr[: max(st.iterations - (1 if res.status == SolveStatus.Converged else 0), 0)])
    return res


def apply_map_single(p: Partition, g: InverseGaps, anchor: int, z, ctx: Optional[Context] = None) -> np.ndarray:
    """f_i(z) = e_i + g_i o (z (Delta z)_i - Delta z) (solver.cpp:122-130)."""
    _check_sizes(p, g, anchor)
    n = p.size()
    z = np.asarray(z)
    if z.shape != (n,):
        raise ValueError("apply_map_single: size mismatch")
    delta = p.delta.to_dense() if isinstance(p.delta, CsrMatrix) else p.delta
    ctx = ctx or default_context()
    dr, di = _planar(p.d)
    ar, ai = _planar(delta)
    zr, zi = _planar(z)
    cx = _out_complex(p, z)
    fr = np.empty(n)
    fi = np.empty(n) if cx else None
    check(_lib.load().ipt_apply_map_single_dense(ctx.handle, n, dptr(dr), dptr(di), dptr(ar), dptr(ai),
                                                 int(anchor), dptr(zr), dptr(zi), dptr(fr), dptr(fi)))
    return _combine(fr, fi, cx)


# ----------------------------------------------------------------- kernels::


class kernels:  # noqa: N801  (namespace ipt::kernels)
    @staticmethod
    def matmul(a, b, ctx: Optional[Context] = None) -> np.ndarray:
        """C = A B (kernels.cpp:175-181); deterministic run to run."""
        if isinstance(a, CsrMatrix):
            a = a.to_dense()
        a, b = np.asarray(a), np.asarray(b)
        if a.shape[1] != b.shape[0]:
            raise ValueError("matmul: inner dimensions differ")
        ctx = ctx or default_context()
        m, k = a.shape
        n = b.shape[1]
        ar, ai = _planar(a)
        br, bi = _planar(b)
        cx = np.iscomplexobj(a) or np.iscomplexobj(b)
        cr = np.empty((m, n))
        ci = np.empty((m, n)) if cx else None
        check(_lib.load().ipt_gemm(ctx.handle, m, k, n, dptr(ar), dptr(ai), dptr(br), dptr(bi), dptr(cr), dptr(ci)))
        return _combine(cr, ci, cx)

    @staticmethod
    def matmul_ozaki(a, b, ctx: Optional[Context] = None) -> np.ndarray:
        """C = A B for real A, B by Ozaki scheme II on the INT8 tensor cores (B200
        extension; the product of `product="ozaki"`): each row of A and column of B is
        scaled by a power of two to 53-bit integers and every C_ij is the correctly rounded
        exact dot product of those integers, scaled back."""
        a, b = np.asarray(a), np.asarray(b)
        if np.iscomplexobj(a) or np.iscomplexobj(b):
            raise ValueError("matmul_ozaki: real operands only")
        if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
            raise ValueError("matmul_ozaki: inner dimensions differ")
        ctx = ctx or default_context()
        m, k = a.shape
        n = b.shape[1]
        ar = np.ascontiguousarray(a, dtype=np.float64)
        bt = np.ascontiguousarray(b.T, dtype=np.float64)
        c = np.empty((m, n))
        check(_lib.load().ipt_ozaki_dgemm(ctx.handle, m, n, k, dptr(ar), dptr(bt), dptr(c), 0, None))
        return c

    @staticmethod
    def matvec(a: Matrix, x, ctx: Optional[Context] = None) -> np.ndarray:
        """y = A x, dense or CSR (kernels.cpp:112-140)."""
        ctx = ctx or default_context()
        x = np.asarray(x)
        xr, xi = _planar(x)
        lib = _lib.load()
        if isinstance(a, CsrMatrix):
            m, n = a.shape
            vr, vi = _planar(a.values)
            cx = np.iscomplexobj(a.values) or np.iscomplexobj(x)
            yr = np.empty(m)
            yi = np.empty(m) if cx else None
            check(lib.ipt_matvec_csr(ctx.handle, m, n, i64ptr(a.row_offsets), i32ptr(a.col_indices), dptr(vr),
                                     dptr(vi), dptr(xr), dptr(xi), dptr(yr), dptr(yi)))
        else:
            a = np.asarray(a)
            m, n = a.shape
            ar, ai = _planar(a)
            cx = np.iscomplexobj(a) or np.iscomplexobj(x)
            yr = np.empty(m)
            yi = np.empty(m) if cx else None
            check(lib.ipt_matvec_dense(ctx.handle, m, n, dptr(ar), dptr(ai), dptr(xr), dptr(xi), dptr(yr), dptr(yi)))
        return _combine(yr, yi, cx)

    @staticmethod
    def frobenius_norm(m) -> float:
        v = m.values if isinstance(m, CsrMatrix) else np.asarray(m)
        return float(np.sqrt(np.sum(np.abs(v) ** 2)))

    @staticmethod
    def nrm2(v) -> float:
        return float(np.sqrt(np.sum(np.abs(np.asarray(v)) ** 2)))

    @staticmethod
    def max_abs(v) -> float:
        return float(np.max(np.abs(np.asarray(v)))) if np.asarray(v).size else 0.0
