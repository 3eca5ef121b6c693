"""CPU oracle for the IPT hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the timed
CPU baseline. The product (paper_2012_14702_b200) never imports it.

Two arms:
  ref  : the unmodified reference library (oracle/_ref/libipt_ref.so, built by
         oracle/Makefile from the sources under /root/reference/proj/src) via
         the extern "C" shim oracle/ref_driver.cpp;
  port : our plain-C restatement (oracle/ipt_oracle.c -> oracle/libipt_oracle.so).
The port is pinned against the ref arm and the reference's known answers in
tests/test_oracle_pins.py (parity pinned, not assumed).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libipt_ref.so")
PORT_SO = os.path.join(HERE, "libipt_oracle.so")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def build(ref: bool = True) -> None:
    """Compile the restatement (and the reference build when /root/reference exists)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _c(a):
    """contiguous complex128 (interleaved re/im doubles) copy or view."""
    return np.ascontiguousarray(a, dtype=np.complex128)


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _csr_args(delta):
    rp = np.ascontiguousarray(delta.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(delta.col_indices, dtype=np.int64)
    va = _c(delta.values)
    return rp, ci, va


class _Arm:
    def __init__(self, path):
        if not os.path.exists(path):
            raise OSError(f"{path} missing: run `make -C {HERE}`")
        self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)


class RefArm(_Arm):
    """The reference implementation itself (proj/src/*.cpp, -O3 -fopenmp)."""

    def __init__(self):
        super().__init__(REF_SO)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_sigma_min.restype = C.c_double
        L.ref_condition_estimate.restype = C.c_double

    def _chk(self, rc):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            if rc == -3:
                raise ArithmeticError(msg)
            raise ValueError(msg) if rc == -1 else RuntimeError(msg)

    def solve_full(self, d, delta, tol=100 * np.finfo(float).eps, max_iter=1000, div_thr=1e8,
                   degeneracy_tol=-1.0, record_trace=False, warm=None, stop_rule="rel_fro"):
        n = len(d)
        d, delta = _c(d), _c(delta)
        z = np.empty((n, n), np.complex128)
        lam = np.empty(n, np.complex128)
        stats = np.zeros(8)
        trace = np.zeros(max_iter)
        if stop_rule == "max_abs":
            self._chk(self.lib.ref_solve_full_maxabs(C.c_int64(n), _p(d), _p(delta), C.c_double(tol),
                                                     C.c_int(max_iter), C.c_double(div_thr), _p(z), _p(lam),
                                                     _p(stats), _p(trace)))
        else:
            w = None if warm is None else _c(warm)
            self._chk(self.lib.ref_solve_full(C.c_int64(n), _p(d), _p(delta), C.c_double(degeneracy_tol),
                                              C.c_double(tol), C.c_int(max_iter), C.c_double(div_thr),
                                              C.c_int(1 if record_trace else 0), _p(w), _p(z), _p(lam),
                                              _p(stats), _p(trace)))
        it = int(stats[0])
        return dict(Z=z, eigenvalues=lam, iterations=it, status=int(stats[1]), final_step=stats[2],
                    residual_frobenius=stats[3], sigma_min=stats[4], matmul_count=int(stats[5]),
                    seconds=stats[6], final_max_abs=stats[7], trace=trace[:it].copy())

    def solve_single(self, d, delta, anchor, tol=100 * np.finfo(float).eps, max_iter=1000, div_thr=1e8,
                     degeneracy_tol=-1.0, record_trace=False, mode="plain", alpha=0.9, memory=5,
                     residual_tol=1e-8, warm=None):
        n = len(d)
        d = _c(d)
        is_csr = hasattr(delta, "row_offsets")
        if is_csr:
            rp, ci, va = _csr_args(delta)
            dense = None
        else:
            dense = _c(delta)
            rp = ci = va = None
        z = np.empty(n, np.complex128)
        lam = np.empty(1, np.complex128)
        stats = np.zeros(6)
        trace = np.zeros(max_iter)
        w = None if warm is None else _c(warm)
        m = {"plain": 0, "continuation": 1, "accelerated": 2}[mode]
        self._chk(self.lib.ref_solve_single(
            C.c_int64(n), _p(d), C.c_int(1 if is_csr else 0), _p(dense),
            None if rp is None else rp.ctypes.data_as(_i64p), None if ci is None else ci.ctypes.data_as(_i64p),
            _p(va), C.c_double(degeneracy_tol), C.c_int64(anchor), C.c_double(tol), C.c_int(max_iter),
            C.c_double(div_thr), C.c_double(residual_tol), C.c_int(1 if record_trace else 0), C.c_int(m),
            C.c_double(alpha), C.c_int(memory), _p(w), _p(z), _p(lam), _p(stats), _p(trace)))
        it = int(stats[0])
        return dict(z=z, eigenvalue=lam[0], iterations=it, status=int(stats[1]), final_step=stats[2],
                    residual=stats[3], matvec_count=int(stats[4]), seconds=stats[5], trace=trace[:it].copy())

    def solve_single_multi(self, d, delta, anchors, tol=100 * np.finfo(float).eps, max_iter=1000):
        """solve_single for several anchors on one partition (builds the reference's
        ComplexMatrix once). Returns (z[n, count], iterations, status, eigenvalues)."""
        n = len(d)
        anchors = np.ascontiguousarray(anchors, dtype=np.int64)
        k = anchors.size
        dd = _c(d)
        dense = _c(delta)
        z = np.empty((k, n), np.complex128)
        meta = np.zeros((k, 4))
        self._chk(self.lib.ref_solve_single_multi(C.c_int64(n), _p(dd), _p(dense), anchors.ctypes.data_as(_i64p),
                                                  C.c_int64(k), C.c_double(tol), C.c_int(max_iter), _p(z), _p(meta)))
        return z.T.copy(), meta[:, 0].astype(int), meta[:, 1].astype(int), meta[:, 2] + 1j * meta[:, 3]

    def solve_full_csr(self, d, delta, tol=100 * np.finfo(float).eps, max_iter=1000, div_thr=1e8):
        """solve_full on a CSR Delta (the reference's sparse product, kernels.cpp:88-108)."""
        n = len(d)
        rp, ci, va = _csr_args(delta)
        z = np.empty((n, n), np.complex128)
        lam = np.empty(n, np.complex128)
        stats = np.zeros(8)
        self._chk(self.lib.ref_solve_full_csr(C.c_int64(n), _p(_c(d)), rp.ctypes.data_as(_i64p),
                                              ci.ctypes.data_as(_i64p), _p(va), C.c_double(tol),
                                              C.c_int(max_iter), C.c_double(div_thr), _p(z), _p(lam),
                                              _p(stats)))
        return dict(Z=z, eigenvalues=lam, iterations=int(stats[0]), status=int(stats[1]), final_step=stats[2],
                    residual_frobenius=stats[3], sigma_min=stats[4], matmul_count=int(stats[5]),
                    seconds=stats[6])

    def apply_map_full_csr(self, d, delta, z):
        n = len(d)
        rp, ci, va = _csr_args(delta)
        out = np.empty((n, n), np.complex128)
        self._chk(self.lib.ref_apply_map_full_csr(C.c_int64(n), _p(_c(d)), rp.ctypes.data_as(_i64p),
                                                  ci.ctypes.data_as(_i64p), _p(va), _p(_c(z)), _p(out)))
        return out

    def lu_factor(self, a):
        a = _c(a)
        n = a.shape[0]
        lu = np.empty((n, n), np.complex128)
        perm = np.empty(n, np.int64)
        sing = C.c_int()
        self._chk(self.lib.ref_lu_factor(C.c_int64(n), _p(a), _p(lu), perm.ctypes.data_as(_i64p), C.byref(sing)))
        return lu, perm, bool(sing.value)

    def lu_solve(self, a, b, adjoint=False):
        a = _c(a)
        b = _c(b)
        n = a.shape[0]
        b2 = b.reshape(n, -1)
        x = np.empty_like(b2)
        self._chk(self.lib.ref_lu_solve(C.c_int64(n), _p(a), C.c_int64(b2.shape[1]), _p(b2),
                                        C.c_int(1 if adjoint else 0), _p(x)))
        return x.reshape(b.shape)

    def condition_estimate(self, a):
        a = _c(a)
        return self.lib.ref_condition_estimate(C.c_int64(a.shape[0]), _p(a))

    def apply_map_full(self, d, delta, z):
        n = len(d)
        out = np.empty((n, n), np.complex128)
        self._chk(self.lib.ref_apply_map_full(C.c_int64(n), _p(_c(d)), _p(_c(delta)), _p(_c(z)), _p(out)))
        return out

    def apply_map_single(self, d, delta, anchor, z):
        n = len(d)
        out = np.empty(n, np.complex128)
        self._chk(self.lib.ref_apply_map_single(C.c_int64(n), _p(_c(d)), _p(_c(delta)), C.c_int64(anchor),
                                                _p(_c(z)), _p(out)))
        return out

    def matmul(self, a, b, serial=False):
        a, b = _c(a), _c(b)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), np.complex128)
        self._chk(self.lib.ref_matmul(C.c_int64(m), C.c_int64(k), C.c_int64(n), _p(a), _p(b), _p(c),
                                      C.c_int(1 if serial else 0)))
        return c

    def matvec(self, a, x):
        n = len(x)
        y = np.empty(n, np.complex128)
        if hasattr(a, "row_offsets"):
            rp, ci, va = _csr_args(a)
            self._chk(self.lib.ref_matvec(C.c_int64(n), C.c_int(1), None, rp.ctypes.data_as(_i64p),
                                          ci.ctypes.data_as(_i64p), _p(va), _p(_c(x)), _p(y)))
        else:
            self._chk(self.lib.ref_matvec(C.c_int64(n), C.c_int(0), _p(_c(a)), None, None, None, _p(_c(x)),
                                          _p(y)))
        return y

    def sigma_min(self, z, max_iters=50, tol=1e-4):
        z = _c(z)
        return self.lib.ref_sigma_min(C.c_int64(z.shape[0]), _p(z), C.c_int(max_iters), C.c_double(tol))

    def gen_near_diagonal(self, n, eps, symmetric, seed):
        out = np.empty((n, n), np.complex128)
        self._chk(self.lib.ref_gen_near_diagonal(C.c_int64(n), C.c_double(eps), C.c_int(1 if symmetric else 0),
                                                 C.c_uint64(seed), _p(out)))
        return out

    def gen_fci_like(self, n, density, gap_scale, seed):
        """testgen.cpp:174-194, partitioned: (d, CSR off-diagonal part) as real arrays."""
        from paper_2012_14702_b200.ipt import CsrMatrix

        nnz = C.c_int64()
        self._chk(self.lib.ref_gen_fci_like(C.c_int64(n), C.c_double(density), C.c_double(gap_scale),
                                            C.c_uint64(seed), C.byref(nnz), None, None, None, None))
        d = np.empty(n)
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz.value, np.int64)
        va = np.empty(nnz.value)
        self._chk(self.lib.ref_gen_fci_like(C.c_int64(n), C.c_double(density), C.c_double(gap_scale),
                                            C.c_uint64(seed), C.byref(nnz), _p(d), rp.ctypes.data_as(_i64p),
                                            ci.ctypes.data_as(_i64p), _p(va)))
        return d, CsrMatrix(n, n, rp, ci.astype(np.int32), va)

    def dense_eigenvalues(self, m):
        m = _c(m)
        out = np.empty(m.shape[0], np.complex128)
        self._chk(self.lib.ref_dense_eigenvalues(C.c_int64(m.shape[0]), _p(m), _p(out)))
        return out

    def rng_draws(self, seed, kind, count, stream=None, bound=0):
        out = np.empty(count, dtype=np.uint64 if kind in (0, 3) else np.float64)
        self.lib.ref_rng_draws(C.c_uint64(seed), C.c_uint64(0 if stream is None else stream),
                               C.c_int(0 if stream is None else 1), C.c_int(kind), C.c_uint64(bound),
                               C.c_int64(count), out.ctypes.data_as(C.c_void_p))
        return out


class PortArm(_Arm):
    """The plain-C restatement (oracle/ipt_oracle.c)."""

    def __init__(self):
        super().__init__(PORT_SO)
        self.lib.orc_sigma_min.restype = C.c_double
        self.lib.orc_full_final_block.restype = C.c_double

    def gemm(self, a, b):
        a, b = _c(a), _c(b)
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), np.complex128)
        self.lib.orc_gemm(C.c_int64(m), C.c_int64(k), C.c_int64(n), _p(a), _p(b), _p(c))
        return c

    def matvec(self, a, x):
        n = len(x)
        y = np.empty(n, np.complex128)
        if hasattr(a, "row_offsets"):
            rp, ci, va = _csr_args(a)
            self.lib.orc_matvec(C.c_int64(n), C.c_int(1), None, rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i64p),
                                _p(va), _p(_c(x)), _p(y))
        else:
            self.lib.orc_matvec(C.c_int64(n), C.c_int(0), _p(_c(a)), None, None, None, _p(_c(x)), _p(y))
        return y

    def dense_uniform(self, n, eps, seed=42):
        """Configs 1-3 inputs (d, Delta) from the reference's generator restated in C
        (rng.hpp:13-82, SURVEY 8(d) draw order): no product library involved."""
        d = np.empty(n)
        delta = np.empty((n, n))
        rc = self.lib.orc_dense_uniform(C.c_int64(n), C.c_double(eps), C.c_uint64(seed), _p(d), _p(delta))
        if rc != 0:
            raise ValueError("orc_dense_uniform: bad size")
        return d, delta

    def full_map_block(self, d, delta, c0, z_block):
        """One map application on the column block [c0, c0+nc) (z_block: n x nc)."""
        n = len(d)
        zb = _c(z_block)
        nc = zb.shape[1]
        f = np.empty((n, nc), np.complex128)
        sums = np.zeros(4)
        self.lib.orc_full_map_block(C.c_int64(n), _p(_c(d)), _p(_c(delta)), C.c_int64(c0), C.c_int64(nc),
                                    _p(zb), _p(f), _p(sums))
        return f, sums

    def full_final_block(self, d, delta, c0, z_block):
        n = len(d)
        zb = _c(z_block)
        nc = zb.shape[1]
        lam = np.empty(nc, np.complex128)
        r2 = self.lib.orc_full_final_block(C.c_int64(n), _p(_c(d)), _p(_c(delta)), C.c_int64(c0), C.c_int64(nc),
                                           _p(zb), _p(lam))
        return lam, r2

    def solve_full(self, d, delta, tol=100 * np.finfo(float).eps, max_iter=1000, div_thr=1e8,
                   stop_rule="rel_fro", sigma=True):
        n = len(d)
        z = np.empty((n, n), np.complex128)
        lam = np.empty(n, np.complex128)
        stats = np.zeros(7)
        trace = np.zeros(max_iter)
        self.lib.orc_solve_full(C.c_int64(n), _p(_c(d)), _p(_c(delta)), C.c_double(tol), C.c_int(max_iter),
                                C.c_double(div_thr), C.c_int(1 if stop_rule == "max_abs" else 0),
                                C.c_int(1 if sigma else 0), _p(z), _p(lam), _p(stats), _p(trace))
        it = int(stats[0])
        return dict(Z=z, eigenvalues=lam, iterations=it, status=int(stats[1]), final_step=stats[2],
                    residual_frobenius=stats[3], sigma_min=stats[4], matmul_count=int(stats[5]),
                    final_max_abs=stats[6], trace=trace[:it].copy())

    def solve_single(self, d, delta, anchor, tol=100 * np.finfo(float).eps, max_iter=1000, div_thr=1e8,
                     mode="plain", alpha=0.9, warm=None):
        n = len(d)
        is_csr = hasattr(delta, "row_offsets")
        if is_csr:
            rp, ci, va = _csr_args(delta)
            dense = None
        else:
            dense = _c(delta)
            rp = ci = va = None
        z = np.empty(n, np.complex128)
        lam = np.zeros(2)
        stats = np.zeros(5)
        trace = np.zeros(max_iter)
        w = None if warm is None else _c(warm)
        self.lib.orc_solve_single(
            C.c_int64(n), _p(_c(d)), C.c_int(1 if is_csr else 0), _p(dense),
            None if rp is None else rp.ctypes.data_as(_i64p), None if ci is None else ci.ctypes.data_as(_i64p),
            _p(va), C.c_int64(anchor), C.c_double(tol), C.c_int(max_iter), C.c_double(div_thr),
            C.c_int(1 if mode == "continuation" else 0), C.c_double(alpha), _p(w), _p(z), _p(lam), _p(stats),
            _p(trace))
        it = int(stats[0])
        return dict(z=z, eigenvalue=complex(lam[0], lam[1]), iterations=it, status=int(stats[1]),
                    final_step=stats[2], residual=stats[3], matvec_count=int(stats[4]), trace=trace[:it].copy())

    def sigma_min(self, z, max_iters=50, tol=1e-4):
        z = _c(z)
        return self.lib.orc_sigma_min(C.c_int64(z.shape[0]), _p(z), C.c_int(max_iters), C.c_double(tol))

    def solve_single_real_dense(self, d, delta, anchor, tol=100 * np.finfo(float).eps, max_iter=1000,
                                div_thr=1e8):
        """run_single on a real dense operator in place (no complex copy; config 4 at N=65536)."""
        n = len(d)
        d = np.ascontiguousarray(d, dtype=np.float64)
        delta = np.ascontiguousarray(delta, dtype=np.float64)
        z = np.empty(n)
        lam = np.zeros(1)
        stats = np.zeros(5)
        self.lib.orc_solve_single_real_dense(C.c_int64(n), _p(d), _p(delta), C.c_int64(anchor), C.c_double(tol),
                                             C.c_int(max_iter), C.c_double(div_thr), _p(z), _p(lam), _p(stats))
        return dict(z=z, eigenvalue=lam[0], iterations=int(stats[0]), status=int(stats[1]), final_step=stats[2],
                    residual=stats[3], matvec_count=int(stats[4]))


_ref = _port = None


def ref() -> RefArm:
    global _ref
    if _ref is None:
        _ref = RefArm()
    return _ref


def port() -> PortArm:
    global _port
    if _port is None:
        _port = PortArm()
    return _port


def have_ref() -> bool:
    return os.path.exists(REF_SO)
