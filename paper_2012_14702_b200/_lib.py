"""ctypes binding of libipt_b200.so (include/ipt_cuda.h, include/ipt_synth.h).

The shared library is built in-tree by `make -C paper_2012_14702_b200` (or
`__graft_entry__.build()`). There is no fallback: if the library is missing or
fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IPT_B200_LIB") or os.path.join(_HERE, "libipt_b200.so")

IPT_OK = 0
IPT_ERR_INVALID = -1
IPT_ERR_CUDA = -2
IPT_ERR_NCCL = -4
IPT_ERR_INTERNAL = -5

STOP_REL_FRO = 0
STOP_MAX_ABS = 1
SCHEDULE_PLAIN = 0
SCHEDULE_CONTINUATION = 1

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_vp = C.c_void_p


PRODUCT_DMMA = 0
PRODUCT_OZAKI = 1
OUTPUT_ROOT = 0
OUTPUT_LOCAL_COLUMNS = 1


class Params(C.Structure):
    _fields_ = [
        ("tolerance", C.c_double),
        ("max_iterations", C.c_int32),
        ("divergence_threshold", C.c_double),
        ("record_trace", C.c_int32),
        ("stop_rule", C.c_int32),
        ("want_sigma_min", C.c_int32),
        ("schedule", C.c_int32),
        ("shrink_alpha", C.c_double),
        ("ignore_convergence", C.c_int32),
        ("product", C.c_int32),
        ("output_mode", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("status", C.c_int32),
        ("final_step", C.c_double),
        ("final_max_abs", C.c_double),
        ("residual", C.c_double),
        ("min_singular_value_estimate", C.c_double),
        ("product_count", C.c_int64),
        ("eigenvalue_re", C.c_double),
        ("eigenvalue_im", C.c_double),
        ("trace", _dp),
        ("trace_max_abs", _dp),
        ("ms_upload", C.c_double),
        ("ms_loop", C.c_double),
        ("ms_final", C.c_double),
        ("ms_sigma", C.c_double),
        ("ms_download", C.c_double),
    ]


# name -> (restype, argtypes); mirrors include/ipt_cuda.h and include/ipt_synth.h
SIGNATURES = {
    "ipt_last_error": (C.c_char_p, []),
    "ipt_default_params": (None, [C.POINTER(Params)]),
    "ipt_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ipt_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "ipt_ctx_destroy": (None, [_vp]),
    "ipt_ctx_device": (C.c_int, [_vp]),
    "ipt_nccl_get_unique_id": (C.c_int, [_vp]),
    "ipt_ctx_init_comm": (C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    "ipt_ctx_rank": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ipt_ctx_synchronize": (C.c_int, [_vp]),
    "ipt_ctx_trim": (C.c_int, [_vp]),
    "ipt_local_group_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "ipt_local_group_destroy": (None, [_vp]),
    "ipt_ctx_init_local_comm": (C.c_int, [_vp, _vp, C.c_int]),
    "ipt_ctx_comm_kind": (C.c_char_p, [_vp]),
    "ipt_operator_create_dense": (C.c_int, [_vp, C.c_int64, _dp, _dp, C.POINTER(_vp)]),
    "ipt_operator_create_csr": (C.c_int, [_vp, C.c_int64, _i64p, _i32p, _dp, _dp, C.POINTER(_vp)]),
    "ipt_operator_matvec": (C.c_int, [_vp, _vp, _dp, _dp, _dp, _dp]),
    "ipt_operator_bytes": (C.c_int64, [_vp]),
    "ipt_operator_free": (None, [_vp]),
    "ipt_gemm_operand_create": (C.c_int, [_vp, C.c_int64, C.c_int64, _dp, _dp, C.POINTER(_vp)]),
    "ipt_gemm_operand_apply": (C.c_int, [_vp, _vp, C.c_int64, _dp, _dp, _dp, _dp]),
    "ipt_gemm_operand_free": (None, [_vp]),
    "ipt_full_solve": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, C.POINTER(Params),
                                 _dp, _dp, _dp, _dp, C.POINTER(Stats)]),
    "ipt_full_upload": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, C.POINTER(_vp)]),
    "ipt_full_reset": (C.c_int, [_vp, _vp, _dp, _dp]),
    "ipt_full_iterate": (C.c_int, [_vp, _vp, C.POINTER(Params), C.POINTER(Stats)]),
    "ipt_full_finalize": (C.c_int, [_vp, _vp, C.POINTER(Params), C.POINTER(Stats)]),
    "ipt_full_download": (C.c_int, [_vp, _vp, _dp, _dp, _dp, _dp]),
    "ipt_full_set_product": (C.c_int, [_vp, C.c_int32]),
    "ipt_full_solve_interleaved_start": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, C.POINTER(Params), C.POINTER(_vp),
                                                   C.POINTER(Stats)]),
    "ipt_full_solve_interleaved_finish": (C.c_int, [_vp, _vp, C.POINTER(Params), _dp, _dp, C.POINTER(Stats)]),
    "ipt_full_ozaki_moduli": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "ipt_single_debug_peers": (C.c_int, [_vp, C.c_int32]),
    "ipt_single_debug_peer_z": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp]),
    "ipt_full_local_columns": (C.c_int, [_vp, _i64p, _i64p]),
    "ipt_full_free": (None, [_vp]),
    "ipt_apply_map_full": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
    "ipt_full_upload_columns": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, C.c_int64, C.c_int64,
                                          C.POINTER(_vp)]),
    "ipt_full_upload_csr_columns": (C.c_int, [_vp, C.c_int64, _dp, _i64p, _i32p, _dp, C.c_int64, C.c_int64,
                                              C.POINTER(_vp)]),
    "ipt_full_download_block": (C.c_int, [_vp, _vp, _dp, _dp, _dp, _dp]),
    "ipt_full_solve_csr": (C.c_int, [_vp, C.c_int64, _dp, _dp, _i64p, _i32p, _dp, _dp, _dp, _dp,
                                     C.POINTER(Params), _dp, _dp, _dp, _dp, C.POINTER(Stats)]),
    "ipt_full_upload_csr": (C.c_int, [_vp, C.c_int64, _dp, _dp, _i64p, _i32p, _dp, _dp, C.POINTER(_vp)]),
    "ipt_apply_map_full_csr": (C.c_int, [_vp, C.c_int64, _dp, _dp, _i64p, _i32p, _dp, _dp, _dp, _dp,
                                         _dp, _dp]),
    "ipt_i8_gemm": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp, C.c_int32, _dp]),
    "ipt_ozaki_dgemm": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _dp, _dp, _dp, C.c_int32, _dp]),
    "ipt_lu_factor": (C.c_int, [_vp, C.c_int64, _dp, _dp, C.POINTER(_vp)]),
    "ipt_lu_from_host": (C.c_int, [_vp, C.c_int64, _dp, _dp, _i64p, C.c_int, C.POINTER(_vp)]),
    "ipt_lu_info": (C.c_int, [_vp, _i64p, C.POINTER(C.c_int)]),
    "ipt_lu_download": (C.c_int, [_vp, _vp, _dp, _dp, _i64p]),
    "ipt_lu_solve": (C.c_int, [_vp, _vp, C.c_int64, _dp, _dp, _dp, _dp]),
    "ipt_lu_solve_adjoint": (C.c_int, [_vp, _vp, C.c_int64, _dp, _dp, _dp, _dp]),
    "ipt_lu_free": (None, [_vp]),
    "ipt_sigma_min": (C.c_int, [_vp, C.c_int64, _dp, _dp, C.c_int32, C.c_double, _dp]),
    "ipt_single_solve_dense": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, C.c_int64, _dp, _dp,
                                         C.POINTER(Params), _dp, _dp, C.POINTER(Stats)]),
    "ipt_single_solve_csr": (C.c_int, [_vp, C.c_int64, _dp, _dp, _i64p, _i32p, _dp, _dp, C.c_int64,
                                       _dp, _dp, C.POINTER(Params), _dp, _dp, C.POINTER(Stats)]),
    "ipt_single_upload_dense": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, C.POINTER(_vp)]),
    "ipt_single_upload_csr": (C.c_int, [_vp, C.c_int64, _dp, _dp, _i64p, _i32p, _dp, _dp,
                                        C.POINTER(_vp)]),
    "ipt_single_upload_csr_shared": (C.c_int, [_vp, C.c_int64, _dp, _dp, _i64p, _i32p, _dp, _dp,
                                        C.POINTER(_vp)]),
    "ipt_single_upload_dense_rows": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, C.c_int64, C.c_int64,
                                               C.POINTER(_vp)]),
    "ipt_single_upload_csr_rows": (C.c_int, [_vp, C.c_int64, _dp, _dp, _i64p, _i32p, _dp, _dp, C.c_int64,
                                             C.c_int64, C.POINTER(_vp)]),
    "ipt_single_reset": (C.c_int, [_vp, _vp, C.c_int64, _dp, _dp]),
    "ipt_single_iterate": (C.c_int, [_vp, _vp, C.POINTER(Params), C.POINTER(Stats)]),
    "ipt_single_finalize": (C.c_int, [_vp, _vp, C.POINTER(Stats)]),
    "ipt_single_download": (C.c_int, [_vp, _vp, _dp, _dp]),
    "ipt_single_free": (None, [_vp]),
    "ipt_apply_map_single_dense": (C.c_int, [_vp, C.c_int64, _dp, _dp, _dp, _dp, C.c_int64, _dp,
                                             _dp, _dp, _dp]),
    "ipt_gemm": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp]),
    "ipt_matvec_dense": (C.c_int, [_vp, C.c_int64, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp]),
    "ipt_matvec_csr": (C.c_int, [_vp, C.c_int64, C.c_int64, _i64p, _i32p, _dp, _dp, _dp, _dp, _dp,
                                 _dp]),
    "ipt_single_solve_accelerated_dense": (C.c_int, [_vp, C.c_int64, _dp, _dp, C.c_int64, C.POINTER(Params),
                                                     C.c_int32, C.c_double, _dp, C.POINTER(Stats)]),
    "ipt_single_solve_accelerated_csr": (C.c_int, [_vp, C.c_int64, _dp, _i64p, _i32p, _dp, C.c_int64,
                                                   C.POINTER(Params), C.c_int32, C.c_double, _dp, C.POINTER(Stats)]),
    "ipt_full_run_maps": (C.c_int, [_vp, _vp, C.c_int32, _dp, _dp]),
    "ipt_single_run_steps": (C.c_int, [_vp, _vp, C.c_int32, _dp, _dp]),
    "ipt_kernel_launch_count": (C.c_int64, []),
    "ipt_guard_violations": (C.c_int64, []),
    "ipt_fp64_issue_probe": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "ipt_guard_selftest": (C.c_int64, []),
    "ipt_guard_checked": (C.c_int64, []),
    "ipt_synth_dense_uniform": (C.c_int, [C.c_int64, C.c_double, C.c_uint64, _dp, _dp]),
    "ipt_synth_dense_normal": (C.c_int, [C.c_int64, C.c_double, C.c_uint64, C.c_int, _dp, _dp]),
    "ipt_synth_csr_ci_plan": (C.c_int, [C.c_int64, C.c_int, C.c_uint64, C.POINTER(_vp), _i64p]),
    "ipt_synth_csr_ci_fill": (C.c_int, [_vp, C.c_double, _dp, _i64p, _i32p, _dp]),
    "ipt_synth_rng_draws": (None, [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_int64,
                                   _vp]),
}

_lock = threading.Lock()
_lib = None


class IptError(RuntimeError):
    """A CUDA / NCCL / internal failure reported by the C ABI (std::runtime_error)."""


def load() -> C.CDLL:
    """Load libipt_b200.so (raises OSError if it is absent: there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise OSError(f"{LIB_PATH} is missing; build it with `make -C {_HERE}`")
            lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def check(rc: int) -> None:
    """Map IPT_ERR_* to the reference's exception types (solver.cpp raises invalid_argument)."""
    if rc == IPT_OK:
        return
    msg = load().ipt_last_error().decode(errors="replace")
    if rc == IPT_ERR_INVALID:
        raise ValueError(msg)
    raise IptError(f"[{rc}] {msg}")


def default_params() -> Params:
    p = Params()
    load().ipt_default_params(C.byref(p))
    return p


def dptr(a):
    """double* of a contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def i64ptr(a):
    return None if a is None else a.ctypes.data_as(_i64p)


def i32ptr(a):
    return None if a is None else a.ctypes.data_as(_i32p)
