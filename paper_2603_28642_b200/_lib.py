"""ctypes binding of librowsplit_b200.so (the C ABI in include/rowsplit_b200.h).

The library is built in-tree by ``paper_2603_28642_b200.build.build()``
(``make -C paper_2603_28642_b200/csrc``).  There is no CPU fallback: if the
library or a CUDA device is missing, the device entry points raise.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "librowsplit_b200.so")

RSB_OK, RSB_EINVAL, RSB_ESINGULAR, RSB_ECUDA, RSB_ENOMEM, RSB_ESTATE = range(6)
RSB_HOST, RSB_DEVICE, RSB_DEVICE_ASYNC = 0, 1, 2
RSB_DOT_EXACT, RSB_DOT_TREE = 0, 1
TRI_LOWER, TRI_LOWER_UNIT, TRI_UPPER, TRI_LOWER_T, TRI_LOWER_T_UNIT, TRI_UPPER_T = range(6)
S_DENSE, S_CG, S_IDENTITY = 0, 1, 2
Y_EXPLICIT, Y_IMPLICIT = 0, 1

i64 = ctypes.c_int64
i32 = ctypes.c_int32
f64 = ctypes.c_double
vp = ctypes.c_void_p
i64p = ctypes.POINTER(ctypes.c_int64)
f64p = ctypes.POINTER(ctypes.c_double)


class CglsCfgC(ctypes.Structure):
    _fields_ = [("norm_A", f64), ("delta", f64), ("max_iters", i64),
                ("estimator_delay", i32), ("ratio_raw", i32)]


class ReportC(ctypes.Structure):
    _fields_ = [("its", i64), ("iters_run", i64), ("converged", i32), ("breakdown", i32),
                ("ratio_pt_final", f64), ("residual_norm", f64), ("gradient_norm", f64),
                ("history_len", i64)]


# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGS = {
    "rsb_last_error": [],
    "rsb_version": [],
    "rsb_device_count": [ctypes.POINTER(ctypes.c_int)],
    "rsb_ctx_create": [ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)],
    "rsb_ctx_destroy": [vp],
    "rsb_ctx_sync": [vp],
    "rsb_ctx_stream": [vp, ctypes.POINTER(vp)],
    "rsb_ctx_kernel_launches": [vp, i64p, ctypes.c_int],
    "rsb_ctx_mem_bytes": [vp, i64p],
    "rsb_host_alloc": [i64, ctypes.POINTER(vp)],
    "rsb_host_free": [vp],
    "rsb_device_alloc": [vp, i64, ctypes.POINTER(vp)],
    "rsb_device_free": [vp, vp],
    "rsb_memcpy": [vp, vp, vp, i64, ctypes.c_int],
    "rsb_event_mark": [vp, ctypes.c_int],
    "rsb_event_elapsed": [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)],
    "rsb_mat_create": [vp, i64, i64, vp, vp, vp, ctypes.POINTER(vp)],
    "rsb_mat_destroy": [vp],
    "rsb_mat_info": [vp, i64p, i64p, i64p],
    "rsb_matvec": [vp, vp, vp, ctypes.c_int],
    "rsb_matvec_transpose": [vp, vp, vp, ctypes.c_int],
    "rsb_trsv": [vp, ctypes.c_int, vp, vp, ctypes.c_int],
    "rsb_trsv_levels": [vp, ctypes.c_int, i64p, i64p],
    "rsb_trsv_variant": [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
    "rsb_trsv_profile_levels": [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong), i64],
    "rsb_trsv_profile": [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)],
    "rsb_power_norm2": [vp, vp, ctypes.c_int, f64p],
    "rsb_dot": [vp, i64, vp, vp, f64p, ctypes.c_int],
    "rsb_chol_solve": [vp, i64, vp, vp, vp, ctypes.c_int],
    "rsb_pre_create": [vp, i64, i64, vp, vp, vp, vp, vp, vp, i64, ctypes.c_int, ctypes.c_int,
                       ctypes.c_int, ctypes.POINTER(vp)],
    "rsb_pre_destroy": [vp],
    "rsb_pre_apply": [vp, vp, vp, vp, ctypes.c_int],
    "rsb_pre_y_apply": [vp, vp, vp, ctypes.c_int],
    "rsb_pre_y_apply_transpose": [vp, vp, vp, ctypes.c_int],
    "rsb_pre_s_matvec": [vp, vp, vp, ctypes.c_int],
    "rsb_solver_create": [vp, vp, ctypes.POINTER(vp)],
    "rsb_solver_create_on": [vp, vp, vp, ctypes.POINTER(vp)],
    "rsb_solver_destroy": [vp],
    "rsb_solver_start": [vp, vp, ctypes.c_int, ctypes.POINTER(CglsCfgC), ctypes.POINTER(ctypes.c_int)],
    "rsb_solver_iterate": [vp, i64, i64p, ctypes.POINTER(ctypes.c_int)],
    "rsb_solver_get_x": [vp, vp, ctypes.c_int],
    "rsb_solver_finish": [vp, ctypes.POINTER(ReportC), vp, i64],
    "rsb_pcgls": [vp, vp, ctypes.c_int, ctypes.POINTER(CglsCfgC), vp, ctypes.POINTER(ReportC), vp, i64],
    "rsb_pcgls_many": [ctypes.c_int, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.c_int, ctypes.POINTER(CglsCfgC),
                       ctypes.POINTER(vp), ctypes.POINTER(ReportC), vp, i64],
    "rsb_solver_bench": [vp, i64, ctypes.c_int, f64p, f64p, i64p, i64p, ctypes.POINTER(ctypes.c_int)],
    "rsb_solver_bench_products": [vp, f64p, i64p],
    "rsb_l2_flush": [vp],
    "rsb_bsolver_create": [vp, vp, ctypes.POINTER(vp)],
    "rsb_bsolver_destroy": [vp],
    "rsb_bsolver_start": [vp, ctypes.c_int, vp, ctypes.c_int, ctypes.POINTER(CglsCfgC), ctypes.POINTER(ctypes.c_int)],
    "rsb_bsolver_iterate": [vp, i64, ctypes.POINTER(ctypes.c_int)],
    "rsb_bsolver_finish": [vp, vp, ctypes.c_int, ctypes.POINTER(ReportC), vp, i64],
    "rsb_pcgls_batch8": [vp, ctypes.c_int, vp, ctypes.c_int, ctypes.POINTER(CglsCfgC), vp, ctypes.POINTER(ReportC),
                         vp, i64],
    "rsb_bsolver_bench": [vp, i64, ctypes.c_int, f64p, f64p, i64p, i64p, ctypes.POINTER(ctypes.c_int)],
    "rsb_ilup_factorize": [i64, i64, vp, vp, vp, i64, f64, f64, f64, ctypes.POINTER(vp)],
    "rsb_ilup_sizes": [vp, i64p, i64p, i64p, i64p],
    "rsb_ilup_copy": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
    "rsb_ilup_destroy": [vp],
    "rsb_build_y_explicit": [i64, i64, vp, vp, vp, vp, vp, vp, i64p, vp, vp, vp],
    "rsb_cholesky_factorize": [i64, vp],
    "rsb_column_scale": [i64, vp, vp, vp, vp],
    "rsb_column_scale_device": [vp, i64, vp, vp, vp, vp],
    "rsb_dense_build": [vp, vp, ctypes.c_int, ctypes.POINTER(vp)],
    "rsb_dense_build_sizes": [vp, i64p, i64p, i64p, f64p],
    "rsb_dense_build_copy": [vp, vp, vp, vp, vp, vp],
    "rsb_dense_build_destroy": [vp],
    "rsb_cholesky_factorize_device": [vp, i64, vp, ctypes.c_int],
}
_RESTYPES = {"rsb_last_error": ctypes.c_char_p}

_lib = None
_lock = threading.Lock()


class LibraryMissingError(RuntimeError):
    pass


def lib():
    """Load librowsplit_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissingError(
                    f"{LIB_PATH} is not built; run paper_2603_28642_b200.build.build() "
                    "(there is no CPU fallback for the solve path)")
            L = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(rc):
    """Map an RSB status to the reference's exception types."""
    if rc == RSB_OK:
        return
    msg = lib().rsb_last_error().decode(errors="replace")
    if rc == RSB_EINVAL:
        raise ValueError(msg)
    if rc == RSB_ESINGULAR:
        raise np.linalg.LinAlgError(msg)
    raise RuntimeError(f"rowsplit_b200 error {rc}: {msg}")


def ptr(a):
    """Raw data pointer of a contiguous numpy array (None for empty arrays is avoided)."""
    return ctypes.c_void_p(a.ctypes.data)


def f64c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64c(a):
    return np.ascontiguousarray(a, dtype=np.int64)
