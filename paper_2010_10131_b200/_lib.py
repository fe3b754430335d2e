"""ctypes binding of libatk_cuda.so (include/atk.h).

The product path loads ONLY this in-tree library; if it is missing the import
fails loudly (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libatk_cuda.so"

ATK_MAX_ORDER = 8
ATK_F32, ATK_F64 = 0, 1
SOLVER_EIG, SOLVER_ALS, SOLVER_SVD = 0, 1, 2

u64 = C.c_uint64
dptr = C.POINTER(C.c_double)
u64ptr = C.POINTER(C.c_uint64)

SELECTOR_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64)


HOST_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_uint64)
HOST_BROADCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int)


class HostCollectives(C.Structure):
    _fields_ = [("allreduce_f64", HOST_ALLREDUCE_FN), ("broadcast", HOST_BROADCAST_FN),
                ("user", C.c_void_p)]


class RooflineParams(C.Structure):
    _fields_ = [("hbm_gbs", C.c_double), ("tf32_tflops", C.c_double), ("fp64_tflops", C.c_double),
                ("eig_small_ms", C.c_double), ("eig_large_ms", C.c_double),
                ("als_iter_overhead_ms", C.c_double), ("dtype", C.c_int), ("num_iters", C.c_int),
                ("als_fused_factor", C.c_double), ("als_fused_overhead_ms", C.c_double),
                ("num_sms", C.c_int)]


class AlsOpts(C.Structure):
    _fields_ = [("num_iters", C.c_int), ("rel_tol", C.c_double), ("seed", C.c_uint64)]


class StageTimes(C.Structure):
    _fields_ = [("gram_ms", C.c_double), ("eig_ms", C.c_double), ("ttm_ms", C.c_double),
                ("als_ms", C.c_double), ("comm_ms", C.c_double), ("total_ms", C.c_double)]


class ModeReportC(C.Structure):
    _fields_ = [("mode", C.c_int), ("solver_used", C.c_int), ("iterations_run", C.c_int),
                ("eig_method", C.c_int), ("selector_decision_time", C.c_double),
                ("solver_time", C.c_double), ("predicted_cost_eig", C.c_double),
                ("predicted_cost_als", C.c_double), ("dims_before", C.c_uint64 * ATK_MAX_ORDER),
                ("dims_after", C.c_uint64 * ATK_MAX_ORDER), ("times", StageTimes)]


class AllocStats(C.Structure):
    _fields_ = [("alloc_count", C.c_int64), ("live_elems", C.c_int64), ("peak_elems", C.c_int64),
                ("live_watched", C.c_int64), ("peak_watched", C.c_int64)]


# name -> (restype, argtypes); every atk_status-returning entry in atk.h.
_SIGS = {
    "atk_version": (C.c_char_p, []),
    "atk_last_error": (C.c_char_p, []),
    "atk_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "atk_ctx_destroy": (C.c_int, [C.c_void_p]),
    "atk_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "atk_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "atk_ctx_launch_count": (C.c_uint64, [C.c_void_p]),
    "atk_ctx_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_double]),
    "atk_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "atk_comm_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "atk_comm_destroy": (C.c_int, [C.c_void_p]),
    "atk_dten_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), u64ptr]),
    "atk_tensor_read_dten": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "atk_tensor_write_dten": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p]),
    "atk_comm_init_host": (C.c_int, [C.c_void_p, C.POINTER(HostCollectives), C.c_int, C.c_int]),
    "atk_comm_get_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64 * 4)]),
    "atk_comm_reset_stats": (C.c_int, [C.c_void_p]),
    "atk_tensor_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, u64ptr, C.POINTER(C.c_void_p)]),
    "atk_tensor_wrap": (C.c_int, [C.c_void_p, C.c_int, C.c_int, u64ptr, C.c_void_p, C.POINTER(C.c_void_p)]),
    "atk_tensor_from_host": (C.c_int, [C.c_void_p, C.c_int, C.c_int, u64ptr, C.c_void_p, C.POINTER(C.c_void_p)]),
    "atk_tensor_to_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "atk_tensor_free": (C.c_int, [C.c_void_p]),
    "atk_tensor_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), u64ptr, C.POINTER(C.c_void_p)]),
    "atk_fill_uniform": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64]),
    "atk_axpy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p]),
    "atk_frobenius_norm": (C.c_int, [C.c_void_p, C.c_void_p, dptr]),
    "atk_gram": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, dptr]),
    "atk_ttm": (C.c_int, [C.c_void_p, C.c_void_p, dptr, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]),
    "atk_ttt": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, dptr]),
    "atk_sym_eig_top_r": (C.c_int, [C.c_void_p, dptr, C.c_uint64, C.c_uint64, dptr, dptr]),
    "atk_thin_qr": (C.c_int, [C.c_void_p, dptr, C.c_uint64, C.c_uint64, dptr, dptr]),
    "atk_spd_solve": (C.c_int, [C.c_void_p, dptr, C.c_uint64, dptr, C.c_uint64, dptr]),
    "atk_eig_mode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, dptr, C.POINTER(C.c_void_p), C.POINTER(StageTimes)]),
    "atk_als_mode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.POINTER(AlsOpts), dptr, dptr,
                               C.POINTER(C.c_void_p), C.POINTER(C.c_int), C.POINTER(StageTimes)]),
    "atk_als_iterate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, dptr, C.c_uint64, C.POINTER(AlsOpts), dptr,
                                  C.POINTER(C.c_void_p), C.POINTER(C.c_int)]),
    "atk_svd_mode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, dptr, C.POINTER(C.c_void_p), C.POINTER(StageTimes)]),
    "atk_sthosvd": (C.c_int, [C.c_void_p, C.c_void_p, u64ptr, SELECTOR_FN, C.c_void_p, C.POINTER(AlsOpts),
                              C.POINTER(C.c_void_p), dptr, C.POINTER(ModeReportC)]),
    "atk_sthosvd_host": (C.c_int, [C.c_void_p, C.c_int, C.c_int, u64ptr, C.c_void_p, u64ptr, SELECTOR_FN, C.c_void_p,
                                   C.POINTER(AlsOpts), C.c_void_p, dptr, C.POINTER(ModeReportC)]),
    "atk_reconstruct": (C.c_int, [C.c_void_p, C.c_void_p, dptr, u64ptr, C.POINTER(C.c_void_p)]),
    "atk_relative_error": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, dptr, dptr]),
    "atk_reset_gemm_counters": (None, []),
    "atk_gemm_calls": (C.c_longlong, []),
    "atk_gemm_flops": (C.c_longlong, []),
    "atk_alloc_tracking_enable": (None, [C.c_uint64]),
    "atk_alloc_tracking_disable": (None, []),
    "atk_alloc_tracking_stats": (C.c_int, [C.POINTER(AllocStats)]),
    "atk_cost_eig": (C.c_double, [C.c_double, C.c_double, C.c_double]),
    "atk_cost_als": (C.c_double, [C.c_double, C.c_double, C.c_double, C.c_int]),
    "atk_roofline_params_default": (None, [C.POINTER(RooflineParams), C.c_int, C.c_int]),
    "atk_roofline_time_eig": (C.c_double, [C.POINTER(RooflineParams), C.c_double, C.c_double, C.c_double]),
    "atk_roofline_time_als": (C.c_double, [C.POINTER(RooflineParams), C.c_double, C.c_double, C.c_double]),
    "atk_roofline_time_als_mode": (C.c_double, [C.POINTER(RooflineParams), C.c_int, C.c_double, C.c_double,
                                                C.c_double]),
    "atk_roofline_selector": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]),
}

_lib = None


def load() -> C.CDLL:
    """Load libatk_cuda.so (built in-tree by paper_2010_10131_b200.build)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -m paper_2010_10131_b200.build` "
                "(the engine has no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(code: int) -> None:
    if code:
        msg = load().atk_last_error()
        raise_for_status(code, msg.decode() if msg else f"atk status {code}")
