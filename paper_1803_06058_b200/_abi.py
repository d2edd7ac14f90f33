"""ctypes mirror of include/love.h (argument marshalling only; no arithmetic here)."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblove.so")

LOVE_OK, LOVE_ERR_ARG, LOVE_ERR_RANGE, LOVE_ERR_NOT_PD, LOVE_ERR_ZERO_PROBE = 0, 1, 2, 3, 4
LOVE_ERR_CUDA, LOVE_ERR_NCCL, LOVE_ERR_OOM, LOVE_ERR_STATE = 5, 6, 7, 8
STATUS_NAMES = {0: "OK", 1: "ERR_ARG", 2: "ERR_RANGE", 3: "ERR_NOT_PD", 4: "ERR_ZERO_PROBE",
                5: "ERR_CUDA", 6: "ERR_NCCL", 7: "ERR_OOM", 8: "ERR_STATE"}
LOVE_FP32, LOVE_FP64 = 0, 1
LOVE_PROBE_Y, LOVE_PROBE_AVGCOL = 0, 1
LOVE_PRIOR_SKI, LOVE_PRIOR_EXACT = 0, 1
LOVE_EXPORT_RC, LOVE_EXPORT_MEAN, LOVE_EXPORT_S, LOVE_EXPORT_PERM = 0, 1, 2, 3
LOVE_CACHE_FP64_AUTO, LOVE_CACHE_FP64_ON, LOVE_CACHE_FP64_OFF = 0, 1, 2
PROF_NAMES = ["setup", "scatter", "kuu", "gather", "reorth_dots", "reorth_update", "scalars_rc",
              "finish", "query", "sample_cache", "sample", "comm", "fused_pass", "sample_gemm"]


class love_grid(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("m", ctypes.c_int64 * 3), ("lo", ctypes.c_double * 3), ("h", ctypes.c_double * 3)]


class love_rbf(ctypes.Structure):
    _fields_ = [("outputscale", ctypes.c_double), ("lengthscale", ctypes.c_double * 3)]


class love_opts(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_int32), ("probe", ctypes.c_int32), ("prior", ctypes.c_int32),
                ("reorth_passes", ctypes.c_int32), ("breakdown_tol", ctypes.c_double),
                ("k_sample", ctypes.c_int32), ("lanczos_mode", ctypes.c_int32), ("var_blocks", ctypes.c_int32),
                ("reorth_tol", ctypes.c_double), ("cache_fp64", ctypes.c_int32), ("reserved1", ctypes.c_int32)]


class love_axis(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("lo", ctypes.c_double), ("h", ctypes.c_double),
                ("lengthscale", ctypes.c_double), ("outputscale", ctypes.c_double)]


class love_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p)]


class love_info(ctypes.Structure):
    _fields_ = [("k_eff", ctypes.c_int32), ("k_pad", ctypes.c_int32),
                ("k_sample_eff", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("n_local", ctypes.c_int64), ("n_global", ctypes.c_int64),
                ("m_total", ctypes.c_int64), ("n_items", ctypes.c_int64),
                ("b_norm", ctypes.c_double),
                ("alpha", ctypes.POINTER(ctypes.c_double)), ("beta", ctypes.POINTER(ctypes.c_double)),
                ("n_negative_var", ctypes.c_int64), ("n_out_of_range", ctypes.c_int64), ("n_reorth_steps", ctypes.c_int32), ("cache_precision", ctypes.c_int32)]


# name -> (restype, argtypes); every symbol include/love.h declares
SIGNATURES = {
    "love_build_cache": (ctypes.c_int, [ctypes.POINTER(love_grid), ctypes.POINTER(love_rbf), ctypes.c_double,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                        ctypes.POINTER(love_opts), ctypes.POINTER(love_dist), ctypes.c_void_p,
                                        ctypes.POINTER(ctypes.c_void_p)]),
    "love_build_cache_additive": (ctypes.c_int, [ctypes.POINTER(love_axis), ctypes.c_int32, ctypes.c_double,
                                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                                 ctypes.POINTER(love_opts), ctypes.POINTER(love_dist),
                                                 ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "love_predict_var": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "love_predict_covar": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "love_sample": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "love_cache_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(love_info)]),
    "love_free": (None, [ctypes.c_void_p]),
    "love_last_error": (ctypes.c_char_p, []),
    "love_ski_mvm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "love_kuu_mvm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "love_cache_export": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p]),
    "love_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "love_launch_count": (ctypes.c_int64, []),
    "love_abi_version": (ctypes.c_int32, []),
    "love_profile_enable": (None, [ctypes.c_int32]),
    "love_profile_read": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]),
}

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load liblove.so (in-tree; LOVE_LIB overrides the path for A/B builds of the same
    sources).  Raises if it has not been built: there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("LOVE_LIB", path)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run `make -C paper_1803_06058_b200` "
                           "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
