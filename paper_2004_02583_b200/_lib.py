"""ctypes binding of libtenkit_b200.so (include/tenkit_b200.h).

The shared library is built in-tree by paper_2004_02583_b200/build.py. There
is no fallback: if the library cannot be built or loaded, or no CUDA device
is present, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtenkit_b200.so")
SYNTH_PATH = os.path.join(PKG, "libtkg_synth.so")

MAX_ORDER = 64
MAX_HISTORY = 64


class TkgError(C.Structure):
    _fields_ = [("code", C.c_int32), ("subtype", C.c_int32), ("message", C.c_char * 512)]


class TkgAlsConfig(C.Structure):
    _fields_ = [("eta", C.c_double), ("max_iters", C.c_int32), ("seed", C.c_uint64),
                ("init", C.POINTER(C.c_double)), ("init_rows", C.c_uint64), ("init_cols", C.c_uint64)]


class TkgFactorEngine(C.Structure):
    _fields_ = [("kind", C.c_int32), ("als", TkgAlsConfig)]


ENGINE_KINDS = {"svd": 0, "eig": 1, "als": 2}


class TkgModeReport(C.Structure):
    _fields_ = [("mode", C.c_int32), ("iterations", C.c_int32), ("status", C.c_int32),
                ("history_len", C.c_int32), ("achieved_eta", C.c_double), ("seconds", C.c_double),
                ("residual_history", C.c_double * MAX_HISTORY)]


class TkgReport(C.Structure):
    _fields_ = [("order", C.c_int32), ("n_modes", C.c_int32),
                ("per_mode", TkgModeReport * MAX_ORDER), ("relative_residual", C.c_double),
                ("seconds", C.c_double), ("h2d_seconds", C.c_double),
                ("d2h_seconds", C.c_double), ("residual_seconds", C.c_double),
                ("kernel_launches", C.c_uint64), ("tensor_passes", C.c_uint64),
                ("algorithmic_bytes", C.c_uint64)]


class TkgKernelStats(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("launches", C.c_uint64 * 8), ("bytes", C.c_double * 8),
                ("flops", C.c_double * 8)]


_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_ctxp = C.c_void_p

# (name, restype, argtypes) for every symbol include/tenkit_b200.h declares.
SIGNATURES = [
    ("tkg_version", C.c_char_p, []),
    ("tkg_create", C.c_int, [C.POINTER(_ctxp), C.c_int, C.POINTER(TkgError)]),
    ("tkg_destroy", C.c_int, [_ctxp]),
    ("tkg_t_hosvd", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, _u64p,
                              C.POINTER(TkgAlsConfig), C.c_int32, _dp, _dp,
                              C.POINTER(TkgReport), C.POINTER(TkgError)]),
    ("tkg_st_hosvd", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, _u64p, _u32p,
                               C.POINTER(TkgAlsConfig), _dp, _dp, C.POINTER(TkgReport),
                               C.POINTER(TkgError)]),
    ("tkg_t_hosvd_engine", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, _u64p,
                                     C.POINTER(TkgFactorEngine), C.c_int32, _dp, _dp,
                                     C.POINTER(TkgReport), C.POINTER(TkgError)]),
    ("tkg_st_hosvd_engine", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, _u64p, _u32p,
                                      C.POINTER(TkgFactorEngine), _dp, _dp, C.POINTER(TkgReport),
                                      C.POINTER(TkgError)]),
    ("tkg_hooi", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, _u64p, _dp, _dp, C.c_double,
                           C.c_int32, _dp, _dp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), _dp, _dp,
                           C.POINTER(TkgError)]),
    ("tkg_device_alloc", C.c_int, [_ctxp, C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(TkgError)]),
    ("tkg_device_free", C.c_int, [_ctxp, C.c_void_p]),
    ("tkg_device_copy", C.c_int, [_ctxp, C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(TkgError)]),
    ("tkg_read_tnsr_shape", C.c_int, [C.c_char_p, C.POINTER(C.c_int32), _u64p, C.POINTER(TkgError)]),
    ("tkg_read_tnsr", C.c_int, [_ctxp, C.c_char_p, C.c_void_p, C.c_int, C.POINTER(TkgError)]),
    ("tkg_write_tnsr", C.c_int, [C.c_char_p, C.c_int32, _u64p, _dp, C.POINTER(TkgError)]),
    ("tkg_write_tukr", C.c_int, [C.c_char_p, C.c_int32, _u64p, _u64p, _dp, _dp, C.POINTER(TkgError)]),
    ("tkg_multi_mode_product", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, C.c_int32, _u32p, C.POINTER(_dp), _u64p,
                                         _u64p, _dp, C.POINTER(TkgError)]),
    ("tkg_reconstruct", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, _u64p, _dp, _dp, C.POINTER(TkgError)]),
    ("tkg_mode_gram", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, C.c_uint32, _dp, C.POINTER(TkgError)]),
    ("tkg_sym_eig", C.c_int, [_ctxp, _dp, C.c_uint64, C.c_uint64, _dp, _dp, C.POINTER(TkgError)]),
    ("tkg_residual_history", C.c_int, [_ctxp, C.c_int32, _dp, C.c_uint64, _u64p, C.POINTER(TkgError)]),
    ("tkg_select_order", C.c_int, [C.c_int32, _u64p, _u64p, _u32p, C.POINTER(TkgError)]),
    ("tkg_nccl_unique_id", C.c_int, [C.c_void_p, C.POINTER(TkgError)]),
    ("tkg_comm_init_nccl", C.c_int, [_ctxp, C.c_int, C.c_int, C.c_void_p, C.POINTER(TkgError)]),
    ("tkg_local_group_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p), C.POINTER(TkgError)]),
    ("tkg_local_group_destroy", None, [C.c_void_p]),
    ("tkg_comm_init_local", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.POINTER(TkgError)]),
    ("tkg_comm_init_shm", C.c_int, [_ctxp, C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.POINTER(TkgError)]),
    ("tkg_shard_range", C.c_int, [C.c_uint64, C.c_int, C.c_int, _u64p, _u64p]),
    ("tkg_t_hosvd_sharded", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, C.c_uint64, C.c_uint64,
                                      _u64p, C.POINTER(TkgAlsConfig), C.c_int32, _dp, _dp,
                                      C.POINTER(TkgReport), C.POINTER(TkgError)]),
    ("tkg_st_hosvd_sharded", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, C.c_uint64, C.c_uint64,
                                       _u64p, _u32p, C.POINTER(TkgAlsConfig), _dp, _dp, C.POINTER(TkgReport),
                                       C.POINTER(TkgError)]),
    ("tkg_als_low_rank", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, C.c_uint32,
                                   C.c_uint64, C.POINTER(TkgAlsConfig), _dp, _dp,
                                   C.POINTER(TkgModeReport), C.POINTER(TkgError)]),
    ("tkg_als_init", C.c_int, [_ctxp, C.c_void_p, C.c_int, C.c_int32, _u64p, C.c_uint32,
                               C.c_uint64, C.c_uint64, _dp, C.POINTER(TkgError)]),
    ("tkg_als_sweep", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, C.c_uint32, _dp, C.c_uint64, _dp, _dp, _dp,
                                C.POINTER(TkgError)]),
    ("tkg_unfold_times", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, C.c_uint32, _dp, C.c_uint64,
                                   _dp, C.POINTER(TkgError)]),
    ("tkg_unfold_t_times", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, C.c_uint32, _dp, C.c_uint64,
                                     _dp, C.POINTER(TkgError)]),
    ("tkg_mode_n_product", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, _dp, C.c_uint64, C.c_uint64,
                                     C.c_uint32, _dp, C.POINTER(TkgError)]),
    ("tkg_frobenius_norm", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, _dp, C.POINTER(TkgError)]),
    ("tkg_relative_error", C.c_int, [_ctxp, _dp, _dp, C.c_int32, _u64p, _dp,
                                     C.POINTER(TkgError)]),
    ("tkg_reduced_qr", C.c_int, [_ctxp, _dp, C.c_uint64, C.c_uint64, _dp, _dp,
                                 C.POINTER(TkgError)]),
    ("tkg_gram", C.c_int, [_ctxp, _dp, C.c_uint64, C.c_uint64, _dp, C.POINTER(TkgError)]),
    ("tkg_recover_singular_vectors", C.c_int, [_ctxp, _dp, C.c_int32, _u64p, C.c_uint32, _dp, C.c_uint64,
                                               C.c_uint64, _dp, C.POINTER(TkgError)]),
    ("tkg_uniform01", C.c_int, [_ctxp, C.c_uint64, C.c_uint32, C.c_uint64, _dp,
                                C.POINTER(TkgError)]),
    ("tkg_set_profiling", C.c_int, [_ctxp, C.c_int]),
    ("tkg_set_fused_sweep", C.c_int, [_ctxp, C.c_int]),
    ("tkg_get_kernel_stats", C.c_int, [_ctxp, C.POINTER(TkgKernelStats)]),
    ("tkg_timer_start", C.c_int, [_ctxp]),
    ("tkg_timer_stop", C.c_int, [_ctxp, _dp]),
    ("tkg_flush_l2", C.c_int, [_ctxp]),
    ("tkg_bench_contractions", C.c_int, [_ctxp, C.c_void_p, C.c_int32, _u64p, C.c_uint32,
                                         C.c_uint32, C.c_int32, _dp, C.POINTER(TkgError)]),
]

_lock = threading.Lock()
_lib = None
_synth = None


def ensure_built() -> str:
    """Build the library in-tree if it is missing (nvcc is in the image)."""
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            path = ensure_built()
            handle = C.CDLL(path)
            for name, res, args in SIGNATURES:
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
        return _lib


def synth_lib():
    global _synth
    with _lock:
        if _synth is None:
            if not os.path.exists(SYNTH_PATH):
                from . import build as _build
                _build.build_synth(force=True)
            h = C.CDLL(SYNTH_PATH)
            h.tkg_synth_tucker.restype = C.c_int
            h.tkg_synth_tucker.argtypes = [C.c_int, _u64p, _u64p, C.c_double, C.c_double,
                                           C.c_uint64, _dp]
            h.tkg_synth_tucker_slab.restype = C.c_int
            h.tkg_synth_tucker_slab.argtypes = [C.c_int, _u64p, _u64p, C.c_double, C.c_uint64,
                                                C.c_uint64, C.c_uint64, _dp, _dp]
            h.tkg_synth_add_noise.restype = C.c_int
            h.tkg_synth_add_noise.argtypes = [C.c_int, _u64p, C.c_uint64, C.c_uint64, C.c_uint64,
                                              C.c_double, _dp]
            h.tkg_synth_noise_scale.restype = C.c_double
            h.tkg_synth_noise_scale.argtypes = [C.c_uint64, _dp, C.c_double]
            _synth = h
        return _synth


def u64(seq):
    return (C.c_uint64 * len(seq))(*[int(x) for x in seq])


def u32(seq):
    return (C.c_uint32 * len(seq))(*[int(x) for x in seq])
