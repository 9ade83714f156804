"""ctypes binding of the dcdg C ABI (include/dcdg.h).

Loads the in-tree ``libdcdg.so`` built by ``paper_1902_08653_b200.build``.
There is no fallback: if the library is missing the import fails, and if no
CUDA device is present every call raises ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("DCDG_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdcdg.so")

DCDG_OK, DCDG_EINVAL, DCDG_ENUMERIC, DCDG_ECUDA, DCDG_ENCCL = 0, 1, 2, 3, 4
FP32, FP16 = 0, 1
FUSION_OPTIMAL, FUSION_UNIFORM = 0, 1
ALG_SWEEP, ALG_GRAM = 0, 1


class DcdgError(Exception):
    status = -1


class InvalidArgument(DcdgError, ValueError):
    """std::invalid_argument in the reference."""
    status = DCDG_EINVAL


class NumericError(DcdgError, RuntimeError):
    """std::runtime_error in the reference (zero row, zero beamformer, singular Gram)."""
    status = DCDG_ENUMERIC


class CudaError(DcdgError, RuntimeError):
    status = DCDG_ECUDA


class NcclError(DcdgError, RuntimeError):
    status = DCDG_ENCCL


_ERR = {DCDG_EINVAL: InvalidArgument, DCDG_ENUMERIC: NumericError, DCDG_ECUDA: CudaError, DCDG_ENCCL: NcclError}

_vp = C.c_void_p
_fp = C.POINTER(C.c_float)

# name -> (restype, argtypes); every symbol include/dcdg.h declares
SIGNATURES = {
    "dcdg_abi_version": (C.c_int, []),
    "dcdg_device_count": (C.c_int, []),
    "dcdg_init": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "dcdg_destroy": (C.c_int, [_vp]),
    "dcdg_last_error": (C.c_char_p, []),
    "dcdg_last_error_problem": (C.c_longlong, []),
    "dcdg_ul_detect": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.c_double, C.c_double, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "dcdg_dl_precode": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_double, C.c_int, _vp, _vp, _vp, _vp]),
    "dcdg_post_eq_variance": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                        _vp, _vp]),
    "dcdg_ul_trace": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                _vp, _vp, _vp]),
    "dcdg_dl_trace": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "dcdg_fuse": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp]),
    "dcdg_gain_reduce": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "dcdg_fuse_finalize": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, _vp]),
    "dcdg_gain_part": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "dcdg_power_scale": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_double, C.c_int, _vp]),
    "dcdg_fusion_weights": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp]),
    "dcdg_sync_status": (C.c_int, [_vp, _vp]),
    "dcdg_status_enqueue": (C.c_int, [_vp, _vp, _vp]),
    "dcdg_status_decode": (C.c_int, [_vp, C.c_ulonglong]),
    "dcdg_launch_count": (C.c_uint64, [_vp]),
    "dcdg_round_fp16": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "dcdg_mmse_bias": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _vp,
                                 _vp]),
    "dcdg_slice": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int64, C.c_int, C.c_double, _vp, _vp]),
    "dcdg_bit_errors": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int, _vp, _vp]),
    "dcdg_dl_receive": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_double, _vp, _vp, _vp, _vp]),
    "dcdg_convert": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, C.c_int64, _vp]),
    "dcdg_synth": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                             C.c_uint64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dcdg_mf_detect": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "dcdg_mf_precode": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _vp, _vp]),
    "dcdg_lmmse_exact": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, _vp,
                                   _vp]),
    "dcdg_zf_exact": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _vp, _vp]),
    "dcdg_kernel_name": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int]),
    "dcdg_ctx_kernel_name": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int]),
    "dcdg_set_fp16_algorithm": (C.c_int, [C.c_void_p, C.c_int]),
    "dcdg_xwin_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int64, C.POINTER(_vp)]),
    "dcdg_xwin_handle": (C.c_int, [_vp, _vp]),
    "dcdg_xwin_open": (C.c_int, [_vp, C.c_int, _vp]),
    "dcdg_xwin_set_timeout": (C.c_int, [_vp, C.c_int64]),
    "dcdg_xwin_destroy": (C.c_int, [_vp]),
    "dcdg_ul_detect_xchg": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _vp, _vp]),
    "dcdg_dl_precode_xchg": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_double, C.c_int, _vp, _vp, _vp]),
}

XWIN_HANDLE_BYTES = 64

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1902_08653_b200.build` "
                              "(there is no CPU fallback for the CD kernels)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == DCDG_OK:
        return
    msg = lib().dcdg_last_error().decode()
    err = _ERR.get(rc, DcdgError)(msg)
    err.problem = int(lib().dcdg_last_error_problem())
    raise err


def kernel_name(direction: int, bc: int, u: int, fmt: int) -> str:
    buf = C.create_string_buffer(96)
    lib().dcdg_kernel_name(direction, bc, u, fmt, buf, 96)
    return buf.value.decode()
