"""ctypes binding of libbandchol_b200.so (the C ABI declared in include/bandchol_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).  If it
is missing, or no CUDA device is visible, every entry point raises DeviceError:
there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes
import os

from .errors import BandCholError, DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BCG_LIB") or os.path.join(_HERE, "libbandchol_b200.so")

# (name, restype, argtypes) -- must match include/bandchol_b200.h
_i64, _i32p, _dp, _vp, _sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t
SIGNATURES = {
    "bcg_version": (ctypes.c_int, []),
    "bcg_last_error": (ctypes.c_char_p, []),
    "bcg_dpbtrf_workspace_size": (_sz, [_i64, _i64, _i64]),
    "bcg_dpbtrf": (ctypes.c_int, [_i64, _i64, _dp, _i64, _i32p, _vp, _sz, _vp]),
    "bcg_dpbtrf_batched_workspace_size": (_sz, [_i64, _i64, _i64, _i64]),
    "bcg_dpbsv_batched_workspace_size": (_sz, [_i64, _i64, _i64, _i64]),
    "bcg_dpbtrf_batched": (ctypes.c_int, [_i64, _i64, _dp, _i64, _i64, _i64, _i32p, _vp, _sz, _vp]),
    "bcg_dpbtrs": (ctypes.c_int, [_i64, _i64, _dp, _i64, _dp, _i64, _i64, _i32p, _vp]),
    "bcg_dpbtrs_batched": (ctypes.c_int, [_i64, _i64, _dp, _i64, _i64, _dp, _i64, _i64, _i32p, _vp]),
    "bcg_dpbtrs_batched_nrhs": (ctypes.c_int, [_i64, _i64, _dp, _i64, _i64, _dp, _i64, _i64, _i64, _i64, _i32p,
                                               _vp]),
    "bcg_dpbsv_batched": (ctypes.c_int, [_i64, _i64, _dp, _i64, _i64, _dp, _i64, _i64, _i32p, _vp, _sz, _vp]),
    "bcg_dpbtrf_fwd_batched": (ctypes.c_int, [_i64, _i64, _dp, _i64, _i64, _dp, _i64, _i64, _i32p, _dp, _vp]),
    "bcg_dpbtrs_bwd_batched": (ctypes.c_int, [_i64, _i64, _dp, _i64, _i64, _dp, _dp, _i64, _i64, _i32p, _vp]),
    "bcg_probe_fp64_peak": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double)]),
    "bcg_set_trace": (ctypes.c_int, [_vp, _sz]),
    "bcg_band_residual_workspace_size": (_sz, []),
    "bcg_band_residual": (ctypes.c_int, [_i64, _i64, _dp, _i64, _dp, _i64, _dp, _vp, _sz, _vp]),
    "bcg_band_residual_batched_workspace_size": (_sz, [_i64]),
    "bcg_band_residual_batched": (ctypes.c_int, [_i64, _i64, _dp, _i64, _i64, _dp, _i64, _i64, _i64, _dp, _vp,
                                                 _sz, _vp]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the CUDA library (raises DeviceError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code to an exception."""
    if rc == 0:
        return
    msg = load().bcg_last_error().decode(errors="replace")
    if rc < 0:
        raise BandCholError(f"{what}: illegal argument {-rc}: {msg}")
    raise DeviceError(f"{what}: CUDA error {rc}: {msg}")
