"""ctypes binding of libsbp.so (the C ABI in include/sbp.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_1010_0012_b200/csrc``).  There is no fallback: if the shared object is
missing or cannot be loaded, importing the engine raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

# SBP_LIB selects another in-tree build of the same C ABI (kernel A/B runs).
LIB_PATH = Path(__file__).resolve().parent / os.environ.get("SBP_LIB", "libsbp.so")

SBP_OK, SBP_EINVAL, SBP_ECUDA, SBP_EUNSUPPORTED = 0, -1, -2, -3
SBP_SUM, SBP_MAX = 0, 1
SBP_POT_BAND, SBP_POT_ELL, SBP_POT_DENSE = 0, 1, 2
SBP_MAX_R = 32
SBP_ERR_NONE = 0xFFFFFFFFFFFFFFFF
SBP_ITER_FIRST = 1
SBP_ACC_F32, SBP_ACC_F64 = 0, 1


SBP_DEVICE_AUTO = -1


class SbpGrid(ctypes.Structure):
    _fields_ = [("H", ctypes.c_int), ("W", ctypes.c_int), ("M", ctypes.c_int),
                ("Ms", ctypes.c_int), ("r0", ctypes.c_int), ("rows", ctypes.c_int),
                ("device", ctypes.c_int)]


class SbpPotential(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("domain", ctypes.c_int), ("floor_term", ctypes.c_int),
                ("R", ctypes.c_int), ("m_max", ctypes.c_int),
                ("fbar", ctypes.c_float * 2),
                ("band_w", (ctypes.c_float * (2 * SBP_MAX_R + 1)) * 2),
                ("ell_idx", ctypes.c_void_p * 2), ("ell_w", ctypes.c_void_p * 2),
                ("dense_t", ctypes.c_void_p * 2),
                ("n_pot", ctypes.c_int), ("fbar_all", ctypes.c_void_p),
                ("pid_h", ctypes.c_void_p), ("pid_v", ctypes.c_void_p),
                ("accumulate", ctypes.c_int), ("fbar64", ctypes.c_double * 2),
                ("ell_w_lo", ctypes.c_void_p * 2)]


class SbpError(RuntimeError):
    """A libsbp call failed (bad arguments, unsupported shape or CUDA error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"libsbp error {code}: {msg}")
        self.code = code


class UnsupportedByKernel(SbpError):
    pass


_lib = None

# (name, restype, argtypes) -- mirrors include/sbp.h
_P = ctypes.c_void_p
_i = ctypes.c_int
_PROTOS = {
    "sbp_version": (_i, []),
    "sbp_last_error": (ctypes.c_char_p, []),
    "sbp_reload_config": (_i, []),
    "sbp_padded_labels": (_i, [_i]),
    "sbp_band_radius": (_i, [_i, _i]),
    "sbp_init_msgs": (_i, [ctypes.POINTER(SbpGrid), _i, _i, _P, _P]),
    "sbp_load_values": (_i, [ctypes.POINTER(SbpGrid), _i, _P, _P, _P]),
    "sbp_stereo_values": (_i, [ctypes.POINTER(SbpGrid), _i, _P, _P, ctypes.c_double,
                               ctypes.c_double, _P, _P]),
    "sbp_iterate": (_i, [ctypes.POINTER(SbpGrid), ctypes.POINTER(SbpPotential), _P, _P, _P,
                         _i, _i, _i, _i, _P, _P]),
    "sbp_iterate_delta": (_i, [ctypes.POINTER(SbpGrid), ctypes.POINTER(SbpPotential), _P, _P,
                               _P, _i, _i, _i, _i, _P, _P, _P]),
    "sbp_sweep_delta": (_i, [ctypes.POINTER(SbpGrid), ctypes.POINTER(SbpPotential), _P, _P, _i,
                             _P, _P, _P]),
    "sbp_fused_stamp_words": (_i, [ctypes.POINTER(SbpGrid)]),
    "sbp_iterate_fused": (_i, [ctypes.POINTER(SbpGrid), ctypes.POINTER(SbpPotential), _P, _P, _P,
                               _i, _i, _i, _P, ctypes.c_uint, _i, _i, _P, _P]),
    "sbp_sweep": (_i, [ctypes.POINTER(SbpGrid), ctypes.POINTER(SbpPotential), _P, _P, _i, _P,
                       _P]),
    "sbp_plan_name": (_i, [ctypes.POINTER(SbpGrid), ctypes.POINTER(SbpPotential), _i,
                           ctypes.c_char_p, _i]),
    "sbp_beliefs": (_i, [ctypes.POINTER(SbpGrid), _i, _P, _P, _P, _P, _P, _P, _P]),
    "sbp_gather_store": (_i, [ctypes.POINTER(SbpGrid), _P, _P, _P]),
    "sbp_max_abs_diff": (_i, [ctypes.POINTER(SbpGrid), _P, _P, _P, _P]),
}


def lib():
    """Load libsbp.so once; raises if it is absent (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                              "(there is no CPU fallback)")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _PROTOS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc != SBP_OK:
        msg = lib().sbp_last_error().decode(errors="replace")
        if rc == SBP_EUNSUPPORTED:
            raise UnsupportedByKernel(rc, msg)
        raise SbpError(rc, msg)


def exported_symbols() -> list[str]:
    return list(_PROTOS)
