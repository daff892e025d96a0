"""ctypes binding of libmact_cuda.so (the C ABI declared in include/mact_cuda.h).

This is the only door into the CUDA implementation.  There is no CPU
fallback: if the shared library is missing or no CUDA device is visible the
first call raises ``MactError`` loudly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import MactError, UnknownApproximant

_PKG = Path(__file__).resolve().parent
# MACT_LIB selects an alternative build (tuning variants); default: the in-tree library
LIB_PATH = Path(os.environ["MACT_LIB"]) if os.environ.get("MACT_LIB") else _PKG / "libmact_cuda.so"

MACT_OK, MACT_EBADARG, MACT_EUNKNOWN_APPROX, MACT_ECUDA = 0, 1, 2, 3
SPACES = {"lab": 0, "hsi": 1, "sct": 2}
LAYOUTS = {"interleaved": 0, "planar": 1}
DTYPE_U8, DTYPE_F32, DTYPE_F64 = 0, 1, 2
METHODS = {"trilinear": 0, "prism": 1, "pyramidal": 2, "tetrahedral": 3}
METRIC_DISTANCE, METRIC_COMPONENT = 0, 1
CAND_FAST, CAND_LUT, CAND_ARRAY, CAND_FAST_F64 = 0, 1, 2, 3
MAX_COEFFS = 8

_c_double8 = C.c_double * MAX_COEFFS


class MactCoeffs(C.Structure):
    _fields_ = [("cbrt_num_deg", C.c_int32), ("cbrt_den_deg", C.c_int32),
                ("hsi_deg", C.c_int32), ("asin_deg", C.c_int32), ("acos_deg", C.c_int32),
                ("atan_deg", C.c_int32),
                ("cbrt_num", _c_double8), ("cbrt_den", _c_double8), ("atan_sqrt3", _c_double8),
                ("asin_half", _c_double8), ("acos_half", _c_double8), ("atan_f", _c_double8),
                ("atan_g", _c_double8)]


class MactErrStats(C.Structure):
    _fields_ = [("sum", C.c_double), ("max", C.c_double), ("count", C.c_uint64),
                ("argmax", C.c_uint64), ("nan_count", C.c_uint64), ("_pad", C.c_uint64)]


class MactErrSpec(C.Structure):
    _fields_ = [("space", C.c_int32), ("metric", C.c_int32), ("candidate", C.c_int32),
                ("lut_grid_n", C.c_int32), ("lut_method", C.c_int32), ("cand_dtype", C.c_int32),
                ("lut_lattice", C.c_void_p), ("cand_array", C.c_void_p),
                ("ref_array", C.c_void_p), ("ref_dtype", C.c_int32), ("_pad", C.c_int32)]


class MactApproxSpec(C.Structure):
    _fields_ = [("fn", C.c_int32), ("a_deg", C.c_int32), ("b_deg", C.c_int32), ("_pad", C.c_int32),
                ("a", _c_double8), ("b", _c_double8)]


POLY_MAX = 32


class MactPolySpec(C.Structure):
    _fields_ = [("num_deg", C.c_int32), ("den_deg", C.c_int32),
                ("num", C.c_double * POLY_MAX), ("den", C.c_double * POLY_MAX)]


FN_FORM, FN_ATAN_SQRT3, FN_ACOS, FN_ATAN_UNIT = 0, 1, 2, 3
ELEM_INVERSE_GAMMA, ELEM_RGB_TO_XYZ, ELEM_LAB_F, ELEM_XYZ_TO_LAB, ELEM_ANGULAR_LERP = 0, 1, 2, 3, 4
# TargetFn.exact (approximants.py:101-115)
ELEM_TARGET = {"cbrt": 5, "atan_sqrt3": 6, "asin_half": 7, "acos_half": 8, "atan_f": 9, "atan_g": 10}
SPACE_HSI_ARCCOS = 3
LAB_PATH_SEG, LAB_PATH_MONIC, LAB_PATH_PQ = 1, 2, 3

_vp, _i, _i64, _u64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
_SIGNATURES = {
    "mact_lab_fast": (_i, [_vp, _i, _vp, _i64, C.POINTER(MactCoeffs), _i, _vp]),
    "mact_hsi_fast": (_i, [_vp, _i, _vp, _i64, C.POINTER(MactCoeffs), _i, _vp]),
    "mact_sct_fast": (_i, [_vp, _i, _vp, _i64, C.POINTER(MactCoeffs), _i, _vp]),
    "mact_all_fast": (_i, [_vp, _vp, _vp, _vp, _i64, C.POINTER(MactCoeffs), _i, _vp]),
    "mact_exact": (_i, [_i, _vp, _i, _vp, _i, _i64, _vp]),
    "mact_sct_to_rgb": (_i, [_vp, _vp, _i64, _vp]),
    "mact_distance": (_i, [_i, _vp, _i, _vp, _i, _vp, _i64, _vp]),
    "mact_lut_build": (_i, [_i, _i, _vp, _vp, _vp]),
    "mact_lut_interp": (_i, [_vp, _i, _i, _vp, _vp, _i64, _i, _vp]),
    "mact_lut_interp_angular": (_i, [_vp, _i, _i, _i, _vp, _vp, _i64, _i, _vp]),
    "mact_lut_interp_real": (_i, [_vp, _i, _i, _i, _vp, _i, _vp, _i, _i64, _i, _vp]),
    "mact_lut_cache_build": (_i, [_vp, _i, _vp, _vp, _vp]),
    "mact_lut_interp_cached": (_i, [_vp, _vp, _vp, _i, _i, _i, _vp, _i, _vp, _i, _i64, _i, _vp]),
    "mact_lut_nodes_timed": (_i, [_i, _i, _vp, _i64, _vp, _vp, _vp]),
    "mact_lut_nodes": (_i, [_i, _i, _vp, _i64, _vp, _vp, _vp]),
    "mact_lut_nodes_real": (_i, [_i, _i, _vp, _i, _i64, _vp, _vp, _vp]),
    "mact_err_workspace_bytes": (C.c_size_t, []),
    "mact_err_reduce": (_i, [C.POINTER(MactErrSpec), C.POINTER(MactCoeffs), _vp, _i64, _i64,
                             _i64, _vp, _vp, _vp]),
    "mact_cube_fill": (_i, [_vp, _i64, _i64, _vp]),
    "mact_call_counts": (_i, [_vp, _vp]),
    "mact_approx_eval": (_i, [C.POINTER(MactApproxSpec), _vp, _vp, _vp, _i64, _vp, _vp]),
    "mact_poly_eval": (_i, [C.POINTER(MactPolySpec), _vp, _vp, _i64, _vp, _vp]),
    "mact_exact_elem": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    "mact_exact_f32": (_i, [_i, _vp, _vp, _i64, _i, _vp]),
    "mact_fast_f64": (_i, [_i, _vp, _i, _vp, _i64, C.POINTER(MactCoeffs), _i, _vp]),
    "mact_probe_expand": (_i, [_vp, _vp, _i64, _vp]),
    "mact_host_ctx_create": (_i, [_i, _i64, _i, C.POINTER(_vp)]),
    "mact_host_ctx_destroy": (_i, [_vp]),
    "mact_transform_host": (_i, [_vp, _i, _vp, _vp, _i64, C.POINTER(MactCoeffs), _i]),
    "mact_transform_host_f64": (_i, [_vp, _i, _vp, _vp, _i64, C.POINTER(MactCoeffs), _i]),
    "mact_lut_interp_host": (_i, [_vp, _vp, _i, _i, _vp, _vp, _i64, _i]),
    "mact_last_error": (C.c_char_p, []),
    "mact_version": (_i, []),
    "mact_lab_eval_path": (_i, [C.POINTER(MactCoeffs)]),
    "mact_launch_count": (_u64, []),
    "mact_launch_count_reset": (None, []),
}
EXPORTS = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load (once) and type the shared library.  Loading needs no GPU."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise MactError(
                f"{p} is missing: build it with `python -m paper_1009_0854_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a C status to the reference's exception conventions."""
    if rc == MACT_OK:
        return
    msg = (load().mact_last_error() or b"").decode(errors="replace")
    if rc == MACT_EBADARG:
        raise ValueError(msg)
    if rc == MACT_EUNKNOWN_APPROX:
        raise UnknownApproximant(msg)
    raise MactError(msg or f"libmact_cuda error {rc}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
