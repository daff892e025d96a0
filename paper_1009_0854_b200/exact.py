"""Exact (fp64) transforms and distances on B200 — drop-in for ``mact.exact``.

    rgb_to_lab_exact / rgb_to_hsi_exact / rgb_to_sct_exact   (exact.py:86-149)
    rgb_to_hsi_arccos                                        (exact.py:104-116)
    inverse_gamma / rgb_to_xyz / lab_f / xyz_to_lab          (exact.py:52-83)
    sct_to_rgb                                               (exact.py:152-160)
    lab_distance / hsi_distance / sct_distance_indirect      (exact.py:163-190)

These compute in float64 on the device with libdevice cbrt/pow/atan/acos/
atan2/sincos and return float64 (the reference's dtype).  Device tensors in ->
device tensors out; numpy in -> numpy out.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _lib

TWO_PI = 2.0 * np.pi
GAMMA_KNEE, GAMMA_SLOPE, GAMMA_OFFSET, GAMMA_SCALE, GAMMA_POWER = 0.081, 4.5, 0.099, 1.099, 1.0 / 0.45
RGB_TO_XYZ_MATRIX = np.array([[0.412391, 0.357584, 0.180481],
                              [0.212639, 0.715169, 0.072192],
                              [0.019331, 0.119195, 0.950532]])
WHITE_X, WHITE_Y, WHITE_Z = 0.950456, 1.0, 1.089058
LAB_KNEE, LAB_LINEAR_SLOPE, LAB_LINEAR_OFFSET = 0.008856, 7.787, 16.0 / 116.0


def _exact(space: str, pixels, out_dtype: str = "float64"):
    import torch

    t, code, lead, on_dev = _dev.as_device_pixels(pixels)
    tdt = torch.float64 if out_dtype == "float64" else torch.float32
    res = torch.empty(lead + (3,), dtype=tdt, device=t.device)
    _lib.call("mact_exact", _lib.SPACES[space], t.data_ptr(), code, res.data_ptr(),
              _lib.DTYPE_F64 if out_dtype == "float64" else _lib.DTYPE_F32, t.numel() // 3,
              _dev.stream_ptr())
    return _dev.to_caller(res, on_dev)


def rgb_to_lab_exact(pixels, *, out_dtype: str = "float64"):
    """RGB (0..255, integer or real) -> CIELAB (exact.py:86-92)."""
    return _exact("lab", pixels, out_dtype)


def rgb_to_hsi_exact(pixels, *, out_dtype: str = "float64"):
    """RGB -> HSI, arctangent hue case analysis, NaN hue on grays (exact.py:119-137)."""
    return _exact("hsi", pixels, out_dtype)


def rgb_to_sct_exact(pixels, *, out_dtype: str = "float64"):
    """RGB -> spherical coordinates (L, angle_a, angle_b) (exact.py:140-149)."""
    return _exact("sct", pixels, out_dtype)


def exact_f32(space: str, pixels, *, layout: str = "interleaved"):
    """The exact transform formulas in fp32 libdevice arithmetic (mact_exact_f32):
    the B200 comparator for the paper's Table 4 gain.  uint8 pixels, fp32 out."""
    t, code, lead, on_dev = _dev.as_device_pixels(pixels)
    if code != _lib.DTYPE_U8:
        raise ValueError("exact_f32 takes 8-bit pixels")
    res = _dev.empty_out(lead, layout, t.device)
    _lib.call("mact_exact_f32", _lib.SPACES[space], t.data_ptr(), res.data_ptr(), t.numel() // 3,
              _lib.LAYOUTS[layout], _dev.stream_ptr())
    return _dev.to_caller(res, on_dev)


def rgb_to_hsi_arccos(pixels, *, out_dtype: str = "float64"):
    """RGB -> HSI via the inverse-cosine hue formula (exact.py:104-116)."""
    import torch

    t, code, lead, on_dev = _dev.as_device_pixels(pixels)
    tdt = torch.float64 if out_dtype == "float64" else torch.float32
    res = torch.empty(lead + (3,), dtype=tdt, device=t.device)
    _lib.call("mact_exact", _lib.SPACE_HSI_ARCCOS, t.data_ptr(), code, res.data_ptr(),
              _lib.DTYPE_F64 if out_dtype == "float64" else _lib.DTYPE_F32, t.numel() // 3,
              _dev.stream_ptr())
    return _dev.to_caller(res, on_dev)


def _f64_args(*xs):
    """Broadcast fp64 device copies of the arguments; on_dev if the first was a CUDA tensor."""
    import torch

    on_dev = _dev.is_device_tensor(xs[0])
    ts = [_as_f64_device(x)[0] for x in xs]
    if len(ts) > 1:
        ts = [t.contiguous() for t in torch.broadcast_tensors(*ts)]
    return ts, on_dev


def _elem(op: int, *xs, outs: int = 1, stacked: bool = False):
    import torch

    ts, on_dev = _f64_args(*xs)
    shape = ts[0].shape + ((3,) if stacked else ())
    res = [torch.empty(shape, dtype=torch.float64, device=ts[0].device) for _ in range(outs)]
    ptr = [t.data_ptr() for t in ts] + [None] * (3 - len(ts))
    optr = [r.data_ptr() for r in res] + [None] * (3 - len(res))
    _lib.call("mact_exact_elem", op, *ptr, *optr, ts[0].numel(), _dev.stream_ptr())
    out = [_dev.to_caller(r, on_dev) for r in res]
    return out[0] if outs == 1 else tuple(out)


def inverse_gamma(k_prime):
    """Nonlinear 0..1 channel value -> linear intensity, BT.709 (exact.py:52-57)."""
    return _elem(_lib.ELEM_INVERSE_GAMMA, k_prime)


def rgb_to_xyz(r, g, b):
    """Linear RGB in [0,1] -> (X, Y, Z) (exact.py:60-66)."""
    return _elem(_lib.ELEM_RGB_TO_XYZ, r, g, b, outs=3)


def lab_f(t):
    """Lightness kernel: cube root above the knee, linear below (exact.py:69-72)."""
    return _elem(_lib.ELEM_LAB_F, t)


def xyz_to_lab(x, y, z):
    """CIEXYZ -> CIELAB, D65 white, stacked (..., 3) (exact.py:75-83)."""
    return _elem(_lib.ELEM_XYZ_TO_LAB, x, y, z, stacked=True)


def _as_f64_device(x):
    import torch

    if _dev.is_device_tensor(x):
        return x.to(torch.float64).contiguous(), True
    _dev.require_cuda()
    a = np.asarray(x, dtype=np.float64)
    if not a.flags.c_contiguous:                     # (np.ascontiguousarray would make 0-d arrays 1-d)
        a = a.copy()
    return torch.from_numpy(a).cuda(), False


def sct_to_rgb(pixels):
    """Spherical coordinates -> real RGB; undefined angle_b acts as 0 (exact.py:152-160)."""
    import torch

    t, on_dev = _as_f64_device(pixels)
    res = torch.empty_like(t)
    _lib.call("mact_sct_to_rgb", t.data_ptr(), res.data_ptr(), t.numel() // 3, _dev.stream_ptr())
    return _dev.to_caller(res, on_dev)


def _distance(space: str, x, y):
    import torch

    tx, on_dev = _as_f64_device(x)
    ty, _ = _as_f64_device(y)
    if tx.shape != ty.shape:
        tx, ty = torch.broadcast_tensors(tx, ty)
        tx, ty = tx.contiguous(), ty.contiguous()
    res = torch.empty(tx.shape[:-1], dtype=torch.float64, device=tx.device)
    _lib.call("mact_distance", _lib.SPACES[space], tx.data_ptr(), _lib.DTYPE_F64, ty.data_ptr(),
              _lib.DTYPE_F64, res.data_ptr(), tx.numel() // 3, _dev.stream_ptr())
    return _dev.to_caller(res, on_dev)


def lab_distance(x, y):
    """Euclidean ΔE*ab (exact.py:163-166)."""
    return _distance("lab", x, y)


def hsi_distance(x, y):
    """Cylindrical HSI distance, hue on the shorter arc, NaN hue -> 0 (exact.py:169-178)."""
    return _distance("hsi", x, y)


def sct_distance_indirect(x, y):
    """SCT pixels mapped back to clamped RGB, scored in CIELAB (exact.py:181-190)."""
    return _distance("sct", x, y)


DISTANCES = {"lab": lab_distance, "hsi": hsi_distance, "sct": sct_distance_indirect}
