"""MACT fast transforms on B200 — drop-in for ``mact.fast`` (reference fast.py).

Same entry points, same arguments:

    rgb_to_lab_fast(pixels, cfg=DEFAULT_CONFIG)   # fast.py:86-107
    rgb_to_hsi_fast(pixels, cfg=DEFAULT_CONFIG)   # fast.py:125-148
    rgb_to_sct_fast(pixels, cfg=DEFAULT_CONFIG)   # fast.py:188-203

``pixels`` is any ``(..., 3)`` array.  Integer input takes the 8-bit table path,
real input the analytic path, as in the reference.  Differences, all
documented in DESIGN.md:

* results are float32 (the reference returns float64) — within the north-star
  tolerance (1e-4 on L*a*b*, 1e-5 on normalised H/S/I and SCT);
* a CUDA tensor in gives a CUDA tensor out (no host round trip); a numpy
  array in gives a numpy array out, streamed through the native host executor;
* keyword-only extras: ``out=`` (preallocated result) and ``layout=``
  ("interleaved" (...,3) or "planar" (3,...)).

Every call runs libmact_cuda kernels; there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

import numpy as np

from . import _dev, _lib
from .approximants import Rational, TargetFn, hsi_refit, registry_get
from .errors import DegenerateDenominator, UndefinedAngle

TWO_PI = 2.0 * np.pi


def _inverse_gamma_table() -> np.ndarray:
    k = np.arange(256) / 255.0
    with np.errstate(invalid="ignore"):
        curved = ((k + 0.099) / 1.099) ** (1.0 / 0.45)
    return np.where(k < 0.081, k / 4.5, curved)


# Linearised 8-bit channel values (reference fast.py:35); informational — the
# kernels rebuild the same table on device.
GAMMA_TABLE = _inverse_gamma_table()


def _fill(dst, coeffs) -> int:
    for i, c in enumerate(coeffs):
        dst[i] = float(c)
    return len(coeffs) - 1


@dataclass(frozen=True)
class MactConfig:
    """Degree selection (reference fast.py:46-78).  Defaults: CIELAB rational
    (4,4), HSI degree 5, SCT (n_asin, m_acos, r_atan) = (5,5,5)."""

    cielab_degrees: Tuple[int, int] = (4, 4)
    hsi_degree: int = 5
    sct_degrees: Tuple[int, int, int] = (5, 5, 5)

    def __post_init__(self):
        n, m = self.cielab_degrees
        object.__setattr__(self, "cbrt_approx", registry_get(TargetFn.CBRT, (n, m)))
        registry_get(TargetFn.ATAN_SQRT3, (self.hsi_degree,))   # degree must be bundled
        object.__setattr__(self, "atan_sqrt3_approx", hsi_refit(self.hsi_degree))
        a, c, t = self.sct_degrees
        object.__setattr__(self, "asin_approx", registry_get(TargetFn.ASIN_HALF, (a,)))
        object.__setattr__(self, "acos_approx", registry_get(TargetFn.ACOS_HALF, (c,)))
        object.__setattr__(self, "atan_f_approx", registry_get(TargetFn.ATAN_F, (t,)))
        object.__setattr__(self, "atan_g_approx", registry_get(TargetFn.ATAN_G, (t,)))
        object.__setattr__(self, "coeffs", self._pack())

    def _pack(self) -> _lib.MactCoeffs:
        k = _lib.MactCoeffs()
        rat: Rational = self.cbrt_approx.form
        k.cbrt_num_deg = _fill(k.cbrt_num, rat.numerator.coeffs)
        k.cbrt_den_deg = _fill(k.cbrt_den, rat.denominator.coeffs)
        k.hsi_deg = _fill(k.atan_sqrt3, self.atan_sqrt3_approx.form.coeffs)
        k.asin_deg = _fill(k.asin_half, self.asin_approx.form.coeffs)
        k.acos_deg = _fill(k.acos_half, self.acos_approx.form.coeffs)
        k.atan_deg = _fill(k.atan_f, self.atan_f_approx.form.coeffs)
        _fill(k.atan_g, self.atan_g_approx.form.coeffs)
        return k


DEFAULT_CONFIG = MactConfig()

_ENTRY = {"lab": "mact_lab_fast", "hsi": "mact_hsi_fast", "sct": "mact_sct_fast"}


def _host_u8(space: str, arr: np.ndarray, cfg: MactConfig, out, layout: str, out_dtype: str = "float32"):
    """numpy uint8 -> numpy fp32 (or fp64, the fidelity mode) through the native chunked
    H2D/kernel/D2H executor."""
    import torch

    src = np.ascontiguousarray(arr)
    lead = src.shape[:-1]
    n = int(np.prod(lead, dtype=np.int64)) if lead else 1
    out = _dev.host_out(out, lead, layout, np.float64 if out_dtype == "float64" else np.float32)
    _dev.host_call("mact_transform_host_f64" if out_dtype == "float64" else "mact_transform_host",
                   torch.cuda.current_device(), _lib.SPACES[space], _dev.np_ptr(src),
                   _dev.np_ptr(out), n, cfg.coeffs, _lib.LAYOUTS[layout])
    return out


def transform(space: str, pixels, cfg: MactConfig = DEFAULT_CONFIG, *, out=None,
              layout: str = "interleaved", out_dtype: str = "float32"):
    """Run one MACT fast transform (space in lab/hsi/sct) on the GPU.

    out_dtype "float32" (default) is the throughput path; "float64" evaluates
    in the reference's own fp64 arithmetic (mact_fast_f64) and returns what
    mact.fast returns, bit for bit for 8-bit pixels.
    """
    if space not in _ENTRY:
        raise ValueError(f"unknown space {space!r}")
    if layout not in _lib.LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    if out_dtype not in ("float32", "float64"):
        raise ValueError(f"out_dtype must be float32 or float64, got {out_dtype!r}")
    _dev.require_cuda()
    if out_dtype == "float64" and not _dev.is_device_tensor(pixels):
        arr = np.asarray(pixels)
        if arr.dtype == np.uint8 and arr.ndim >= 1 and arr.shape[-1] == 3:
            return _host_u8(space, arr, cfg, out, layout, out_dtype)
    if out_dtype == "float64":
        import torch

        t, code, lead, on_dev = _dev.as_device_pixels(pixels)
        res = _dev.empty_out(lead, layout, t.device, dtype=torch.float64)
        _lib.call("mact_fast_f64", _lib.SPACES[space], t.data_ptr(), code, res.data_ptr(), t.numel() // 3,
                  cfg.coeffs, _lib.LAYOUTS[layout], _dev.stream_ptr())
        return _dev.to_caller(res, on_dev)
    if not _dev.is_device_tensor(pixels):
        arr = np.asarray(pixels)
        if arr.dtype == np.uint8 and arr.ndim >= 1 and arr.shape[-1] == 3:
            return _host_u8(space, arr, cfg, out, layout)
    t, code, lead, on_dev = _dev.as_device_pixels(pixels)
    n = t.numel() // 3
    res = (_dev.check_out(out, lead, layout, t.device) if (out is not None and on_dev)
           else _dev.empty_out(lead, layout, t.device))
    _lib.call(_ENTRY[space], t.data_ptr(), code, res.data_ptr(), n, cfg.coeffs,
              _lib.LAYOUTS[layout], _dev.stream_ptr())
    if not on_dev and out is not None:
        out[...] = res.cpu().numpy()
        return out
    return _dev.to_caller(res, on_dev)


# ------------------------------------------------ scalar approximant functions
def _approx(fn: int, a, b, x, y=None):
    """Evaluate one approximant family elementwise on the GPU (mact_approx_eval)."""
    import torch

    from .exact import _f64_args

    ts, on_dev = _f64_args(x) if y is None else _f64_args(x, y)
    spec = _lib.MactApproxSpec()
    spec.fn = fn
    spec.a_deg = _fill(spec.a, a)
    spec.b_deg = _fill(spec.b, b) if b is not None else -1
    out = torch.empty(ts[0].shape, dtype=torch.float64, device=ts[0].device)
    flag = torch.zeros(1, dtype=torch.int32, device=ts[0].device)
    _lib.call("mact_approx_eval", spec, ts[0].data_ptr(), ts[1].data_ptr() if y is not None else None,
              out.data_ptr(), ts[0].numel(), flag.data_ptr(), _dev.stream_ptr())
    if fn == _lib.FN_FORM and b is not None and int(flag.item()):
        raise DegenerateDenominator("denominator vanished inside evaluation batch")
    return _dev.to_caller(out, on_dev)


def _form_coeffs(form):
    if isinstance(form, Rational):
        return form.numerator.coeffs, form.denominator.coeffs
    return form.coeffs, None


def cbrt_fast(t, approx):
    """Approximate t**(1/3) with ``approx`` (polynomial or rational) (fast.py:81-83;
    approximants.eval_poly / eval_rational, approximants.py:55-82)."""
    a, b = _form_coeffs(approx.form)
    return _approx(_lib.FN_FORM, a, b, t)


def atan_sqrt3_fast(x, approx):
    """arctan(sqrt(3) x) for |x| <= 1, odd-extended (fast.py:118-122)."""
    return _approx(_lib.FN_ATAN_SQRT3, approx.form.coeffs, None, x)


def acos_fast(x, cfg: MactConfig = DEFAULT_CONFIG):
    """arccos on [0, 1]: direct fit below 0.5, folded arcsin at and above (fast.py:151-162)."""
    return _approx(_lib.FN_ACOS, cfg.acos_approx.form.coeffs, cfg.asin_approx.form.coeffs, x)


def atan_unit_fast(g, r, cfg: MactConfig = DEFAULT_CONFIG):
    """arctan(g/r) for g, r >= 0 via the split-domain fits; NaN at g = r = 0, and
    UndefinedAngle for that scalar input (fast.py:165-185)."""
    if np.ndim(g) == 0 and np.ndim(r) == 0 and not _dev.is_device_tensor(g) \
            and float(g) == 0.0 and float(r) == 0.0:
        raise UndefinedAngle("arctan(g/r) undefined at g = r = 0")
    return _approx(_lib.FN_ATAN_UNIT, cfg.atan_f_approx.form.coeffs, cfg.atan_g_approx.form.coeffs, g, r)


def rgb_to_lab_fast(pixels, cfg: MactConfig = DEFAULT_CONFIG, **kw):
    """RGB -> CIELAB with the minimax rational cube root (reference fast.py:86-107)."""
    return transform("lab", pixels, cfg, **kw)


def rgb_to_hsi_fast(pixels, cfg: MactConfig = DEFAULT_CONFIG, **kw):
    """RGB -> HSI with the minimax hue arctangent (reference fast.py:125-148)."""
    return transform("hsi", pixels, cfg, **kw)


def rgb_to_sct_fast(pixels, cfg: MactConfig = DEFAULT_CONFIG, **kw):
    """RGB -> spherical coordinates with minimax arccos/arctan (reference fast.py:188-203)."""
    return transform("sct", pixels, cfg, **kw)


def rgb_to_all_fast(pixels, cfg: MactConfig = DEFAULT_CONFIG, *, layout: str = "interleaved",
                    spaces=("lab", "hsi", "sct")):
    """Several transforms from one read of the pixels (BASELINE configs 5 and 2).

    uint8 pixels in -> one output per name in ``spaces`` (a subset of lab, hsi,
    sct), returned in the order given; each equals the single transform.
    """
    t, code, lead, on_dev = _dev.as_device_pixels(pixels)
    if code != _lib.DTYPE_U8:
        raise ValueError("rgb_to_all_fast takes 8-bit pixels")
    spaces = tuple(spaces)
    if not spaces or any(s not in ("lab", "hsi", "sct") for s in spaces) or len(set(spaces)) != len(spaces):
        raise ValueError(f"spaces must be distinct names from lab, hsi, sct; got {spaces}")
    n = t.numel() // 3
    outs = {s: _dev.empty_out(lead, layout, t.device) for s in spaces}
    ptrs = [outs[s].data_ptr() if s in outs else None for s in ("lab", "hsi", "sct")]
    _lib.call("mact_all_fast", t.data_ptr(), *ptrs, n, cfg.coeffs, _lib.LAYOUTS[layout], _dev.stream_ptr())
    return tuple(_dev.to_caller(outs[s], on_dev) for s in spaces)
