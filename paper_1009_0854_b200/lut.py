"""3D-LUT interpolators on B200 — drop-in for ``mact.lut``.

    build_lut(space, grid_n) -> Lut3D          (lut.py:82-95)
    node_weights(lut, pixels, method)          (lut.py:115-199)
    interpolate(lut, pixels, method, variant)  (lut.py:341-350)

The lattice is built on device from the fp64 exact transforms; interpolation
and node selection run in libmact_cuda (integer cell location, bit-exact
node indices).  Angular destination components (HSI hue, SCT angles) are
blended on the circle as the reference does (lut.py:202-262).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Optional, Tuple

import numpy as np

from . import _dev, _lib
from .errors import CacheMissing

METHODS = ("trilinear", "prism", "pyramidal", "tetrahedral")
VARIANTS = ("standard", "caching")
NEIGHBOR_COUNT = {"trilinear": 8, "prism": 6, "pyramidal": 5, "tetrahedral": 4}
SPACES = ("lab", "hsi", "sct")
ANGULAR_MASKS = {"lab": (False, False, False), "hsi": (True, False, False),
                 "sct": (False, True, True)}


@dataclass
class Lut3D:
    grid_n: int
    spacing: float
    destination_space: str
    values: np.ndarray                      # (n, n, n, 3) float64, r-major (host copy)
    angular_mask: Tuple[bool, bool, bool]
    cache: Optional[Dict[str, object]] = None
    _device: Dict[int, object] = field(default_factory=dict, repr=False, compare=False)

    @property
    def flat_values(self) -> np.ndarray:
        return self.values.reshape(-1, 3)

    def lattice(self, device=None):
        """fp32 (n^3, 4) device lattice consumed by the kernels — node = (c0, c1,
        c2, 0), one 16-byte load — cached per device."""
        import torch

        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        key = dev.index if dev.index is not None else torch.cuda.current_device()
        if key not in self._device:
            v = np.zeros((self.grid_n ** 3, 4), dtype=np.float32)
            v[:, :3] = self.values.reshape(-1, 3)
            self._device[key] = torch.from_numpy(v).to(dev)
        return self._device[key]

    def lattice64(self, device=None):
        """fp64 (n^3, 3) device lattice used by angular destinations."""
        import torch

        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        key = ("f64", dev.index if dev.index is not None else torch.cuda.current_device())
        if key not in self._device:
            self._device[key] = torch.from_numpy(
                np.ascontiguousarray(self.values.reshape(-1, 3), dtype=np.float64)).to(dev)
        return self._device[key]


def lattice_coordinates(grid_n: int) -> np.ndarray:
    return np.arange(grid_n) * (255.0 / (grid_n - 1))


def build_lut(space: str, grid_n: int) -> Lut3D:
    """Lattice of exact transforms at k*255/(n-1), NaN -> 0 (lut.py:82-95), built on device."""
    import torch

    if space not in SPACES:
        raise ValueError(f"unknown destination space {space!r}")
    if grid_n not in (9, 17, 33):
        raise ValueError("grid_n must be one of 9, 17, 33")
    _dev.require_cuda()
    total = grid_n ** 3
    f64 = torch.empty((total, 3), dtype=torch.float64, device="cuda")
    f32 = torch.empty((total, 4), dtype=torch.float32, device="cuda")
    _lib.call("mact_lut_build", _lib.SPACES[space], grid_n, f64.data_ptr(), f32.data_ptr(),
              _dev.stream_ptr())
    lut = Lut3D(grid_n=grid_n, spacing=255.0 / (grid_n - 1), destination_space=space,
                values=f64.cpu().numpy().reshape(grid_n, grid_n, grid_n, 3),
                angular_mask=ANGULAR_MASKS[space])
    lut._device[f32.device.index] = f32
    return lut


def _method_code(method: str) -> int:
    if method not in METHODS:
        raise ValueError(f"unknown interpolation method {method!r}")
    return _lib.METHODS[method]


def _is_u8(pixels) -> bool:
    """Integer pixels take the uint8 path (as _dev.as_device_pixels converts them)."""
    if _dev.is_device_tensor(pixels):
        return not pixels.dtype.is_floating_point
    return np.asarray(pixels).dtype.kind in "iub"


def _u8_pixels(pixels):
    t, code, lead, on_dev = _dev.as_device_pixels(pixels)
    if code != _lib.DTYPE_U8:
        raise ValueError("LUT kernels take 8-bit pixels (integer RGB in [0, 255])")
    return t, lead, on_dev


def node_weights(lut: Lut3D, pixels, method: str):
    """(flat node indices int32 (..., k), float64 weights (..., k)), bit-identical to
    the reference for every pixel dtype (lut.py:115-199)."""
    import torch

    m = _method_code(method)
    t, code, lead, on_dev = _dev.as_device_pixels(pixels)
    k = NEIGHBOR_COUNT[method]
    nodes = torch.empty(lead + (k,), dtype=torch.int32, device=t.device)
    w = torch.empty(lead + (k,), dtype=torch.float64, device=t.device)   # the reference's fp64 weights
    _lib.call("mact_lut_nodes_real", lut.grid_n, m, t.data_ptr(), code, t.numel() // 3,
              nodes.data_ptr(), w.data_ptr(), _dev.stream_ptr())
    return _dev.to_caller(nodes, on_dev), _dev.to_caller(w, on_dev)


def build_cache(lut: Lut3D) -> Lut3D:
    """A LUT carrying the per-cell cache of every method (lut.py:265-291), built on the GPU
    (mact_lut_cache_build, the reference's operation order: bit-identical).

    ``cache["trilinear"]`` holds the 8 trilinear polynomial coefficients and
    ``cache["corner_diff"]`` the 8 corner differences of every cell, both
    (n-1, n-1, n-1, 8, 3) float64 like the reference's.  The device copies
    stay with the returned LUT for ``interpolate(..., variant="caching")``.
    """
    import torch

    _dev.require_cuda()
    g = lut.grid_n
    dev = torch.device("cuda", torch.cuda.current_device())
    shape = (g - 1, g - 1, g - 1, 8, 3)
    tri = torch.empty(shape, dtype=torch.float64, device=dev)
    cdiff = torch.empty(shape, dtype=torch.float64, device=dev)
    _lib.call("mact_lut_cache_build", lut.lattice64(dev).data_ptr(), g, tri.data_ptr(), cdiff.data_ptr(),
              _dev.stream_ptr())
    out = Lut3D(grid_n=g, spacing=lut.spacing, destination_space=lut.destination_space, values=lut.values,
                angular_mask=lut.angular_mask,
                cache={"trilinear": tri.cpu().numpy(), "corner_diff": cdiff.cpu().numpy()},
                _device=dict(lut._device))
    out._device[("cache", dev.index)] = (tri, cdiff)
    return out


def _cache_device(lut: Lut3D, device):
    """Device copies of the cache arrays (uploaded once if the cache came from the host)."""
    import torch

    key = ("cache", device.index if device.index is not None else torch.cuda.current_device())
    if key not in lut._device:
        tri = torch.from_numpy(np.ascontiguousarray(lut.cache["trilinear"], dtype=np.float64)).to(device)
        cdiff = torch.from_numpy(np.ascontiguousarray(lut.cache["corner_diff"], dtype=np.float64)).to(device)
        lut._device[key] = (tri, cdiff)
    return lut._device[key]


def angular_lerp(theta0, theta1, alpha):
    """Circular interpolation between two angles, wrapped to [0, 2 pi); a
    vanishing blended direction resolves to theta0 mod 2 pi (lut.py:202-216)."""
    from .exact import _elem

    return _elem(_lib.ELEM_ANGULAR_LERP, theta0, theta1, alpha)


def _host_interp(lut: Lut3D, method_code: int, arr: np.ndarray, out, layout: str):
    """numpy uint8 -> numpy fp32 through the native chunked H2D/kernel/D2H executor."""
    import torch

    _dev.require_cuda()
    src = np.ascontiguousarray(arr)
    lead = src.shape[:-1]
    n = int(np.prod(lead, dtype=np.int64)) if lead else 1
    out = _dev.host_out(out, lead, layout)
    dev = torch.cuda.current_device()
    lat = lut.lattice(torch.device("cuda", dev))
    torch.cuda.current_stream().synchronize()          # the executor runs on its own streams
    _dev.host_call("mact_lut_interp_host", dev, lat.data_ptr(), lut.grid_n, method_code,
                   _dev.np_ptr(src), _dev.np_ptr(out), n, _lib.LAYOUTS[layout])
    return out


def interpolate(lut: Lut3D, pixels, method: str = "tetrahedral", variant: str = "standard", *,
                out=None, layout: str = "interleaved", out_dtype: str = "float32"):
    """Interpolate destination triples for RGB in [0, 255] (lut.py:341-350).

    out_dtype "float32" (default) is the throughput path (fp32 lattice in
    shared memory); "float64" evaluates on the fp64 lattice in the reference's
    arithmetic, bit-identical for linear destinations.
    """
    m = _method_code(method)
    if out_dtype not in ("float32", "float64"):
        raise ValueError(f"out_dtype must be float32 or float64, got {out_dtype!r}")
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if variant == "caching" and lut.cache is None:
        raise CacheMissing("caching interpolation requested without a cache; call build_cache first")
    if layout not in _lib.LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    mask = sum(1 << c for c, ang in enumerate(lut.angular_mask) if ang)
    if variant == "caching" and (out_dtype == "float64" or mask or not _is_u8(pixels)):
        # the caching arithmetic itself (lut.py:294-331); for uint8 pixels into fp32 the
        # throughput kernel below serves both variants (they agree to 1e-12)
        import torch

        t, code, lead, on_dev = _dev.as_device_pixels(pixels)
        res = _dev.empty_out(lead, layout, t.device,
                             dtype=torch.float64 if out_dtype == "float64" else torch.float32)
        tri, cdiff = _cache_device(lut, t.device)
        _lib.call("mact_lut_interp_cached", lut.lattice64(t.device).data_ptr(), tri.data_ptr(), cdiff.data_ptr(),
                  lut.grid_n, m, mask, t.data_ptr(), code, res.data_ptr(),
                  _lib.DTYPE_F64 if out_dtype == "float64" else _lib.DTYPE_F32, t.numel() // 3,
                  _lib.LAYOUTS[layout], _dev.stream_ptr())
        return _dev.to_caller(res, on_dev)
    if out_dtype == "float64":
        import torch

        t, code, lead, on_dev = _dev.as_device_pixels(pixels)
        res = _dev.empty_out(lead, layout, t.device, dtype=torch.float64)
        lat = lut.lattice64(t.device)
        _lib.call("mact_lut_interp_real", lat.data_ptr(), lut.grid_n, m, mask, t.data_ptr(), code,
                  res.data_ptr(), _lib.DTYPE_F64, t.numel() // 3, _lib.LAYOUTS[layout], _dev.stream_ptr())
        return _dev.to_caller(res, on_dev)
    if not mask and not _dev.is_device_tensor(pixels):
        arr = np.asarray(pixels)
        if arr.dtype == np.uint8 and arr.ndim >= 1 and arr.shape[-1] == 3:
            return _host_interp(lut, m, arr, out, layout)
    t, code, lead, on_dev = _dev.as_device_pixels(pixels)
    res = (_dev.check_out(out, lead, layout, t.device) if (out is not None and on_dev)
           else _dev.empty_out(lead, layout, t.device))
    if code != _lib.DTYPE_U8:
        # real-valued pixels: fp64 cell location and weights (lut.py:98-199)
        lat = lut.lattice64(t.device)
        _lib.call("mact_lut_interp_real", lat.data_ptr(), lut.grid_n, m, mask, t.data_ptr(), code,
                  res.data_ptr(), _lib.DTYPE_F32, t.numel() // 3, _lib.LAYOUTS[layout], _dev.stream_ptr())
    elif mask:
        lat = lut.lattice64(t.device)
        _lib.call("mact_lut_interp_angular", lat.data_ptr(), lut.grid_n, m, mask, t.data_ptr(),
                  res.data_ptr(), t.numel() // 3, _lib.LAYOUTS[layout], _dev.stream_ptr())
    else:
        lat = lut.lattice(t.device)
        _lib.call("mact_lut_interp", lat.data_ptr(), lut.grid_n, m, t.data_ptr(), res.data_ptr(),
                  t.numel() // 3, _lib.LAYOUTS[layout], _dev.stream_ptr())
    return _dev.to_caller(res, on_dev)


# ------------------------------------------------------------------ MLUT files
# lut.py:353-383 of the reference: "MLUT" magic, little-endian u32 version,
# grid, space index, angular-mask bits, then (n,n,n,3) float64 values.
_MAGIC = b"MLUT"
_VERSION = 1


def save_lut(lut: Lut3D, path) -> None:
    """Write the lattice (never the cache) in the reference's binary format."""
    import struct

    mask = sum(1 << i for i, a in enumerate(lut.angular_mask) if a)
    with open(path, "wb") as fh:
        fh.write(_MAGIC + struct.pack("<IIII", _VERSION, lut.grid_n,
                                      SPACES.index(lut.destination_space), mask))
        fh.write(np.ascontiguousarray(lut.values, dtype="<f8").tobytes())


def load_lut(path) -> Lut3D:
    """Read an MLUT file; MalformedHeader on a bad magic, version, grid or size."""
    import struct

    from .errors import MalformedHeader

    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < 20 or blob[:4] != _MAGIC:
        raise MalformedHeader("not a LUT file (bad magic)")
    version, grid_n, space_idx, mask = struct.unpack("<IIII", blob[4:20])
    if version != _VERSION:
        raise MalformedHeader(f"unsupported LUT version {version}")
    if space_idx >= len(SPACES) or grid_n not in (9, 17, 33):
        raise MalformedHeader("corrupt LUT header")
    payload = blob[20:]
    if len(payload) != grid_n ** 3 * 3 * 8:
        raise MalformedHeader(f"LUT payload size {len(payload)} != expected {grid_n ** 3 * 24}")
    values = np.frombuffer(payload, dtype="<f8").reshape(grid_n, grid_n, grid_n, 3).astype(np.float64)
    return Lut3D(grid_n=grid_n, spacing=255.0 / (grid_n - 1), destination_space=SPACES[space_idx],
                 values=values, angular_mask=tuple(bool(mask >> i & 1) for i in range(3)))
