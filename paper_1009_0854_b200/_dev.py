"""Device plumbing shared by the public modules: array <-> device tensor
conversion, raw pointers and the current CUDA stream for the C ABI.

torch is used only as the allocator / stream provider; all arithmetic happens
in libmact_cuda.so.
"""

from __future__ import annotations

import threading
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .errors import MactError

try:  # torch provides device memory and streams
    import torch
except Exception:  # pragma: no cover
    torch = None


def require_cuda() -> None:
    if torch is None or not torch.cuda.is_available():
        raise MactError("a CUDA device is required (libmact_cuda has no CPU fallback)")


def is_device_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


_DT = {"uint8": _lib.DTYPE_U8, "float32": _lib.DTYPE_F32, "float64": _lib.DTYPE_F64}


def as_device_pixels(pixels) -> Tuple["torch.Tensor", int, tuple, bool]:
    """(contiguous device tensor, dtype code, leading shape, was_on_device).

    Integer inputs take the 8-bit table path like the reference
    (fast.py:92-95); real inputs keep their precision (f32 or f64).
    """
    require_cuda()
    on_dev = is_device_tensor(pixels)
    if on_dev:
        t = pixels
    else:
        a = np.asarray(pixels)
        if a.dtype.kind in "iub" and a.dtype != np.uint8:
            a = a.astype(np.uint8)
        elif a.dtype.kind == "f" and a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).cuda(non_blocking=False)
    if t.shape[-1] != 3:
        raise ValueError(f"pixels must have a trailing axis of 3 channels, got shape {tuple(t.shape)}")
    if t.dtype in (torch.int8, torch.int16, torch.int32, torch.int64, torch.bool):
        t = t.to(torch.uint8)
    elif t.dtype in (torch.float16, torch.bfloat16):
        t = t.to(torch.float32)
    t = t.contiguous()
    name = str(t.dtype).replace("torch.", "")
    if name not in _DT:
        raise ValueError(f"unsupported pixel dtype {t.dtype}")
    return t, _DT[name], tuple(t.shape[:-1]), on_dev


def empty_out(lead: tuple, layout: str, device, dtype=None):
    dtype = dtype or torch.float32
    shape = lead + (3,) if layout == "interleaved" else (3,) + lead
    return torch.empty(shape, dtype=dtype, device=device)


def check_out(out, lead: tuple, layout: str, device):
    """Validate a caller-supplied device output tensor (shape, dtype, contiguity)."""
    shape = lead + (3,) if layout == "interleaved" else (3,) + lead
    if not is_device_tensor(out) or out.dtype != torch.float32 or tuple(out.shape) != shape \
            or not out.is_contiguous() or out.device != device:
        raise ValueError(f"out must be a contiguous float32 CUDA tensor of shape {shape} on {device}")
    return out


def host_out(out, lead: tuple, layout: str, dtype=np.float32):
    """Validate (or allocate) a numpy float32 / float64 output for the host executor."""
    shape = lead + (3,) if layout == "interleaved" else (3,) + lead
    dtype = np.dtype(dtype)
    if out is None:
        return np.empty(shape, dtype=dtype)
    if not isinstance(out, np.ndarray) or out.dtype != dtype or out.shape != shape \
            or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous {dtype.name} array of shape {shape}")
    return out


def to_caller(t, on_dev: bool):
    """Device result back to the caller's world (numpy for host callers)."""
    if on_dev:
        return t
    return t.cpu().numpy()


# ------------------------------------------------------------------ host executor
_ctx_lock = threading.Lock()
_ctx = {}


def host_ctx(device: int, chunk_px: int = 1 << 23, nstreams: int = 3):
    """Per-(device, chunk, streams) native streaming executor (mact_transform_host)."""
    import ctypes as C

    key = (device, chunk_px, nstreams)
    with _ctx_lock:
        if key not in _ctx:
            h = C.c_void_p()
            _lib.call("mact_host_ctx_create", device, chunk_px, nstreams, C.byref(h))
            _ctx[key] = (h, threading.Lock())
        return _ctx[key][0]


def host_call(name: str, device: int, *args):
    """Call a host-executor entry point on the device's shared context.  A context
    owns streams and staging buffers, so concurrent callers (the reference's
    harness uses a thread pool, harness.py:99-101) are serialised on it; one
    call already keeps both copy engines and the SMs busy."""
    ctx = host_ctx(device)
    with _ctx[(device, 1 << 23, 3)][1]:
        return _lib.call(name, ctx, *args)


def np_ptr(a: np.ndarray) -> int:
    return a.ctypes.data
