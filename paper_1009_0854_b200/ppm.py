"""Binary PPM (P6) I/O — the image format SPEC.md:583-590 names for the
transform path's input (``read_ppm`` / write), declared but not implemented by
the reference (pyproject.toml:18-19).

    read_ppm(path, device=None)  -> (H, W, 3) uint8 numpy array, or a device
                                    tensor when ``device`` is given (one H2D copy
                                    of the payload, ready for rgb_to_*_fast)
    write_ppm(path, image)       -> P6, maxval 255; write -> read is identity

Header grammar (netpbm): magic ``P6``, then width, height, maxval as ASCII
decimals separated by whitespace, ``#`` comments to end of line allowed
between tokens, then exactly one whitespace byte and W*H*3 payload bytes.
Errors: MalformedHeader, UnsupportedMaxval (anything but 255), TruncatedData.
"""

from __future__ import annotations

import os

import numpy as np

from .errors import MalformedHeader, TruncatedData, UnsupportedMaxval

_WS = b" \t\r\n\x0b\x0c"


def _tokens(buf: bytes, count: int, pos: int):
    """Read ``count`` header tokens starting at ``pos``; returns (tokens, pos of
    the single whitespace byte that ends the header)."""
    out = []
    n = len(buf)
    while len(out) < count:
        while pos < n and (buf[pos] in _WS or buf[pos] == ord("#")):
            if buf[pos] == ord("#"):
                while pos < n and buf[pos] not in b"\r\n":
                    pos += 1
            else:
                pos += 1
        start = pos
        while pos < n and buf[pos] not in _WS and buf[pos] != ord("#"):
            pos += 1
        if start == pos:
            raise MalformedHeader("PPM header ends early")
        out.append(buf[start:pos])
    return out, pos


def parse_header(buf: bytes):
    """(width, height, maxval, payload offset) of a P6 file held in ``buf``."""
    if buf[:2] != b"P6":
        raise MalformedHeader("not a binary PPM (magic P6 expected)")
    toks, pos = _tokens(buf, 3, 2)
    try:
        w, h, maxval = (int(t.decode("ascii")) for t in toks)
    except (UnicodeDecodeError, ValueError) as e:
        raise MalformedHeader(f"non-numeric PPM header field: {e}") from None
    if w <= 0 or h <= 0 or maxval <= 0 or maxval >= 65536:
        raise MalformedHeader(f"bad PPM dimensions {w}x{h} maxval {maxval}")
    if maxval != 255:
        raise UnsupportedMaxval(f"maxval {maxval}: only 8-bit (255) PPM images are supported")
    if pos >= len(buf) or buf[pos] not in _WS:
        raise MalformedHeader("PPM header must end with one whitespace byte")
    return w, h, maxval, pos + 1


def read_ppm(path, device=None):
    """(H, W, 3) uint8 image; on ``device`` (torch) if given."""
    with open(path, "rb") as fh:
        buf = fh.read()
    w, h, _, off = parse_header(buf)
    need = w * h * 3
    if len(buf) - off < need:
        raise TruncatedData(f"PPM payload has {len(buf) - off} bytes, header promises {need}")
    img = np.frombuffer(buf, dtype=np.uint8, count=need, offset=off).reshape(h, w, 3)
    if device is None:
        return img.copy()
    import torch

    return torch.from_numpy(img.copy()).to(device)


def write_ppm(path, image) -> None:
    """Write an (H, W, 3) uint8 image (numpy or tensor) as P6, maxval 255."""
    if hasattr(image, "detach"):
        image = image.detach().cpu().numpy()
    a = np.asarray(image)
    if a.ndim != 3 or a.shape[2] != 3 or a.dtype != np.uint8:
        raise ValueError(f"write_ppm needs an (H, W, 3) uint8 image, got {a.shape} {a.dtype}")
    tmp = f"{os.fspath(path)}.tmp"
    with open(tmp, "wb") as fh:
        fh.write(b"P6\n%d %d\n255\n" % (a.shape[1], a.shape[0]))
        fh.write(np.ascontiguousarray(a).tobytes())
    os.replace(tmp, path)
