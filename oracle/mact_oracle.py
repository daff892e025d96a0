"""CPU oracle for the MACT per-pixel colour-transform path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``mact`` 0.1.0
(``/root/reference/pkg/src/mact``) for exactly the functions on the hot path
(SURVEY.md §8a rows A1–A21).  It exists to *check* the CUDA path, never to be
it: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product package
(``paper_1009_0854_b200``) never imports anything under ``oracle/``.

Parity pinning: every function here is checked against golden vectors produced
by the real reference (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/mact`` in the build container and writes
``tests/golden/*.npz|json``); ``tests/test_oracle_golden.py`` asserts bit
equality (or ≤1e-12 where the reference itself is order-sensitive).

Arithmetic follows the reference operation-for-operation (numpy float64, no
FMA contraction, Horner highest coefficient first) so results are bit-identical
to the reference on the same numpy build.  Citations are ``file:line`` into
``/root/reference/pkg/src/mact``.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Callable, Dict, Sequence, Tuple

import numpy as np

TWO_PI = 2.0 * np.pi

# ---------------------------------------------------------------------------
# A1 — constants (exact.py:21-40, approximants.py:163)
# ---------------------------------------------------------------------------
GAMMA_KNEE = 0.081
GAMMA_SLOPE = 4.5
GAMMA_OFFSET = 0.099
GAMMA_SCALE = 1.099
GAMMA_POWER = 1.0 / 0.45
RGB_TO_XYZ = np.array([[0.412391, 0.357584, 0.180481],
                       [0.212639, 0.715169, 0.072192],
                       [0.019331, 0.119195, 0.950532]])
WHITE = (0.950456, 1.0, 1.089058)
LAB_KNEE = 0.008856
LAB_LINEAR_SLOPE = 7.787
LAB_LINEAR_OFFSET = 16.0 / 116.0

# ---------------------------------------------------------------------------
# Coefficient tables (approximants.py:168-265), published decimal strings
# parsed to the nearest double.  Tuples are a_0 .. a_n (ascending powers).
# ---------------------------------------------------------------------------
# Cube-root polynomials on [0, 1] (approximants.py:168-177; PAPER Table 1).
CBRT_POLYS: Dict[int, Tuple[str, ...]] = {
    2: ("1.268979e-01", "2.393873", "-1.647669"),
    3: ("9.787826e-02", "4.057495", "-7.388864", "4.331370"),
    4: ("8.111133e-02", "5.926004", "-2.017165e+01", "2.833070e+01", "-1.324728e+01"),
    5: ("7.002910e-02", "7.961214", "-4.329352e+01", "1.063182e+02", "-1.135685e+02", "4.358268e+01"),
}
CBRT_RATIONALS: Dict[Tuple[int, int], Tuple[Tuple[str, ...], Tuple[str, ...]]] = {
    (2, 2): (("6.309655e-03", "5.785782e-01", "1.591005"),
             ("4.482646e-02", "1.175862", "9.596879e-01")),
    (2, 3): (("2.500705e-03", "3.447113e-01", "1.942708"),
             ("1.978701e-02", "8.542797e-01", "1.664540", "-2.503267e-01")),
    (3, 2): (("1.776519e-03", "2.632323e-01", "1.751297", "3.836709e-01"),
             ("1.432256e-02", "6.779998e-01", "1.706260")),
    (2, 4): (("1.317899e-03", "2.390113e-01", "2.099395"),
             ("1.124254e-02", "6.726679e-01", "2.184656", "-7.511150e-01", "2.229717e-01")),
    (3, 3): (("4.370889e-04", "9.526952e-02", "1.252009", "1.302733"),
             ("3.912364e-03", "2.954084e-01", "1.717143", "6.343408e-01")),
    (4, 2): (("7.589302e-04", "1.519784e-01", "1.663584", "8.368075e-01", "-1.657269e-01"),
             ("6.644723e-03", "4.506424e-01", "2.030622")),
    (3, 4): (("1.683667e-04", "4.667675e-02", "9.106812e-01", "1.810577"),
             ("1.610864e-03", "1.617974e-01", "1.494070", "1.218468", "-1.079451e-01")),
    (4, 3): (("1.349673e-04", "3.832079e-02", "7.870174e-01", "1.799062", "2.071170e-01"),
             ("1.299250e-03", "1.345420e-01", "1.330358", "1.365369")),
    (4, 4): (("3.927283e-05", "1.392318e-02", "4.114739e-01", "1.734853", "8.679223e-01"),
             ("4.022100e-04", "5.414536e-02", "8.221526e-01", "1.800167", "3.513617e-01")),
}
ASIN_HALF = {4: ("2.097797e-05", "1.412840", "1.429881e-02", "6.704361e-02", "6.909677e-02"),
             5: ("-2.370048e-06", "1.414434", "-3.300037e-03", "1.354670e-01",
                 "-3.994259e-02", "6.099502e-02")}
ACOS_HALF = {4: ("1.570786", "-9.990285e-01", "-1.429899e-02", "-9.481335e-02", "-1.381942e-01"),
             5: ("1.570798", "-1.000156", "3.299810e-03", "-1.915780e-01",
                 "7.988231e-02", "-1.725177e-01")}
ATAN_F = {4: ("-1.036508e-04", "1.003740", "-1.773538e-02", "-3.390563e-01", "1.386796e-01"),
          5: ("2.073866e-05", "9.982666e-01", "2.352573e-02", "-4.506862e-01",
              "2.635050e-01", "-4.920822e-02")}
ATAN_G = {4: ("1.570917", "-1.004004", "1.885694e-02", "3.373159e-01", "-1.377930e-01"),
          5: ("1.570769", "-9.981253e-01", "-2.440212e-02", "4.528921e-01",
              "-2.659181e-01", "5.016228e-02")}
# Bundled ATAN_SQRT3 degrees (approximants.py:219-229) only gate which HSI
# degrees are legal (fast.py:64); the pipeline evaluates the [0,1] refit
# (fast.py:38-43).  These are the refit outputs of remez_poly(ATAN_SQRT3,
# (0,1), n) as produced by the reference in the build container, frozen as
# exact float64 values (tests/golden/hsi_refit.json pins them).
HSI_REFIT = {
    2: (0.006284947651693185, 1.780260485842989, -0.7464821732923941),
    3: (-0.003692653108724686, 1.8851978201283177, -0.984841853121039, 0.14684158418931897),
    4: (-0.0013203887844437379, 1.7981353035694578, -0.5047931910004136,
        -0.6755157658048955, 0.43201198200133645),
    5: (-0.00018962050654047768, 1.7398783026013234, -0.02536381417376224,
        -2.0498061861186665, 2.032735308062768, -0.6502460591750653),
}


def _f(seq) -> Tuple[float, ...]:
    return tuple(float(s) for s in seq)


@dataclass(frozen=True)
class OracleConfig:
    """Restates MactConfig (fast.py:46-78): degree selection -> coefficient sets."""

    cielab_degrees: Tuple[int, int] = (4, 4)
    hsi_degree: int = 5
    sct_degrees: Tuple[int, int, int] = (5, 5, 5)

    @property
    def cbrt_num(self):
        return _f(CBRT_RATIONALS[tuple(self.cielab_degrees)][0])

    @property
    def cbrt_den(self):
        return _f(CBRT_RATIONALS[tuple(self.cielab_degrees)][1])

    @property
    def atan_sqrt3(self):
        return HSI_REFIT[self.hsi_degree]

    @property
    def asin(self):
        return _f(ASIN_HALF[self.sct_degrees[0]])

    @property
    def acos(self):
        return _f(ACOS_HALF[self.sct_degrees[1]])

    @property
    def atan_f(self):
        return _f(ATAN_F[self.sct_degrees[2]])

    @property
    def atan_g(self):
        return _f(ATAN_G[self.sct_degrees[2]])


DEFAULT = OracleConfig()


def horner(coeffs: Sequence[float], x):
    """eval_poly (approximants.py:55-71): acc = a_n; acc = acc*x + a_k, k descending."""
    x = np.asarray(x, dtype=np.float64)
    acc = np.full(x.shape, coeffs[-1], dtype=np.float64)
    for c in coeffs[-2::-1]:
        acc *= x
        acc += c
    return acc


# ---------------------------------------------------------------------------
# A2/A3/A13 — exact transforms (exact.py:46-149)
# ---------------------------------------------------------------------------
def channels(pixels):
    a = np.asarray(pixels, dtype=np.float64)
    return a[..., 0], a[..., 1], a[..., 2]


def stack3(c0, c1, c2):
    return np.stack(np.broadcast_arrays(c0, c1, c2), axis=-1)


def inverse_gamma(kp):
    """BT.709 inverse gamma (exact.py:52-57)."""
    k = np.asarray(kp, dtype=np.float64)
    with np.errstate(invalid="ignore"):
        curved = ((k + GAMMA_OFFSET) / GAMMA_SCALE) ** GAMMA_POWER
    return np.where(k < GAMMA_KNEE, k / GAMMA_SLOPE, curved)


GAMMA_TABLE = inverse_gamma(np.arange(256) / 255.0)   # fast.py:35


def rgb_to_xyz(r, g, b):
    """exact.py:60-66 — row-wise m0*r + m1*g + m2*b, left to right."""
    m = RGB_TO_XYZ
    return (m[0, 0] * r + m[0, 1] * g + m[0, 2] * b,
            m[1, 0] * r + m[1, 1] * g + m[1, 2] * b,
            m[2, 0] * r + m[2, 1] * g + m[2, 2] * b)


def lab_f(t):
    """exact.py:69-72."""
    t = np.asarray(t, dtype=np.float64)
    return np.where(t > LAB_KNEE, np.cbrt(t), LAB_LINEAR_SLOPE * t + LAB_LINEAR_OFFSET)


def xyz_to_lab(x, y, z):
    """exact.py:75-83."""
    fx = lab_f(np.asarray(x, dtype=np.float64) / WHITE[0])
    fy = lab_f(np.asarray(y, dtype=np.float64) / WHITE[1])
    fz = lab_f(np.asarray(z, dtype=np.float64) / WHITE[2])
    return stack3(116.0 * fy - 16.0, 500.0 * (fx - fy), 200.0 * (fy - fz))


def rgb_to_lab_exact(pixels):
    """exact.py:86-92 (analytic gamma on r/255 for any dtype)."""
    r, g, b = channels(pixels)
    return xyz_to_lab(*rgb_to_xyz(inverse_gamma(r / 255.0), inverse_gamma(g / 255.0),
                                  inverse_gamma(b / 255.0)))


def hsi_sat_int(r, g, b):
    """exact.py:95-101."""
    total = r + g + b
    low = np.minimum(np.minimum(r, g), b)
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(total > 0.0, 1.0 - 3.0 * low / total, 0.0)
    return s, total / 3.0


def _kender_cases(r, g, b):
    """Hue case analysis shared by exact.py:127-130 and fast.py:133-136."""
    c1 = (r > b) & (g > b)
    c2 = ~c1 & (g > r)
    c3 = ~c1 & ~c2 & (b > g)
    c4 = ~c1 & ~c2 & ~c3 & (r > b)
    return c1, c2, c3, c4


def rgb_to_hsi_exact(pixels):
    """exact.py:119-137 (arctangent form, NaN hue on the gray axis)."""
    r, g, b = channels(pixels)
    r, g, b = r / 255.0, g / 255.0, b / 255.0
    s3 = np.sqrt(3.0)
    c1, c2, c3, c4 = _kender_cases(r, g, b)
    with np.errstate(divide="ignore", invalid="ignore"):
        h1 = np.pi / 3.0 + np.arctan(s3 * (g - r) / ((g - b) + (r - b)))
        h2 = np.pi + np.arctan(s3 * (b - g) / ((b - r) + (g - r)))
        h3 = 5.0 * np.pi / 3.0 + np.arctan(s3 * (r - b) / ((r - g) + (b - g)))
    h = np.select([c1, c2, c3, c4], [h1, h2, h3, 0.0], default=np.nan)
    s, i = hsi_sat_int(r, g, b)
    return stack3(h, s, i)


def rgb_to_hsi_arccos(pixels):
    """exact.py:104-116 — inverse-cosine hue (property check Kender ≡ arccos)."""
    r, g, b = channels(pixels)
    r, g, b = r / 255.0, g / 255.0, b / 255.0
    num = 0.5 * ((r - g) + (r - b))
    den_sq = (r - g) ** 2 + (r - b) * (g - b)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = num / np.sqrt(den_sq)
    h = np.arccos(np.clip(ratio, -1.0, 1.0))
    h = np.where(b > g, TWO_PI - h, h)
    h = np.where(den_sq > 0.0, h, np.nan)
    s, i = hsi_sat_int(r, g, b)
    return stack3(h, s, i)


def rgb_to_sct_exact(pixels):
    """exact.py:140-149."""
    r, g, b = channels(pixels)
    length = np.sqrt(r * r + g * g + b * b)
    safe = np.where(length > 0.0, length, 1.0)
    ang_a = np.where(length > 0.0, np.arccos(np.clip(b / safe, -1.0, 1.0)), 0.0)
    ang_b = np.arctan2(g, r)
    ang_b = np.where((r == 0.0) & (g == 0.0), np.nan, ang_b)
    return stack3(length, ang_a, ang_b)


def sct_to_rgb(pixels):
    """exact.py:152-160."""
    length, a, b = channels(pixels)
    b = np.where(np.isnan(b), 0.0, b)
    sa = np.sin(a)
    return stack3(length * sa * np.cos(b), length * sa * np.sin(b), length * np.cos(a))


# ---------------------------------------------------------------------------
# A19 — distances (exact.py:163-190)
# ---------------------------------------------------------------------------
def lab_distance(x, y):
    d = np.asarray(x, dtype=np.float64) - np.asarray(y, dtype=np.float64)
    return np.sqrt(np.sum(d * d, axis=-1))


def hsi_distance(x, y):
    hx, sx, ix = channels(x)
    hy, sy, iy = channels(y)
    hx = np.where(np.isnan(hx), 0.0, hx)
    hy = np.where(np.isnan(hy), 0.0, hy)
    th = np.abs(hx - hy)
    th = np.where(th > np.pi, TWO_PI - th, th)
    d2 = sx * sx + sy * sy - 2.0 * sx * sy * np.cos(th) + (ix - iy) ** 2
    return np.sqrt(np.maximum(d2, 0.0))


def sct_distance_indirect(x, y):
    rx = np.clip(sct_to_rgb(x), 0.0, 255.0)
    ry = np.clip(sct_to_rgb(y), 0.0, 255.0)
    return lab_distance(rgb_to_lab_exact(rx), rgb_to_lab_exact(ry))


DISTANCES = {"lab": lab_distance, "hsi": hsi_distance, "sct": sct_distance_indirect}

# ---------------------------------------------------------------------------
# A4–A12 — MACT fast transforms (fast.py:81-203)
# ---------------------------------------------------------------------------
def _lab_f_fast(t, cfg: OracleConfig):
    """fast.py:110-115 with cbrt_fast -> eval_rational (approximants.py:74-82)."""
    t = np.asarray(t, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        approx = horner(cfg.cbrt_num, t) / horner(cfg.cbrt_den, t)
    return np.where(t > LAB_KNEE, approx, LAB_LINEAR_SLOPE * t + LAB_LINEAR_OFFSET)


def rgb_to_lab_fast(pixels, cfg: OracleConfig = DEFAULT):
    """fast.py:86-107 — integer input takes the 256-entry gamma table."""
    arr = np.asarray(pixels)
    if arr.dtype.kind in "iu":
        r, g, b = GAMMA_TABLE[arr[..., 0]], GAMMA_TABLE[arr[..., 1]], GAMMA_TABLE[arr[..., 2]]
    else:
        k = arr.astype(np.float64) / 255.0
        r, g, b = inverse_gamma(k[..., 0]), inverse_gamma(k[..., 1]), inverse_gamma(k[..., 2])
    x, y, z = rgb_to_xyz(r, g, b)
    fx = _lab_f_fast(x / WHITE[0], cfg)
    fy = _lab_f_fast(y / WHITE[1], cfg)
    fz = _lab_f_fast(z / WHITE[2], cfg)
    return stack3(116.0 * fy - 16.0, 500.0 * (fx - fy), 200.0 * (fy - fz))


def cbrt_fast(t, num, den=None):
    """fast.py:81-83 -> approximants.eval_poly / eval_rational (approximants.py:55-82):
    numerator / denominator Horner, one division (ValueError stands in for
    DegenerateDenominator on |q| < 1e-300)."""
    if den is None:
        return horner(num, t)
    q = horner(den, t)
    if np.any(np.abs(q) < 1e-300):
        raise ValueError("denominator vanished inside evaluation batch")
    return horner(num, t) / q


def atan_sqrt3_fast(x, coeffs):
    """fast.py:118-122 — odd extension of the [0,1] polynomial."""
    x = np.asarray(x, dtype=np.float64)
    mag = horner(coeffs, np.abs(x))
    return np.where(x < 0.0, -mag, mag)


def rgb_to_hsi_fast(pixels, cfg: OracleConfig = DEFAULT):
    """fast.py:125-148."""
    r, g, b = channels(pixels)
    r, g, b = r / 255.0, g / 255.0, b / 255.0
    c1, c2, c3, c4 = _kender_cases(r, g, b)
    num = np.select([c1, c2, c3], [g - r, b - g, r - b], default=0.0)
    den = np.select([c1, c2, c3], [(g - b) + (r - b), (b - r) + (g - r), (r - g) + (b - g)],
                    default=1.0)
    base = np.select([c1, c2, c3], [np.pi / 3.0, np.pi, 5.0 * np.pi / 3.0], default=0.0)
    h = base + atan_sqrt3_fast(num / den, cfg.atan_sqrt3)
    h = np.select([c1 | c2 | c3, c4], [h, 0.0], default=np.nan)
    h = np.where(h < 0.0, h + TWO_PI, h)
    h = np.where(h >= TWO_PI, h - TWO_PI, h)
    s, i = hsi_sat_int(r, g, b)
    return stack3(h, s, i)


def acos_fast(x, cfg: OracleConfig = DEFAULT):
    """fast.py:151-162."""
    x = np.asarray(x, dtype=np.float64)
    upper = horner(cfg.asin, np.sqrt(np.maximum(1.0 - x, 0.0)))
    lower = horner(cfg.acos, x)
    return np.where(x < 0.5, lower, upper)


def atan_unit_fast(g, r, cfg: OracleConfig = DEFAULT):
    """fast.py:165-185 (array form: NaN at g = r = 0)."""
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    g, r = np.broadcast_arrays(g, r)
    direct = g < r
    with np.errstate(divide="ignore", invalid="ignore"):
        arg = np.where(direct, g / np.where(r > 0.0, r, 1.0),
                       np.where(g > 0.0, r / np.where(g > 0.0, g, 1.0), 0.0))
    out = np.where(direct, horner(cfg.atan_f, arg), horner(cfg.atan_g, arg))
    return np.where((g == 0.0) & (r == 0.0), np.nan, out)


def rgb_to_sct_fast(pixels, cfg: OracleConfig = DEFAULT):
    """fast.py:188-203."""
    r, g, b = channels(pixels)
    length = np.sqrt(r * r + g * g + b * b)
    safe = np.where(length > 0.0, length, 1.0)
    ang_a = np.where(length > 0.0, acos_fast(b / safe, cfg), 0.0)
    ang_b = atan_unit_fast(g, r, cfg)
    ang_a = np.clip(ang_a, 0.0, 0.5 * np.pi)
    ang_b = np.where(np.isnan(ang_b), np.nan, np.clip(ang_b, 0.0, 0.5 * np.pi))
    return stack3(length, ang_a, ang_b)


FAST = {"lab": rgb_to_lab_fast, "hsi": rgb_to_hsi_fast, "sct": rgb_to_sct_fast}
EXACT = {"lab": rgb_to_lab_exact, "hsi": rgb_to_hsi_exact, "sct": rgb_to_sct_exact}

# ---------------------------------------------------------------------------
# A14–A17 — 3D LUT (lut.py:63-246)
# ---------------------------------------------------------------------------
METHODS = ("trilinear", "prism", "pyramidal", "tetrahedral")
NEIGHBORS = {"trilinear": 8, "prism": 6, "pyramidal": 5, "tetrahedral": 4}
ANGULAR_MASKS = {"lab": (False, False, False), "hsi": (True, False, False),
                 "sct": (False, True, True)}


def build_lut_values(space: str, grid_n: int) -> np.ndarray:
    """lut.py:77-95 — exact transform at k*255/(n-1), NaN -> 0; (n,n,n,3) r-major."""
    if space not in EXACT:
        raise ValueError(f"unknown destination space {space!r}")
    if grid_n not in (9, 17, 33):
        raise ValueError("grid_n must be one of 9, 17, 33")
    coords = np.arange(grid_n) * (255.0 / (grid_n - 1))
    r, g, b = np.meshgrid(coords, coords, coords, indexing="ij")
    vals = EXACT[space](np.stack([r, g, b], axis=-1))
    return np.nan_to_num(vals, nan=0.0)


def locate(grid_n: int, pixels):
    """lut.py:98-105 — floor(p/spacing) clamped to [0, n-2]; frac = x - base."""
    x = np.asarray(pixels, dtype=np.float64) / (255.0 / (grid_n - 1))
    base = np.maximum(np.minimum(np.floor(x).astype(np.int64), grid_n - 2), 0)
    return base, x - base


def node_weights(grid_n: int, pixels, method: str):
    """lut.py:115-199 — flat node indices (…,k) and weights (…,k)."""
    base, frac = locate(grid_n, pixels)
    n = grid_n
    dr, dg, db = frac[..., 0], frac[..., 1], frac[..., 2]
    bf = (base[..., 0] * n + base[..., 1]) * n + base[..., 2]
    sr, sg, sb = n * n, n, 1
    if method == "trilinear":
        nodes, ws = [], []
        for c in range(8):
            br, bg, bb = c >> 2 & 1, c >> 1 & 1, c & 1
            nodes.append(bf + br * sr + bg * sg + bb * sb)
            ws.append((dr if br else 1.0 - dr) * (dg if bg else 1.0 - dg) * (db if bb else 1.0 - db))
        return np.stack(nodes, -1), np.stack(ws, -1)
    if method == "prism":
        up = dg >= db
        ta = np.where(up, 1.0 - dg, 1.0 - db)
        tb = np.where(up, dg - db, db - dg)
        tc = np.where(up, db, dg)
        mid = np.where(up, sg, sb)
        far = sg + sb
        nodes = np.stack([bf, bf + mid, bf + far, bf + sr, bf + mid + sr, bf + far + sr], -1)
        w = np.stack([ta * (1.0 - dr), tb * (1.0 - dr), tc * (1.0 - dr),
                      ta * dr, tb * dr, tc * dr], -1)
        return nodes, w
    if method == "pyramidal":
        sel_r = (dg > dr) & (db > dr)
        sel_g = ~sel_r & (dr >= dg) & (db >= dg)
        dm = np.select([sel_r, sel_g], [dr, dg], default=db)
        du = np.select([sel_r, sel_g], [dg, dr], default=dr)
        dv = np.select([sel_r, sel_g], [db, db], default=dg)
        nu = np.select([sel_r, sel_g], [sg, sr], default=sr)
        nv = np.select([sel_r, sel_g], [sb, sb], default=sg)
        nodes = np.stack([bf, bf + nu, bf + nv, bf + nu + nv, bf + sr + sg + sb], -1)
        w = np.stack([(1.0 - du) * (1.0 - dv), du * (1.0 - dv), dv * (1.0 - du),
                      du * dv - dm, dm], -1)
        return nodes, w
    if method == "tetrahedral":
        d = np.stack([dr, dg, db], -1)
        order = np.argsort(-d, axis=-1, kind="stable")
        ds = np.take_along_axis(d, order, -1)
        strides = np.array([sr, sg, sb], dtype=np.int64)
        first = strides[order[..., 0]]
        second = first + strides[order[..., 1]]
        nodes = np.stack([bf, bf + first, bf + second, bf + sr + sg + sb], -1)
        w = np.stack([1.0 - ds[..., 0], ds[..., 0] - ds[..., 1], ds[..., 1] - ds[..., 2],
                      ds[..., 2]], -1)
        return nodes, w
    raise ValueError(f"unknown interpolation method {method!r}")


def angular_lerp(t0, t1, a):
    """lut.py:202-216."""
    t0 = np.asarray(t0, dtype=np.float64)
    t1 = np.asarray(t1, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    c = (1.0 - a) * np.cos(t0) + a * np.cos(t1)
    s = (1.0 - a) * np.sin(t0) + a * np.sin(t1)
    out = np.arctan2(s, c)
    out = np.where(out < 0.0, out + TWO_PI, out)
    return np.where(np.hypot(c, s) < 1e-12, np.mod(t0, TWO_PI), out)


def circular_blend(angles, weights):
    """lut.py:219-228."""
    c = np.sum(weights * np.cos(angles), axis=-1)
    s = np.sum(weights * np.sin(angles), axis=-1)
    out = np.arctan2(s, c)
    out = np.where(out < 0.0, out + TWO_PI, out)
    heavy = np.take_along_axis(angles, np.argmax(weights, axis=-1)[..., None], -1)[..., 0]
    return np.where(np.hypot(c, s) < 1e-12, np.mod(heavy, TWO_PI), out)


def interpolate(values: np.ndarray, pixels, method: str = "tetrahedral",
                angular_mask=(False, False, False)):
    """lut.py:231-262, 341-350 (standard variant)."""
    if method not in METHODS:
        raise ValueError(f"unknown interpolation method {method!r}")
    n = values.shape[0]
    flat = values.reshape(-1, 3)
    nodes, w = node_weights(n, pixels, method)
    out = np.zeros(w.shape[:-1] + (3,), dtype=np.float64)
    for j in range(w.shape[-1]):
        out += w[..., j, None] * flat[nodes[..., j]]
    if any(angular_mask):
        base, frac = locate(n, pixels)
        for comp, ang in enumerate(angular_mask):
            if not ang:
                continue
            if method == "trilinear":
                out[..., comp] = _trilinear_angular(flat, n, base, frac, comp)
            else:
                out[..., comp] = circular_blend(flat[nodes, comp], w)
    return out


def _trilinear_angular(flat, n, base, frac, comp):
    """lut.py:249-262 — cascade r, then g, then b."""
    bf = (base[..., 0] * n + base[..., 1]) * n + base[..., 2]
    vals = [flat[bf + (c >> 2 & 1) * n * n + (c >> 1 & 1) * n + (c & 1), comp] for c in range(8)]
    dr, dg, db = frac[..., 0], frac[..., 1], frac[..., 2]
    r0 = {(gb, bb): angular_lerp(vals[gb << 1 | bb], vals[4 | gb << 1 | bb], dr)
          for gb in (0, 1) for bb in (0, 1)}
    g0 = angular_lerp(r0[(0, 0)], r0[(1, 0)], dg)
    g1 = angular_lerp(r0[(0, 1)], r0[(1, 1)], dg)
    return angular_lerp(g0, g1, db)


def build_cache(values: np.ndarray):
    """lut.py:265-291 — per-cell trilinear polynomial coefficients and corner
    differences, each (n-1, n-1, n-1, 8, 3), in the reference's expression order."""
    m = values.shape[0] - 1
    c = [values[(k >> 2 & 1):(k >> 2 & 1) + m, (k >> 1 & 1):(k >> 1 & 1) + m, (k & 1):(k & 1) + m]
         for k in range(8)]
    tri = np.stack([c[0], c[4] - c[0], c[2] - c[0], c[1] - c[0],
                    c[6] - c[4] - c[2] + c[0], c[5] - c[4] - c[1] + c[0], c[3] - c[2] - c[1] + c[0],
                    c[7] - c[6] - c[5] - c[3] + c[4] + c[2] + c[1] - c[0]], axis=-2)
    return {"trilinear": tri, "corner_diff": np.stack([c[k] - c[0] for k in range(8)], axis=-2)}


def interpolate_caching(values: np.ndarray, cache, pixels, method: str = "tetrahedral",
                        angular_mask=(False, False, False)):
    """lut.py:294-331 — the caching variant: linear components from the cache
    (trilinear polynomial terms summed in order; simplex methods as base node
    plus weighted corner differences), angular components as the standard variant."""
    if method not in METHODS:
        raise ValueError(f"unknown interpolation method {method!r}")
    n = values.shape[0]
    flat = values.reshape(-1, 3)
    base, frac = locate(n, pixels)
    dr, dg, db = frac[..., 0], frac[..., 1], frac[..., 2]
    cell = (base[..., 0], base[..., 1], base[..., 2])
    nodes, w = node_weights(n, pixels, method)
    if method == "trilinear":
        c = cache["trilinear"][cell]
        terms = [np.ones_like(dr), dr, dg, db, dr * dg, dr * db, dg * db, dr * dg * db]
        out = c[..., 0, :] * terms[0][..., None]
        for k in range(1, 8):
            out = out + c[..., k, :] * terms[k][..., None]
    else:
        diff = cache["corner_diff"][cell]
        bf = (base[..., 0] * n + base[..., 1]) * n + base[..., 2]
        local = nodes - bf[..., None]
        rows = (local // (n * n)) << 2 | ((local % (n * n)) // n) << 1 | (local % n)
        out = flat[bf].astype(np.float64).copy()
        for j in range(w.shape[-1]):
            out += w[..., j, None] * np.take_along_axis(diff, rows[..., j][..., None, None], axis=-2)[..., 0, :]
    if any(angular_mask):
        for comp, ang in enumerate(angular_mask):
            if not ang:
                continue
            if method == "trilinear":
                out[..., comp] = _trilinear_angular(flat, n, base, frac, comp)
            else:
                out[..., comp] = circular_blend(flat[nodes, comp], w)
    return out


# ---------------------------------------------------------------------------
# A18/A20/A21 — harness semantics (harness.py:25-122)
# ---------------------------------------------------------------------------
CUBE_SIZE = 1 << 24
CHUNK = 1 << 20


def cube_chunk(start: int, size: int) -> np.ndarray:
    """harness.py:35-46 — pixel i = (i>>16, i>>8 & 255, i & 255)."""
    idx = np.arange(start, min(start + size, CUBE_SIZE), dtype=np.uint32)
    out = np.empty((idx.size, 3), dtype=np.uint8)
    out[:, 0] = idx >> 16
    out[:, 1] = (idx >> 8) & 0xFF
    out[:, 2] = idx & 0xFF
    return out


@dataclass(frozen=True)
class Stats:
    avg: float
    max: float
    count: int
    argmax_pixel: Tuple[int, int, int]


def _score(pixels, cand, ref, dist):
    """harness.py:71-74."""
    d = dist(cand(pixels), ref(pixels))
    j = int(np.argmax(d))
    return float(np.sum(d)), float(d[j]), tuple(int(v) for v in np.asarray(pixels)[j]), d.shape[0]


def measure_error(space: str, cand: Callable, ref: Callable, population=None,
                  chunk_size: int = CHUNK, threads: int = 1) -> Stats:
    """harness.py:77-122 — fsum of chunk sums, strict '>' keeps the earliest max."""
    dist = DISTANCES[space]
    if population is None:
        chunks = [cube_chunk(s, chunk_size) for s in range(0, CUBE_SIZE, chunk_size)]
    elif isinstance(population, np.ndarray):
        chunks = [population]
    else:
        chunks = list(population)
    job = lambda p: _score(p, cand, ref, dist)  # noqa: E731
    if threads > 1 and len(chunks) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            results = list(pool.map(job, chunks))
    else:
        results = [job(p) for p in chunks]
    sums, worst, wpx, count = [], -1.0, (0, 0, 0), 0
    for s, mx, px, n in results:
        sums.append(s)
        count += n
        if mx > worst:
            worst, wpx = mx, px
    if count == 0:
        raise ValueError("empty population")
    return Stats(math.fsum(sums) / count, worst, count, wpx)


def component_abs_error(space: str, fast_out, exact_out):
    """SURVEY A21 (not in the reference): per-component |fast - exact|.

    HSI hue uses the circular difference min(d, 2π - d); pixels whose exact
    value is NaN (gray hue / undefined ∠B) are excluded and counted.
    Returns a list of dicts {sum, count, max, argmax, nan} per component.
    """
    f = np.asarray(fast_out, dtype=np.float64)
    e = np.asarray(exact_out, dtype=np.float64)
    res = []
    for c in range(3):
        d = np.abs(f[..., c] - e[..., c]).reshape(-1)
        if space == "hsi" and c == 0:
            d = np.minimum(d, TWO_PI - d)
        nan = np.isnan(e[..., c]).reshape(-1) | np.isnan(f[..., c]).reshape(-1)
        d = np.where(nan, -np.inf, d)
        j = int(np.argmax(d))
        valid = d[~nan]
        res.append({"sum": float(np.sum(valid)), "count": int(valid.size),
                    "max": float(d[j]) if valid.size else 0.0, "argmax": j,
                    "nan": int(nan.sum())})
    return res


CALL_SITES = ("cbrt_x", "cbrt_y", "cbrt_z", "arcsin", "arccos", "arctan")


def call_counts() -> Dict[str, int]:
    """harness.py:137-175 — full-cube call-site counts of the approximated functions.

    Restated by brute force over every colour (not the reference's row/plane
    counting), with the same fp64 evaluation order: X/X0 > knee is
    m[row,0]*gamma[r] + (m[row,1]*gamma[g] + m[row,2]*gamma[b]) > LAB_KNEE*white[row]
    (harness.py:146-156); arcsin <=> 3b^2 >= r^2+g^2 in integers (:158-170);
    arctan defined unless r = g = 0 (:174).
    """
    gamma = inverse_gamma(np.arange(256) / 255.0)
    out = {}
    for row, name in enumerate(("cbrt_x", "cbrt_y", "cbrt_z")):
        tr, tg, tb = (RGB_TO_XYZ[row, k] * gamma for k in range(3))
        plane = tg[:, None] + tb[None, :]
        thr = LAB_KNEE * WHITE[row]
        out[name] = int(sum(np.count_nonzero(tr[r] + plane > thr) for r in range(256)))
    i = np.arange(256, dtype=np.int64)
    rg2 = (i[:, None] ** 2 + i[None, :] ** 2).reshape(-1)
    out["arcsin"] = int(sum(np.count_nonzero(3 * b * b >= rg2) for b in range(256)))
    out["arccos"] = CUBE_SIZE - out["arcsin"]
    out["arctan"] = CUBE_SIZE - 256
    return out


# ---------------------------------------------------------------------------
# CPU baseline runner (bench.py cpu_baseline / --impl reference).  Mirrors
# the reference's only concurrency: a ThreadPoolExecutor over fixed pixel
# chunks (harness.py:92-103).
# ---------------------------------------------------------------------------
def run_chunked(fn: Callable, pixels: np.ndarray, threads: int, chunk: int = 1 << 18):
    flat = pixels.reshape(-1, 3)
    parts = [flat[s:s + chunk] for s in range(0, flat.shape[0], chunk)]
    if threads <= 1:
        return [fn(p) for p in parts]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        return list(pool.map(fn, parts))


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
