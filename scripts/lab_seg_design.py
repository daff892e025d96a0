"""Design study for the segmented fp32 evaluation of the CIELAB lightness
rational: emulates the kernel's fp32 arithmetic on the full
2^24 RGB cube and reports the worst |error| of L*, a*, b* against the
reference fast transform (the oracle, fp64).

    python scripts/lab_seg_design.py [SEGS_PER_BINADE] [DEGREE] [lo|nolo] [N,M]

The rational R = P/Q (fast.py:110-115, approximants.py:74-82) is replaced on
t in (knee, 1] by a piecewise polynomial in u = t - t_seg (t_seg = t with its
mantissa bits below the segment index cleared, so u is exact), with the
constant term split into an fp32 (hi, lo) pair.  Then
    a* = 500 ((hi_x - hi_y) + (d_x - d_y)),   d = lo + u (c1 + u c2 ...)
so the 500x amplification sees the small parts' rounding only.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import mact_oracle as O  # noqa: E402

f32 = np.float32


def fmaf(a, b, c):
    return (a.astype(np.float64) * np.float64(b) + np.float64(c)).astype(f32) if isinstance(a, np.ndarray) \
        else f32(np.float64(a) * np.float64(b) + np.float64(c))


def fma_arr(a, b, c):
    return (np.asarray(a, np.float64) * np.asarray(b, np.float64) + np.asarray(c, np.float64)).astype(f32)


def build_table(num, den, segs, deg, lo_split=True):
    """Segment i covers [t_i, t_i + w_i); t_i = 2^(e) (1 + k/segs), e from -7."""
    shift = 23 - int(np.log2(segs))
    base = (np.array([2.0 ** -7], f32).view(np.uint32)[0]) >> shift
    top = (np.array([1.0], f32).view(np.uint32)[0] >> shift) - base + 1
    tab = np.zeros((top, 4), f32)
    def R(t):
        return O.horner(num, t) / O.horner(den, t)
    fit_err = 0.0
    for i in range(top):
        t0 = float((np.uint32((base + i) << shift)).view(f32))
        t1 = float((np.uint32((base + i + 1) << shift)).view(f32))
        w = t1 - t0
        k = np.arange(deg + 1)
        nodes = 0.5 * w * (1 - np.cos((2 * k + 1) * np.pi / (2 * (deg + 1))))
        coef = np.polyfit(nodes, R(t0 + nodes), deg)[::-1]  # c0 .. cdeg
        uu = np.linspace(0, w, 2001)
        fit_err = max(fit_err, float(np.max(np.abs(np.polyval(coef[::-1], uu) - R(t0 + uu)))))
        hi = f32(coef[0])
        lo = f32(coef[0] - np.float64(hi)) if lo_split else f32(0)
        row = [hi, lo] + [f32(c) for c in coef[1:]]
        tab[i, :len(row[:4])] = row[:4]
        if deg == 3:
            tab[i] = [hi, f32(coef[1]), f32(coef[2]), f32(coef[3])]
    return tab, base, shift, fit_err


def seg_eval(t, tab, base, shift, deg, lo_split):
    bits = t.view(np.uint32)
    idx = (bits >> shift).astype(np.int64) - int(base)
    idx = np.clip(idx, 0, tab.shape[0] - 1)
    tseg = ((bits >> shift) << shift).view(f32)
    u = (t - tseg).astype(f32)
    e = tab[idx]
    if deg == 2:
        d = fma_arr(u, fma_arr(u, e[:, 3], e[:, 2]), e[:, 1])
    else:
        d = (fma_arr(u, fma_arr(u, e[:, 3], e[:, 2]), e[:, 1]) * u).astype(f32)
    return e[:, 0], d


def main():
    segs = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    deg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    lo_split = (sys.argv[3] != "nolo") if len(sys.argv) > 3 else True
    degs = tuple(int(v) for v in sys.argv[4].split(",")) if len(sys.argv) > 4 else (4, 4)
    cfg = O.OracleConfig(cielab_degrees=degs)
    num, den = cfg.cbrt_num, cfg.cbrt_den
    tab, base, shift, fit_err = build_table(num, den, segs, deg, lo_split)
    print(f"segments {tab.shape[0]}, degree {deg}, lo {lo_split}, max fit error {fit_err:.3e}")
    gam = O.GAMMA_TABLE.astype(f32)
    m = np.array([[O.RGB_TO_XYZ[r, c] / O.WHITE[r] for c in range(3)] for r in range(3)]).astype(f32)
    knee = f32(O.LAB_KNEE)
    slope = f32(O.LAB_LINEAR_SLOPE)
    off_hi = f32(O.LAB_LINEAR_OFFSET)
    off_lo = f32(O.LAB_LINEAR_OFFSET - np.float64(off_hi))
    worst = np.zeros(3)
    chunk = 1 << 22
    for s in range(0, 1 << 24, chunk):
        px = O.cube_chunk(s, chunk)
        ref = O.rgb_to_lab_fast(px, cfg)
        gr, gg, gb = gam[px[:, 0]], gam[px[:, 1]], gam[px[:, 2]]
        ts = []
        for r in range(3):
            ts.append(fma_arr(m[r, 2], gb, fma_arr(m[r, 1], gg, (m[r, 0] * gr).astype(f32))))
        hs, ds = [], []
        for t in ts:
            h, d = seg_eval(t, tab, base, shift, deg, lo_split)
            low = ~(t > knee)
            h = np.where(low, off_hi, h)
            d = np.where(low, fma_arr(slope, t, off_lo), d)
            hs.append(h)
            ds.append(d)
        (hx, hy, hz), (dx, dy, dz) = hs, ds
        L = fma_arr(f32(116), dy, fma_arr(f32(116), hy, f32(-16)))
        A = (f32(500) * ((hx - hy) + (dx - dy))).astype(f32)
        B = (f32(200) * ((hy - hz) + (dy - dz))).astype(f32)
        got = np.stack([L, A, B], -1).astype(np.float64)
        err = np.max(np.abs(got - ref), axis=0)
        worst = np.maximum(worst, err)
    print(f"max |err| L* a* b*: {worst[0]:.3e} {worst[1]:.3e} {worst[2]:.3e}  (tolerance 1e-4)")


if __name__ == "__main__":
    main()
