"""CPU tests of the host-side logic of the package (no GPU needed)."""

import numpy as np
import pytest

from oracle import mact_oracle as O
from paper_1009_0854_b200 import approximants, lut
from paper_1009_0854_b200.errors import MalformedHeader, UnknownApproximant
from paper_1009_0854_b200.fast import DEFAULT_CONFIG, MactConfig


def test_config_resolves_like_reference():
    c = DEFAULT_CONFIG
    assert (c.cielab_degrees, c.hsi_degree, c.sct_degrees) == ((4, 4), 5, (5, 5, 5))
    k = c.coeffs
    assert (k.cbrt_num_deg, k.cbrt_den_deg, k.hsi_deg, k.asin_deg, k.acos_deg, k.atan_deg) == (4, 4, 5, 5, 5, 5)
    # the HSI pipeline evaluates the [0,1] refit, not the bundled Table 3 set (fast.py:38-43)
    assert tuple(k.atan_sqrt3[:6]) == O.HSI_REFIT[5]
    assert tuple(k.cbrt_num[:5]) == tuple(float(x) for x in O.CBRT_RATIONALS[(4, 4)][0])


@pytest.mark.parametrize("kw", [dict(cielab_degrees=(5, 5)), dict(hsi_degree=6),
                                dict(sct_degrees=(3, 5, 5)), dict(cielab_degrees=(4,))])
def test_unknown_degrees_raise(kw):
    with pytest.raises((UnknownApproximant, ValueError)):
        MactConfig(**kw)


def test_registry_matches_oracle_tables():
    for (n, m), (num, den) in O.CBRT_RATIONALS.items():
        a = approximants.registry_get(approximants.TargetFn.CBRT, (n, m))
        assert a.form.numerator.coeffs == tuple(map(float, num))
        assert a.form.denominator.coeffs == tuple(map(float, den))
    for deg in (4, 5):
        assert approximants.registry_get(approximants.TargetFn.ASIN_HALF, (deg,)).form.coeffs == \
            tuple(map(float, O.ASIN_HALF[deg]))
        assert approximants.registry_get(approximants.TargetFn.ATAN_G, (deg,)).form.coeffs == \
            tuple(map(float, O.ATAN_G[deg]))
    assert len(approximants.registry_keys()) == 25


def test_mlut_roundtrip_and_errors(tmp_path):
    vals = O.build_lut_values("hsi", 9)
    L = lut.Lut3D(9, 255 / 8, "hsi", vals, lut.ANGULAR_MASKS["hsi"])
    p = tmp_path / "a.mlut"
    lut.save_lut(L, p)
    R = lut.load_lut(p)
    assert R.grid_n == 9 and R.destination_space == "hsi" and R.angular_mask == (True, False, False)
    np.testing.assert_array_equal(R.values, vals)
    raw = p.read_bytes()
    for bad in (b"XXXX" + raw[4:], raw[:4] + (2).to_bytes(4, "little") + raw[8:], raw[:-8]):
        q = tmp_path / "bad.mlut"
        q.write_bytes(bad)
        with pytest.raises(MalformedHeader):
            lut.load_lut(q)


def test_mlut_bytes_match_reference(tmp_path):
    """save_lut writes byte-identical files to the reference's (lut.py:353-361)."""
    import os
    ref = os.path.join(os.path.dirname(__file__), "golden", "ref_hsi9.mlut")
    L = lut.Lut3D(9, 255 / 8, "hsi", O.build_lut_values("hsi", 9), lut.ANGULAR_MASKS["hsi"])
    p = tmp_path / "ours.mlut"
    lut.save_lut(L, p)
    assert p.read_bytes() == open(ref, "rb").read()
    R = lut.load_lut(ref)
    np.testing.assert_array_equal(R.values, L.values)


def _lab_seg_model():
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts", "lab_seg_design.py")
    spec = importlib.util.spec_from_file_location("lab_seg_design", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("degs", [(4, 4), (2, 2)])
def test_lab_segmented_fp32_model(degs):
    """CPU model of the segmented fp32 CIELAB kernel (scripts/lab_seg_design.py:
    16 segments per binade, cubic, (hi, small part) epilogue) on the degenerate
    probe sets of SURVEY §4.4 plus 2^20 cube colours: inside the 1e-4 tolerance."""
    M = _lab_seg_model()
    cfg = O.OracleConfig(cielab_degrees=degs)
    tab, base, shift, fit_err = M.build_table(cfg.cbrt_num, cfg.cbrt_den, 16, 3, lo_split=False)
    assert fit_err < 1e-8
    f32 = np.float32
    grays = np.repeat(np.arange(256, dtype=np.uint8)[:, None], 3, axis=1)
    rg0 = np.stack([np.zeros(256), np.zeros(256), np.arange(256)], 1).astype(np.uint8)
    face = np.random.default_rng(3).integers(0, 256, (4096, 3)).astype(np.uint8)
    face[:, 0] = 255
    px = np.concatenate([grays, rg0, face, O.cube_chunk(7 << 20, 1 << 20)])
    ref = O.rgb_to_lab_fast(px, cfg)
    gam = O.GAMMA_TABLE.astype(f32)
    m = np.array([[O.RGB_TO_XYZ[r, c] / O.WHITE[r] for c in range(3)] for r in range(3)]).astype(f32)
    gr, gg, gb = gam[px[:, 0]], gam[px[:, 1]], gam[px[:, 2]]
    hs, ds = [], []
    for r in range(3):
        t = M.fma_arr(m[r, 2], gb, M.fma_arr(m[r, 1], gg, (m[r, 0] * gr).astype(f32)))
        h, d = M.seg_eval(t, tab, base, shift, 3, False)
        low = ~(t > f32(O.LAB_KNEE))
        off_hi = f32(O.LAB_LINEAR_OFFSET)
        hs.append(np.where(low, off_hi, h))
        ds.append(np.where(low, M.fma_arr(f32(O.LAB_LINEAR_SLOPE), t, f32(O.LAB_LINEAR_OFFSET - np.float64(off_hi))), d))
    (hx, hy, hz), (dx, dy, dz) = hs, ds
    L = M.fma_arr(f32(116), dy, M.fma_arr(f32(116), hy, f32(-16)))
    A = (f32(500) * ((hx - hy) + (dx - dy))).astype(f32)
    B = (f32(200) * ((hy - hz) + (dy - dz))).astype(f32)
    err = np.abs(np.stack([L, A, B], -1).astype(np.float64) - ref)
    assert err.max() <= 1e-4, err.max(axis=0)


def test_shift_free_div255_magic():
    """lut_locate / the 17^3 ghost-plane locate divide x = p (n-1) by 255 as
    hi(x * 0x01010102) (csrc/mact_lut.cuh): exact for every x <= 8160 (33^3)."""
    x = np.arange(0, 8161, dtype=np.uint64)
    assert np.array_equal((x * np.uint64(0x01010102)) >> np.uint64(32), x // np.uint64(255))


def test_lut_cell_is_a_shift_for_byte_pixels():
    """lut_locate (csrc/mact_lut.cuh) for n = 9 / 17 / 33: the reference's cell
    min(p (n-1) div 255, n-2) (lut.py:98-105) equals p >> log2(256 / (n-1)) for
    every byte p, the clamp at p = 255 included."""
    p = np.arange(256)
    for n, s in ((9, 5), (17, 4), (33, 3)):
        assert np.array_equal(np.minimum(p * (n - 1) // 255, n - 2), p >> s)
