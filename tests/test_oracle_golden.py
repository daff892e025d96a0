"""Pin the CPU oracle (oracle/mact_oracle.py) against the real reference's outputs.

The fixtures in tests/golden/ were produced by tests/golden/make_golden.py
importing /root/reference/pkg/src/mact.  The oracle must reproduce them
bit-for-bit (same numpy operation order), except where noted.
"""

import json
import os

import numpy as np
import pytest

from oracle import mact_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def eq(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


def test_hsi_refit_frozen():
    with open(os.path.join(HERE, "golden", "hsi_refit.json")) as fh:
        ref = json.load(fh)["coeffs"]
    for n in (2, 3, 4, 5):
        assert tuple(ref[str(n)]) == O.HSI_REFIT[n]


def test_fast_transforms_bit_exact(golden):
    p = golden["probe"]
    eq(O.rgb_to_lab_fast(p), golden["lab_fast"])
    eq(O.rgb_to_hsi_fast(p), golden["hsi_fast"])
    eq(O.rgb_to_sct_fast(p), golden["sct_fast"])
    eq(O.rgb_to_lab_fast(golden["small_float"]), golden["lab_fast_float"])


def test_other_degrees_bit_exact(golden):
    s = golden["small"]
    for n, m in [(2, 2), (2, 3), (3, 2), (2, 4), (3, 3), (4, 2), (3, 4), (4, 3)]:
        eq(O.rgb_to_lab_fast(s, O.OracleConfig(cielab_degrees=(n, m))), golden[f"lab_fast_{n}{m}"])
    for n in (2, 3, 4):
        eq(O.rgb_to_hsi_fast(s, O.OracleConfig(hsi_degree=n)), golden[f"hsi_fast_{n}"])
    for d in [(4, 4, 4), (4, 5, 4), (5, 4, 4), (5, 5, 4), (4, 4, 5), (4, 5, 5), (5, 4, 5)]:
        eq(O.rgb_to_sct_fast(s, O.OracleConfig(sct_degrees=d)),
           golden["sct_fast_" + "".join(map(str, d))])


def test_exact_and_distances_bit_exact(golden):
    p = golden["probe"]
    eq(O.rgb_to_lab_exact(p), golden["lab_exact"])
    eq(O.rgb_to_hsi_exact(p), golden["hsi_exact"])
    eq(O.rgb_to_hsi_arccos(p), golden["hsi_arccos"])
    eq(O.rgb_to_sct_exact(p), golden["sct_exact"])
    eq(O.lab_distance(golden["lab_fast"], golden["lab_exact"]), golden["lab_dist"])
    eq(O.hsi_distance(golden["hsi_fast"], golden["hsi_exact"]), golden["hsi_dist"])
    eq(O.sct_distance_indirect(golden["sct_fast"], golden["sct_exact"]), golden["sct_dist"])
    eq(O.sct_to_rgb(golden["sct_exact"]), golden["sct_to_rgb"])


def test_known_answers(golden):
    """SURVEY §8c KAT pixels (values printed by the reference)."""
    lab = O.rgb_to_lab_fast(np.array([[255, 0, 0], [37, 201, 88]], np.uint8))
    np.testing.assert_allclose(lab[0], [53.2364392, 80.0948249, 67.2005027], atol=1e-6)
    np.testing.assert_allclose(lab[1], [73.6499493, -61.4765821, 40.5739238], atol=1e-6)
    h = O.rgb_to_hsi_fast(np.array([[255, 0, 0], [0, 0, 1]], np.uint8))
    np.testing.assert_allclose(h[0], [0, 1, 1 / 3], atol=1e-12)
    np.testing.assert_allclose(h[1, 0], 4.18897983, atol=1e-7)
    s = O.rgb_to_sct_fast(np.array([[255, 0, 0]], np.uint8))
    np.testing.assert_allclose(s[0], [255, np.pi / 2, 2.073866e-5], atol=1e-6)
    assert abs(O.rgb_to_lab_exact(np.array([128, 128, 128], np.uint8))[0] - 58.1774072) < 1e-6
    assert abs(O.rgb_to_sct_exact(np.array([100, 100, 100], np.uint8))[1] - 0.955317) < 1e-6


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_lut_lattices(golden, space):
    for n in (9, 17):
        eq(O.build_lut_values(space, n), golden[f"lut_{space}_{n}"])
    v = O.build_lut_values(space, 33)
    eq(v.reshape(-1, 3)[golden[f"lut_{space}_33_sample_idx"]], golden[f"lut_{space}_33_sample"])
    np.testing.assert_allclose(v.sum(axis=(0, 1, 2)), golden[f"lut_{space}_33_sum"][0], rtol=1e-13)


@pytest.mark.parametrize("n", [9, 17, 33])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut_nodes_and_interp(golden, n, method):
    s = golden["small"]
    nodes, w = O.node_weights(n, s, method)
    eq(nodes, golden[f"nodes_{n}_{method}"])
    eq(w, golden[f"weights_{n}_{method}"])
    vals = O.build_lut_values("lab", n)
    eq(O.interpolate(vals, s, method), golden[f"interp_lab_{n}_{method}"])
    # caching variant ≡ standard: reference agrees to 1e-12
    np.testing.assert_allclose(golden[f"interp_lab_{n}_{method}_caching"],
                               golden[f"interp_lab_{n}_{method}"], atol=1e-12)


@pytest.mark.parametrize("space", ["hsi", "sct"])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut_angular_interp(golden, space, method):
    s = golden["small"]
    for n in (9, 17, 33):
        vals = O.build_lut_values(space, n)
        eq(O.interpolate(vals, s, method, O.ANGULAR_MASKS[space]),
           golden[f"interp_{space}_{n}_{method}"])


def test_c1_figures(figures):
    c1 = np.random.default_rng(0).integers(0, 256, size=(512, 512, 3), dtype=np.uint8)
    assert int(c1.astype(np.int64).sum()) == figures["c1_sum"]
    st = O.measure_error("lab", O.rgb_to_lab_fast, O.rgb_to_lab_exact, c1.reshape(-1, 3))
    ref = figures["c1_lab"]
    assert st.avg == pytest.approx(ref["avg"], rel=1e-13)
    assert st.max == ref["max"] and list(st.argmax_pixel) == ref["argmax_pixel"]
    assert st.count == ref["count"]


def test_cube_chunk_enumeration():
    c = O.cube_chunk((1 << 24) - 3, 10)
    assert c.shape == (3, 3)
    eq(c[-1], [255, 255, 255])
    eq(O.cube_chunk(0, 2)[1], [0, 0, 1])
    eq(O.cube_chunk(65536 + 256 + 1, 1)[0], [1, 1, 1])


@pytest.mark.slow
def test_cube_hsi_figure(figures):
    """Full-cube HSI n=5 error figure (Table 10 row; ~10 s on 8 threads)."""
    st = O.measure_error("hsi", O.rgb_to_hsi_fast, O.rgb_to_hsi_exact, threads=O.host_threads())
    ref = figures["cube"]["hsi_5"]
    assert st.avg == pytest.approx(ref["avg"], rel=1e-13)
    assert st.max == ref["max"] and list(st.argmax_pixel) == ref["argmax_pixel"]


def test_call_counts_vs_reference(figures):
    """Oracle brute-force call-site counts == reference harness.call_probabilities."""
    got = O.call_counts()
    for k, v in figures["call_probabilities"].items():
        assert got[k] == v["count"], k
        assert got[k] / O.CUBE_SIZE == v["p"], k


@pytest.fixture(scope="module")
def elem():
    return np.load(os.path.join(HERE, "golden", "elem_outputs.npz"))


def test_scalar_approximants_vs_reference(elem):
    """cbrt_fast / atan_sqrt3_fast / acos_fast / atan_unit_fast (fast.py:81-185), bit-exact."""
    t, x = elem["t"], elem["x"]
    for n, m in [(2, 2), (3, 4), (4, 4)]:
        num, den = (O._f(c) for c in O.CBRT_RATIONALS[(n, m)])
        with np.errstate(all="ignore"):
            eq(O.cbrt_fast(t, num, den), elem[f"cbrt_{n}{m}"])
    for n in (3, 5):
        eq(O.cbrt_fast(t, O._f(O.CBRT_POLYS[n])), elem[f"cbrt_poly{n}"])
    for n in (2, 3, 4, 5):
        eq(O.atan_sqrt3_fast(x, O.HSI_REFIT[n]), elem[f"atan_sqrt3_{n}"])
    for d in [(4, 4, 4), (5, 5, 5), (4, 5, 4)]:
        cfg = O.OracleConfig(sct_degrees=d)
        key = "".join(map(str, d))
        with np.errstate(all="ignore"):
            eq(O.acos_fast(x, cfg), elem[f"acos_{key}"])
        eq(O.atan_unit_fast(elem["g"], elem["r"], cfg), elem[f"atan_unit_{key}"])


def test_exact_building_blocks_vs_reference(elem):
    """inverse_gamma / rgb_to_xyz / lab_f / xyz_to_lab (exact.py:52-83), bit-exact."""
    eq(O.inverse_gamma(elem["k"]), elem["inverse_gamma"])
    eq(np.stack(O.rgb_to_xyz(*elem["rgb_lin"])), elem["rgb_to_xyz"])
    eq(O.lab_f(elem["t"][:-1]), elem["lab_f"])
    eq(O.xyz_to_lab(*(elem["rgb_lin"] * np.array([[0.95], [1.0], [1.09]]))), elem["xyz_to_lab"])


def test_angular_lerp_vs_reference(elem):
    eq(O.angular_lerp(*elem["lerp_in"]), elem["angular_lerp"])


def test_float_pixels_vs_reference(elem):
    """Oracle fast/exact transforms on real-valued pixels == the reference's (bit-exact)."""
    for sp in ("lab", "hsi", "sct"):
        eq(O.FAST[sp](elem["float_px"]), elem[f"{sp}_fast_float"])
        eq(O.EXACT[sp](elem["float_px"]), elem[f"{sp}_exact_float"])


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_lut_real_pixels_vs_reference(elem, space):
    for n in (9, 17, 33):
        vals = O.build_lut_values(space, n)
        for m in O.METHODS:
            got = O.interpolate(vals, elem["lut_px"], m, angular_mask=O.ANGULAR_MASKS[space])
            eq(got, elem[f"lutf_{space}_{n}_{m}"])


def test_lut_node_weights_real_pixels_vs_reference(elem):
    for n in (9, 17, 33):
        for m in O.METHODS:
            nodes, w = O.node_weights(n, elem["lut_px"], m)
            eq(nodes, elem[f"nodesf_{n}_{m}"])
            eq(w, elem[f"weightsf_{n}_{m}"])


def test_cache_arrays_bit_exact(caching_golden):
    """oracle.build_cache (lut.py:265-291) equals the reference's arrays."""
    import hashlib
    for n in (9, 17, 33):
        c = O.build_cache(O.build_lut_values("lab", n))
        for key in ("trilinear", "corner_diff"):
            assert hashlib.sha256(np.ascontiguousarray(c[key]).tobytes()).digest() == \
                caching_golden[f"cache_sha_{n}_{key}"].tobytes(), (n, key)
    eq(O.build_cache(O.build_lut_values("lab", 9))["trilinear"], caching_golden["cache_9_trilinear"])


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_caching_interp_bit_exact(caching_golden, space):
    """oracle.interpolate_caching (lut.py:294-331) on uint8 and real-valued pixels."""
    for n in (9, 17, 33):
        vals = O.build_lut_values(space, n)
        cache = O.build_cache(vals)
        for method in O.METHODS:
            for key, px in (("cach", caching_golden["px"]), ("cachf", caching_golden["fpx"])):
                got = O.interpolate_caching(vals, cache, px, method, O.ANGULAR_MASKS[space])
                eq(got, caching_golden[f"{key}_{space}_{n}_{method}"])
