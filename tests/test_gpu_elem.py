"""GPU parity of the reference's scalar building blocks (mact_approx_eval,
mact_exact_elem, mact_exact HSI-arccos) against the reference's own outputs
(tests/golden/elem_outputs.npz, reference_outputs.npz)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def elem():
    return np.load(os.path.join(HERE, "golden", "elem_outputs.npz"))


@pytest.fixture(scope="module")
def M():
    from paper_1009_0854_b200 import _lib, approximants, exact, fast
    _lib.load()
    return {"fast": fast, "exact": exact, "A": approximants}


def eq(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


def test_cbrt_fast_bit_exact(M, elem):
    A, fast = M["A"], M["fast"]
    for n, m in [(2, 2), (3, 4), (4, 4)]:
        eq(fast.cbrt_fast(elem["t"], A.registry_get(A.TargetFn.CBRT, (n, m))), elem[f"cbrt_{n}{m}"])
    for n in (3, 5):
        eq(fast.cbrt_fast(elem["t"], A.registry_get(A.TargetFn.CBRT, (n,))), elem[f"cbrt_poly{n}"])


def test_trig_approximants_bit_exact(M, elem):
    A, fast = M["A"], M["fast"]
    for n in (2, 3, 4, 5):
        eq(fast.atan_sqrt3_fast(elem["x"], A.hsi_refit(n)), elem[f"atan_sqrt3_{n}"])
    for d in [(4, 4, 4), (5, 5, 5), (4, 5, 4)]:
        cfg = fast.MactConfig(sct_degrees=d)
        key = "".join(map(str, d))
        eq(fast.acos_fast(elem["x"], cfg), elem[f"acos_{key}"])
        eq(fast.atan_unit_fast(elem["g"], elem["r"], cfg), elem[f"atan_unit_{key}"])


def test_device_in_device_out_and_broadcast(M, elem):
    fast = M["fast"]
    x = torch.from_numpy(elem["x"]).cuda()
    y = fast.acos_fast(x)
    assert isinstance(y, torch.Tensor) and y.is_cuda and y.dtype == torch.float64
    eq(y.cpu().numpy(), elem["acos_555"])
    # scalar r broadcast against an array of g
    g = np.linspace(0, 2, 101)
    eq(fast.atan_unit_fast(g, 1.0), fast.atan_unit_fast(g, np.ones_like(g)))
    assert np.asarray(fast.acos_fast(0.25)).shape == ()


def test_error_conventions(M):
    from paper_1009_0854_b200.approximants import Approximant, Polynomial, Rational, TargetFn
    from paper_1009_0854_b200.errors import DegenerateDenominator, UndefinedAngle
    fast = M["fast"]
    bad = Approximant(Rational(Polynomial((1.0,)), Polynomial((1.0, -1.0))), (0.0, 2.0), 0.0, TargetFn.CBRT)
    with pytest.raises(DegenerateDenominator):
        fast.cbrt_fast(np.array([0.5, 1.0]), bad)
    fast.cbrt_fast(np.array([0.5, 0.75]), bad)                     # no vanishing point: fine
    with pytest.raises(UndefinedAngle):
        fast.atan_unit_fast(0.0, 0.0)
    assert np.isnan(fast.atan_unit_fast(np.array([0.0]), np.array([0.0]))[0])


def test_exact_building_blocks(M, elem):
    """libdevice pow/cbrt vs libm: within a few ulp; the rest is bit-exact."""
    ex = M["exact"]
    np.testing.assert_allclose(ex.inverse_gamma(elem["k"]), elem["inverse_gamma"], rtol=4e-16, atol=0)
    eq(np.stack(ex.rgb_to_xyz(*elem["rgb_lin"])), elem["rgb_to_xyz"])
    np.testing.assert_allclose(ex.lab_f(elem["t"][:-1]), elem["lab_f"], rtol=4e-16, atol=0)
    xyz = elem["rgb_lin"] * np.array([[0.95], [1.0], [1.09]])
    np.testing.assert_allclose(ex.xyz_to_lab(*xyz), elem["xyz_to_lab"], rtol=0, atol=1e-12)


def test_hsi_arccos_vs_reference(M, golden):
    got = M["exact"].rgb_to_hsi_arccos(golden["probe"])
    ref = golden["hsi_arccos"]
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12, equal_nan=True)


def test_angular_lerp(elem):
    from paper_1009_0854_b200 import lut
    got = lut.angular_lerp(*elem["lerp_in"])
    ref = elem["angular_lerp"]
    d = np.abs(got - ref)
    d = np.minimum(d, 2 * np.pi - d)                 # 0 and 2 pi are the same angle
    assert d.max() < 1e-12
    assert np.isclose(got[0], 0.0)                   # antipodal at alpha 0.5 -> theta0


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_exact_f32_comparator(M, space):
    """fp32 libdevice exact transforms (Table 4 comparator) stay inside the
    north-star tolerance of the fp64 reference on the full cube."""
    from oracle import mact_oracle as O
    from tests.parity_util import CHECK
    from paper_1009_0854_b200 import harness
    cube = harness.cube_chunk(0, 1 << 24, device="cuda")
    got = M["exact"].exact_f32(space, cube).cpu().numpy()
    host = cube.cpu().numpy()
    for s in range(0, 1 << 24, 1 << 22):
        CHECK[space](got[s:s + (1 << 22)], O.EXACT[space](host[s:s + (1 << 22)]))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_float_pixels_fast_and_exact(M, elem, space, dtype):
    """Real-valued pixels: analytic gamma / real-channel formulas (fast.py:91-99, exact.py)."""
    from tests.parity_util import CHECK
    px = elem["float_px"].astype(dtype)
    ref_px = px.astype(np.float64)                      # the reference computes on the fp64 values
    fast_ref = elem[f"{space}_fast_float"] if dtype == np.float64 else \
        __import__("oracle.mact_oracle", fromlist=["x"]).FAST[space](ref_px)
    CHECK[space](getattr(M["fast"], f"rgb_to_{space}_fast")(px), fast_ref)
    exact_ref = elem[f"{space}_exact_float"] if dtype == np.float64 else \
        __import__("oracle.mact_oracle", fromlist=["x"]).EXACT[space](ref_px)
    got = getattr(M["exact"], f"rgb_to_{space}_exact")(px)
    CHECK[space](got, exact_ref)


@pytest.mark.parametrize("grid", [9, 17, 33])
@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_lut_real_valued_pixels(elem, space, grid):
    """lut.interpolate on float pixels (fp64 cell location, lut.py:98-199), every
    method, linear and angular destinations, including extrapolation outside [0, 255]."""
    from tests.parity_util import CHECK
    from paper_1009_0854_b200 import lut
    L = lut.build_lut(space, grid)
    for dtype in (np.float64, np.float32):
        px = elem["lut_px"].astype(dtype)
        for m in ("trilinear", "prism", "pyramidal", "tetrahedral"):
            if dtype == np.float64:
                ref = elem[f"lutf_{space}_{grid}_{m}"]          # the reference itself
            else:                                               # fp32 pixels: oracle on their fp64 values
                from oracle import mact_oracle as O
                ref = O.interpolate(O.build_lut_values(space, grid), px.astype(np.float64), m,
                                    angular_mask=O.ANGULAR_MASKS[space])
            CHECK[space](lut.interpolate(L, px, m), ref)


@pytest.mark.parametrize("grid", [9, 17, 33])
def test_lut_node_weights_real_pixels_bit_exact(elem, grid):
    """node_weights on float pixels: indices and fp64 weights bit-identical to the reference."""
    from paper_1009_0854_b200 import lut
    L = lut.build_lut("lab", grid)
    for m in ("trilinear", "prism", "pyramidal", "tetrahedral"):
        nodes, w = lut.node_weights(L, elem["lut_px"], m)
        eq(nodes, elem[f"nodesf_{grid}_{m}"])
        eq(w, elem[f"weightsf_{grid}_{m}"])


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_fast_f64_bit_identical_to_reference(M, golden, space):
    """out_dtype="float64": the reference's own arithmetic, bit for bit on the probe set."""
    got = getattr(M["fast"], f"rgb_to_{space}_fast")(golden["probe"], out_dtype="float64")
    assert got.dtype == np.float64
    eq(got, golden[f"{space}_fast"])


def test_fast_f64_other_degrees_and_layouts(M, golden):
    fast = M["fast"]
    s = golden["small"]
    for n, m in [(2, 2), (3, 4), (4, 3)]:
        eq(fast.rgb_to_lab_fast(s, fast.MactConfig(cielab_degrees=(n, m)), out_dtype="float64"),
           golden[f"lab_fast_{n}{m}"])
    for n in (2, 3, 4):
        eq(fast.rgb_to_hsi_fast(s, fast.MactConfig(hsi_degree=n), out_dtype="float64"), golden[f"hsi_fast_{n}"])
    for d in [(4, 4, 4), (4, 5, 5)]:
        eq(fast.rgb_to_sct_fast(s, fast.MactConfig(sct_degrees=d), out_dtype="float64"),
           golden["sct_fast_" + "".join(map(str, d))])
    planar = fast.rgb_to_hsi_fast(torch.from_numpy(s).cuda(), out_dtype="float64", layout="planar")
    eq(planar.cpu().numpy().T, fast.rgb_to_hsi_fast(s, out_dtype="float64"))


def test_fast_f64_real_valued_pixels(M, elem):
    fast = M["fast"]
    for sp in ("hsi", "sct"):                    # basic operations only: bit-identical
        eq(getattr(fast, f"rgb_to_{sp}_fast")(elem["float_px"], out_dtype="float64"), elem[f"{sp}_fast_float"])
    lab = fast.rgb_to_lab_fast(elem["float_px"], out_dtype="float64")   # libdevice pow: within ulps
    np.testing.assert_allclose(lab, elem["lab_fast_float"], rtol=0, atol=1e-12)


def test_fast_f64_full_cube_vs_oracle(M):
    """All 2^24 colours, fp64 mode, bit-identical to the oracle (itself pinned to the reference)."""
    from oracle import mact_oracle as O
    from paper_1009_0854_b200 import harness
    cube = harness.cube_chunk(0, 1 << 24, device="cuda")
    host = cube.cpu().numpy()
    for sp in ("lab", "hsi", "sct"):
        got = getattr(M["fast"], f"rgb_to_{sp}_fast")(cube, out_dtype="float64").cpu().numpy()
        for s in range(0, 1 << 24, 1 << 22):
            eq(got[s:s + (1 << 22)], O.FAST[sp](host[s:s + (1 << 22)]))


@pytest.mark.parametrize("grid", [9, 17, 33])
def test_lut_f64_bit_identical_to_reference(golden, elem, grid):
    """interpolate(out_dtype="float64"): linear destination bit-identical to lut.interpolate,
    for 8-bit and real-valued pixels."""
    from paper_1009_0854_b200 import lut
    L = lut.build_lut("lab", grid)
    for m in ("trilinear", "prism", "pyramidal", "tetrahedral"):
        got = lut.interpolate(L, golden["small"], m, out_dtype="float64")
        assert got.dtype == np.float64
        # the lattice is built on the GPU (libdevice cbrt/pow): compare against the oracle on OUR lattice
        from oracle import mact_oracle as O
        vals = L.values
        eq(got, O.interpolate(vals, golden["small"], m))
        eq(lut.interpolate(L, elem["lut_px"], m, out_dtype="float64"), O.interpolate(vals, elem["lut_px"], m))
