"""GPU parity of the drop-in names added for the reference's public surface:

* eval_poly / eval_rational and callable Polynomial / Rational / Approximant
  (approximants.py:40-82, :138), bit-identical to the reference;
* TargetFn.exact (approximants.py:101-115), libdevice vs numpy libm;
* harness.DISTANCES (harness.py:28-32);
* lut.build_cache and interpolate(..., variant="caching") (lut.py:265-331),
  bit-identical for linear destinations with fp64 output.

Fixtures: tests/golden/caching_outputs.npz, written by the live reference
(tests/golden/make_golden.py --caching-only).
"""

import hashlib

import numpy as np
import pytest

from oracle import mact_oracle as O
from tests.parity_util import CHECK

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_1009_0854_b200 as pkg
    from paper_1009_0854_b200 import _lib, approximants, exact, harness, lut
    _lib.load()
    return {"pkg": pkg, "ap": approximants, "exact": exact, "harness": harness, "lut": lut}


def test_eval_poly_rational_bit_exact(P, caching_golden):
    ap = P["ap"]
    x = caching_golden["poly_x"]
    for fn, deg in ap.registry_keys():
        a = ap.registry_get(fn, deg)
        ref = caching_golden[f"poly_{fn.value}_{'_'.join(map(str, deg))}"]
        np.testing.assert_array_equal(a(x), ref)                       # Approximant.__call__
        np.testing.assert_array_equal(a.form(x), ref)                  # Polynomial / Rational.__call__
        if isinstance(a.form, ap.Rational):
            np.testing.assert_array_equal(P["pkg"].eval_rational(a.form, x), ref)
        else:
            np.testing.assert_array_equal(P["pkg"].eval_poly(a.form, x), ref)
        # device tensors stay on the device
        d = a(torch.from_numpy(x).cuda())
        assert d.is_cuda
        np.testing.assert_array_equal(d.cpu().numpy(), ref)


def test_eval_poly_scalars_and_shapes(P):
    ap = P["ap"]
    p = ap.Polynomial((1.0, -2.0, 0.5))
    v = ap.eval_poly(p, 0.3)
    assert isinstance(v, float) and v == (0.5 * 0.3 + -2.0) * 0.3 + 1.0
    x = np.linspace(0, 1, 24).reshape(2, 3, 4)
    assert ap.eval_poly(p, x).shape == (2, 3, 4)
    np.testing.assert_array_equal(ap.eval_poly(ap.Polynomial((7.0,)), x), np.full(x.shape, 7.0))
    big = ap.Polynomial(tuple(1.0 / (k + 1) for k in range(20)))           # beyond the registry's degrees
    ref = np.full(x.shape, big.coeffs[-1])
    for c in big.coeffs[-2::-1]:
        ref *= x
        ref += c
    np.testing.assert_array_equal(ap.eval_poly(big, x), ref)


def test_degenerate_denominator(P):
    from paper_1009_0854_b200.errors import DegenerateDenominator
    ap = P["ap"]
    r = ap.Rational(ap.Polynomial((1.0,)), ap.Polynomial((-0.5, 1.0)))
    with pytest.raises(DegenerateDenominator):
        ap.eval_rational(r, np.array([0.1, 0.5, 0.9]))
    with pytest.raises(DegenerateDenominator):
        r(0.5)
    assert r(1.0) == 2.0


def test_target_fn_exact(P, caching_golden):
    x = caching_golden["target_x"]
    for fn in P["ap"].TargetFn:
        got = fn.exact(x)
        np.testing.assert_allclose(got, caching_golden[f"target_{fn.value}"], rtol=4e-16, atol=1e-300)
    assert isinstance(P["ap"].TargetFn.CBRT.exact(0.125), float)
    assert P["ap"].TargetFn.CBRT.exact(0.125) == 0.5


def test_measured_max_error(P):
    a = P["ap"].registry_get(P["ap"].TargetFn.CBRT, (4, 4))
    e = a.measured_max_error(20001)
    assert 0.5 * a.eps_max <= e <= 1.5 * a.eps_max


def test_distances_table(P, golden):
    D = P["harness"].DISTANCES
    assert set(D) == {"lab", "hsi", "sct"}
    np.testing.assert_allclose(D["lab"](golden["lab_fast"], golden["lab_exact"]), golden["lab_dist"],
                               rtol=1e-9, atol=1e-12)


def _ref_lut(P, space, n):
    lut = P["lut"]
    return lut.Lut3D(n, 255.0 / (n - 1), space, O.build_lut_values(space, n), lut.ANGULAR_MASKS[space])


@pytest.mark.parametrize("n", [9, 17, 33])
def test_build_cache_arrays(P, caching_golden, n):
    """Device-built cache arrays, reference-shaped and bit-identical (on the reference's lattice)."""
    c = P["lut"].build_cache(_ref_lut(P, "lab", n))
    for key in ("trilinear", "corner_diff"):
        arr = c.cache[key]
        assert arr.shape == (n - 1, n - 1, n - 1, 8, 3) and arr.dtype == np.float64
        assert hashlib.sha256(np.ascontiguousarray(arr).tobytes()).digest() == \
            caching_golden[f"cache_sha_{n}_{key}"].tobytes(), key


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
@pytest.mark.parametrize("n", [9, 17, 33])
def test_caching_variant(P, caching_golden, space, n):
    lut = P["lut"]
    L = _ref_lut(P, space, n)
    C = lut.build_cache(L)
    for method in O.METHODS:
        for key in ("cach", "cachf"):
            px = caching_golden["px" if key == "cach" else "fpx"]
            ref = caching_golden[f"{key}_{space}_{n}_{method}"]
            got = lut.interpolate(C, px, method, "caching", out_dtype="float64")
            if space == "lab":
                np.testing.assert_array_equal(got, ref)          # linear destination: bit-identical
            else:
                CHECK[space](got, ref, atol=1e-9)                # angular blend: libdevice sincos/atan2
            got32 = lut.interpolate(C, torch.from_numpy(px).cuda(), method, "caching").cpu().numpy()
            CHECK[space](got32, ref)
    # a host-side (reference-built) cache is uploaded and used as is
    C2 = lut.Lut3D(n, L.spacing, space, L.values, L.angular_mask,
                   cache={k: v.copy() for k, v in C.cache.items()})
    np.testing.assert_array_equal(
        lut.interpolate(C2, caching_golden["fpx"], "tetrahedral", "caching", out_dtype="float64"),
        lut.interpolate(C, caching_golden["fpx"], "tetrahedral", "caching", out_dtype="float64"))
