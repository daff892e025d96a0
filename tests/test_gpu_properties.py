"""Property-based parity (hypothesis): random shapes, dtypes, degrees, layouts and
LUT methods against the oracle, plus size-independent properties."""

import numpy as np
import pytest

from oracle import mact_oracle as O
from tests.parity_util import CHECK, check_lab

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402

SETTINGS = settings(max_examples=150, deadline=None, suppress_health_check=list(HealthCheck))

DEGREES = {"lab": [dict(cielab_degrees=d) for d in [(2, 2), (3, 3), (4, 4), (2, 4), (4, 3)]],
           "hsi": [dict(hsi_degree=d) for d in (2, 3, 4, 5)],
           "sct": [dict(sct_degrees=d) for d in [(4, 4, 4), (5, 5, 5), (4, 5, 4)]]}
ORACLE_CFG = {"lab": lambda k: O.OracleConfig(cielab_degrees=k["cielab_degrees"]),
              "hsi": lambda k: O.OracleConfig(hsi_degree=k["hsi_degree"]),
              "sct": lambda k: O.OracleConfig(sct_degrees=k["sct_degrees"])}


@pytest.fixture(scope="module")
def M():
    from paper_1009_0854_b200 import _lib, fast, lut
    _lib.load()
    return {"fast": fast, "lut": lut}


@st.composite
def images(draw):
    shape = draw(st.sampled_from([(1,), (7,), (3, 5), (64, 65), (2, 3, 129), (4099,)]))
    seed = draw(st.integers(0, 2 ** 31 - 1))
    return np.random.default_rng(seed).integers(0, 256, shape + (3,), dtype=np.uint8)


@SETTINGS
@given(img=images(), space=st.sampled_from(["lab", "hsi", "sct"]), di=st.integers(0, 4),
       layout=st.sampled_from(["interleaved", "planar"]), on_dev=st.booleans())
def test_fast_transforms_random(M, img, space, di, layout, on_dev):
    kw = DEGREES[space][di % len(DEGREES[space])]
    cfg = M["fast"].MactConfig(**kw)
    x = torch.from_numpy(img).cuda() if on_dev else img
    got = getattr(M["fast"], f"rgb_to_{space}_fast")(x, cfg, layout=layout)
    got = got.cpu().numpy() if on_dev else got
    if layout == "planar":
        got = np.moveaxis(got, 0, -1)
    assert got.shape == img.shape
    CHECK[space](got, O.FAST[space](img, ORACLE_CFG[space](kw)))


@SETTINGS
@given(img=images(), grid=st.sampled_from([9, 17, 33]),
       method=st.sampled_from(["trilinear", "prism", "pyramidal", "tetrahedral"]))
def test_lut_random(M, img, grid, method):
    L = M["lut"].build_lut("lab", grid)
    got = M["lut"].interpolate(L, img, method)
    vals = O.build_lut_values("lab", grid).astype(np.float32).astype(np.float64)
    check_lab(got, O.interpolate(vals, img, method))
    idx, _ = M["lut"].node_weights(L, img, method)
    ref_idx, _ = O.node_weights(grid, img.reshape(-1, 3), method)
    np.testing.assert_array_equal(np.asarray(idx).reshape(ref_idx.shape), ref_idx)


@SETTINGS
@given(img=images(), space=st.sampled_from(["lab", "hsi", "sct"]))
def test_permutation_equivariance(M, img, space):
    """Per-pixel independence: transforming a permuted stream permutes the result."""
    flat = img.reshape(-1, 3)
    perm = np.random.default_rng(flat.shape[0]).permutation(flat.shape[0])
    fn = getattr(M["fast"], f"rgb_to_{space}_fast")
    a = fn(flat)[perm]
    b = fn(np.ascontiguousarray(flat[perm]))
    np.testing.assert_array_equal(a, b)


@st.composite
def device_views(draw):
    """A device image of 1 .. 400k pixels as a view at a byte offset of 0..3 into its buffer (16-byte
    aligned, 4-byte aligned or unaligned input), with a colour distribution that is uniform, confined
    to one r-half, or mostly in one r-half (the 33^3 kernel's CTAs split the pixels by bit 7 of r)."""
    n = draw(st.one_of(st.integers(1, 700), st.integers(3000, 20000), st.integers(100_000, 400_000)))
    off = draw(st.sampled_from([0, 0, 4, 8, 1, 3]))
    kind = draw(st.sampled_from(["uniform", "dark", "bright", "mostly_dark", "runs"]))
    seed = draw(st.integers(0, 2 ** 31 - 1))
    rng = np.random.default_rng(seed)
    img = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    if kind == "dark":
        img[:, 0] &= 0x7F
    elif kind == "bright":
        img[:, 0] |= 0x80
    elif kind == "mostly_dark":
        img[rng.random(n) < 0.9, 0] &= 0x7F
    elif kind == "runs":                       # runs of ~200 pixels alternating between the halves
        img[(np.arange(n) // 200) % 2 == 0, 0] &= 0x7F
        img[(np.arange(n) // 200) % 2 == 1, 0] |= 0x80
    return img, off


@settings(max_examples=200, deadline=None, suppress_health_check=list(HealthCheck))
@given(view=device_views(), grid=st.sampled_from([17, 33, 33]),
       method=st.sampled_from(["trilinear", "prism", "pyramidal", "tetrahedral"]),
       layout=st.sampled_from(["interleaved", "planar"]))
def test_lut_device_views_random(M, view, grid, method, layout):
    """The streaming / split LUT kernels on device buffers of arbitrary size and alignment: every
    combination matches the oracle within the tolerance."""
    img, off = view
    n = img.shape[0]
    buf = torch.zeros(3 * n + 16, dtype=torch.uint8, device="cuda")
    buf[off:off + 3 * n] = torch.from_numpy(img.reshape(-1)).cuda()
    x = buf[off:off + 3 * n].view(n, 3)
    L = M["lut"].build_lut("lab", grid)
    got = M["lut"].interpolate(L, x, method, layout=layout).cpu().numpy()
    if layout == "planar":
        got = got.T
    vals = O.build_lut_values("lab", grid).astype(np.float32).astype(np.float64)
    check_lab(got, O.interpolate(vals, img, method))
