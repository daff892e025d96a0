"""GPU parity of the MACT fast transforms (K1-K3, fused triple) against the
reference golden vectors and the CPU oracle, through the C ABI."""

import numpy as np
import pytest

from oracle import mact_oracle as O
from tests.parity_util import CHECK, check_hsi, check_lab, check_sct

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    from paper_1009_0854_b200 import _lib, exact, fast, harness, lut
    _lib.load()
    return {"fast": fast, "exact": exact, "lut": lut, "harness": harness}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_probe_vs_reference_golden(P, golden, space):
    got = getattr(P["fast"], f"rgb_to_{space}_fast")(dev(golden["probe"])).cpu().numpy()
    CHECK[space](got, golden[f"{space}_fast"])


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_full_cube_vs_oracle(P, space):
    """All 2^24 colours (BASELINE config 2 population) against the oracle."""
    cube = P["harness"].cube_chunk(0, 1 << 24, device="cuda")
    got = getattr(P["fast"], f"rgb_to_{space}_fast")(cube).cpu().numpy()
    host = cube.cpu().numpy()
    np.testing.assert_array_equal(host, O.cube_chunk(0, 1 << 24))
    for s in range(0, 1 << 24, 1 << 22):
        CHECK[space](got[s:s + (1 << 22)], O.FAST[space](host[s:s + (1 << 22)]))


@pytest.mark.parametrize("degs", [(2, 2), (2, 3), (3, 2), (2, 4), (3, 3), (4, 2), (3, 4), (4, 3)])
def test_lab_full_cube_every_degree(P, degs):
    """The segmented fp32 lightness kernel is fitted per configuration: every
    bundled rational, all 2^24 colours, against the oracle (default (4,4) is
    test_full_cube_vs_oracle)."""
    from paper_1009_0854_b200 import _lib
    fast = P["fast"]
    cfg = fast.MactConfig(cielab_degrees=degs)
    import ctypes
    assert _lib.load().mact_lab_eval_path(ctypes.byref(cfg._pack())) == _lib.LAB_PATH_SEG
    cube = P["harness"].cube_chunk(0, 1 << 24, device="cuda")
    got = fast.rgb_to_lab_fast(cube, cfg).cpu().numpy()
    host = cube.cpu().numpy()
    ocfg = O.OracleConfig(cielab_degrees=degs)
    for s in range(0, 1 << 24, 1 << 22):
        check_lab(got[s:s + (1 << 22)], O.rgb_to_lab_fast(host[s:s + (1 << 22)], ocfg))


@pytest.mark.parametrize("degs", [(4, 4), (3, 3)])
def test_lab_fp64_fallback_full_cube(P, degs, monkeypatch):
    """MACT_LAB_EVAL=fp64 keeps the fp64 evaluation (monic (4,4) quotient, P/Q
    otherwise) -- the path a configuration whose segment fit fails takes."""
    import ctypes
    from paper_1009_0854_b200 import _lib
    monkeypatch.setenv("MACT_LAB_EVAL", "fp64")
    fast = P["fast"]
    cfg = fast.MactConfig(cielab_degrees=degs)
    want = _lib.LAB_PATH_MONIC if degs == (4, 4) else _lib.LAB_PATH_PQ
    assert _lib.load().mact_lab_eval_path(ctypes.byref(cfg._pack())) == want
    cube = P["harness"].cube_chunk(0, 1 << 24, device="cuda")
    got = fast.rgb_to_lab_fast(cube, cfg).cpu().numpy()
    host = cube.cpu().numpy()
    ocfg = O.OracleConfig(cielab_degrees=degs)
    for s in range(0, 1 << 24, 1 << 22):
        check_lab(got[s:s + (1 << 22)], O.rgb_to_lab_fast(host[s:s + (1 << 22)], ocfg))


def test_other_degrees(P, golden):
    fast = P["fast"]
    s = dev(golden["small"])
    for n, m in [(2, 2), (2, 3), (3, 2), (2, 4), (3, 3), (4, 2), (3, 4), (4, 3)]:
        check_lab(fast.rgb_to_lab_fast(s, fast.MactConfig(cielab_degrees=(n, m))).cpu().numpy(),
                  golden[f"lab_fast_{n}{m}"])
    for n in (2, 3, 4):
        check_hsi(fast.rgb_to_hsi_fast(s, fast.MactConfig(hsi_degree=n)).cpu().numpy(),
                  golden[f"hsi_fast_{n}"])
    for d in [(4, 4, 4), (4, 5, 4), (5, 4, 4), (5, 5, 4), (4, 4, 5), (4, 5, 5), (5, 4, 5)]:
        check_sct(fast.rgb_to_sct_fast(s, fast.MactConfig(sct_degrees=d)).cpu().numpy(),
                  golden["sct_fast_" + "".join(map(str, d))])


def test_float_input_path(P, golden):
    got = P["fast"].rgb_to_lab_fast(dev(golden["small_float"])).cpu().numpy()
    check_lab(got, golden["lab_fast_float"])


@pytest.mark.parametrize("n", [0, 1, 3, 5, 2047, 2048, 2049, 4097, 100003])
@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_ragged_sizes_and_tail(P, n, space):
    rng = np.random.default_rng(n)
    px = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    got = getattr(P["fast"], f"rgb_to_{space}_fast")(dev(px)).cpu().numpy()
    assert got.shape == (n, 3) and got.dtype == np.float32
    if n:
        CHECK[space](got, O.FAST[space](px))


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_unaligned_and_planar(P, space):
    rng = np.random.default_rng(7)
    px = rng.integers(0, 256, (65536 + 1, 3), dtype=np.uint8)
    d = dev(px)
    fn = getattr(P["fast"], f"rgb_to_{space}_fast")
    full = fn(d).cpu().numpy()
    sub = fn(d[1:]).cpu().numpy()          # 3-byte offset: not 16-B aligned -> generic kernel
    np.testing.assert_array_equal(sub, full[1:])
    planar = fn(d[:65536], layout="planar").cpu().numpy()
    np.testing.assert_array_equal(planar.T, full[:65536])


@pytest.mark.parametrize("spaces", [("hsi", "sct"), ("lab", "hsi"), ("sct", "lab"), ("hsi",)])
def test_fused_subsets_match_single(P, spaces):
    """mact_all_fast with NULL outputs: every subset equals the single transforms."""
    fast = P["fast"]
    rng = np.random.default_rng(12)
    d = dev(rng.integers(0, 256, ((1 << 20) + 77, 3), dtype=np.uint8))
    got = fast.rgb_to_all_fast(d, spaces=spaces)
    for sp, g in zip(spaces, got):
        np.testing.assert_array_equal(g.cpu().numpy(), getattr(fast, f"rgb_to_{sp}_fast")(d).cpu().numpy())
    planar = fast.rgb_to_all_fast(d[:65536], spaces=spaces, layout="planar")
    for sp, g in zip(spaces, planar):
        np.testing.assert_array_equal(g.cpu().numpy().T, getattr(fast, f"rgb_to_{sp}_fast")(d[:65536]).cpu().numpy())
    with pytest.raises(ValueError):
        fast.rgb_to_all_fast(d, spaces=("hsi", "hsi"))


def test_fused_all_matches_single(P):
    fast = P["fast"]
    rng = np.random.default_rng(11)
    d = dev(rng.integers(0, 256, (1 << 20, 3), dtype=np.uint8))
    lab, hsi, sct = fast.rgb_to_all_fast(d)
    np.testing.assert_array_equal(lab.cpu().numpy(), fast.rgb_to_lab_fast(d).cpu().numpy())
    np.testing.assert_array_equal(hsi.cpu().numpy(), fast.rgb_to_hsi_fast(d).cpu().numpy())
    np.testing.assert_array_equal(sct.cpu().numpy(), fast.rgb_to_sct_fast(d).cpu().numpy())


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_host_executor_matches_device(P, space):
    """numpy in -> numpy out through mact_transform_host (pageable and pinned)."""
    fn = getattr(P["fast"], f"rgb_to_{space}_fast")
    rng = np.random.default_rng(5)
    n = (1 << 24) + 12345                     # > 2 host chunks + ragged tail
    px = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    ref = fn(dev(px)).cpu().numpy()
    got = fn(px)
    assert isinstance(got, np.ndarray) and got.dtype == np.float32
    np.testing.assert_array_equal(got, ref)
    pin_in = torch.empty((n, 3), dtype=torch.uint8).pin_memory()
    pin_in.numpy()[...] = px
    pin_out = torch.empty((n, 3), dtype=torch.float32).pin_memory()
    fn(pin_in.numpy(), out=pin_out.numpy())
    np.testing.assert_array_equal(pin_out.numpy(), ref)
    planar = fn(px[:4096], layout="planar")
    np.testing.assert_array_equal(planar.T, ref[:4096])


def test_known_answers(P):
    fast = P["fast"]
    lab = fast.rgb_to_lab_fast(np.array([[255, 0, 0], [37, 201, 88]], np.uint8))
    np.testing.assert_allclose(lab[0], [53.2364392, 80.0948249, 67.2005027], atol=1e-4)
    np.testing.assert_allclose(lab[1], [73.6499493, -61.4765821, 40.5739238], atol=1e-4)
    h = fast.rgb_to_hsi_fast(np.array([[255, 0, 0], [0, 0, 1], [9, 9, 9]], np.uint8))
    np.testing.assert_allclose(h[0], [0, 1, 1 / 3], atol=1e-6)
    assert abs(h[1, 0] - 4.18897983) < 1e-5 and np.isnan(h[2, 0])
    s = fast.rgb_to_sct_fast(np.array([[255, 0, 0], [0, 0, 7], [0, 0, 0]], np.uint8))
    np.testing.assert_allclose(s[0], [255, np.pi / 2, 2.073866e-5], atol=1e-5)
    assert np.isnan(s[1, 2]) and s[2, 0] == 0 and s[2, 1] == 0 and np.isnan(s[2, 2])


def test_determinism(P):
    d = dev(np.random.default_rng(3).integers(0, 256, (1 << 21, 3), dtype=np.uint8))
    for sp in ("lab", "hsi", "sct"):
        fn = getattr(P["fast"], f"rgb_to_{sp}_fast")
        a, b = fn(d).cpu().numpy(), fn(d).cpu().numpy()
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))


def test_unknown_approximant_and_bad_args(P):
    from paper_1009_0854_b200.errors import UnknownApproximant
    fast = P["fast"]
    with pytest.raises(UnknownApproximant):
        fast.MactConfig(cielab_degrees=(5, 5))
    with pytest.raises(ValueError):
        fast.rgb_to_lab_fast(np.zeros((4, 2), np.uint8))
    with pytest.raises(ValueError):
        fast.transform("xyz", np.zeros((4, 3), np.uint8))


@pytest.mark.parametrize("degenerate", [False, True])
def test_corpus_images_vs_oracle(P, degenerate):
    """BASELINE configs 4/5 content: correlated synthetic images (config 5 adds 10 %
    saturated channels and 5 % exact grays, exercising the hue singularity)."""
    from paper_1009_0854_b200 import corpus
    img = corpus.correlated_image(3, 270, 480, degenerate=degenerate)      # 1/8-scale 1080p
    host = img.cpu().numpy()
    flat = host.reshape(-1, 3)
    if degenerate:
        gray = (flat[:, 0] == flat[:, 1]) & (flat[:, 1] == flat[:, 2])
        assert gray.mean() > 0.04 and ((flat == 0) | (flat == 255)).any(axis=1).mean() > 0.08
    lab, hsi, sct = P["fast"].rgb_to_all_fast(img)
    CHECK["lab"](lab.cpu().numpy(), O.rgb_to_lab_fast(host))
    CHECK["hsi"](hsi.cpu().numpy(), O.rgb_to_hsi_fast(host))
    CHECK["sct"](sct.cpu().numpy(), O.rgb_to_sct_fast(host))
    # the same bytes through the single-transform kernels
    np.testing.assert_array_equal(P["fast"].rgb_to_hsi_fast(img).cpu().numpy(), hsi.cpu().numpy())


def test_corpus_deterministic_per_image_seed(P):
    """Image i has the same bytes whatever the shard (sharding by image)."""
    from paper_1009_0854_b200 import corpus
    a = corpus.batch(range(2, 5), 64, 96)
    b = corpus.batch([4], 64, 96)
    np.testing.assert_array_equal(a[2].cpu().numpy(), b[0].cpu().numpy())


@pytest.mark.parametrize("space", ["lab", "sct"])
def test_beyond_int32_pixel_count(P, space):
    """One call over 2^31 + 4099 pixels (BASELINE config 5 is 2.12 G px per GPU):
    64-bit indexing in the tile, tail and store paths.  Pixels repeat the cube
    enumeration, so any output position can be checked against the oracle."""
    n = (1 << 31) + 4099
    x = P["harness"].cube_chunk(0, 1 << 24, device="cuda").repeat((n >> 24) + 1, 1)[:n]
    out = getattr(P["fast"], f"rgb_to_{space}_fast")(x)
    idx = np.r_[0:64, (1 << 31) - 64:(1 << 31) + 64, n - 4099 - 64:n]
    got = out[torch.from_numpy(idx).cuda()].cpu().numpy()
    CHECK[space](got, O.FAST[space](O.cube_chunk(0, 1 << 24)[idx % (1 << 24)]))
    del out, x
    torch.cuda.empty_cache()
