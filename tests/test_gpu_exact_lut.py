"""GPU parity of the exact transforms, distances (K5) and the 3D LUT (K4)."""

import os
import numpy as np
import pytest

from oracle import mact_oracle as O
from tests.parity_util import check_lab

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    from paper_1009_0854_b200 import _lib, exact, fast, harness, lut
    _lib.load()
    return {"fast": fast, "exact": exact, "lut": lut, "harness": harness}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def close(a, b, rtol=1e-12, atol=1e-12):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    np.testing.assert_array_equal(np.isnan(a), np.isnan(b))
    np.testing.assert_allclose(np.nan_to_num(a), np.nan_to_num(b), rtol=rtol, atol=atol)


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_exact_vs_reference(P, golden, space):
    got = getattr(P["exact"], f"rgb_to_{space}_exact")(dev(golden["probe"])).cpu().numpy()
    close(got, golden[f"{space}_exact"], rtol=1e-11, atol=1e-11)


def test_exact_real_inputs(P, golden):
    x = golden["small_float"]
    close(P["exact"].rgb_to_lab_exact(dev(x)).cpu().numpy(), O.rgb_to_lab_exact(x), 1e-11, 1e-11)
    close(P["exact"].rgb_to_sct_exact(dev(x)).cpu().numpy(), O.rgb_to_sct_exact(x), 1e-11, 1e-11)
    close(P["exact"].rgb_to_hsi_exact(dev(x)).cpu().numpy(), O.rgb_to_hsi_exact(x), 1e-11, 1e-11)


def test_distances_vs_reference(P, golden):
    ex = P["exact"]
    close(ex.lab_distance(golden["lab_fast"], golden["lab_exact"]), golden["lab_dist"], 1e-9, 1e-12)
    close(ex.hsi_distance(golden["hsi_fast"], golden["hsi_exact"]), golden["hsi_dist"], 1e-6, 1e-9)
    close(ex.sct_distance_indirect(golden["sct_fast"], golden["sct_exact"]), golden["sct_dist"],
          1e-6, 1e-10)
    close(ex.sct_to_rgb(golden["sct_exact"]), golden["sct_to_rgb"], 1e-11, 1e-10)


@pytest.mark.parametrize("space", ["lab", "hsi", "sct"])
def test_lut_build(P, golden, space):
    for n in (9, 17):
        lt = P["lut"].build_lut(space, n)
        close(lt.values, golden[f"lut_{space}_{n}"], 1e-11, 1e-11)
    lt = P["lut"].build_lut(space, 33)
    flat = lt.values.reshape(-1, 3)
    close(flat[golden[f"lut_{space}_33_sample_idx"]], golden[f"lut_{space}_33_sample"], 1e-11, 1e-11)


@pytest.mark.parametrize("n", [9, 17, 33])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut_nodes_bit_exact(P, golden, n, method):
    lt = P["lut"].build_lut("lab", n)
    nodes, w = P["lut"].node_weights(lt, golden["small"], method)
    np.testing.assert_array_equal(nodes, golden[f"nodes_{n}_{method}"])
    np.testing.assert_array_equal(w, golden[f"weights_{n}_{method}"])     # fp64, bit-identical


@pytest.mark.parametrize("n", [9, 17, 33])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut_nodes_full_cube(P, n, method):
    """Every cube colour: node indices bit-exact against the oracle (C3 rows), both
    for the integer cell location the interpolation kernels use (mact_lut_nodes)
    and for node_weights (fp64 weights, bit-identical)."""
    from paper_1009_0854_b200 import _lib
    lt = P["lut"].build_lut("lab", n)
    cube = P["harness"].cube_chunk(0, 1 << 24, device="cuda")
    k = P["lut"].NEIGHBOR_COUNT[method]
    inodes = torch.empty((1 << 24, k), dtype=torch.int32, device="cuda")
    iw = torch.empty((1 << 24, k), dtype=torch.float32, device="cuda")
    _lib.call("mact_lut_nodes", n, _lib.METHODS[method], cube.data_ptr(), 1 << 24, inodes.data_ptr(),
              iw.data_ptr(), torch.cuda.current_stream().cuda_stream)
    inodes = inodes.cpu().numpy()
    iw = iw.cpu().numpy()
    nodes, w = P["lut"].node_weights(lt, cube, method)
    nodes, w = nodes.cpu().numpy(), w.cpu().numpy()
    host = cube.cpu().numpy()
    step = 1 << 22
    for s in range(0, 1 << 24, step):
        on, ow = O.node_weights(n, host[s:s + step], method)
        np.testing.assert_array_equal(inodes[s:s + step], on)
        np.testing.assert_array_equal(nodes[s:s + step], on)
        np.testing.assert_array_equal(w[s:s + step], ow)
        np.testing.assert_allclose(iw[s:s + step], ow, rtol=0, atol=2e-7)


@pytest.mark.parametrize("n", [9, 17, 33])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut_interp_vs_reference(P, golden, n, method):
    lt = P["lut"].build_lut("lab", n)
    got = P["lut"].interpolate(lt, dev(golden["small"]), method).cpu().numpy()
    check_lab(got, golden[f"interp_lab_{n}_{method}"])
    cache = P["lut"].build_cache(lt)
    got_c = P["lut"].interpolate(cache, dev(golden["small"]), method, "caching").cpu().numpy()
    check_lab(got_c, golden[f"interp_lab_{n}_{method}_caching"])


@pytest.mark.parametrize("n", [17, 33])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut_interp_c3_image(P, n, method):
    """BASELINE config 3 image (4096^2, default_rng(0)) vs the oracle, tail and planar too."""
    img = np.random.default_rng(0).integers(0, 256, (4096, 4096, 3), dtype=np.uint8)
    lt = P["lut"].build_lut("lab", n)
    d = dev(img)
    got = P["lut"].interpolate(lt, d, method).cpu().numpy()
    vals = O.build_lut_values("lab", n).astype(np.float32).astype(np.float64)
    for r0 in (0, 3584):
        check_lab(got[r0:r0 + 512], O.interpolate(vals, img[r0:r0 + 512], method))
    part = P["lut"].interpolate(lt, d.reshape(-1, 3)[5:100005], method, layout="planar").cpu().numpy()
    if n == 33:   # both layouts run the r-split CTAs (same arithmetic); kept as a tolerance check
        check_lab(part.T, O.interpolate(vals, img.reshape(-1, 3)[5:100005], method))
    else:
        np.testing.assert_array_equal(part.T, got.reshape(-1, 3)[5:100005])


def test_lut_errors(P):
    from paper_1009_0854_b200.errors import CacheMissing
    lut = P["lut"]
    with pytest.raises(ValueError):
        lut.build_lut("xyz", 17)
    with pytest.raises(ValueError):
        lut.build_lut("lab", 16)
    lt = lut.build_lut("lab", 9)
    with pytest.raises(ValueError):
        lut.interpolate(lt, np.zeros((2, 3), np.uint8), "cubic")
    with pytest.raises(ValueError):
        lut.interpolate(lt, np.zeros((2, 3), np.uint8), "tetrahedral", "fancy")
    with pytest.raises(CacheMissing):
        lut.interpolate(lt, np.zeros((2, 3), np.uint8), "tetrahedral", "caching")


def _circ(a, b):
    d = np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)) % (2 * np.pi)
    return np.minimum(d, 2 * np.pi - d)


@pytest.mark.parametrize("space", ["hsi", "sct"])
@pytest.mark.parametrize("n", [9, 17, 33])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut_angular_interp_vs_reference(P, golden, space, n, method):
    """Angular destinations (lut.py:202-262): hue / SCT angles blended on the circle."""
    lt = P["lut"].build_lut(space, n)
    got = P["lut"].interpolate(lt, dev(golden["small"]), method).cpu().numpy().astype(np.float64)
    ref = golden[f"interp_{space}_{n}_{method}"]
    mask = O.ANGULAR_MASKS[space]
    scale = [2 * np.pi, 1.0, 1.0] if space == "hsi" else [255 * np.sqrt(3), np.pi / 2, np.pi / 2]
    for c in range(3):
        err = (_circ(got[:, c], ref[:, c]) if mask[c] else np.abs(got[:, c] - ref[:, c])) / scale[c]
        assert err.max() <= 1e-5, (c, float(err.max()), int(err.argmax()))


@pytest.mark.parametrize("grid,method", [(17, "tetrahedral"), (33, "trilinear"), (9, "pyramidal")])
def test_lut_interp_host_executor(grid, method):
    """numpy in -> numpy out through mact_lut_interp_host (pageable, pinned, planar)
    equals the device-tensor path."""
    from paper_1009_0854_b200 import lut
    rng = np.random.default_rng(grid)
    n = (1 << 23) + 12345                         # two executor chunks + a ragged tail
    px = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    L = lut.build_lut("lab", grid)
    ref = lut.interpolate(L, torch.from_numpy(px).cuda(), method).cpu().numpy()
    got = lut.interpolate(L, px, method)
    assert isinstance(got, np.ndarray) and got.dtype == np.float32
    np.testing.assert_array_equal(got, ref)
    pin_in = torch.empty((n, 3), dtype=torch.uint8).pin_memory()
    pin_in.numpy()[...] = px
    pin_out = torch.empty((n, 3), dtype=torch.float32).pin_memory()
    lut.interpolate(L, pin_in.numpy(), method, out=pin_out.numpy())
    np.testing.assert_array_equal(pin_out.numpy(), ref)
    planar = lut.interpolate(L, px[:5000], method, layout="planar").T
    if grid == 33:   # (older 33^3 families mixed fp32 and fixed-point nodes; kept as a tolerance check)
        check_lab(planar, ref[:5000])
    else:
        np.testing.assert_array_equal(planar, ref[:5000])


@pytest.mark.parametrize("kernel", ["split", "pair", "comp"])
@pytest.mark.parametrize("n", [4096 * 37 + 8, 4096 * 5 + 3, 1000])
@pytest.mark.parametrize("method", ["trilinear", "tetrahedral"])
def test_lut33_planar_equals_interleaved(monkeypatch, kernel, n, method):
    """33^3 planar output == interleaved output within one kernel family (forced
    with MACT_LUT33_KERNEL; tails and odd sizes take the per-pixel kernel of the
    same arithmetic).  The default is "split" for both layouts;
    test_lut33_both_kernels checks every family against the oracle."""
    from paper_1009_0854_b200 import lut
    monkeypatch.setenv("MACT_LUT33_KERNEL", kernel)
    px = torch.from_numpy(np.random.default_rng(n).integers(0, 256, (n, 3), dtype=np.uint8)).cuda()
    L = lut.build_lut("lab", 33)
    inter = lut.interpolate(L, px, method).cpu().numpy()
    planar = lut.interpolate(L, px, method, layout="planar").cpu().numpy()
    np.testing.assert_array_equal(planar.T, inter)


@pytest.mark.parametrize("grid", [9, 17, 33])
def test_lut_unaligned_views_and_step_edges(grid):
    """Unaligned buffers take the generic kernel, step-multiple edges the tails:
    every path agrees bit for bit with the aligned interleaved result."""
    from paper_1009_0854_b200 import lut
    L = lut.build_lut("lab", grid)
    px = torch.from_numpy(np.random.default_rng(grid).integers(0, 256, (4096 * 8 + 7, 3), dtype=np.uint8)).cuda()
    full = lut.interpolate(L, px, "tetrahedral").cpu().numpy()
    sub = lut.interpolate(L, px[1:], "tetrahedral").cpu().numpy()          # 3-byte offset input
    np.testing.assert_array_equal(sub, full[1:])
    for n in (4096 * 8 - 1, 4096 * 8 + 1, 4096 * 3, 4095):
        np.testing.assert_array_equal(lut.interpolate(L, px[:n], "tetrahedral").cpu().numpy(), full[:n])
    out = torch.empty((px.shape[0] + 1, 3), dtype=torch.float32, device="cuda")[1:]   # 12-byte offset output
    lut.interpolate(L, px, "tetrahedral", out=out)
    np.testing.assert_array_equal(out.cpu().numpy(), full)


@pytest.mark.parametrize("grid", [17, 33])
def test_lut_beyond_int32_pixel_count(grid):
    """One interpolation over 2^31 + 4099 pixels (64-bit step and tile indexing)."""
    from paper_1009_0854_b200 import harness, lut
    L = lut.build_lut("lab", grid)
    n = (1 << 31) + 4099
    cube = harness.cube_chunk(0, 1 << 24, device="cuda")
    ref = lut.interpolate(L, cube, "tetrahedral")
    x = cube.repeat((n >> 24) + 1, 1)[:n]
    out = lut.interpolate(L, x, "tetrahedral")
    idx = torch.from_numpy(np.r_[0:64, (1 << 31) - 64:(1 << 31) + 64, n - 4099 - 64:n]).cuda()
    np.testing.assert_array_equal(out[idx].cpu().numpy(), ref[idx % (1 << 24)].cpu().numpy())
    del out, x
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("n", [9, 17, 33])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut_interp_full_cube(P, n, method):
    """The TIMED uint8 kernels (9^3 bank-private copies, 17^3 fixed-point nodes
    in the reference's cells, 33^3 r-split independent CTAs for both layouts) on
    all 2^24 colours vs the oracle on the same fp32 lattice values; 9^3 / 17^3
    planar output bit-identical to interleaved.  The fixed-point formats stay
    inside 1e-4 (quantisation half-step <= 4.4e-5)."""
    lt = P["lut"].build_lut("lab", n)
    cube = P["harness"].cube_chunk(0, 1 << 24, device="cuda")
    got = P["lut"].interpolate(lt, cube, method).cpu().numpy()
    planar = P["lut"].interpolate(lt, cube, method, layout="planar").cpu().numpy().T
    if n != 33:
        np.testing.assert_array_equal(planar, got)
    host = cube.cpu().numpy()
    vals = lt.values.astype(np.float32).astype(np.float64)
    worst = 0.0
    for s in range(0, 1 << 24, 1 << 22):
        ref = O.interpolate(vals, host[s:s + (1 << 22)], method)
        worst = max(worst, check_lab(got[s:s + (1 << 22)], ref))
        if n == 33:
            check_lab(planar[s:s + (1 << 22)], ref)
    print(f"{n}^3 {method}: max |dLab| {worst:.3e}")


def _sorted_nonzero(nodes, w, tiny):
    """Per pixel: the (node, weight) pairs with |weight| > tiny, sorted by node (zeros -> sentinel)."""
    nodes = np.where(np.abs(w) > tiny, nodes, np.iinfo(np.int32).max).astype(np.int64)
    order = np.argsort(nodes, axis=1, kind="stable")
    return np.take_along_axis(nodes, order, 1), np.take_along_axis(w, order, 1)


@pytest.mark.slow
@pytest.mark.parametrize("n", [9, 17, 33])
@pytest.mark.parametrize("method", O.METHODS)
def test_timed_kernel_selection_full_cube(P, n, method):
    """Cells and simplices of the INTERPOLATION kernels (their own select():
    tetrahedral order from max/min keys) on all 2^24 colours: the cells are the
    reference's, and the nodes carrying nonzero weight are exactly the
    reference's (lut.py:98-199), with the same weights to fp32 rounding.  Only a
    zero-weight node may differ (a tie's middle corner); fmaf(0, v, a) == a, so
    it cannot change a sum of finite nodes."""
    from paper_1009_0854_b200 import _lib
    k = P["lut"].NEIGHBOR_COUNT[method]
    cube = P["harness"].cube_chunk(0, 1 << 24, device="cuda")
    nodes = torch.empty((1 << 24, k), dtype=torch.int32, device="cuda")
    w = torch.empty((1 << 24, k), dtype=torch.float32, device="cuda")
    _lib.call("mact_lut_nodes_timed", n, _lib.METHODS[method], cube.data_ptr(), 1 << 24, nodes.data_ptr(),
              w.data_ptr(), torch.cuda.current_stream().cuda_stream)
    nodes, w, host = nodes.cpu().numpy(), w.cpu().numpy(), cube.cpu().numpy()
    step = 1 << 21
    for s in range(0, 1 << 24, step):
        on, ow = O.node_weights(n, host[s:s + step], method)
        gn, gw = _sorted_nonzero(nodes[s:s + step], w[s:s + step], 0.0)
        rn, rw = _sorted_nonzero(on, ow, 1e-12)     # the pyramid's u v - m may round to +-1e-19 in fp64
        np.testing.assert_array_equal(gn, rn)
        np.testing.assert_allclose(gw, rw, rtol=0, atol=2e-7)


@pytest.mark.parametrize("n", [17, 33])
def test_lut_nonfinite_lattice(P, n):
    """A lattice with inf / NaN nodes keeps the reference's cells (no ghost-cell
    0 * inf) and gathers in fp32: the non-finite pattern and every finite value
    match the oracle on the same fp32 values."""
    import dataclasses
    lt = P["lut"].build_lut("lab", n)
    vals = lt.values.copy()
    vals[n - 1, n - 1, n - 1, 0] = np.inf          # the white corner
    vals[n - 1, 0, :, 1] = -np.inf                 # a face edge
    vals[n // 2, n // 2, n // 2, 2] = np.nan       # an interior node
    bad = dataclasses.replace(lt, values=vals, _device={})
    rng = np.random.default_rng(n)
    img = np.concatenate([rng.integers(0, 256, (1 << 16, 3), dtype=np.uint8),
                          np.array([[255, 255, 255], [255, 0, 0], [255, 0, 255], [128, 128, 128]], np.uint8)])
    ref = O.interpolate(vals.astype(np.float32).astype(np.float64), img, "tetrahedral")
    for method in O.METHODS:
        ref = O.interpolate(vals.astype(np.float32).astype(np.float64), img, method)
        got = P["lut"].interpolate(bad, dev(img), method).cpu().numpy().astype(np.float64)
        np.testing.assert_array_equal(np.isnan(got), np.isnan(ref), err_msg=method)
        np.testing.assert_array_equal(np.isinf(got), np.isinf(ref), err_msg=method)
        fin = np.isfinite(ref)
        np.testing.assert_allclose(got[fin], ref[fin], rtol=2e-6, atol=1e-4, err_msg=method)


@pytest.mark.parametrize("kernel", ["comp", "pair", "split"])
def test_lut33_wide_range_lattice_falls_back(P, monkeypatch, kernel):
    """33^3 lattice too wide for the fixed-point nodes (x1000): the component
    kernels stage fp32 components, the pair kernel gathers the fp32 lattice from
    L2; both match the oracle."""
    import dataclasses
    monkeypatch.setenv("MACT_LUT33_KERNEL", kernel)
    lt = P["lut"].build_lut("lab", 33)
    wide = dataclasses.replace(lt, values=lt.values * 1000.0, _device={})
    img = np.random.default_rng(5).integers(0, 256, (1 << 18, 3), dtype=np.uint8)
    vals = wide.values.astype(np.float32).astype(np.float64)
    for method in O.METHODS:
        got = P["lut"].interpolate(wide, dev(img), method).cpu().numpy()
        np.testing.assert_allclose(got, O.interpolate(vals, img, method), rtol=2e-6, atol=1e-2)


def test_lut17_wide_range_lattice_keeps_fp32(P):
    """A lattice whose value range is too wide for the fixed-point format
    (x1000) takes the fp32 planes: the result still matches the oracle to fp32
    accuracy."""
    import dataclasses
    lt = P["lut"].build_lut("lab", 17)
    wide = dataclasses.replace(lt, values=lt.values * 1000.0, _device={})
    img = np.random.default_rng(5).integers(0, 256, (1 << 16, 3), dtype=np.uint8)
    got = P["lut"].interpolate(wide, dev(img), "tetrahedral").cpu().numpy()
    vals = wide.values.astype(np.float32).astype(np.float64)
    ref = O.interpolate(vals, img, "tetrahedral")
    np.testing.assert_allclose(got, ref, rtol=2e-6, atol=1e-2)


@pytest.mark.parametrize("n", [17, 33])
@pytest.mark.parametrize("scale", [0.25, 1.0, 1.1, 1.2, 3.0])
@pytest.mark.parametrize("method", ["pyramidal", "tetrahedral"])
def test_lut_error_bound_either_format(P, n, scale, method):
    """Lattices scaled around the fixed-point threshold (half-step 5e-5: the
    CIELAB lattice x1.14): below it the 64-bit nodes are used, above it the
    fp32 planes.  Either way |interp - oracle| <= 1.5 * 5e-5 (pyramid sum|w|)
    plus fp32 rounding of the values."""
    import dataclasses
    lt = P["lut"].build_lut("lab", n)
    sc = dataclasses.replace(lt, values=lt.values * scale, _device={})
    img = np.random.default_rng(11).integers(0, 256, (1 << 18, 3), dtype=np.uint8)
    got = P["lut"].interpolate(sc, dev(img), method).cpu().numpy().astype(np.float64)
    vals = sc.values.astype(np.float32).astype(np.float64)
    ref = O.interpolate(vals, img, method)
    bound = 1.5 * 5e-5 + 4e-7 * np.abs(ref).max()
    assert np.abs(got - ref).max() <= bound


@pytest.mark.parametrize("kernel", ["comp", "pair", "split"])
@pytest.mark.parametrize("method", O.METHODS)
def test_lut33_both_kernels(P, monkeypatch, kernel, method):
    """Every 33^3 interpolation kernel family -- the r-split independent CTAs (the
    default for both layouts), the r-split cluster pairs and the component-split
    CTAs (MACT_LUT33_KERNEL=pair / comp) -- against the oracle on the
    same fp32 lattice: 2^20 random colours plus the cube's corners and faces,
    interleaved, planar and unaligned (per-pixel kernel) outputs."""
    monkeypatch.setenv("MACT_LUT33_KERNEL", kernel)
    lt = P["lut"].build_lut("lab", 33)
    rng = np.random.default_rng(33)
    edge = np.array([[a, b, c] for a in (0, 127, 128, 255) for b in (0, 128, 255) for c in (0, 1, 254, 255)], np.uint8)
    img = np.concatenate([rng.integers(0, 256, ((1 << 20) + 5, 3), dtype=np.uint8), edge])
    ref = O.interpolate(lt.values.astype(np.float32).astype(np.float64), img, method)
    d = dev(img)
    got = P["lut"].interpolate(lt, d, method).cpu().numpy()
    check_lab(got, ref)
    n4 = img.shape[0] // 4 * 4
    planar = P["lut"].interpolate(lt, d[:n4], method, layout="planar").cpu().numpy()
    check_lab(planar.T, ref[:n4])
    check_lab(P["lut"].interpolate(lt, d[1:], method).cpu().numpy(), ref[1:])


@pytest.mark.parametrize("layout", ["interleaved", "planar"])
def test_lut33_tiny_and_ragged_sizes(P, layout):
    """33^3 on sizes around the 128-pixel slice and the empty input (one launch
    per size through the default kernel): every size matches the oracle."""
    lt = P["lut"].build_lut("lab", 33)
    vals = lt.values.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(128)
    for n in (0, 1, 2, 3, 5, 127, 128, 129, 255, 257, 4095, 4097):
        img = rng.integers(0, 256, (n, 3), dtype=np.uint8)
        got = P["lut"].interpolate(lt, dev(img), "tetrahedral", layout=layout).cpu().numpy()
        if layout == "planar":
            got = got.T
        assert got.shape == (n, 3)
        if n:
            check_lab(got, O.interpolate(vals, img, "tetrahedral"))


@pytest.mark.parametrize("skew", ["dark", "bright", "mostly_dark", "half_image"])
def test_lut33_split_skewed_images(P, skew):
    """k_lut33_split on images whose pixels sit mostly or wholly in one r-half
    (one CTA of each pair then only scans): all-dark, all-bright, 95 % dark and
    dark-first-half images against the oracle, interleaved == planar bit for
    bit, ragged size."""
    lt = P["lut"].build_lut("lab", 33)
    rng = np.random.default_rng(len(skew))
    n = (1 << 21) + 77
    img = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    if skew == "dark":
        img[:, 0] &= 0x7F
    elif skew == "bright":
        img[:, 0] |= 0x80
    elif skew == "mostly_dark":
        img[rng.random(n) < 0.95, 0] &= 0x7F
    else:
        img[: n // 2, 0] &= 0x7F
        img[n // 2:, 0] |= 0x80
    vals = lt.values.astype(np.float32).astype(np.float64)
    d = dev(img)
    for method in ("trilinear", "tetrahedral"):
        got = P["lut"].interpolate(lt, d, method).cpu().numpy()
        check_lab(got, O.interpolate(vals, img, method))
        n4 = n // 4 * 4
        planar = P["lut"].interpolate(lt, d[:n4], method, layout="planar").cpu().numpy()
        np.testing.assert_array_equal(planar.T, got[:n4])


_SKEW_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1009_0854_b200 import lut
from oracle import mact_oracle as O
rng = np.random.default_rng(7)
n = 128 * 4096
px = rng.integers(0, 256, (n, 3), dtype=np.uint8)
blk = px.reshape(-1, 128, 3)
kind = np.arange(blk.shape[0]) % 5          # per 128-px slice: all rank 0 / all rank 1 / mixed / runs
blk[kind == 0, :, 0] &= 0x7F
blk[kind == 1, :, 0] |= 0x80
blk[kind == 3, :64, 0] &= 0x7F
blk[kind == 3, 64:, 0] |= 0x80
blk[kind == 4, :64, 0] |= 0x80
blk[kind == 4, 64:, 0] &= 0x7F
lt = lut.build_lut("lab", 33)
vals = lt.values.astype(np.float32).astype(np.float64)
d = torch.from_numpy(px).cuda()
for m in ("trilinear", "tetrahedral"):
    for rep in range(3):
        got = lut.interpolate(lt, d, m).cpu().numpy()
    err = np.abs(got - O.interpolate(vals, px, m)).max()
    assert err <= 1e-4, (m, err)
print("ok")
"""


@pytest.mark.parametrize("kernel", ["pair", "split"])
@pytest.mark.parametrize("cap", ["", "2", "6"])
def test_lut33_pair_one_sided_slices(cap, kernel):
    """The r-split pairs on slices owned entirely by one rank (sends in one
    direction only), alternating with mixed and half/half slices, repeated
    launches and few clusters (MACT_GRID_CAP): the exchange must neither
    deadlock nor mix up transfers.  Runs in a child with a timeout, so a
    protocol regression fails instead of hanging the suite."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MACT_LUT33_KERNEL=kernel)
    if cap:
        env["MACT_GRID_CAP"] = cap
    r = subprocess.run([sys.executable, "-c", _SKEW_CHILD, root], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
