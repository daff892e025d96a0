"""Robustness of the native path: no writes outside the output, concurrent
callers on separate streams/threads, CUDA-graph capture (bench's C1 mode)."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CANARY = 1234.5


@pytest.fixture(scope="module")
def P():
    from paper_1009_0854_b200 import _dev, _lib, fast, harness, lut
    lib = _lib.load()
    return {"fast": fast, "lut": lut, "harness": harness, "lib": lib, "_lib": _lib, "dev": _dev}


def _guarded(n, pad=4096):
    """fp32 buffer with canary bands around an (n,3) window; window is 16-B aligned."""
    buf = torch.full((3 * n + 2 * pad,), CANARY, dtype=torch.float32, device="cuda")
    return buf, buf[pad:pad + 3 * n]


def _check_bands(buf, pad=4096):
    b = buf.cpu().numpy()
    assert (b[:pad] == CANARY).all() and (b[-pad:] == CANARY).all(), "write outside the output"


@pytest.mark.parametrize("n", [1, 4095, 65536 + 3, 1000003])
def test_no_out_of_bounds_writes(P, n):
    lib, _lib, fast = P["lib"], P["_lib"], P["fast"]
    rng = np.random.default_rng(n)
    x = torch.from_numpy(rng.integers(0, 256, (n, 3), dtype=np.uint8)).cuda()
    cf = fast.DEFAULT_CONFIG.coeffs
    st = torch.cuda.current_stream().cuda_stream
    for fn in (lib.mact_lab_fast, lib.mact_hsi_fast, lib.mact_sct_fast):
        for layout in (0, 1):
            buf, win = _guarded(n)
            _lib.check(fn(x.data_ptr(), 0, win.data_ptr(), n, cf, layout, st))
            torch.cuda.synchronize()
            _check_bands(buf)
    bufs = [_guarded(n) for _ in range(3)]
    _lib.check(lib.mact_all_fast(x.data_ptr(), *[w.data_ptr() for _, w in bufs], n, cf, 0, st))
    _lib.check(lib.mact_all_fast(x.data_ptr(), None, bufs[1][1].data_ptr(), bufs[2][1].data_ptr(),
                                 n, cf, 1, st))
    torch.cuda.synchronize()
    for b, _ in bufs:
        _check_bands(b)
    for g in (9, 17, 33):
        lat = P["lut"].build_lut("lab", g).lattice("cuda")
        for m in range(4):
            buf, win = _guarded(n)
            _lib.check(lib.mact_lut_interp(lat.data_ptr(), g, m, x.data_ptr(), win.data_ptr(), n, 0, st))
            torch.cuda.synchronize()
            _check_bands(buf)


def test_concurrent_threads_and_streams(P):
    """The reference harness calls transforms from a thread pool (harness.py:99-101):
    8 threads, each on its own stream and config, agree with sequential results."""
    fast = P["fast"]
    rng = np.random.default_rng(8)
    x = torch.from_numpy(rng.integers(0, 256, (1 << 21, 3), dtype=np.uint8)).cuda()
    cfgs = [fast.MactConfig(cielab_degrees=d) for d in [(4, 4), (3, 3), (2, 4), (4, 2)]] * 2
    spaces = ["lab", "hsi", "sct", "lab", "lab", "sct", "hsi", "lab"]
    ref = [getattr(fast, f"rgb_to_{s}_fast")(x, c).cpu().numpy() for s, c in zip(spaces, cfgs)]
    got = [None] * 8
    errs = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    y = getattr(fast, f"rgb_to_{spaces[i]}_fast")(x, cfgs[i])
                s.synchronize()
                got[i] = y.cpu().numpy()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


def test_cuda_graph_capture_and_replay(P):
    """All stream-ordered entry points are capture-safe (no sync, no allocation)."""
    fast, lib, _lib = P["fast"], P["lib"], P["_lib"]
    rng = np.random.default_rng(9)
    x = torch.from_numpy(rng.integers(0, 256, (512 * 512, 3), dtype=np.uint8)).cuda()
    lat = P["lut"].build_lut("lab", 17).lattice("cuda")
    o1 = torch.empty((x.shape[0], 3), device="cuda")
    o2 = torch.empty_like(o1)
    eager1, eager2 = fast.rgb_to_lab_fast(x), P["lut"].interpolate(P["lut"].build_lut("lab", 17), x)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        st = torch.cuda.current_stream().cuda_stream
        _lib.check(lib.mact_lab_fast(x.data_ptr(), 0, o1.data_ptr(), x.shape[0],
                                     fast.DEFAULT_CONFIG.coeffs, 0, st))
        _lib.check(lib.mact_lut_interp(lat.data_ptr(), 17, 3, x.data_ptr(), o2.data_ptr(),
                                       x.shape[0], 0, st))
    o1.zero_()
    o2.zero_()
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(o1.cpu().numpy(), eager1.cpu().numpy())
    np.testing.assert_array_equal(o2.cpu().numpy(), eager2.cpu().numpy())


def test_concurrent_host_callers(P):
    """numpy callers from a thread pool (harness.py:99-101) share the host executor safely."""
    from concurrent.futures import ThreadPoolExecutor
    fast = P["fast"]
    rng = np.random.default_rng(21)
    imgs = [rng.integers(0, 256, ((1 << 22) + 17 * k, 3), dtype=np.uint8) for k in range(6)]
    ref = [fast.rgb_to_lab_fast(torch.from_numpy(im).cuda()).cpu().numpy() for im in imgs]
    with ThreadPoolExecutor(max_workers=6) as pool:
        got = list(pool.map(fast.rgb_to_lab_fast, imgs))
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)
