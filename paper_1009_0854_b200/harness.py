"""Error measurement on B200 — drop-in for ``mact.harness`` (hot-path parts).

    cube_chunk, rgb16million, CUBE_SIZE                (harness.py:25-52)
    measure_error(space, candidate, reference, population=None)   (harness.py:77-122)
    ErrorStats                                         (harness.py:63-68)
    component_error(...)   per-component |fast - exact|  (not in the reference)
    call_probabilities()  CallProbabilities             (harness.py:125-175)
    measure_gain(...)     GainStats, device-timed        (harness.py:176-221)

``measure_error`` keeps the reference's plugin seam — any callable
``pixels -> (..., 3)`` — and fuses the whole evaluation into one kernel
(candidate + fp64 exact transform + distance + reduction, K6) whenever it
recognises the candidate as one of this package's fast transforms or LUT
interpolators and the reference as the matching exact transform.  Arbitrary
callables are evaluated on device tensors and scored by the same reduction
kernel.  Statistics semantics match the reference: mean = sum / count,
max with the FIRST pixel attaining it.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import numpy as np

from . import _dev, _lib, exact, fast
from .errors import CorpusEmpty

CUBE_SIZE = 1 << 24
_CHUNK = 1 << 20

# harness.DISTANCES (harness.py:28-32): the metric each space is scored with
DISTANCES = exact.DISTANCES


@dataclass(frozen=True)
class ErrorStats:
    avg: float
    max: float
    count: int
    argmax_pixel: Tuple[int, int, int]


@dataclass(frozen=True)
class ComponentStats:
    mean: float
    max: float
    count: int
    nan_count: int
    argmax_index: int
    argmax_pixel: Tuple[int, int, int]


def cube_pixel(i: int) -> Tuple[int, int, int]:
    """Pixel i of the R-major cube enumeration (harness.py:35-46)."""
    return (int(i) >> 16 & 255, int(i) >> 8 & 255, int(i) & 255)


def cube_chunk(start: int, size: int, *, device: Optional[str] = None):
    """Pixels start .. start+size of the cube, generated on the GPU.

    Returns numpy (the reference's type) unless ``device`` is given, in which
    case the uint8 (size, 3) tensor stays on that device.
    """
    import torch

    _dev.require_cuda()
    n = max(0, min(start + size, CUBE_SIZE) - start)
    t = torch.empty((n, 3), dtype=torch.uint8, device=device or "cuda")
    if n:
        _lib.call("mact_cube_fill", t.data_ptr(), start, n, _dev.stream_ptr())
    return t if device is not None else t.cpu().numpy()


def rgb16million(chunk_size: int = _CHUNK, *, device: Optional[str] = None):
    for start in range(0, CUBE_SIZE, chunk_size):
        yield cube_chunk(start, chunk_size, device=device)


# ------------------------------------------------------------------ candidates
class LutCandidate:
    """Callable LUT interpolator that measure_error can fuse (lut.interpolate)."""

    def __init__(self, lut, method: str = "tetrahedral"):
        from . import lut as _lut

        _lut._method_code(method)
        self.lut, self.method = lut, method

    def __call__(self, pixels):
        from . import lut as _lut

        return _lut.interpolate(self.lut, pixels, self.method)


def fast_candidate(space: str, cfg: "fast.MactConfig" = None, *, out_dtype: str = "float32"):
    """The fast transform of ``space`` bound to ``cfg`` (fusable by measure_error).
    out_dtype "float64" scores the reference's own fp64 arithmetic."""
    fn = {"lab": fast.rgb_to_lab_fast, "hsi": fast.rgb_to_hsi_fast, "sct": fast.rgb_to_sct_fast}[space]
    if out_dtype == "float64":
        return functools.partial(fn, cfg=cfg or fast.DEFAULT_CONFIG, out_dtype="float64")
    return functools.partial(fn, cfg=cfg or fast.DEFAULT_CONFIG)


_FAST_FN = {fast.rgb_to_lab_fast: "lab", fast.rgb_to_hsi_fast: "hsi", fast.rgb_to_sct_fast: "sct"}
_EXACT_FN = {exact.rgb_to_lab_exact: "lab", exact.rgb_to_hsi_exact: "hsi",
             exact.rgb_to_sct_exact: "sct"}


def _classify(space: str, candidate):
    """-> (kind, payload) with kind in fast/lut/array."""
    fn, cfg, odt = candidate, fast.DEFAULT_CONFIG, "float32"
    if isinstance(candidate, functools.partial):
        fn = candidate.func
        if candidate.args:
            cfg = candidate.args[0]
        cfg = candidate.keywords.get("cfg", cfg)
        odt = candidate.keywords.get("out_dtype", odt)
        extra = set(candidate.keywords) - {"cfg", "out_dtype"}
        if extra or len(candidate.args) > 1:
            fn = None                                     # other bound arguments: evaluate as-is
    if _FAST_FN.get(fn) == space and isinstance(cfg, fast.MactConfig):
        return ("fast64" if odt == "float64" else "fast"), cfg
    if (isinstance(candidate, LutCandidate) and space == candidate.lut.destination_space
            and not any(candidate.lut.angular_mask)):
        return "lut", candidate                # fused (linear destinations); angular -> array path
    return "array", None


# ------------------------------------------------------------------ reduction
def _workspace(device):
    import torch

    return torch.empty(int(_lib.load().mact_err_workspace_bytes()), dtype=torch.uint8, device=device)


def reduce_partials(space: str, candidate, reference, pixels=None, *, cube_start: int = -1,
                    n: int = 0, index_base: int = 0, metric: str = "distance"):
    """Run the fused reduction over one shard; returns a list of raw partial
    dicts {sum, max, count, argmax, nan} (1 for distance, 3 for component)."""
    import torch

    _dev.require_cuda()
    kind, payload = _classify(space, candidate)
    spec = _lib.MactErrSpec()
    spec.space = _lib.SPACES[space]
    spec.metric = _lib.METRIC_COMPONENT if metric == "component" else _lib.METRIC_DISTANCE
    keep = []
    t = None
    if pixels is not None:
        t, code, lead, _ = _dev.as_device_pixels(pixels)
        if code != _lib.DTYPE_U8:
            raise ValueError("measure_error populations are 8-bit RGB")
        n = t.numel() // 3
    elif cube_start < 0:
        raise ValueError("no population")
    if n <= 0:
        raise ValueError("empty population")
    device = t.device if t is not None else torch.device("cuda", torch.cuda.current_device())
    cfg = fast.DEFAULT_CONFIG
    if kind in ("fast", "fast64"):
        spec.candidate = _lib.CAND_FAST_F64 if kind == "fast64" else _lib.CAND_FAST
        cfg = payload
    elif kind == "lut":
        # score the THROUGHPUT kernel's own fp32 output (mact_lut_interp, the kernel bench.py
        # times), not a re-implementation: run it over the shard, then reduce the array
        px = t if t is not None else cube_chunk(cube_start, n, device=str(device))
        c = torch.empty((n, 3), dtype=torch.float32, device=device)
        lat = payload.lut.lattice(device)
        _lib.call("mact_lut_interp", lat.data_ptr(), payload.lut.grid_n, _lib.METHODS[payload.method],
                  px.data_ptr(), c.data_ptr(), n, _lib.LAYOUTS["interleaved"], _dev.stream_ptr())
        keep += [px, c, lat]
        spec.candidate = _lib.CAND_ARRAY
        spec.cand_array = c.data_ptr()
        spec.cand_dtype = _lib.DTYPE_F32
    else:
        px = t if t is not None else cube_chunk(cube_start, n, device=str(device))
        c = candidate(px)
        c = c if _dev.is_device_tensor(c) else torch.from_numpy(np.ascontiguousarray(c)).to(device)
        c = c.to(torch.float64).contiguous()
        keep.append(c)
        spec.candidate = _lib.CAND_ARRAY
        spec.cand_array = c.data_ptr()
        spec.cand_dtype = _lib.DTYPE_F64
    if _EXACT_FN.get(reference) != space and reference is not None:
        px = t if t is not None else cube_chunk(cube_start, n, device=str(device))
        r = reference(px)
        r = r if _dev.is_device_tensor(r) else torch.from_numpy(np.ascontiguousarray(r)).to(device)
        r = r.to(torch.float64).contiguous()
        keep.append(r)
        spec.ref_array = r.data_ptr()
        spec.ref_dtype = _lib.DTYPE_F64
    nout = 3 if metric == "component" else 1
    out = torch.empty(nout * 6, dtype=torch.float64, device=device)
    ws = _workspace(device)
    _lib.call("mact_err_reduce", spec, cfg.coeffs, t.data_ptr() if t is not None else None,
              cube_start if t is None else -1, n, index_base, out.data_ptr(), ws.data_ptr(),
              _dev.stream_ptr())
    raw = out.cpu().numpy().view(np.uint64).reshape(nout, 6)
    f = out.cpu().numpy().reshape(nout, 6)
    return [{"sum": float(f[c, 0]), "max": float(f[c, 1]), "count": int(raw[c, 2]),
             "argmax": int(raw[c, 3]), "nan": int(raw[c, 4])} for c in range(nout)]


def combine_partials(parts: List[dict]) -> dict:
    """Fold partials in order: fsum of sums, strict '>' keeps the earliest max
    (harness.py:104-121)."""
    sums, best, arg, count, nan = [], -1.0, -1, 0, 0
    for p in parts:
        sums.append(p["sum"])
        count += p["count"]
        nan += p["nan"]
        if p["count"] and p["max"] > best:
            best, arg = p["max"], p["argmax"]
    return {"sum": math.fsum(sums), "max": best, "count": count, "argmax": arg, "nan": nan}


def _populations(population, chunk_size: int):
    """-> iterable of (pixels or None, cube_start, n) shards in index order."""
    if population is None:
        return [(None, s, min(chunk_size, CUBE_SIZE - s)) for s in range(0, CUBE_SIZE, chunk_size)]
    if isinstance(population, np.ndarray) or _dev.is_device_tensor(population):
        return [(population.reshape(-1, 3), -1, 0)]
    return [(np.asarray(p).reshape(-1, 3) if not _dev.is_device_tensor(p) else p.reshape(-1, 3), -1, 0)
            for p in population]


def _pixel_at(shards, gidx: int):
    if gidx < 0:
        return (0, 0, 0)
    off = 0
    for px, start, n in shards:
        if px is None:
            if gidx < off + n:
                return cube_pixel(start + gidx - off)
            off += n
            continue
        m = px.shape[0]
        if gidx < off + m:
            v = px[gidx - off]
            v = v.cpu().numpy() if _dev.is_device_tensor(v) else v
            return tuple(int(x) for x in v)
        off += m
    return (0, 0, 0)


def measure_error(space: str, candidate: Callable, reference: Callable, population=None,
                  chunk_size: int = CUBE_SIZE) -> ErrorStats:
    """Average / maximum distance between two transforms over a population
    (reference harness.py:77-122).  ``population`` None = the full 2^24 cube."""
    if space not in ("lab", "hsi", "sct"):
        raise KeyError(space)
    shards = _populations(population, chunk_size)
    parts, off = [], 0
    for px, start, n in shards:
        m = px.shape[0] if px is not None else n
        if m == 0:
            continue
        parts.append(reduce_partials(space, candidate, reference, px, cube_start=start, n=n,
                                     index_base=off)[0])
        off += m
    tot = combine_partials(parts)
    if tot["count"] == 0:
        raise ValueError("empty population")
    return ErrorStats(avg=tot["sum"] / tot["count"], max=tot["max"], count=tot["count"],
                      argmax_pixel=_pixel_at(shards, tot["argmax"]))


def component_error(space: str, candidate: Callable = None, reference: Callable = None,
                    population=None, chunk_size: int = CUBE_SIZE) -> List[ComponentStats]:
    """Per-component |candidate - exact| statistics: hue uses the
    circular difference, pixels whose exact component is NaN are excluded and
    counted."""
    candidate = candidate or fast_candidate(space)
    reference = reference or {"lab": exact.rgb_to_lab_exact, "hsi": exact.rgb_to_hsi_exact,
                              "sct": exact.rgb_to_sct_exact}[space]
    shards = _populations(population, chunk_size)
    per = [[], [], []]
    off = 0
    for px, start, n in shards:
        m = px.shape[0] if px is not None else n
        if m == 0:
            continue
        res = reduce_partials(space, candidate, reference, px, cube_start=start, n=n,
                              index_base=off, metric="component")
        for c in range(3):
            per[c].append(res[c])
        off += m
    out = []
    for c in range(3):
        tot = combine_partials(per[c])
        cnt = tot["count"]
        out.append(ComponentStats(mean=tot["sum"] / cnt if cnt else 0.0,
                                  max=tot["max"] if cnt else 0.0, count=cnt, nan_count=tot["nan"],
                                  argmax_index=tot["argmax"],
                                  argmax_pixel=_pixel_at(shards, tot["argmax"])))
    return out


@dataclass(frozen=True)
class CallProbabilities:
    """Relative full-cube frequencies of the approximated-function call sites
    (harness.py:125-134)."""

    cbrt_x: float
    cbrt_y: float
    cbrt_z: float
    arcsin: float
    arccos: float
    arctan: float


def call_counts(device=None) -> dict:
    """Exact call-site counts over all 2^24 colours, counted on the GPU
    (mact_call_counts; harness.py:137-175)."""
    import torch

    _dev.require_cuda()
    buf = torch.empty(6, dtype=torch.int64, device=device or "cuda")
    _lib.call("mact_call_counts", buf.data_ptr(), _dev.stream_ptr())
    vals = buf.cpu().tolist()
    return dict(zip(("cbrt_x", "cbrt_y", "cbrt_z", "arcsin", "arccos", "arctan"), vals))


def call_probabilities() -> CallProbabilities:
    """harness.call_probabilities (harness.py:137-175): counts / 2^24."""
    c = call_counts()
    return CallProbabilities(**{k: v / CUBE_SIZE for k, v in c.items()})


@dataclass(frozen=True)
class GainStats:
    """harness.py:176-183."""

    min: float
    max: float
    mean: float
    stdev: float
    median: float
    per_image: Tuple[float, ...]


def _mean_device_seconds(fn: Callable, image, repeats: int) -> float:
    """Mean device time of fn(image) over ``repeats`` calls: CUDA events on the
    current stream around each call (the reference's perf_counter, harness.py:188-194)."""
    import torch

    st = torch.cuda.current_stream()
    total = 0.0
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn(image)
        b.record(st)
        b.synchronize()
        total += a.elapsed_time(b) / 1e3
    return total / repeats


def measure_gain(space: str, fast: Callable, exact_fn: Callable, corpus, repeats_exact: int = 3,
                 repeats_fast: int = 3) -> GainStats:
    """Per-image speedup of ``fast`` over ``exact_fn`` (harness.py:197-221; PAPER Table 4).

    Images are pre-loaded into device memory (the reference pre-loads host
    arrays), both callables get a warm-up call, then each is timed with CUDA
    events and the gain is mean exact time / mean fast time.
    """
    import torch

    corpus = list(corpus)
    if len(corpus) == 0:
        raise CorpusEmpty("gain measurement needs at least one image")
    if repeats_exact < 3 or repeats_fast < 3:
        raise ValueError("timing needs at least 3 repeats per transform")
    _dev.require_cuda()
    gains = []
    for image in corpus:
        img = image if _dev.is_device_tensor(image) else torch.from_numpy(np.ascontiguousarray(image)).cuda()
        fast(img)
        exact_fn(img)
        t_exact = _mean_device_seconds(exact_fn, img, repeats_exact)
        t_fast = _mean_device_seconds(fast, img, repeats_fast)
        gains.append(t_exact / t_fast)
    arr = np.asarray(gains)
    return GainStats(min=float(arr.min()), max=float(arr.max()), mean=float(arr.mean()),
                     stdev=float(arr.std(ddof=1)) if arr.size > 1 else 0.0,
                     median=float(np.median(arr)), per_image=tuple(float(v) for v in arr))
