"""Benchmark of the B200 MACT path — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c1|c2|c3|c5] [--lut-grid 9|17|33] [--lut-method M]
                    [--e2e-steps E] [--no-cpu-baseline] [--graph | --no-graph]

Default workload = BASELINE.json config 4 (the config the metric is quoted on
"at 1/2/4/8 B200"): 64 images of 3840x2160 uint8 RGB, spatially correlated
synthetic content, RGB->CIELAB via MACT (4,4), sharded by image across ranks
(fixed 64-image batch -> strong scaling).  A step = one pass of the transform
over the rank's images, inputs and outputs resident in HBM (1.59 GB in +
6.37 GB out at N=1, far larger than the 126 MB L2, so no flush is needed;
smaller workloads rotate over enough buffer copies to exceed 2x L2).
roofline.achieved counts the algorithmic bytes of the step's one launch:
3 B in + 12 B out per pixel and transform (27 B fused C2, 39 B fused C5).

--gpus N > 1 without torchrun re-launches itself as N ranks through
torch.distributed.run (one process per GPU, NCCL); under torchrun WORLD_SIZE
must equal --gpus.  Every rank processes its shard; the timed window runs from
a common barrier through the K steps AND the final combine of the error
partials (all-gather + rank-order fold); time = max over ranks of the CUDA-event
time.  --share-gpu runs the N ranks on cuda:0 with a gloo combine: a host-logic
test for a 1-GPU box, not an N-GPU number.  --impl reference times the
unmodified reference package (baseline/_ref/mact, pure Python + numpy) on all
host threads on a bounded sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
HBM_FALLBACK = 6650.0          # GB/s, B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)
L2_POOL_BYTES = 512 << 20      # per-step footprint below this rotates over buffer copies

WORKLOADS = {
    "c4": dict(kind="images", images=64, h=2160, w=3840, space="lab", degenerate=False,
               desc="BASELINE config 4: 64 x 3840x2160 uint8 RGB, correlated synthetic content, "
                    "RGB->CIELAB MACT (4,4), sharded by image"),
    "c5": dict(kind="images", images=1024, h=1080, w=1920, space="all", degenerate=True,
               desc="BASELINE config 5: 1024 x 1920x1080 uint8 RGB + 10% saturated + 5% grays, "
                    "CIELAB+HSI+SCT MACT from one read, sharded by image"),
    "c1": dict(kind="random", n=512 * 512, space="lab",
               desc="BASELINE config 1: one 512x512 uint8 image, default_rng(0), RGB->CIELAB MACT"),
    "c2": dict(kind="cube", n=1 << 24, space="hsi+sct",
               desc="BASELINE config 2: 2^24 cube, RGB->HSI and RGB->SCT MACT, fused (one read, two outputs)"),
    "c3": dict(kind="random", n=4096 * 4096, space="lut",
               desc="BASELINE config 3: 4096^2 uint8, default_rng(0), {method} {grid}^3 LUT (RGB->CIELAB)"),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    return HBM_FALLBACK, "B200_PROFILING.md fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------------- CPU legs
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def cpu_functions(kind: str, lut_spec=None):
    """The CPU implementation of the path: kind "reference" = the UNMODIFIED reference package
    installed in baseline/_ref (mact.fast / mact.lut, its own public API); kind "port" = the oracle's
    numpy restatement.  Returns ({space: fn}, kind actually used)."""
    if kind == "reference" and os.path.isdir(os.path.join(REF_DIR, "mact")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from mact import fast as rf
        from mact import lut as rl

        fns = {"lab": rf.rgb_to_lab_fast, "hsi": rf.rgb_to_hsi_fast, "sct": rf.rgb_to_sct_fast}
        if lut_spec is not None:
            L = rl.build_lut("lab", lut_spec[0])
            fns["lut"] = lambda p, L=L: rl.interpolate(L, p, lut_spec[1])
        return fns, "reference"
    from oracle import mact_oracle as O

    fns = {"lab": O.rgb_to_lab_fast, "hsi": O.rgb_to_hsi_fast, "sct": O.rgb_to_sct_fast}
    if lut_spec is not None:
        vals = O.build_lut_values("lab", lut_spec[0])
        fns["lut"] = lambda p, vals=vals: O.interpolate(vals, p, lut_spec[1])
    return fns, "port"


def host_threads() -> int:
    """All host threads, capped at 64 like MACT_THREADS (harness.py:60)."""
    return max(1, min(64, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()))


def run_chunked(fn, pixels, threads: int, chunk: int = 1 << 18):
    """fn over 2^18-px chunks on a thread pool (the reference's own harness.py:92-103 pattern)."""
    from concurrent.futures import ThreadPoolExecutor

    flat = pixels.reshape(-1, 3)
    parts = [flat[i:i + chunk] for i in range(0, flat.shape[0], chunk)]
    if threads <= 1:
        return [fn(p) for p in parts]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, parts))


def cpu_run(fns, space: str, images, budget_s: float, threads: int):
    """The CPU implementation over host images until budget_s."""
    spaces = ["lab", "hsi", "sct"] if space == "all" else [space]
    px, t0 = 0, time.perf_counter()
    i = 0
    while True:
        img = images[i % len(images)]
        for sp in spaces:
            run_chunked(fns[sp], img, threads)
        px += img.size // 3
        i += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return px, dt


def pcie_bandwidth(dev, nbytes: int = 1 << 30, reps: int = 3):
    """Pinned host <-> device copy bandwidth (GB/s), CUDA events, best of `reps`:
    each direction alone and both at once on two streams."""
    import torch

    h_a = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_b = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {"h2d": 0.0, "d2h": 0.0, "h2d_concurrent": 0.0, "d2h_concurrent": 0.0}

    def run(h2d: bool, d2h: bool):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize(dev)
        if h2d:
            ev[0].record(s1)
            with torch.cuda.stream(s1):
                d_a.copy_(h_a, non_blocking=True)
            ev[1].record(s1)
        if d2h:
            ev[2].record(s2)
            with torch.cuda.stream(s2):
                h_b.copy_(d_b, non_blocking=True)
            ev[3].record(s2)
        torch.cuda.synchronize(dev)
        bw = lambda a, b: nbytes / (a.elapsed_time(b) / 1e3) / 1e9
        return (bw(ev[0], ev[1]) if h2d else 0.0), (bw(ev[2], ev[3]) if d2h else 0.0)

    for _ in range(reps + 1):
        res["h2d"] = max(res["h2d"], run(True, False)[0])
        res["d2h"] = max(res["d2h"], run(False, True)[1])
        a, b = run(True, True)
        res["h2d_concurrent"], res["d2h_concurrent"] = max(res["h2d_concurrent"], a), max(res["d2h_concurrent"], b)
    del h_a, h_b, d_a, d_b
    return res


# --------------------------------------------------------------------- our arm
def run_ours(args, wl):
    import numpy as np
    import torch

    from paper_1009_0854_b200 import _lib, corpus, fast, harness, lut, parallel

    rank, world, local = parallel.init("nccl", share_device=args.share_gpu)
    dev = torch.device("cuda", local)
    cdev = parallel.collective_device(dev)          # NCCL: the GPU; gloo (--share-gpu): the host
    lib = _lib.load()
    cfg = fast.DEFAULT_CONFIG
    hbm, hbm_src = peaks()
    st = torch.cuda.current_stream(dev)

    # ---------------- inputs (device-resident) for this rank
    if wl["kind"] == "images":
        my = parallel.shard_range(wl["images"], world, rank)
        x = corpus.batch(my, wl["h"], wl["w"], device=dev, degenerate=wl["degenerate"])
        n_local = len(my) * wl["h"] * wl["w"]
        n_total = wl["images"] * wl["h"] * wl["w"]
        base = my.start * wl["h"] * wl["w"]
    elif wl["kind"] == "cube":
        my = parallel.shard_range(wl["n"], world, rank)
        x = harness.cube_chunk(my.start, len(my), device=str(dev))
        n_local, n_total, base = len(my), wl["n"], my.start
    else:
        full = np.random.default_rng(0).integers(0, 256, (wl["n"], 3), dtype=np.uint8)
        my = parallel.shard_range(wl["n"], world, rank)
        x = torch.from_numpy(full[my.start:my.stop]).to(dev)
        n_local, n_total, base = len(my), wl["n"], my.start
    xf = x.reshape(-1, 3)
    space = wl["space"]
    n_out = 3 if space == "all" else (2 if space == "hsi+sct" else 1)
    f64 = args.out_dtype == "float64"
    out_b = 24 if f64 else 12                       # bytes per pixel and transform written
    outs = [torch.empty((n_local, 3), dtype=torch.float64 if f64 else torch.float32, device=dev)
            for _ in range(n_out)]
    # L2 rule: a step whose inputs + outputs are below 2x the 126 MB L2 rotates
    # over a pool of copies (distinct input and output buffers) whose footprint
    # exceeds 512 MB, so every step reads and writes lines that are not L2-resident.
    step_bytes = n_local * (3 + out_b * n_out)
    pool_n = 1 if step_bytes >= L2_POOL_BYTES else -(-L2_POOL_BYTES // step_bytes)
    pool = [(xf, outs)] + [(xf.clone(), [torch.empty_like(o) for o in outs]) for _ in range(pool_n - 1)]
    lt = lut.build_lut("lab", args.lut_grid) if space == "lut" else None
    lut_code = lut._method_code(args.lut_method)
    step_i = [0]

    def step():
        xf, outs = pool[step_i[0] % pool_n]
        step_i[0] += 1
        sp_ptr = torch.cuda.current_stream(dev).cuda_stream   # capture-safe (graph mode)
        if space == "all":
            _lib.check(lib.mact_all_fast(xf.data_ptr(), outs[0].data_ptr(), outs[1].data_ptr(),
                                         outs[2].data_ptr(), n_local, cfg.coeffs, 0, sp_ptr))
        elif space == "hsi+sct":     # fused pair: one read, two outputs (lab = NULL)
            _lib.check(lib.mact_all_fast(xf.data_ptr(), None, outs[0].data_ptr(), outs[1].data_ptr(),
                                         n_local, cfg.coeffs, 0, sp_ptr))
        elif space == "lab" and f64:     # fidelity mode: the reference's fp64 arithmetic
            _lib.check(lib.mact_fast_f64(_lib.SPACES["lab"], xf.data_ptr(), _lib.DTYPE_U8, outs[0].data_ptr(),
                                         n_local, cfg.coeffs, 0, sp_ptr))
        elif space == "lab":
            _lib.check(lib.mact_lab_fast(xf.data_ptr(), 0, outs[0].data_ptr(), n_local, cfg.coeffs, 0, sp_ptr))
        elif f64:
            lat = lt.lattice64(dev)
            _lib.check(lib.mact_lut_interp_real(lat.data_ptr(), args.lut_grid, lut_code, 0, xf.data_ptr(),
                                                _lib.DTYPE_U8, outs[0].data_ptr(), _lib.DTYPE_F64, n_local, 0,
                                                sp_ptr))
        else:
            lat = lt.lattice(dev)
            _lib.check(lib.mact_lut_interp(lat.data_ptr(), args.lut_grid, lut_code, xf.data_ptr(),
                                           outs[0].data_ptr(), n_local, 0, sp_ptr))

    # ---------------- per-rank error partials (the reduction pass is reporting, not
    # throughput: SURVEY §8(d) excludes it from the metric; its device time is in the
    # line as error.reduce_ms).  The cross-rank all-gather + rank-order fold of these
    # partials -- the job's only exchange -- runs INSIDE the timed window below.
    partial_sets = []
    ev_r0, ev_r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_r0.record(st)
    if space in ("lab", "all", "lut"):
        if space == "lut":
            cand = (harness.LutCandidate(lt, args.lut_method) if not f64 else
                    (lambda p: lut.interpolate(lt, p, args.lut_method, out_dtype="float64")))
        else:
            cand = harness.fast_candidate("lab", out_dtype=args.out_dtype)
        partial_sets.append(("lab", harness.reduce_partials("lab", cand, None, xf, index_base=base)))
        if space == "lut":   # config 3: "compared with MACT on the same pixels"
            partial_sets.append(("mact", harness.reduce_partials("lab", harness.fast_candidate("lab"), None, xf,
                                                                 index_base=base)))
    if space in ("all", "hsi+sct"):   # configs 2 and 5: per-component |fast - exact|
        for sp in ("hsi", "sct"):
            partial_sets.append((sp, harness.reduce_partials(sp, harness.fast_candidate(sp), None, xf,
                                                             index_base=base, metric="component")))
    ev_r1.record(st)
    torch.cuda.synchronize(dev)
    reduce_ms = parallel.max_over_ranks(ev_r0.elapsed_time(ev_r1), cdev)
    flat_parts = [p for _, ps in partial_sets for p in ps]

    transforms = {"all": 3, "hsi+sct": 2}.get(space, 1)
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    # The K steps are captured once into a CUDA graph and replayed in the timed
    # region: short steps are launch-latency bound (C1: 262 K px = ~1 us of HBM
    # time; the ~0.1 ms C2/C3 steps lose ~9 us each to launch gaps), and even C4's
    # 1.8 ms steps gain 0.6 %.  --no-graph times stream launches with per-step events.
    use_graph = args.graph is not False
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(st)
        lib.mact_launch_count_reset()
        with torch.cuda.graph(graph, stream=cap):
            for _ in range(args.steps):
                step()
        graph_launches = int(lib.mact_launch_count())
        graph.replay()                                   # warm replay
        torch.cuda.synchronize(dev)

    # ---------------- timed region: common barrier -> K steps -> the final stat
    # combine (all-gather of the error partials + rank-order fold), SURVEY §8(d);
    # CUDA events on the launching stream, max over ranks.
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    parallel.barrier(cdev)
    torch.cuda.synchronize(dev)
    lib.mact_launch_count_reset()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        tk = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        if graph is not None:
            graph.replay()
        else:
            for k in range(args.steps):
                evs[k][0].record(st)
                step()
                evs[k][1].record(st)
        tk.record(st)
        per_rank = parallel.all_gather_partials(flat_parts, cdev) if flat_parts else []
        folded = parallel.combine(per_rank) if per_rank else []
        t1.record(st)
        torch.cuda.synchronize(dev)
    launches = graph_launches if graph is not None else int(lib.mact_launch_count())
    parallel.barrier(cdev)
    local_ms = t0.elapsed_time(t1)
    total_ms = parallel.max_over_ranks(local_ms, cdev)
    steps_ms = t0.elapsed_time(tk)
    combine_ms = parallel.max_over_ranks(tk.elapsed_time(t1), cdev)
    step_ms = ([steps_ms / args.steps] * args.steps if graph is not None
               else [a.elapsed_time(b) for a, b in evs])

    # ---------------- error statistics from the folded partials
    err = None
    it = iter(folded)
    for name, ps in partial_sets:
        got = [next(it) for _ in ps]
        if name == "lab":
            tot = got[0]
            err = {"dE_mean": tot["sum"] / tot["count"], "dE_max": tot["max"],
                   "dE_argmax_index": tot["argmax"], "pixels": tot["count"]}
        elif name == "mact":
            err["mact_dE_mean"], err["mact_dE_max"] = got[0]["sum"] / got[0]["count"], got[0]["max"]
        else:
            err = err or {}
            err[name] = [{"mean": c["sum"] / max(c["count"], 1), "max": c["max"],
                          "excluded_nan": c["nan"]} for c in got]
    if err is not None:
        err["reduce_ms"] = round(reduce_ms, 3)
        err["combine_ms_in_timed_region"] = round(combine_ms, 4)
    # every workload is ONE launch per step (C2/C5 run the transforms fused from one read)
    kern_ms = statistics.mean(step_ms)
    value = n_total * transforms * args.steps / (total_ms / 1e3) / 1e9
    bytes_px = 3 + out_b * transforms                        # uint8 in once + (N,3) out per transform
    achieved = n_local * bytes_px / (kern_ms / 1e3) / 1e9
    traffic, traffic_b, traffic_src = None, None, None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    tkey = args.workload + (f"_{args.lut_grid}_{args.lut_method}" if space == "lut" else "") + ("_f64" if f64 else "")
    if os.path.exists(prof) and world == 1:
        t = json.load(open(prof)).get(tkey)
        if t:   # ncu dram bytes per launch of this kernel (one --set full capture), over the live launch time
            traffic_b = t["bytes_per_launch"]
            traffic = round(traffic_b / (kern_ms / 1e3) / 1e9, 1)
            traffic_src = (f"profiles/traffic.json[{tkey}]: {t.get('source')} ({t.get('kernel', '')[:40]}), "
                           f"captured at commit {t.get('commit', 'unrecorded')}")

    # ---------------- end to end through the public API with HOST buffers
    e2e = None
    if args.e2e_steps > 0:
        sp1 = {"lab": "lab", "all": "lab", "hsi+sct": "hsi"}.get(space, "lut")
        od = {"out_dtype": "float64"} if f64 else {}
        fn = {"lab": lambda p, out: fast.rgb_to_lab_fast(p, out=out, **od),
              "hsi": fast.rgb_to_hsi_fast,
              "lut": lambda p, out: lut.interpolate(lt, p, args.lut_method, out=out, **od)}[sp1]
        h_in = torch.empty((n_local, 3), dtype=torch.uint8).pin_memory()
        h_in.copy_(xf.cpu())
        h_out = torch.empty((n_local, 3), dtype=torch.float64 if f64 else torch.float32).pin_memory()
        hi, ho = h_in.numpy(), h_out.numpy()
        # warm the executor: a whole untimed call for the small workloads (their chunking differs from
        # a 4 Mpx prefix's), a 4 Mpx prefix for the large ones
        nwarm = n_local if n_local <= (1 << 26) else (1 << 22)
        fn(hi[:nwarm], out=ho[:nwarm])
        torch.cuda.synchronize(dev)
        parallel.barrier(cdev)
        t = time.perf_counter()
        for _ in range(args.e2e_steps):
            fn(hi, out=ho)
        torch.cuda.synchronize(dev)
        dt = parallel.max_over_ranks(time.perf_counter() - t, cdev)
        bw = pcie_bandwidth(dev)
        # the executor overlaps H2D, kernel and D2H on separate engines, so the ceiling is
        # the slower direction at its own best pinned-copy bandwidth (the concurrent
        # figures are reported beside it)
        e2e_peak = min(bw["h2d"] / 3, bw["d2h"] / out_b)      # Gpix/s per GPU
        e2e_val = n_total * args.e2e_steps / dt / 1e9
        e2e = {"value": e2e_val, "unit": "Gpixels/s",
               "h2d_bytes_per_step": n_total * 3, "d2h_bytes_per_step": n_total * out_b,
               "roofline": {"bound": "pcie", "achieved": round(e2e_val / world, 3), "peak": round(e2e_peak, 3),
                            "unit": "Gpixels/s per GPU", "frac": round(e2e_val / world / e2e_peak, 4),
                            **{k + "_gbs": round(v, 1) for k, v in bw.items()},
                            "method": "pinned 1 GiB copies, CUDA events, best of 3: each direction alone "
                                      "(the ceiling) and both at once"},
               "api": (f"paper_1009_0854_b200.fast.rgb_to_{sp1}_fast" if sp1 != "lut" else
                       "paper_1009_0854_b200.lut.interpolate") + "(numpy pinned, out=numpy pinned)",
               "steps": args.e2e_steps, "transform": sp1}
        del h_in, h_out

    # ---------------- CPU baseline (rank 0, N=1 only): the reference itself (baseline/_ref)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = [xf[i * 2_073_600:(i + 1) * 2_073_600].cpu().numpy() for i in range(2)]
        threads = host_threads()
        sp = {"lab": "lab", "all": "lab", "hsi+sct": "hsi"}.get(space, "lut")
        fns, kind = cpu_functions("reference", (args.lut_grid, args.lut_method) if sp == "lut" else None)
        px, dt = cpu_run(fns, sp, sample, args.cpu_seconds, threads)
        what = f"rgb_to_{sp}_fast" if sp != "lut" else f"lut.interpolate({args.lut_method}, {args.lut_grid}^3)"
        src = ("baseline/_ref/mact (the unmodified reference package, its public API)" if kind == "reference"
               else "oracle/mact_oracle.py (numpy restatement of the reference)")
        cpu = {"value": px / dt / 1e9, "unit": "Gpixels/s", "cores": threads, "kind": kind,
               "sample": f"{src} {what} over 2,073,600-px slices of the same workload, {px} px in "
                         f"{dt:.1f} s, ThreadPoolExecutor x{threads} over 2^18-px chunks (harness.py:92-103)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Gpixels/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(total_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8->f64" if f64 else "u8->f32",
            "data": "synthetic (generated on device, seeded per image)",
            "config": {"workload": f"{args.workload}: {wl['desc']}", "pixels": n_total,
                       "transforms_per_step": transforms, "layout": "interleaved (N,3) fp32",
                       "parallelism": (f"dp{world} (shard by {'image' if wl['kind'] == 'images' else 'pixel range'}, "
                                       "no data-path collective; one all-gather of the error partials "
                                       f"over {'gloo' if args.share_gpu else 'NCCL'} inside the timed window)"),
                       "devices": ("all ranks share cuda:0 (--share-gpu host-logic test: NOT an N-GPU number)"
                                   if args.share_gpu else f"{world} x cuda, one process per GPU"),
                       "launch": "CUDA graph of the K steps" if graph is not None else "stream launches",
                       "l2": ("inputs+outputs > 2x the 126 MB L2 (no flush needed)" if pool_n == 1 else
                              f"steps rotate over {pool_n} input/output copies ({pool_n * step_bytes / 1e6:.0f} MB "
                              "> 2x the 126 MB L2), so no step finds its data in L2")},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                         "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
                         "traffic_bytes_per_launch": traffic_b, "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": n_local * bytes_px,
                         "peak_source": hbm_src, "algorithmic_bytes_per_px": bytes_px,
                         "kernel_ms_per_launch": round(kern_ms, 4),
                         "gpix_per_s_per_gpu_kernel": round(n_local * transforms / (kern_ms / 1e3) / 1e9, 2)},
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clk.summary(), "error": err,
        }
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- reference arm
def run_reference(args, wl):
    """The reference arm: the UNMODIFIED reference package (baseline/_ref/mact, pure Python +
    numpy, no GPU code) through its own public API, on all host threads, one bounded sample of
    the workload per step.  Rank 0 only; the oracle port is timed once beside it as a cross-check."""
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if rank != 0:
        return
    import numpy as np

    threads = host_threads()
    space = wl["space"]
    # bounded sample of the same workload: one image-sized slice per step
    if wl["kind"] == "images":
        try:
            import torch
            if torch.cuda.is_available():
                from paper_1009_0854_b200 import corpus
                img = corpus.correlated_image(0, wl["h"], wl["w"], degenerate=wl["degenerate"]).cpu().numpy()
            else:
                raise RuntimeError
        except Exception:
            img = np.random.default_rng(0).integers(0, 256, (wl["h"], wl["w"], 3), dtype=np.uint8)
        sample = img.reshape(-1, 3)[: 2_073_600]
    elif wl["kind"] == "cube":
        idx = np.arange(1 << 21, dtype=np.uint32)                     # harness.cube_chunk(0, 2^21)
        sample = np.stack([idx >> 16, (idx >> 8) & 255, idx & 255], -1).astype(np.uint8)
    else:
        sample = np.random.default_rng(0).integers(0, 256, (min(wl["n"], 1 << 21), 3), dtype=np.uint8)
    lut_spec = (args.lut_grid, args.lut_method) if space == "lut" else None
    spaces = {"lab": ["lab"], "all": ["lab", "hsi", "sct"], "hsi+sct": ["hsi", "sct"]}.get(space, ["lut"])

    def timed(kind, steps, warmup):
        fns, used = cpu_functions(kind, lut_spec)
        for _ in range(warmup):
            for sp in spaces:
                run_chunked(fns[sp], sample, threads)
        times = []
        for _ in range(steps):
            t = time.perf_counter()
            for sp in spaces:
                run_chunked(fns[sp], sample, threads)
            times.append(time.perf_counter() - t)
        return sample.shape[0] * len(spaces) * steps / sum(times) / 1e9, sum(times), used

    value, total, kind = timed("reference", args.steps, max(args.warmup, 1))
    port_value = timed("port", 1, 0)[0] if kind == "reference" else None
    px = sample.shape[0]
    what = ("baseline/_ref/mact (the unmodified reference package, pip-installed from /root/reference; "
            f"{', '.join('mact.fast.rgb_to_%s_fast' % sp if sp != 'lut' else 'mact.lut.interpolate' for sp in spaces)})"
            if kind == "reference" else "oracle/mact_oracle.py (numpy restatement; baseline/_ref missing)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gpixels/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 1),
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {wl['desc']}",
                   "sample_pixels_per_step": px},
        "cpu_baseline": {"value": round(value, 6), "unit": "Gpixels/s", "cores": threads, "kind": kind,
                         "sample": f"{px} px of the workload per step through {what}, "
                                   f"ThreadPoolExecutor x{threads} over 2^18-px chunks (harness.py:92-103)",
                         "port_value": None if port_value is None else round(port_value, 6)},
        "e2e": {"value": round(value, 6), "unit": "Gpixels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _relaunch(n: int) -> int:
    """--gpus N without torchrun: re-exec this command as N ranks through torch.distributed.run."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    print(f"bench.py: launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--lut-grid", type=int, choices=[9, 17, 33], default=17, help="c3 only")
    ap.add_argument("--lut-method", choices=["trilinear", "prism", "pyramidal", "tetrahedral"],
                    default="tetrahedral", help="c3 only")
    ap.add_argument("--out-dtype", choices=["float32", "float64"], default="float32",
                    help="float64 = fidelity mode (the reference's fp64 arithmetic, 24 B/px out); c1/c3/c4")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=None,
                    help="capture the K steps in a CUDA graph (default: on)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="run every rank on cuda:0 with a gloo combine (N-rank host-logic test on a 1-GPU box)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to report a mismatched line",
              file=sys.stderr)
        sys.exit(2)
    if args.out_dtype == "float64" and WORKLOADS[args.workload]["space"] not in ("lab", "lut"):
        ap.error("--out-dtype float64 is measured on the single-transform workloads c1 / c3 / c4")
    wl = dict(WORKLOADS[args.workload])
    wl["desc"] = wl["desc"].format(grid=args.lut_grid, method=args.lut_method)
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
