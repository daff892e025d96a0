"""BASELINE config 4 (and a config-5 subset) error figures: the fused GPU
reduction against the CPU oracle on the same bytes ("oracle ε
computed once on CPU").  "gpu" scores the fp32 throughput outputs (so it
includes their output rounding), "gpu_f64" the fp64 fidelity candidate.
Run on the GPU box; writes one JSON line.

    python scripts/c4_oracle_eps.py [--images 64] [--c5-every 16]
"""
import argparse
import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import mact_oracle as O  # noqa: E402
from paper_1009_0854_b200 import corpus, harness, parallel  # noqa: E402


def oracle_eps(space, images, threads):
    """harness.measure_error semantics over host images: fsum of chunk sums, first max."""
    def chunk(p):
        if space == "lab":
            d = O.lab_distance(O.rgb_to_lab_fast(p), O.rgb_to_lab_exact(p))
            j = int(np.argmax(d))
            return [(float(np.sum(d)), float(d[j]), j, d.size, 0)]
        f, e = O.FAST[space](p), O.EXACT[space](p)
        return [(c["sum"], c["max"], c["argmax"], c["count"], c["nan"]) for c in O.component_abs_error(space, f, e)]

    parts, base = [], 0
    jobs = []
    for img in images:
        flat = img.reshape(-1, 3)
        for s in range(0, flat.shape[0], 1 << 20):
            jobs.append((base + s, flat[s:s + (1 << 20)]))
        base += flat.shape[0]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        res = list(pool.map(lambda j: (j[0], chunk(j[1])), jobs))
    ncomp = len(res[0][1])
    out = []
    for c in range(ncomp):
        sums, best, arg, count, nan = [], -1.0, -1, 0, 0
        for off, r in res:
            s_, m_, a_, n_, z_ = r[c]
            sums.append(s_); count += n_; nan += z_
            if m_ > best:
                best, arg = m_, off + a_
        out.append({"mean": math.fsum(sums) / max(count, 1), "max": best, "argmax": arg, "count": count, "nan": nan})
    return out


def gpu_eps(space, x, metric, out_dtype="float32"):
    parts = harness.reduce_partials(space, harness.fast_candidate(space, out_dtype=out_dtype), None, x,
                                    metric=metric)
    return [{"mean": p["sum"] / max(p["count"], 1), "max": p["max"], "argmax": p["argmax"], "count": p["count"],
             "nan": p["nan"]} for p in parts]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=64)
    ap.add_argument("--c5-every", type=int, default=16)
    a = ap.parse_args()
    threads = O.host_threads()
    t0 = time.time()
    res = {"threads": threads}
    x = corpus.batch(range(a.images), 2160, 3840, device="cuda")
    res["c4_lab"] = {"gpu": gpu_eps("lab", x.reshape(-1, 3), "distance")[0],
                     "gpu_f64": gpu_eps("lab", x.reshape(-1, 3), "distance", "float64")[0],
                     "oracle": oracle_eps("lab", list(x.cpu().numpy()), threads)[0]}
    del x
    idx = list(range(0, 1024, a.c5_every))
    y = corpus.batch(idx, 1080, 1920, device="cuda", degenerate=True)
    host = list(y.cpu().numpy())
    yf = y.reshape(-1, 3)
    res["c5_subset_images"] = idx
    res["c5_lab"] = {"gpu": gpu_eps("lab", yf, "distance")[0], "gpu_f64": gpu_eps("lab", yf, "distance", "float64")[0],
                     "oracle": oracle_eps("lab", host, threads)[0]}
    for sp in ("hsi", "sct"):
        res[f"c5_{sp}"] = {"gpu": gpu_eps(sp, yf, "component"), "gpu_f64": gpu_eps(sp, yf, "component", "float64"),
                           "oracle": oracle_eps(sp, host, threads)}
    res["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
