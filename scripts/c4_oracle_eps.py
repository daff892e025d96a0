"""BASELINE config 4 (and a config-5 subset) error figures: the fused GPU
reduction against the CPU oracle on the same bytes ("oracle ε
computed once on CPU").  "gpu" scores the fp32 throughput outputs (so it
includes their output rounding), "gpu_f64" the fp64 fidelity candidate.
Run on the GPU box; writes one JSON line.

    python scripts/c4_oracle_eps.py [--images 64] [--c5-every 16]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import mact_oracle as O  # noqa: E402
from paper_1009_0854_b200 import corpus  # noqa: E402


from tests.test_gpu_full_scale import gpu_eps, oracle_eps  # noqa: E402  (the slow -m gpu test runs the same)


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
