"""Small driver for ncu / timing of one libmact_cuda kernel.

    python scripts/prof_kernel.py --op lab|hsi|sct|all|lut17|lut33|lut9 [--n PIXELS] [--iters K]
      [--method tetrahedral] [--input random|corr|cube] [--time]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1009_0854_b200 import _lib, corpus, fast, harness, lut  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="lab")
ap.add_argument("--n", type=int, default=1 << 26)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--method", default="tetrahedral")
ap.add_argument("--input", default="random")
ap.add_argument("--time", action="store_true")
ap.add_argument("--planar", action="store_true")
a = ap.parse_args()

lib = _lib.load()
n = a.n
if a.input == "cube":
    x = harness.cube_chunk(0, n, device="cuda")
elif a.input == "corr":
    h, w = 2160, 3840
    k = max(1, n // (h * w))
    x = corpus.batch(range(k), h, w).reshape(-1, 3)
    n = x.shape[0]
else:
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    x = torch.randint(0, 256, (n, 3), dtype=torch.uint8, device="cuda", generator=g)
nout = 3 if a.op == "all" else 1
outs = [torch.empty((n, 3), dtype=torch.float32, device="cuda") for _ in range(nout)]
cfg = fast.DEFAULT_CONFIG
st = torch.cuda.current_stream().cuda_stream
lt = lut.build_lut("lab", int(a.op[3:])) if a.op.startswith("lut") else None


def run():
    if a.op == "all":
        _lib.check(lib.mact_all_fast(x.data_ptr(), outs[0].data_ptr(), outs[1].data_ptr(),
                                     outs[2].data_ptr(), n, cfg.coeffs, 0, st))
    elif a.op.startswith("exactf32_"):
        sp = {"exactf32_lab": 0, "exactf32_hsi": 1, "exactf32_sct": 2}[a.op]
        _lib.check(lib.mact_exact_f32(sp, x.data_ptr(), outs[0].data_ptr(), n, int(a.planar), st))
    elif a.op.startswith("exact_"):
        sp = {"exact_lab": 0, "exact_hsi": 1, "exact_sct": 2}[a.op]
        _lib.check(lib.mact_exact(sp, x.data_ptr(), 0, outs[0].data_ptr(), 1, n, st))
    elif a.op == "probe":
        _lib.check(lib.mact_probe_expand(x.data_ptr(), outs[0].data_ptr(), n, st))
    elif a.op in ("lab", "hsi", "sct"):
        _lib.check(getattr(lib, f"mact_{a.op}_fast")(x.data_ptr(), 0, outs[0].data_ptr(), n,
                                                     cfg.coeffs, 0, st))
    else:
        lat = lt.lattice()
        _lib.check(lib.mact_lut_interp(lat.data_ptr(), lt.grid_n, _lib.METHODS[a.method],
                                       x.data_ptr(), outs[0].data_ptr(), n, int(a.planar), st))


for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
if a.time:
    gbs = n * 15 * nout / (ms / 1e3) / 1e9 if nout == 1 else n * 39 / (ms / 1e3) / 1e9
    print(f"{a.op} n={n} {ms:.4f} ms  {n / ms / 1e6:.1f} Gpix/s  {gbs:.0f} GB/s")
