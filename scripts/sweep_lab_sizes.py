"""Lab fast-transform throughput vs image size with cold L2 (rotating over
distinct input/output copies whose total exceeds 2x the 126 MB L2), to place
the direct-kernel / streaming-kernel crossovers (mact_fast.cu launchers).

    MACT_LIB=... python scripts/sweep_lab_sizes.py [--space lab|hsi|sct]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1009_0854_b200 import _lib, fast  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--space", default="lab")
ap.add_argument("--sizes", default="262144,524288,1048576,2097152,4194304,8388608,16777216,33554432")
a = ap.parse_args()
lib = _lib.load()
fn = getattr(lib, f"mact_{a.space}_fast")
cfg = fast.DEFAULT_CONFIG
st = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda")
g.manual_seed(0)
for n in map(int, a.sizes.split(",")):
    copies = max(2, -(-(300 << 20) // (15 * n)))
    xs = [torch.randint(0, 256, (n, 3), dtype=torch.uint8, device="cuda", generator=g) for _ in range(copies)]
    ys = [torch.empty((n, 3), dtype=torch.float32, device="cuda") for _ in range(copies)]
    iters = max(copies, min(2000, (1 << 30) // n))

    def run(i):
        _lib.check(fn(xs[i % copies].data_ptr(), 0, ys[i % copies].data_ptr(), n, cfg.coeffs, 0, st))

    for i in range(copies):
        run(i)
    torch.cuda.synchronize()
    # one CUDA graph over all copies, replayed: launch gaps of the host loop excluded
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        st = side.cuda_stream
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=side):
            for i in range(copies):
                run(i)
    st = torch.cuda.current_stream().cuda_stream
    reps = max(1, iters // copies)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * copies)
    print(f"{a.space} n={n:>9} copies={copies:>3} {ms * 1e3:9.2f} us  {n / ms / 1e6:7.1f} Gpix/s", flush=True)
    del xs, ys
