import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1009_0854_b200 import lut, harness
seq = sys.argv[1]
cube = harness.cube_chunk(0, 1 << 24, device="cuda")
def run(n, layout, m="trilinear"):
    lt = lut.build_lut("lab", n)
    t = time.time()
    o = lut.interpolate(lt, cube, m, layout=layout).cpu()
    print(seq, n, layout, f"{time.time() - t:.3f}s", flush=True)
if seq == "a":
    run(33, "interleaved"); run(33, "planar")
elif seq == "b":
    for n in (9, 17):
        run(n, "interleaved"); run(n, "planar")
    run(33, "interleaved"); run(33, "planar")
elif seq == "c":
    run(33, "planar"); run(33, "interleaved"); run(33, "planar")
elif seq == "d":
    os.environ["MACT_LUT33_KERNEL"] = "comp"; run(33, "planar"); run(33, "interleaved")
