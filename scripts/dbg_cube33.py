import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1009_0854_b200 import lut, harness
lt = lut.build_lut("lab", 33)
for n in [1 << 16, 1 << 20, 1 << 24]:
    cube = harness.cube_chunk(0, n, device="cuda")
    for m in sys.argv[1:] or ["trilinear"]:
        for layout in ("interleaved", "planar"):
            t = time.time()
            o = lut.interpolate(lt, cube, m, layout=layout)
            torch.cuda.synchronize()
            print(n, m, layout, f"{time.time() - t:.3f}s", flush=True)
