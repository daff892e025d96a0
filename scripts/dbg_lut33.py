import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1009_0854_b200 import lut
from oracle import mact_oracle as O
rng = np.random.default_rng(3)
for n in [int(a) for a in sys.argv[2:]] or [4096]:
    px = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    d = torch.from_numpy(px).cuda()
    lt = lut.build_lut("lab", 33)
    for m in ["trilinear", "prism", "pyramidal", "tetrahedral"] if sys.argv[1] == "all" else [sys.argv[1]]:
        o = lut.interpolate(lt, d, m).cpu().numpy()
        torch.cuda.synchronize()
        r = O.interpolate(O.build_lut_values("lab", 33), px, m)
        print(n, m, np.abs(o - r).max(), flush=True)
