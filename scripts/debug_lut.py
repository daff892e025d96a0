import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import mact_oracle as O
from paper_1009_0854_b200 import lut
img = np.random.default_rng(0).integers(0, 256, (4096 * 4096, 3), dtype=np.uint8)
d = torch.from_numpy(img).cuda()
for n, m in [(17, "trilinear"), (33, "tetrahedral"), (17, "tetrahedral")]:
    lt = lut.build_lut("lab", n)
    a = lut.interpolate(lt, d, m).cpu().numpy()
    b = lut.interpolate(lt, d, m).cpu().numpy()
    # generic path: unaligned copy
    buf = torch.empty(img.shape[0] * 3 + 16, dtype=torch.uint8, device="cuda")
    u = buf[1:1 + img.shape[0] * 3].view(-1, 3)
    u.copy_(d)
    g = lut.interpolate(lt, u, m).cpu().numpy()
    vals = O.build_lut_values("lab", n).astype(np.float32).astype(np.float64)
    k = 1 << 20
    ref = O.interpolate(vals, img[:k], m)
    bad = np.nonzero(np.abs(a[:k] - ref).max(1) > 1e-4)[0]
    badg = np.nonzero(np.abs(g[:k] - ref).max(1) > 1e-4)[0]
    print(n, m, "runs equal:", np.array_equal(a, b), "bad tile-path:", bad.size, "bad generic:", badg.size)
    if bad.size:
        print("  first bad idx", bad[:10], "mod1024", bad[:10] % 1024, "px", img[bad[:5]].tolist())
        print("  got", a[bad[:3]].tolist(), "ref", ref[bad[:3]].tolist())
        print("  distinct tiles", np.unique(bad // 1024).size, "pos hist", np.bincount(bad % 1024 // 128, minlength=8))
