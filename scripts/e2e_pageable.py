"""End-to-end throughput of the numpy API with ordinary (pageable) host arrays,
the way a reference user calls it: uint8 (H,W,3) in, fresh float32 array out."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1009_0854_b200 import fast  # noqa: E402
img = np.random.default_rng(0).integers(0, 256, (8, 2160, 3840, 3), dtype=np.uint8)   # 66 Mpx
fast.rgb_to_lab_fast(img[:1])
for mode in ("fresh out", "reused out"):
    out = np.empty(img.shape, np.float32) if mode == "reused out" else None
    if out is not None:
        fast.rgb_to_lab_fast(img, out=out)
    t = time.perf_counter()
    for _ in range(3):
        r = fast.rgb_to_lab_fast(img, out=out) if out is not None else fast.rgb_to_lab_fast(img)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"pageable numpy, {mode}: {img.size // 3 / dt / 1e9:.2f} Gpix/s ({dt * 1e3:.1f} ms per {img.size // 3 / 1e6:.0f} Mpx)")
