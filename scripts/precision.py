"""Full-cube precision of the fast kernels against the CPU oracle (max abs
error per component; HSI/SCT normalised).  python scripts/precision.py [lab hsi sct]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from oracle import mact_oracle as O  # noqa: E402
from paper_1009_0854_b200 import fast, harness  # noqa: E402

spaces = [a for a in sys.argv[1:] if a in ("lab", "hsi", "sct")] or ["lab", "hsi", "sct"]
cube = harness.cube_chunk(0, 1 << 24, device="cuda")
host = cube.cpu().numpy()
scale = {"lab": np.ones(3), "hsi": np.array([2 * np.pi, 1, 1]), "sct": np.array([255 * np.sqrt(3), np.pi / 2, np.pi / 2])}
for sp in spaces:
    got = getattr(fast, f"rgb_to_{sp}_fast")(cube).cpu().numpy().astype(np.float64)
    worst = np.zeros(3)
    where = [None] * 3
    for s in range(0, 1 << 24, 1 << 22):
        ref = O.FAST[sp](host[s:s + (1 << 22)])
        d = np.abs(got[s:s + (1 << 22)] - ref)
        if sp == "hsi":
            d[:, 0] = np.minimum(d[:, 0], 2 * np.pi - d[:, 0])
        d = np.nan_to_num(d) / scale[sp]
        for c in range(3):
            j = int(np.argmax(d[:, c]))
            if d[j, c] > worst[c]:
                worst[c] = d[j, c]
                where[c] = tuple(int(v) for v in host[s + j])
    print(f"{sp}: max err {worst.tolist()} at {where}  (tolerance {'1e-4 abs' if sp == 'lab' else '1e-5 normalised'})")
