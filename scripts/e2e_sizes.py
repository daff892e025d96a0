"""End-to-end time of the public API on pinned numpy buffers vs input size: separates the fixed cost of a
call from the PCIe-bound slope (Lab transform and 33^3 / 17^3 tetrahedral LUT).  Run on the GPU box."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1009_0854_b200 import fast, lut  # noqa: E402

L33, L17 = lut.build_lut("lab", 33), lut.build_lut("lab", 17)
for n in (1 << 18, 1 << 20, 1 << 22, 1 << 24, 1 << 26):
    h_in = torch.randint(0, 256, (n, 3), dtype=torch.uint8).pin_memory()
    h_out = torch.empty((n, 3), dtype=torch.float32).pin_memory()
    a, o = h_in.numpy(), h_out.numpy()
    row = [f"n=2^{n.bit_length() - 1}"]
    for name, fn in (("lab", lambda: fast.rgb_to_lab_fast(a, out=o)),
                     ("lut17", lambda: lut.interpolate(L17, a, "tetrahedral", out=o)),
                     ("lut33", lambda: lut.interpolate(L33, a, "tetrahedral", out=o))):
        fn(); fn()
        reps = 5 if n <= 1 << 24 else 2
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        dt = (time.perf_counter() - t0) / reps
        row.append(f"{name} {dt * 1e3:.3f} ms {n / dt / 1e9:.2f} Gpix/s")
    print("  ".join(row))
