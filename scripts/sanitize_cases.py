"""Small launches of every kernel family for compute-sanitizer (scripts/sanitize.sh).

    MACT_GRID_CAP=4 python scripts/sanitize_cases.py [case ...]

MACT_GRID_CAP caps the persistent grids (and 33^3 cluster counts) so every CTA
loops over several tiles and recycles every ring / staging buffer even on
small inputs -- the hazards racecheck / synccheck look for live in that
recycling.  Each case checks its result against a loose bound so a sanitizer
run also proves the kernels still compute.  Cases: lab all hsi sct lut9 lut17
lut33 err host (default: all).
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1009_0854_b200 import _lib, exact, fast, harness, lut  # noqa: E402


def px(n, seed=7):
    return torch.from_numpy(np.random.default_rng(seed).integers(0, 256, (n, 3), dtype=np.uint8)).cuda()


def close(a, b, tol):
    d = (a.double() - b.double()).abs()
    d = torch.where(torch.isnan(d), torch.zeros_like(d), d)
    assert float(d.max()) <= tol, float(d.max())


N = 4 * 16 * 512 * 4 + 77          # several streaming tiles per CTA under the cap, plus a tail


def case_lab():
    x = px(N)
    close(fast.rgb_to_lab_fast(x), exact.rgb_to_lab_exact(x), 0.1)
    close(fast.rgb_to_lab_fast(x[:4096]), exact.rgb_to_lab_exact(x[:4096]), 0.1)   # small-image path


def case_all():
    x = px(N)
    lab, hsi, sct = (torch.empty((N, 3), dtype=torch.float32, device="cuda") for _ in range(3))
    _lib.call("mact_all_fast", x.data_ptr(), lab.data_ptr(), hsi.data_ptr(), sct.data_ptr(), N,
              fast.DEFAULT_CONFIG.coeffs, 0, torch.cuda.current_stream().cuda_stream)
    close(lab, fast.rgb_to_lab_fast(x), 1e-4)


def case_hsi():
    x = px(N)
    fast.rgb_to_hsi_fast(x), fast.rgb_to_hsi_fast(x[:8192])


def case_sct():
    x = px(N)
    fast.rgb_to_sct_fast(x), fast.rgb_to_sct_fast(x[:8192])


def _lut(n, planar=True):
    x = px(N)
    lt = lut.build_lut("lab", n)
    for m in lut.METHODS:
        a = lut.interpolate(lt, x, m)
        ref = lut.interpolate(lt, x, m, out_dtype="float64")
        close(a, ref, 1e-4)
        if planar:
            close(lut.interpolate(lt, x[:N - 77], m, layout="planar").T, ref[:N - 77], 1e-4)


def case_lut9():
    _lut(9)


def case_lut17():
    _lut(17)


def case_lut33():
    _lut(33)


def case_err():
    x = px(N)
    st = harness.measure_error("lab", fast.rgb_to_lab_fast, exact.rgb_to_lab_exact, population=x)
    assert 0 < st.avg < 0.01
    comp = harness.component_error("hsi", population=x)
    assert len(comp) == 3


def case_host():
    x = px(N).cpu().numpy()
    out = fast.rgb_to_lab_fast(x)
    close(torch.from_numpy(out), exact.rgb_to_lab_exact(torch.from_numpy(x).cuda()).cpu(), 0.1)


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        CASES[name]()
        torch.cuda.synchronize()
        print(f"case {name}: ok", flush=True)
