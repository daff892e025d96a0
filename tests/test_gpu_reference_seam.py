"""The plugin seam exercised from the REFERENCE side.

The unmodified reference package installed in baseline/_ref (`pip install --target
baseline/_ref`) is copied to a scratch directory, INTEGRATION.md's
ctypes stub is dropped in as `mact/_b200.py` -- extracted verbatim from the document,
so the document is what is tested -- and the reference's own harness
(`mact.harness.measure_error`, harness.py:77-122) scores the B200 backend:

- `_b200.rgb_to_{lab,hsi,sct}_fast` agree with `mact.fast` within the north-star
  tolerances on config 1 (512x512, default_rng(0)), and bit for bit with
  out_dtype="float64" (mact_transform_host_f64);
- `mact.harness.measure_error("lab", _b200 backend, mact.exact.rgb_to_lab_exact,
  population=C1)` reproduces the figure the reference itself produced
  (tests/golden/figures.json, written by make_golden.py from the live reference).
"""

import os
import re
import shutil
import subprocess
import sys
import textwrap

import pytest

from tests.parity_util import check_figure

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "mact")

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs cuda"),
              pytest.mark.skipif(not os.path.isdir(REF), reason="baseline/_ref/mact not installed (DESIGN.md §8)")]


def _stub_source():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = doc[doc.index("## 2."):]
    m = re.search(r"```python\n(# mact/_b200.py.*?)```", sec, re.S)
    assert m, "INTEGRATION.md §2 has no mact/_b200.py block"
    return m.group(1)


DRIVER = textwrap.dedent("""
    import json, sys
    import numpy as np
    import mact, mact._b200 as B
    from mact import exact, fast, harness
    assert mact.__file__.startswith(sys.argv[1]), mact.__file__
    c1 = np.random.default_rng(0).integers(0, 256, size=(512, 512, 3), dtype=np.uint8).reshape(-1, 3)
    cfg = fast.DEFAULT_CONFIG
    out = {}
    for sp in ("lab", "hsi", "sct"):
        got = getattr(B, f"rgb_to_{sp}_fast")(c1, cfg)
        ref = getattr(fast, f"rgb_to_{sp}_fast")(c1, cfg)
        assert got.dtype == np.float32 and got.shape == ref.shape
        d = np.abs(got.astype(np.float64) - ref)
        if sp == "hsi":
            assert np.array_equal(np.isnan(got[:, 0]), np.isnan(ref[:, 0]))
            d[:, 0] = np.where(np.isnan(d[:, 0]), 0, np.minimum(d[:, 0], 2 * np.pi - d[:, 0])) / (2 * np.pi)
        if sp == "sct":
            assert np.array_equal(np.isnan(got[:, 2]), np.isnan(ref[:, 2]))
            d = np.nan_to_num(d / np.array([255 * np.sqrt(3), np.pi / 2, np.pi / 2]))
        out[sp] = float(d.max())
        exact64 = getattr(B, f"rgb_to_{sp}_fast")(c1, cfg, "float64")
        assert exact64.dtype == np.float64
        assert np.array_equal(exact64, ref, equal_nan=True), sp      # fidelity mode: bit for bit
    st = harness.measure_error("lab", lambda p: B.rgb_to_lab_fast(p, cfg), exact.rgb_to_lab_exact, population=c1)
    out["c1"] = {"avg": st.avg, "max": st.max, "count": st.count, "argmax_pixel": list(st.argmax_pixel)}
    print(json.dumps(out))
""")


def test_b200_stub_inside_the_reference(tmp_path, figures):
    from paper_1009_0854_b200 import _lib

    pkg = tmp_path / "mact"
    shutil.copytree(REF, pkg)
    (pkg / "_b200.py").write_text(_stub_source())
    (tmp_path / "drive.py").write_text(DRIVER)
    env = dict(os.environ, MACT_CUDA_LIB=str(_lib.LIB_PATH), PYTHONPATH=str(tmp_path))
    r = subprocess.run([sys.executable, str(tmp_path / "drive.py"), str(tmp_path)], env=env,
                       capture_output=True, text=True, timeout=600, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-3000:]
    import json

    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["lab"] <= 1e-4 and res["hsi"] <= 1e-5 and res["sct"] <= 1e-5, res
    ref = figures["c1_lab"]
    check_figure(res["c1"]["avg"], res["c1"]["max"], ref["avg"], ref["max"])
    assert res["c1"]["count"] == ref["count"] and res["c1"]["argmax_pixel"] == ref["argmax_pixel"]
