"""CPU-side checks of the C ABI: the library builds/loads without a GPU, exports
every symbol include/mact_cuda.h declares, and the ctypes structs match the C
layout (checked by compiling the header with gcc)."""

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mact_cuda.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1009_0854_b200 import _lib, build
    if not _lib.LIB_PATH.exists():
        build.build()
    return _lib.load()


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mact_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    from paper_1009_0854_b200 import _lib
    names = header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), f"libmact_cuda.so does not export {n}"
    assert set(names) == set(_lib.EXPORTS), "ctypes signature table out of sync with the header"


def test_version_and_counters_without_gpu(lib):
    assert lib.mact_version() == 100
    lib.mact_launch_count_reset()
    assert lib.mact_launch_count() == 0


def test_struct_layout_matches_c(tmp_path):
    from paper_1009_0854_b200 import _lib
    import ctypes as C
    src = tmp_path / "layout.c"
    src.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "mact_cuda.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(MactCoeffs), offsetof(MactCoeffs, atan_g),
         sizeof(MactErrStats), sizeof(MactErrSpec), offsetof(MactErrSpec, ref_array),
         offsetof(MactErrSpec, ref_dtype), sizeof(MactApproxSpec), offsetof(MactApproxSpec, b));
  return 0;
}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()))
    assert vals == [C.sizeof(_lib.MactCoeffs), _lib.MactCoeffs.atan_g.offset,
                    C.sizeof(_lib.MactErrStats), C.sizeof(_lib.MactErrSpec),
                    _lib.MactErrSpec.ref_array.offset, _lib.MactErrSpec.ref_dtype.offset,
                    C.sizeof(_lib.MactApproxSpec), _lib.MactApproxSpec.b.offset]


def test_bad_arguments_fail_without_touching_the_device(lib):
    from paper_1009_0854_b200 import _lib
    from paper_1009_0854_b200.errors import UnknownApproximant
    with pytest.raises(ValueError):
        _lib.call("mact_lut_build", 0, 16, None, None, None)
    with pytest.raises(ValueError):
        _lib.call("mact_exact", 7, None, 0, None, 2, 1, None)
    c = _lib.MactCoeffs()
    c.cbrt_num_deg = c.cbrt_den_deg = 9
    c.hsi_deg = 5
    c.asin_deg = c.acos_deg = c.atan_deg = 5
    with pytest.raises(UnknownApproximant):
        _lib.call("mact_lab_fast", None, 0, None, 0, C_ptr(c), 0, None)


def C_ptr(c):
    import ctypes as C
    return C.pointer(c)


def test_product_never_imports_oracle():
    """The product package must not reach the CPU oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1009_0854_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*", "", txt).replace('"""', ""), f


def test_gamma_table_header_is_current():
    """csrc/mact_gamma_table.inc == fp32(oracle GAMMA_TABLE) (regenerate with scripts/gen_gamma_table.py)."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("gen", os.path.join(root, "scripts", "gen_gamma_table.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    for bits, name in gen.FILES.items():
        with open(os.path.join(root, "paper_1009_0854_b200", "csrc", name)) as fh:
            assert fh.read() == gen.render(bits), name


def test_plain_c_client_links_and_gets_status_codes(tmp_path, lib):
    """A C program (no Python, no torch) links libmact_cuda.so through the header
    alone and gets the documented status codes for argument errors, which are
    decided before any CUDA call (so this runs without a GPU)."""
    from paper_1009_0854_b200 import _lib
    src = tmp_path / "client.c"
    src.write_text(r'''
#include <stdio.h>
#include <string.h>
#include "mact_cuda.h"
int main(void) {
  MactCoeffs c; memset(&c, 0, sizeof c);
  c.cbrt_num_deg = 4; c.cbrt_den_deg = 4; c.hsi_deg = 5; c.asin_deg = 5; c.acos_deg = 5; c.atan_deg = 5;
  int ok = 1;
  ok &= mact_version() == 100;
  ok &= mact_lab_fast(NULL, MACT_DTYPE_U8, NULL, -1, &c, MACT_LAYOUT_INTERLEAVED, NULL) == MACT_EBADARG;
  ok &= strlen(mact_last_error()) > 0;
  ok &= mact_lab_fast(NULL, MACT_DTYPE_U8, NULL, 0, &c, 7, NULL) == MACT_EBADARG;        /* bad layout */
  c.cbrt_num_deg = 5;                                                                   /* no such set */
  ok &= mact_hsi_fast(NULL, MACT_DTYPE_U8, NULL, 0, &c, MACT_LAYOUT_INTERLEAVED, NULL) == MACT_EUNKNOWN_APPROX;
  ok &= mact_lut_interp(NULL, 17, MACT_LUT_TETRAHEDRAL, NULL, NULL, 0, 0, NULL) == MACT_OK;  /* n = 0: no-op */
  ok &= mact_lut_interp(NULL, 17, 9, NULL, NULL, 0, 0, NULL) == MACT_EBADARG;          /* unknown method */
  ok &= mact_exact(5, NULL, MACT_DTYPE_U8, NULL, MACT_DTYPE_F64, 0, NULL) == MACT_EBADARG;
  printf("%s\n", ok ? "ok" : "FAIL");
  return ok ? 0 : 1;
}
''')
    exe = tmp_path / "client"
    libdir = str(_lib.LIB_PATH.parent)
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                    "-L", libdir, "-l:" + _lib.LIB_PATH.name, "-Wl,-rpath," + libdir], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr


def test_lab_eval_path_segmented_for_every_registry_rational(lib):
    """Host-only: the segmented fp32 lightness kernel is fitted for
    every bundled CIELAB rational (approximants.py:179-211) and passes the
    host-side 1e-8 fit check, so no configuration falls back to fp64."""
    from paper_1009_0854_b200 import _lib, fast
    from oracle import mact_oracle as O
    for degs in O.CBRT_RATIONALS:
        cfg = fast.MactConfig(cielab_degrees=degs)
        assert lib.mact_lab_eval_path(C.byref(cfg._pack())) == _lib.LAB_PATH_SEG, degs


def test_lab_eval_path_env_switch(lib, monkeypatch):
    """MACT_LAB_EVAL=fp64 selects the fp64 evaluation (host-only query)."""
    from paper_1009_0854_b200 import _lib, fast
    monkeypatch.setenv("MACT_LAB_EVAL", "fp64")
    assert lib.mact_lab_eval_path(C.byref(fast.DEFAULT_CONFIG._pack())) == _lib.LAB_PATH_MONIC
    monkeypatch.delenv("MACT_LAB_EVAL")
    assert lib.mact_lab_eval_path(C.byref(fast.DEFAULT_CONFIG._pack())) == _lib.LAB_PATH_SEG


def test_integration_stub_binds_only_exported_symbols(lib):
    """INTEGRATION.md §2's mact/_b200.py (run inside the real reference by
    test_gpu_reference_seam.py) is valid Python and calls only symbols the library exports."""
    import ast

    from tests.test_gpu_reference_seam import _stub_source

    src = _stub_source()
    ast.parse(src)
    used = set(re.findall(r"_lib\.(mact_\w+)", src))
    assert {"mact_transform_host", "mact_host_ctx_create", "mact_last_error"} <= used
    for name in used:
        assert hasattr(lib, name), name
