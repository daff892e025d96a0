"""PPM P6 I/O and the thin CLI (SPEC.md:563-607 examples)."""

import csv

import numpy as np
import pytest

from paper_1009_0854_b200 import ppm
from tests.parity_util import check_figure
from paper_1009_0854_b200.__main__ import main as cli
from paper_1009_0854_b200.errors import MalformedHeader, TruncatedData, UnsupportedMaxval


def test_roundtrip_random(tmp_path):
    img = np.random.default_rng(16).integers(0, 256, (16, 16, 3), dtype=np.uint8)
    p = tmp_path / "a.ppm"
    ppm.write_ppm(p, img)
    np.testing.assert_array_equal(ppm.read_ppm(p), img)
    assert p.read_bytes()[:13] == b"P6\n16 16\n255\n"


def test_single_black_pixel_and_comments(tmp_path):
    p = tmp_path / "b.ppm"
    p.write_bytes(b"P6\n# a comment\n1 # width\n1\n255\n\x00\x00\x00")
    np.testing.assert_array_equal(ppm.read_ppm(p), np.zeros((1, 1, 3), np.uint8))


@pytest.mark.parametrize("data,exc", [
    (b"P6\n1 1\n65535\n" + b"\x00" * 6, UnsupportedMaxval),
    (b"P6\n2 2\n255\n" + b"\x00" * 11, TruncatedData),
    (b"P3\n1 1\n255\n0 0 0", MalformedHeader),
    (b"P6\n1 x\n255\n\x00\x00\x00", MalformedHeader),
    (b"P6\n1 1", MalformedHeader),
    (b"P6\n0 1\n255\n", MalformedHeader),
])
def test_errors(tmp_path, data, exc):
    p = tmp_path / "bad.ppm"
    p.write_bytes(data)
    with pytest.raises(exc):
        ppm.read_ppm(p)


def test_cli_flag_and_io_errors(tmp_path, capsys):
    assert cli(["convert"]) == 2                                  # missing flags
    assert cli(["bogus"]) == 2
    assert cli(["convert", str(tmp_path / "missing.ppm"), str(tmp_path / "o"), "--space", "hsi"]) == 3


@pytest.mark.gpu
def test_cli_convert_errors_probabilities(tmp_path, capsys, figures):
    src = tmp_path / "red.ppm"
    ppm.write_ppm(src, np.array([[[255, 0, 0]]], np.uint8))
    out = tmp_path / "red.f64"
    assert cli(["convert", str(src), str(out), "--space", "hsi", "--backend", "exact"]) == 0
    np.testing.assert_allclose(np.fromfile(out, "<f8"), [0.0, 1.0, 1.0 / 3.0], atol=1e-12)
    assert cli(["convert", str(src), str(out), "--space", "lab", "--backend", "lut:tetrahedral:17",
                "--format", "csv"]) == 0
    capsys.readouterr()
    assert cli(["errors", "--space", "cielab", "--backend", "mact", "--degrees", "4,4"]) == 0
    row = next(iter(csv.reader(capsys.readouterr().out.strip().splitlines()[1:])))
    ref = figures["cube"]["lab_44"]
    check_figure(float(row[3]), float(row[4]), ref["avg"], ref["max"], floor=1e-6)   # SPEC ~0.003201
    assert int(row[5]) == 1 << 24 and row[2] == "4,4"
    assert cli(["probabilities"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()[1:]
    got = {k: float(v) for k, v in (ln.split(",") for ln in lines)}
    assert got == {k: v["p"] for k, v in figures["call_probabilities"].items()}
    assert cli(["lut-build", str(tmp_path / "h.mlut"), "--space", "hsi", "--grid", "9"]) == 0
    ours = (tmp_path / "h.mlut").read_bytes()
    ref = (__import__("pathlib").Path(__file__).parent / "golden" / "ref_hsi9.mlut").read_bytes()
    assert ours[:20] == ref[:20] and len(ours) == len(ref)        # MLUT header + size
    np.testing.assert_allclose(np.frombuffer(ours[20:], "<f8"), np.frombuffer(ref[20:], "<f8"),
                               rtol=1e-12, atol=1e-12)             # GPU fp64 lattice vs numpy
