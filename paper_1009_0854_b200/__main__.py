"""Thin command-line front end over the GPU path (declared but
absent in the reference, pyproject.toml:18-19).  Only the subcommands that
drive the hot path are provided:

    convert        PPM -> destination space via exact | mact | lut:<method>:<grid>
    errors         eps_avg / eps_max of a backend over the cube or a PPM (CSV)
    probabilities  full-cube call-site frequencies (harness.call_probabilities)
    lut-build      build a lattice and write it in the MLUT format

Exit codes follow SPEC.md: 0 ok, 2 flag errors, 3 I/O errors, 4 numerical errors.
Outputs: binary little-endian float64 triples (``--format binary-f64``) or CSV.
"""

from __future__ import annotations

import argparse
import csv
import sys

import numpy as np

SPACES = {"cielab": "lab", "lab": "lab", "hsi": "hsi", "sct": "sct"}


def _backend(spec: str, space: str, degrees):
    from . import exact, fast, lut

    if spec == "exact":
        return getattr(exact, f"rgb_to_{space}_exact")
    if spec == "mact":
        kw = {}
        if degrees:
            d = tuple(int(x) for x in degrees.split(","))
            kw = {"lab": {"cielab_degrees": d}, "hsi": {"hsi_degree": d[0]},
                  "sct": {"sct_degrees": d}}[space]
        cfg = fast.MactConfig(**kw)
        fn = getattr(fast, f"rgb_to_{space}_fast")
        return lambda p: fn(p, cfg)
    if spec.startswith("lut:"):
        _, method, grid = spec.split(":")
        table = lut.build_lut(space, int(grid))
        return lambda p: lut.interpolate(table, p, method)
    raise ValueError(f"unknown backend {spec!r}")


def _emit(arr: np.ndarray, path: str, fmt: str) -> None:
    a = np.asarray(arr, dtype=np.float64).reshape(-1, 3)
    if fmt == "binary-f64":
        a.astype("<f8").tofile(path)
    else:
        np.savetxt(path, a, delimiter=",", fmt="%.17g")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1009_0854_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("convert")
    c.add_argument("input")
    c.add_argument("output")
    c.add_argument("--space", required=True, choices=sorted(SPACES))
    c.add_argument("--backend", default="mact")
    c.add_argument("--degrees")
    c.add_argument("--format", default="binary-f64", choices=["binary-f64", "csv"])
    e = sub.add_parser("errors")
    e.add_argument("--space", required=True, choices=sorted(SPACES))
    e.add_argument("--backend", default="mact")
    e.add_argument("--degrees")
    e.add_argument("--population", default="cube", help="'cube' or a PPM path")
    e.add_argument("--format", default="csv", choices=["csv", "markdown"])
    sub.add_parser("probabilities")
    lb = sub.add_parser("lut-build")
    lb.add_argument("output")
    lb.add_argument("--space", required=True, choices=sorted(SPACES))
    lb.add_argument("--grid", type=int, required=True)
    try:
        args = ap.parse_args(argv)
    except SystemExit as ex:
        return 0 if ex.code == 0 else 2

    from . import exact, harness, lut, ppm
    from .errors import MactError, PpmError, UnknownApproximant

    try:
        if args.cmd == "convert":
            space = SPACES[args.space]
            img = ppm.read_ppm(args.input)
            _emit(_backend(args.backend, space, args.degrees)(img), args.output, args.format)
        elif args.cmd == "errors":
            space = SPACES[args.space]
            pop = None if args.population == "cube" else ppm.read_ppm(args.population).reshape(-1, 3)
            ref = getattr(exact, f"rgb_to_{space}_exact")
            s = harness.measure_error(space, _backend(args.backend, space, args.degrees), ref, pop)
            row = [args.space, args.backend, args.degrees or "default", f"{s.avg:.10g}",
                   f"{s.max:.10g}", str(s.count), "(%d,%d,%d)" % s.argmax_pixel]
            if args.format == "csv":
                w = csv.writer(sys.stdout, lineterminator="\n")
                w.writerow(["space", "backend", "degrees", "eps_avg", "eps_max", "count", "argmax_pixel"])
                w.writerow(row)
            else:
                print("| space | backend | degrees | eps_avg | eps_max | count | argmax |")
                print("|---|---|---|---|---|---|---|")
                print("| " + " | ".join(row) + " |")
        elif args.cmd == "probabilities":
            p = harness.call_probabilities()
            print("call_site,probability")
            for k in ("cbrt_x", "cbrt_y", "cbrt_z", "arcsin", "arccos", "arctan"):
                print(f"{k},{getattr(p, k)!r}")
        elif args.cmd == "lut-build":
            if args.grid not in (9, 17, 33):
                raise ValueError("grid must be one of 9, 17, 33")
            lut.save_lut(lut.build_lut(SPACES[args.space], args.grid), args.output)
    except (ValueError, KeyError, UnknownApproximant) as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 2
    except (OSError, PpmError) as ex:
        print(f"I/O error: {ex}", file=sys.stderr)
        return 3
    except MactError as ex:
        print(f"numerical error: {ex}", file=sys.stderr)
        return 4
    return 0


if __name__ == "__main__":
    sys.exit(main())
