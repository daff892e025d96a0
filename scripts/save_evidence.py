"""Copy the outputs of scripts/evidence.sh (gpurun_out/ev/) into profiles/ (runs here, no GPU):
bench lines, ncu summaries, per-line profiles, the C4 launch list, and profiles/traffic.json
(ncu DRAM bytes per launch of every config's timed kernel, with the capture commit).

    python scripts/save_evidence.py <commit>
"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EV = os.path.join(ROOT, "gpurun_out", "ev")
PR = os.path.join(ROOT, "profiles")
commit = sys.argv[1]


def raw(name):
    """First kernel row of an `ncu --page raw --csv` dump as {metric: (value, unit)}."""
    rows = list(csv.reader(open(os.path.join(EV, name + ".raw.csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v.replace(",", ""), u) for h, u, v in zip(hdr, units, vals)}


def to_bytes(vu):
    v, u = float(vu[0]), vu[1].lower()
    return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}[u]


def to_ns(vu):
    v, u = float(vu[0]), vu[1].lower()
    return v * {"ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "usecond": 1e3, "msecond": 1e6, "nsecond": 1, "second": 1e9}[u]


names = ["c4", "c4_f64", "c1", "c2", "c5"] + [f"c3_{g}_{m}" for g in (17, 33)
                                               for m in ("trilinear", "prism", "pyramidal", "tetrahedral")]
tpath = os.path.join(PR, "traffic.json")
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
summ = [f"# R02 (commit {commit}): ncu --set full --clock-control none of every config's timed kernel "
        "(scripts/evidence.sh)"]
lines = []
for n in names:
    if not os.path.exists(os.path.join(EV, n + ".raw.csv")):
        print("missing", n)
        continue
    r = raw(n)
    rd, wr = to_bytes(r["dram__bytes_read.sum"]), to_bytes(r["dram__bytes_write.sum"])
    traffic[n] = {"bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                  "kernel": r["Kernel Name"][0][:60], "duration_ns_under_ncu": to_ns(r["gpu__time_duration.sum"]),
                  "source": f"gpurun_out/ev/{n}.raw.csv (scripts/evidence.sh)", "commit": commit}
    summ.append(f"## {n}")
    summ.append(open(os.path.join(EV, n + ".summary.txt")).read().rstrip())
    lines.append(f"## {n}")
    lines.append(open(os.path.join(EV, n + ".lines.txt")).read().rstrip())
traffic.pop("c3", None)
json.dump(traffic, open(tpath, "w"), indent=1)
open(os.path.join(PR, "r02_ncu_configs_summary.txt"), "w").write("\n".join(summ) + "\n")
open(os.path.join(PR, "r02_ncu_configs_hot_lines.txt"), "w").write("\n".join(lines) + "\n")
shutil.copy(os.path.join(EV, "configs.jsonl"), os.path.join(PR, "r02_bench_configs.jsonl"))
shutil.copy(os.path.join(EV, "c4_launches.csv"), os.path.join(PR, "r02_bench_c4_launches.csv"))
shutil.copy(os.path.join(EV, "c4.raw.csv"), os.path.join(PR, "r02_ncu_bench_c4_details.csv"))
open(os.path.join(PR, "r02_bench_c4.json"), "w").write(open(os.path.join(EV, "configs.jsonl")).readline())
if os.path.exists(os.path.join(EV, "reference_arm.json")):
    shutil.copy(os.path.join(EV, "reference_arm.json"), os.path.join(PR, "r02_bench_c4_reference_arm.json"))
hz = os.path.join(ROOT, "gpurun_out", "hazard", "summary.txt")
if os.path.exists(hz):
    shutil.copy(hz, os.path.join(PR, "r02_hazard_check.txt"))
print("saved", len(names), "configs at", commit)
