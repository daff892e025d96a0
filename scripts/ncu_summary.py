"""Summarise ncu reports (raw page) into one table: duration, DRAM bytes and
throughput, issue activity, pipe utilisation, occupancy, top stall reasons.

    python scripts/ncu_summary.py gpurun_out/prof_*.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_conflicts",
}
UNIT = {"dur": 1.0}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"name": vals[hdr.index("Kernel Name")][:60]}
        for k, short in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                u = units[i]
                if short == "dur" and u == "us":
                    v = v * 1e3
                if short == "dur" and u == "ms":
                    v = v * 1e6
                if short.startswith("dram_") and short != "dram_pct":
                    v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                d[short] = v
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(vals[i] or 0)
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
        tot = sum(stalls.values()) or 1
        d["stalls"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        res.append(d)
    return res


def main():
    paths = [a for a in sys.argv[1:] if a.endswith(".ncu-rep")]
    allres = {}
    for p in paths:
        for d in load(p):
            allres[p] = d
            print(f"== {p}: {d['name']}")
            print("   dur {:.1f} us  dram rd {:.1f} MB wr {:.1f} MB ({:.1f}% peak)  issue {:.1f}%  warps {:.1f}%  regs {}".format(
                d.get("dur", 0) / 1e3, d.get("dram_rd", 0) / 1e6, d.get("dram_wr", 0) / 1e6, d.get("dram_pct", 0),
                d.get("issue_pct", 0), d.get("warps_pct", 0), d.get("regs")))
            print("   pipes fp64 {fp64_pct} fma {fma_pct} alu {alu_pct} xu {xu_pct} lsu {lsu_pct}  warp-inst {warp_inst:.3g}  smem-conflicts {smem_conflicts}".format(**{k: d.get(k) for k in KEYS.values()}))
            print("   stalls", d["stalls"])
    if "--json" in sys.argv:
        json.dump(allres, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
