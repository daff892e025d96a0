"""Hot SASS instructions of one ncu report (source page, SASS view): top-N by
stall samples and instruction totals by opcode.

    python scripts/ncu_sass_hot.py report.ncu-rep [N]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {k: hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed")}
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        n = float(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    recs.append((r[ix["Address"]], r[ix["Source"]].strip(), s, n))
tot_s = sum(x[2] for x in recs) or 1
tot_n = sum(x[3] for x in recs) or 1
print(f"samples {tot_s:.0f}  warp-inst {tot_n:.3e}")
by_op = collections.Counter()
by_op_s = collections.Counter()
for a, src, s, n in recs:
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    by_op[op] += n
    by_op_s[op] += s
print("opcode          inst%   stall%")
for op, n in by_op.most_common(25):
    print(f"{op:14s} {100 * n / tot_n:6.2f} {100 * by_op_s[op] / tot_s:7.2f}")
print("--- top instructions by stall samples")
for a, src, s, n in sorted(recs, key=lambda x: -x[2])[:top]:
    print(f"{a:>6s} {100 * s / tot_s:5.2f}% n={n:.2e}  {src[:90]}")
