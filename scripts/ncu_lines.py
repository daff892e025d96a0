"""Per-CUDA-source-line totals (warp instructions executed, stall samples) of one
ncu report, from the source page's cuda,sass view.

    python scripts/ncu_lines.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, recs = "?", []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "" or len(r) < 8:
        continue
    try:
        s, n = float(r[4]), float(r[7])
    except ValueError:
        continue
    recs.append((f"{fname}:{r[0]}", r[1].strip()[:80], s, n))
ts = sum(x[2] for x in recs) or 1
tn = sum(x[3] for x in recs) or 1
print(f"stall samples {ts:.0f}, warp-inst {tn:.3e}")
print("--- by instructions")
for k, src, s, n in sorted(recs, key=lambda x: -x[3])[:top]:
    print(f"{k:22s} inst {100 * n / tn:5.2f}%  stall {100 * s / ts:5.2f}%  {src}")
print("--- by stall samples")
for k, src, s, n in sorted(recs, key=lambda x: -x[2])[:top // 2]:
    print(f"{k:22s} inst {100 * n / tn:5.2f}%  stall {100 * s / ts:5.2f}%  {src}")
