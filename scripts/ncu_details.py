"""Key 'details' page rows of an ncu report as a small CSV (section, metric, unit, value)."""
import csv
import io
import subprocess
import sys

KEEP = {"Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Dynamic Shared Memory Per Block", "Executed Ipc Active",
        "Issue Slots Busy", "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "SM Frequency", "DRAM Frequency",
        "Block Size", "Grid Size", "Waves Per SM", "Executed Instructions", "L1/TEX Hit Rate"}
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
si, mi, ui, vi = (hdr.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
w = csv.writer(sys.stdout)
w.writerow(["section", "metric", "unit", "value"])
for r in rows[1:]:
    if len(r) > vi and r[mi] in KEEP:
        w.writerow([r[si], r[mi], r[ui], r[vi]])
