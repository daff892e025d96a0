"""Dynamic opcode mix of one kernel from an ncu report's source page (SASS),
in thread-instructions per unit of work.  python scripts/op_mix.py REPORT UNITS [TOP]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
c = collections.Counter()
tot = 0.0
for r in rows[2:]:
    m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", r[isrc])
    if not m:
        continue
    n = float(r[iex] or 0) * 32 / units
    tot += n
    c[m.group(1) + (m.group(2) or "")[:12]] += n
print(f"thread-instructions per unit: {tot:.1f}")
for k, v in c.most_common(top):
    print(f"  {k:26s} {v:7.2f}")
