"""Per-kernel SASS opcode histogram of libmact_cuda.so (cuobjdump -sass).

    python scripts/sass_stats.py [substring-filter] [--top N]
"""
import collections
import re
import subprocess
import sys

lib = "paper_1009_0854_b200/libmact_cuda.so"
flt = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else ""
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)[1:]
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if flt not in name:
        continue
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f)
    c = collections.Counter(ops)
    print(f"== {name}  ({len(ops)} instr)")
    print("   " + "  ".join(f"{k}:{v}" for k, v in c.most_common(top)))
