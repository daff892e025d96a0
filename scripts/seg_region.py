"""Opcode histogram of the SASS between the tile wait (TRYWAIT) and the first
STS.128 of a k_ws kernel: the per-tile-group hot path of the first layout
block.  MACT_LIB=... python scripts/seg_region.py NAME_SUBSTRING"""
import collections, os, re, subprocess, sys
name = sys.argv[1]
lib = os.environ.get("MACT_LIB", "paper_1009_0854_b200/libmact_cuda.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", out)[1:]:
    fn = f.split("\n", 1)[0]
    if "k_ws" not in fn or name not in fn:
        continue
    lines = f.split("\n")
    i0 = next(i for i, l in enumerate(lines) if "TRYWAIT" in l)
    i1 = next(i for i, l in enumerate(lines) if "STS.128" in l and i > i0)
    ops = [m.group(1) for l in lines[i0:i1] for m in [re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(?:\.[A-Z0-9]+)?)", l)] if m]
    c = collections.Counter(ops)
    print(fn[:80], len(ops), "instr")
    print("  " + "  ".join(f"{k}:{v}" for k, v in c.most_common(40)))
    if len(sys.argv) > 2:
        print("\n".join(lines[i0:i1]))
