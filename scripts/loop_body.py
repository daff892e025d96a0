"""Opcode histogram of the main tile loop of a k_stream kernel (between the
mbarrier TRYWAIT and the bulk-store issue).  python scripts/loop_body.py OpLab"""
import collections, os, re, subprocess, sys
name = sys.argv[1]
out = subprocess.run(["cuobjdump", "-sass", os.environ.get("MACT_LIB", "paper_1009_0854_b200/libmact_cuda.so")], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", out)[1:]:
    fn = f.split("\n", 1)[0]
    if "k_ws" not in fn or name not in fn:
        continue
    lines = f.split("\n")
    i0 = next(i for i, l in enumerate(lines) if "TRYWAIT" in l)
    i1 = next(i for i, l in enumerate(lines) if "UBLKCP.G.S" in l)
    ops = [m.group(1) for l in lines[i0:i1] for m in [re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", l)] if m]
    c = collections.Counter(ops)
    print(fn[:80], len(ops), "instr")
    print("  " + "  ".join(f"{k}:{v}" for k, v in c.most_common(30)))
