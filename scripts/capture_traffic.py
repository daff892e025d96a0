"""Turn an ncu --set full capture of bench.py's dominant kernel into
profiles/traffic.json (dram__bytes_read.sum + dram__bytes_write.sum per launch),
which bench.py reports as roofline.traffic.

    python scripts/capture_traffic.py gpurun_out/prof_bench_c4.ncu-rep c4 [commit]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

rep, workload = sys.argv[1], sys.argv[2]
d = load(rep)[0]
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[workload] = {"bytes_per_launch": d["dram_rd"] + d["dram_wr"], "dram_read": d["dram_rd"],
                  "dram_write": d["dram_wr"], "kernel": d["name"], "duration_ns_under_ncu": d["dur"],
                  "source": os.path.basename(rep)}
if len(sys.argv) > 3:
    data[workload]["commit"] = sys.argv[3]
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[workload]))
