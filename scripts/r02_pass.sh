#!/bin/bash
# Round-2 GPU pass: 33^3 smoke, -m gpu tests (not slow first), smoke(), default bench, 33^3 A/B.
mkdir -p gpurun_out
timeout 300 python scripts/dbg_lut33.py all 4096 1000003 > gpurun_out/dbg_all.log 2>&1; echo "dbg=$?"; cat gpurun_out/dbg_all.log | tail -8
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "bench=$?"
timeout 900 bash scripts/lut33_ab.sh > /dev/null 2>&1; echo "ab=$?"
cat gpurun_out/lut33_ab.jsonl
