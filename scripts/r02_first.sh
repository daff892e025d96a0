#!/bin/bash
# Round-2 first GPU pass: -m gpu tests, smoke, default bench + reference arm, 33^3 A/B.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 600 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "bench=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref=$?"
timeout 900 bash scripts/lut33_ab.sh > /dev/null 2>&1; echo "ab=$?"
cat gpurun_out/bench_ours.json gpurun_out/bench_ref.json gpurun_out/lut33_ab.jsonl
