#!/bin/bash
# Round-2 re-entry pass: full -m gpu suite, smoke, hazard check, default bench + reference arm,
# C4 launch list and one ncu --set full capture of the bench kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
bash scripts/r02_testall.sh
bash scripts/gpu_bench_round.sh
cat gpurun_out/bench_ours.json gpurun_out/bench_ref.json
