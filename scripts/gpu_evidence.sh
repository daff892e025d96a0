#!/bin/bash
# Full evidence pass on one B200 (run through gpurun): GPU tests, the default
# bench line (ours + reference arm), every BASELINE config, the ncu launch list
# of the bench command, one --set full capture of the bench's Lab kernel and of
# each other workload's kernel (DRAM traffic).  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -1 gpurun_out/pytest_gpu.log
bash scripts/gpu_bench_round.sh
bash scripts/bench_all_configs.sh; echo "configs=$?"
bash scripts/capture_traffic_all.sh
