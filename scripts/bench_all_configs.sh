#!/bin/bash
# Every BASELINE config through bench.py (N=1), one JSON line each -> gpurun_out/configs.jsonl
mkdir -p gpurun_out; : > gpurun_out/configs.jsonl
run() { timeout 900 python bench.py "$@" 2>>gpurun_out/configs.err | tail -1 >> gpurun_out/configs.jsonl; }
run --workload c1 --steps 200 --warmup 10 --no-cpu-baseline
run --workload c2 --steps 50 --warmup 5 --no-cpu-baseline
for g in 17 33; do for m in trilinear prism pyramidal tetrahedral; do
  run --workload c3 --lut-grid $g --lut-method $m --steps 50 --warmup 5 --no-cpu-baseline; done; done
run --workload c5 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline
