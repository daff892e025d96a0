#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_reference_seam.py tests/test_gpu_fast.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_p2.log 2>&1; echo "pytest=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_p2.log | tail -5
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench=$?"
timeout 600 python bench.py --steps 20 --warmup 3 --out-dtype float64 --no-cpu-baseline > gpurun_out/bench_c4_f64.json 2> gpurun_out/bench_c4_f64.err; echo "bench64=$?"
cat gpurun_out/bench_c4.json gpurun_out/bench_c4_f64.json
bash scripts/hazard_check.sh
