#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_elem.py tests/test_gpu_reduce.py -m gpu -q -p no:cacheprovider -k "f64 or fidelity" > gpurun_out/pytest_f64.log 2>&1; echo "pytest=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_f64.log | tail -5
bash scripts/r02_evidence.sh
