#!/bin/bash
# 17^3 trilinear pair-node path: parity tests + C3 A/B against the previous build (libmact_cuda_prev.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact_lut.py -m gpu -q -p no:cacheprovider -k "17 or unaligned or planar or nonfinite or wide" > gpurun_out/pytest_tri17.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|max \|dLab\|" gpurun_out/pytest_tri17.log | tail -8
timeout 900 python -m pytest tests/test_gpu_exact_lut.py -m gpu -q -s -p no:cacheprovider -k "full_cube and 17 and interp" > gpurun_out/pytest_tri17_cube.log 2>&1; echo "cube=$?"
grep -E "FAILED|passed|failed|max \|dLab\|" gpurun_out/pytest_tri17_cube.log | tail -8
bash scripts/lut_ab.sh "17" "trilinear" "def prev"
