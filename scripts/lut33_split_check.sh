#!/bin/bash
# 33^3 split kernel: parity tests, then A/B against pair / comp on C3 (interleaved), planar timing via prof_kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact_lut.py -x -q -m gpu -k "lut33" 2>&1 | tail -5
for m in trilinear prism pyramidal tetrahedral; do
  for k in split; do
  MACT_LUT33_KERNEL=$k timeout 300 python bench.py --workload c3 --lut-grid 33 --lut-method $m --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', '$m', d['value'], d['roofline']['frac'], d['error']['dE_max'])"
  done
done
