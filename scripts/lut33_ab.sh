#!/bin/bash
# 33^3 A/B: r-split pair kernel (default) vs the R01 component-split kernels (MACT_LUT33_KERNEL=comp),
# C3 (4096^2 random) bench lines -> gpurun_out/lut33_ab.jsonl
mkdir -p gpurun_out; : > gpurun_out/lut33_ab.jsonl
for m in trilinear prism pyramidal tetrahedral; do
  for k in pair comp; do
    if [ $k = comp ]; then export MACT_LUT33_KERNEL=comp; else unset MACT_LUT33_KERNEL; fi
    timeout 600 python bench.py --workload c3 --lut-grid 33 --lut-method $m --steps 50 --warmup 5 \
      --no-cpu-baseline --e2e-steps 0 2>>gpurun_out/lut33_ab.err | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'kernel':'$k','method':'$m','gpix':d['value'],'frac':d['roofline']['frac'],'err':d['error']}))" >> gpurun_out/lut33_ab.jsonl
  done
done
unset MACT_LUT33_KERNEL
cat gpurun_out/lut33_ab.jsonl
