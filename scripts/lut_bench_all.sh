#!/bin/bash
# all C3 LUT lines (17^3 default kernel, 33^3 with MACT_LUT33_KERNEL=${K33:-split}); optional lib tag as $1; TESTS=1 runs the LUT parity tests first
mkdir -p gpurun_out
lib=paper_1009_0854_b200/libmact_cuda${1:+_$1}.so
if [ -n "$TESTS" ]; then MACT_LIB=$lib timeout 1500 python -m pytest tests/test_gpu_exact_lut.py -x -q -m gpu 2>&1 | tail -4; fi
for g in 17 33; do for m in trilinear prism pyramidal tetrahedral; do
  MACT_LIB=$lib MACT_LUT33_KERNEL=${K33:-split} timeout 300 python bench.py --workload c3 --lut-grid $g --lut-method $m --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${1:-def}', $g, '$m', d['value'], d['roofline']['frac'], d['error']['dE_max'])"
done; done
