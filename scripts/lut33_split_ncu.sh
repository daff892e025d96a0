#!/bin/bash
# ncu --set full of the split kernel (tet + tri) and build-variant A/B: bash scripts/lut33_split_ncu.sh [tags...]
mkdir -p gpurun_out /tmp/reps
export MACT_LUT33_KERNEL=split
for m in tetrahedral trilinear; do
  B="python bench.py --workload c3 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-graph --lut-grid 33 --lut-method $m"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_lut33_split" -s 3 -c 1 -f -o /tmp/reps/s33_$m $B > gpurun_out/s33_$m.log 2>&1; echo "ncu $m=$?"
  python scripts/ncu_summary.py /tmp/reps/s33_$m.ncu-rep > gpurun_out/s33_$m.summary.txt 2>&1
  python scripts/ncu_lines.py /tmp/reps/s33_$m.ncu-rep 40 > gpurun_out/s33_$m.lines.txt 2>&1
  python scripts/ncu_sass_hot.py /tmp/reps/s33_$m.ncu-rep > gpurun_out/s33_$m.sass.txt 2>&1
done
for t in "$@"; do
  for m in trilinear tetrahedral; do
  MACT_LIB=paper_1009_0854_b200/libmact_cuda_$t.so timeout 300 python bench.py --workload c3 --lut-grid 33 --lut-method $m --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '$m', d['value'], d['roofline']['frac'], d['error']['dE_max'])"
  done
done
