#!/bin/bash
mkdir -p gpurun_out
MACT_LUT33_KERNEL=pair timeout 300 python scripts/dbg_lut33.py all 4096 1000003 > gpurun_out/dbg_p33.log 2>&1; echo "dbg=$?"; tail -8 gpurun_out/dbg_p33.log
timeout 900 python -m pytest tests/test_gpu_exact_lut.py -m gpu -q -p no:cacheprovider -k "33" > gpurun_out/pytest_p33.log 2>&1; echo "pytest=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_p33.log | tail -5
for t in def nw16 nw20; do for m in trilinear tetrahedral; do
  MACT_LUT33_KERNEL=pair MACT_LIB=paper_1009_0854_b200/libmact_cuda$([ $t = def ] || echo _$t).so timeout 300 python bench.py --workload c3 --lut-grid 33 --lut-method $m --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '$m', d['value'], d['roofline']['frac'], d['error']['dE_max'])"
done; done
