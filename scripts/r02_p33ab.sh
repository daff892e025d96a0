#!/bin/bash
for k in pair comp; do for m in trilinear prism pyramidal tetrahedral; do
  MACT_LUT33_KERNEL=$k timeout 300 python bench.py --workload c3 --lut-grid 33 --lut-method $m --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', '$m', d['value'], d['roofline']['frac'], d['error']['dE_max'])"
done; done
