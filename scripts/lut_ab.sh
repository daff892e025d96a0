#!/bin/bash
# LUT A/B on C3 (4096^2 random px): bash scripts/lut_ab.sh "<grid>" "<methods>" "<lib tags>" [env for tag 'comp']
# tag "" = default libmact_cuda.so; tag comp = default lib with MACT_LUT33_KERNEL=comp
mkdir -p gpurun_out; OUT=gpurun_out/lut_ab.jsonl; : > $OUT
for g in $1; do for m in $2; do for t in $3; do
  lib=paper_1009_0854_b200/libmact_cuda.so; ev=""
  if [ "$t" = comp ]; then ev="MACT_LUT33_KERNEL=comp"; elif [ "$t" != def ]; then lib=paper_1009_0854_b200/libmact_cuda_$t.so; fi
  env $ev MACT_LIB=$lib timeout 300 python bench.py --workload c3 --lut-grid $g --lut-method $m --steps 50 --warmup 5 \
      --no-cpu-baseline --e2e-steps 0 2>>gpurun_out/lut_ab.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'tag':'$t','grid':$g,'method':'$m','gpix':d['value'],'frac':d['roofline']['frac'],'dE_max':d['error']['dE_max'],'sm_mhz':d['clocks']['sm_mhz']}))" >> $OUT
done; done; done
cat $OUT
