#!/bin/bash
# One GPU session: bench (ours + reference arm), launch list, ncu full capture of
# the bench's dominant kernel (traffic), all outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "bench=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref=$?"
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_bench.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches=$?"
$CMD > gpurun_out/plain_bench2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_ws" -s 3 -c 1 \
     -o gpurun_out/prof_bench_c4 -f $CMD > gpurun_out/ncu_bench_c4.log 2>&1; echo "ncu=$?"
