#!/bin/bash
# ncu --set full of each workload's dominant kernel (bench.py command, run plainly first);
# reports land in gpurun_out/prof_bench_<wl>.ncu-rep for scripts/capture_traffic.py
for wl in c1 c2 c3 c5; do
  CMD="python bench.py --workload $wl --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-graph"
  $CMD > gpurun_out/plain_$wl.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none -k regex:"k_ws|k_lut33" -s 3 -c 1 \
      -o gpurun_out/prof_bench_$wl -f $CMD > gpurun_out/ncu_$wl.log 2>&1; echo "$wl=$?"
done
