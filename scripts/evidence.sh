#!/bin/bash
# Round-2 evidence pass on one B200: every BASELINE config through bench.py (N=1),
# then one `ncu --set full` capture of each config's timed kernel (after its
# plain run exited 0), and the C4 launch list.  Outputs under gpurun_out/ev/.
set -u
O=gpurun_out/ev; R=/tmp/ev_reps; mkdir -p $O $R; : > $O/configs.jsonl
run() { timeout 900 python bench.py "$@" 2>>$O/configs.err | tail -1 >> $O/configs.jsonl; }
run --steps 50 --warmup 5
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>>$O/configs.err | tail -1 > $O/reference_arm.json
run --steps 20 --warmup 3 --out-dtype float64 --no-cpu-baseline
# the minimax rational itself evaluated in fp64 (MACT_LAB_EVAL=fp64) instead of the segmented fp32 cubic of it
MACT_LAB_EVAL=fp64 timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>>$O/configs.err | tail -1 > $O/c4_rational_fp64.json
run --workload c1 --steps 200 --warmup 10 --no-cpu-baseline
run --workload c2 --steps 50 --warmup 5 --no-cpu-baseline
for g in 17 33; do for m in trilinear prism pyramidal tetrahedral; do
  run --workload c3 --lut-grid $g --lut-method $m --steps 50 --warmup 5 --no-cpu-baseline; done; done
run --workload c5 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline
echo "configs: $(wc -l < $O/configs.jsonl) lines"
# ncu captures: name | kernel regex | bench args
cap() {
  local name=$1 rx=$2; shift 2
  local B="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-graph $*"
  $B > /dev/null 2>&1 || { echo "$name plain run failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 3 -c 1 -f -o $R/$name $B \
      > $O/$name.log 2>&1; echo "ncu $name=$?"
  # the reports (~22 MB each) stay on the box: raw metrics, summary and per-line profile come back
  ncu -i $R/$name.ncu-rep --page raw --csv > $O/$name.raw.csv 2>/dev/null
  python scripts/ncu_summary.py $R/$name.ncu-rep > $O/$name.summary.txt 2>&1
  python scripts/ncu_lines.py $R/$name.ncu-rep 30 > $O/$name.lines.txt 2>&1
}
cap c4 "k_ws"
cap c4_f64 "k_fast_ref" --out-dtype float64
cap c1 "k_ws" --workload c1
cap c2 "k_ws" --workload c2
cap c5 "k_ws" --workload c5
for m in trilinear prism pyramidal tetrahedral; do cap c3_17_$m "k_ws" --workload c3 --lut-grid 17 --lut-method $m; done
for m in trilinear prism pyramidal tetrahedral; do cap c3_33_$m "k_lut33" --workload c3 --lut-grid 33 --lut-method $m; done
# C4 launch list (per-launch durations, cold, serialised)
B="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c4_launches.csv $B > $O/c4_launches.log 2>&1; echo "launches=$?"
