#!/bin/bash
# Copies the outputs of scripts/gpu_evidence.sh (gpurun_out/) into profiles/ (runs here, no GPU).
set -e
tail -1 gpurun_out/bench_ours.json > profiles/r01_bench_c4.json
tail -1 gpurun_out/bench_ref.json > profiles/r01_bench_c4_reference_arm.json
cp gpurun_out/configs.jsonl profiles/r01_bench_configs.jsonl
cp gpurun_out/launches.csv profiles/r01_bench_c4_launches.csv
for w in c4 c1 c2 c3 c5; do python scripts/capture_traffic.py gpurun_out/prof_bench_$w.ncu-rep $w > /dev/null; done
(echo "# R01: ncu --set full --clock-control none of the bench's C4 Lab kernel (scripts/gpu_bench_round.sh)"
 python scripts/ncu_summary.py gpurun_out/prof_bench_c4.ncu-rep) > profiles/r01_ncu_bench_c4_summary.txt
python scripts/ncu_details.py gpurun_out/prof_bench_c4.ncu-rep > profiles/r01_ncu_bench_c4_details.csv
(echo "# R01: ncu --set full of the C1/C2/C3/C5 bench kernels (scripts/capture_traffic_all.sh)"
 for w in c1 c2 c3 c5; do python scripts/ncu_summary.py gpurun_out/prof_bench_$w.ncu-rep; done) > profiles/r01_ncu_bench_other_configs_summary.txt
[ -f gpurun_out/precision.txt ] && cp gpurun_out/precision.txt profiles/r01_precision_full_cube.txt
[ -f gpurun_out/gain.txt ] && cp gpurun_out/gain.txt profiles/r01_table4_gain.txt
[ -f gpurun_out/c4eps.txt ] && tail -1 gpurun_out/c4eps.txt > profiles/r01_c4_c5_error_figures.json
echo saved
