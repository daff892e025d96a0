#!/bin/bash
# scripts/gpu_evidence.sh plus the summaries made ON the box (scripts/save_evidence.sh),
# so only small files come back: gpurun_out/profiles/ holds the new profiles/ files;
# the .ncu-rep files stay on the box except the C4 one.
bash scripts/gpu_evidence.sh
python scripts/c4_oracle_eps.py > gpurun_out/c4eps.txt 2>&1
python scripts/precision.py lab > gpurun_out/precision.txt 2>&1
bash scripts/sweep_gain.sh > gpurun_out/gain.txt 2>&1
bash scripts/save_evidence.sh
python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.txt 2>&1
for m in trilinear prism pyramidal tetrahedral; do
  timeout 600 ncu --set full --clock-control none -k regex:"k_ws" -s 2 -c 1 -o gpurun_out/prof_lut17_$m -f \
    python scripts/prof_kernel.py --op lut17 --method $m --iters 1 > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_lut17_$m.ncu-rep >> gpurun_out/lut17_ncu_summary.txt
done
mkdir -p gpurun_out/profiles && cp profiles/* gpurun_out/profiles/
find gpurun_out -name "*.ncu-rep" ! -name "prof_bench_c4.ncu-rep" -delete
du -sh gpurun_out
