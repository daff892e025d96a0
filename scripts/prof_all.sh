#!/bin/bash
# ncu --set full of each streaming kernel (one launch each, 64 Mpx random input).
# Each command runs once plainly first (exit 0 required) before ncu.
set -e
mkdir -p gpurun_out
for spec in ${SPECS:-"probe" "lab" "hsi" "sct" "all" "lut17 --method tetrahedral" "lut17 --method trilinear"}; do
  tag=$(echo $spec | tr -d ' -' | sed 's/method//')
  python scripts/prof_kernel.py --op $spec --iters 1 > gpurun_out/plain_$tag.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"k_ws|k_stream|k_generic|k_err" -s 2 -c 1 \
      -o gpurun_out/prof_$tag -f python scripts/prof_kernel.py --op $spec --iters 1 > gpurun_out/ncu_$tag.log 2>&1
done
