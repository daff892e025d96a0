#!/bin/bash
# ncu --set full of every streaming kernel family at 64 Mpx (R01 evidence), each
# command run plainly first (exit 0) before profiling.
set -e
mkdir -p gpurun_out
run() {  # tag, args...
  tag=$1; shift
  python scripts/prof_kernel.py "$@" --iters 1 > gpurun_out/plain_$tag.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"k_ws|k_lut33" -s 2 -c 1 \
      -o gpurun_out/prof_$tag -f python scripts/prof_kernel.py "$@" --iters 1 > gpurun_out/ncu_$tag.log 2>&1
}
run probe --op probe
run lab --op lab
run hsi --op hsi
run sct --op sct
run all --op all
run lut17tet --op lut17 --method tetrahedral
run lut17tri --op lut17 --method trilinear
run lut33tet --op lut33 --method tetrahedral
run lut33tri --op lut33 --method trilinear
