#!/bin/bash
# ncu --set full of every streaming kernel family at 64 Mpx (R01 evidence), each
# command run plainly first (exit 0) before profiling.  Optional args select a
# subset of the tags (gpurun copies back at most 64 MiB of reports per call).
set -e
mkdir -p gpurun_out
declare -A ARGS=(
  [probe]="--op probe" [lab]="--op lab" [hsi]="--op hsi" [sct]="--op sct" [all]="--op all"
  [lut17tet]="--op lut17 --method tetrahedral" [lut17tri]="--op lut17 --method trilinear"
  [lut33tet]="--op lut33 --method tetrahedral" [lut33tri]="--op lut33 --method trilinear")
TAGS=${@:-probe lab hsi sct all lut17tet lut17tri lut33tet lut33tri}
for tag in $TAGS; do
  python scripts/prof_kernel.py ${ARGS[$tag]} --iters 1 > gpurun_out/plain_$tag.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"k_ws|k_lut33" -s 2 -c 1 \
      -o gpurun_out/prof_$tag -f python scripts/prof_kernel.py ${ARGS[$tag]} --iters 1 > gpurun_out/ncu_$tag.log 2>&1
done
