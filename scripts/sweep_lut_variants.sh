#!/bin/bash
# A/B of LUT tuning builds (libmact_cuda_<tag>.so via MACT_LIB) on 64 Mpx random input
for lib in paper_1009_0854_b200/libmact_cuda_*.so; do
  echo "== $(basename $lib)"
  for g in ${GRIDS:-9 17}; do for m in trilinear prism pyramidal tetrahedral; do
    echo -n "lut$g $m: "; MACT_LIB=$PWD/$lib python scripts/prof_kernel.py --op lut$g --method $m --iters 10 --time; done; done
done
