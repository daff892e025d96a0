#!/bin/bash
# timing sweep of every streaming kernel (CUDA events, 64 Mpx random input unless noted)
set -e
for op in lab hsi sct all; do python scripts/prof_kernel.py --op $op --iters 10 --time; done
python scripts/prof_kernel.py --op lab --input corr --n 33177600 --iters 10 --time
for g in 9 17 33; do for m in trilinear prism pyramidal tetrahedral; do
  echo -n "lut$g $m: "; python scripts/prof_kernel.py --op lut$g --method $m --iters 10 --time; done; done
