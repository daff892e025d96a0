#!/bin/bash
# 33^3 planar output: split vs component CTAs, 2^24 random px
for m in trilinear prism pyramidal tetrahedral; do for k in split comp; do
  echo -n "$k $m planar: "; MACT_LUT33_KERNEL=$k python scripts/prof_kernel.py --op lut33 --method $m --n 16777216 --iters 20 --time --planar | tail -1
done; done
