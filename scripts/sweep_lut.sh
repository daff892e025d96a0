#!/bin/bash
for g in 9 17 33; do for m in trilinear prism pyramidal tetrahedral; do
  echo -n "lut$g $m: "; python scripts/prof_kernel.py --op lut$g --method $m --iters 10 --time; done; done
