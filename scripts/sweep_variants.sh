#!/bin/bash
# A/B timing of tuning builds: libmact_cuda_<tag>.so selected by MACT_LIB
for lib in paper_1009_0854_b200/libmact_cuda*.so; do
  echo "== $lib"
  for op in probe lab hsi sct all; do MACT_LIB=$PWD/$lib python scripts/prof_kernel.py --op $op --iters 10 --time; done
done
