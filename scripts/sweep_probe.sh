#!/bin/bash
for rep in 1 2; do
for lib in paper_1009_0854_b200/libmact_cuda*.so; do
  echo -n "$(basename $lib) "; for op in probe lab hsi sct; do MACT_LIB=$PWD/$lib python scripts/prof_kernel.py --op $op --iters 20 --time | awk '{printf "%s %s  ", $1, $5}'; done; echo
done; done
