#!/bin/bash
# PAPER.md Table 4 restated on B200, same 64 Mpx random pixels:
#   gain = exact time / MACT time, exact = fp64 libdevice (mact_exact) and
#   fp32 libdevice on the same streaming skeleton (mact_exact_f32)
for sp in lab hsi sct; do
  python scripts/prof_kernel.py --op exact_$sp --iters 10 --time
  python scripts/prof_kernel.py --op exactf32_$sp --iters 10 --time
  python scripts/prof_kernel.py --op $sp --iters 10 --time
done
