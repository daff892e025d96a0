#!/bin/bash
# PAPER.md Table 4 restated on B200: exact (fp64 libdevice) vs MACT fast, same pixels
for sp in lab hsi sct; do
  python scripts/prof_kernel.py --op exact_$sp --iters 10 --time
  python scripts/prof_kernel.py --op $sp --iters 10 --time
done
