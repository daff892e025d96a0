#!/bin/bash
for lib in paper_1009_0854_b200/libmact_cuda*.so; do echo -n "$(basename $lib): "; MACT_LIB=$PWD/$lib python scripts/prof_kernel.py --op all --iters 10 --time; done
