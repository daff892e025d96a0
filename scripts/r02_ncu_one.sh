#!/bin/bash
# ncu --set full of one C3 LUT kernel: bash scripts/r02_ncu_one.sh <grid> <method> <kernel regex> <out name> [lib tag]
mkdir -p gpurun_out
lib=paper_1009_0854_b200/libmact_cuda${5:+_$5}.so
B="python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-graph --lut-grid $1 --lut-method $2"
MACT_LIB=$lib $B > /dev/null 2>&1 || echo "plain bench failed"
MACT_LIB=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$3" -s 3 -c 1 -f -o gpurun_out/$4 $B > gpurun_out/$4.log 2>&1; echo "ncu $4=$?"
