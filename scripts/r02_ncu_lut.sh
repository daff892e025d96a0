#!/bin/bash
# ncu --set full of the timed LUT kernels (C3: 4096^2 random px): 33^3 pair + comp tetrahedral, 17^3 trilinear + tetrahedral
mkdir -p gpurun_out
B="python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-graph"
$B --lut-grid 33 --lut-method tetrahedral > /dev/null 2>&1 || echo "plain bench failed"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_lut33_pair" -s 3 -c 1 -f -o gpurun_out/ncu_p33_tet $B --lut-grid 33 --lut-method tetrahedral > gpurun_out/ncu_p33.log 2>&1; echo "p33=$?"
MACT_LUT33_KERNEL=comp timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_lut33_comp" -s 3 -c 1 -f -o gpurun_out/ncu_c33_tet $B --lut-grid 33 --lut-method tetrahedral > gpurun_out/ncu_c33.log 2>&1; echo "c33=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ws" -s 3 -c 1 -f -o gpurun_out/ncu_l17_tri $B --lut-grid 17 --lut-method trilinear > gpurun_out/ncu_l17.log 2>&1; echo "l17=$?"
