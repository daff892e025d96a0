#!/usr/bin/env bash
# Hazard check of libmact_cuda.so.  compute-sanitizer is closed on
# this GPU pool (runs under it left GPUs needing a reset), so:
#   1. the CHECKED build (-DMACT_CHECKS: device asserts on every shared-memory
#      gather index, the 33^3 DSMEM exchange sizes and list bounds) runs the
#      LUT / transform / reduction parity tests under MACT_GRID_CAP=4, so each
#      persistent CTA recycles its ring stages and staging buffers;
#   2. the grid / repeat stress (tests/test_gpu_hazards.py) runs on the product
#      build and on the checked build: every kernel family's output hash must
#      not depend on the grid size.
# Build the checked library first (here or on the box):
#   MACT_LIB_TAG=checks MACT_NVCC_DEFS=-DMACT_CHECKS python -m paper_1009_0854_b200.build
set -u
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/hazard}
mkdir -p "$OUT"
SUM="$OUT/summary.txt"
CHK=paper_1009_0854_b200/libmact_cuda_checks.so
echo "hazard check $(date -u +%FT%TZ) $(nvidia-smi --query-gpu=name,driver_version --format=csv,noheader)" > "$SUM"
[ -f "$CHK" ] || { echo "missing $CHK" | tee -a "$SUM"; exit 2; }
fail=0
run() {  # name, env..., -- cmd
  local name=$1; shift
  timeout 2400 env "$@" > "$OUT/$name.log" 2>&1
  local rc=$?
  [ $rc -ne 0 ] && fail=1
  printf '%-28s rc=%-3s %s\n' "$name" "$rc" "$(grep -E 'passed|failed|MACT_DCHECK' "$OUT/$name.log" | tail -1)" >> "$SUM"
}
run checked_parity_cap4 MACT_LIB=$CHK MACT_GRID_CAP=4 python -m pytest -q -p no:cacheprovider -m gpu \
    tests/test_gpu_exact_lut.py tests/test_gpu_fast.py tests/test_gpu_robust.py tests/test_gpu_elem.py \
    -k "not full_cube and not beyond_int32"
run checked_parity_default MACT_LIB=$CHK python -m pytest -q -p no:cacheprovider -m gpu \
    tests/test_gpu_exact_lut.py tests/test_gpu_reduce.py -k "not full_cube and not beyond_int32"
run checked_grid_stress MACT_LIB=$CHK python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_hazards.py
run product_grid_stress X=1 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_hazards.py
grep -h "MACT_DCHECK" "$OUT"/*.log | sort | uniq -c | head -20 >> "$SUM"
cat "$SUM"
exit $fail
