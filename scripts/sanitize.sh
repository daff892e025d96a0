#!/usr/bin/env bash
# compute-sanitizer over every kernel family of libmact_cuda.so.
#
#   bash scripts/sanitize.sh [outdir] [tool ...]      (default: gpurun_out/sanitize; memcheck racecheck synccheck)
#
# Only the library's own kernels are instrumented (mangled names contain
# "4mact"); MACT_GRID_CAP=4 makes each CTA of a persistent kernel (and each
# 33^3 cluster) loop over several tiles so every ring / staging buffer is
# recycled on these small inputs.  One log per tool and case; the summary
# lists each run's exit status and the sanitizer's final ERROR SUMMARY line.
set -u
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/sanitize}
shift || true
TOOLS=${*:-memcheck racecheck synccheck}
CASES="lab all hsi sct lut9 lut17 lut33 err host"
CS=${COMPUTE_SANITIZER:-/usr/local/cuda/bin/compute-sanitizer}
mkdir -p "$OUT"
SUM="$OUT/summary.txt"
: > "$SUM"
echo "compute-sanitizer $($CS --version | tail -1); $(nvidia-smi --query-gpu=name,driver_version --format=csv,noheader)" >> "$SUM"
fail=0
for tool in $TOOLS; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all --racecheck-memcpy-async yes"
  for c in $CASES; do
    log="$OUT/${tool}_${c}.log"
    MACT_GRID_CAP=4 timeout 1500 "$CS" --tool "$tool" $extra --kernel-name kns=4mact --error-exitcode 9 \
        --print-limit 50 python scripts/sanitize_cases.py "$c" > "$log" 2>&1
    rc=$?
    [ $rc -ne 0 ] && fail=1
    printf '%-10s %-6s rc=%-3s %s\n' "$tool" "$c" "$rc" "$(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$log" | tail -1)" >> "$SUM"
  done
done
cat "$SUM"
exit $fail
