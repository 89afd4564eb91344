#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py
# (every hot kernel on tiny inputs, results checked bitwise against the oracle),
# under both 27-point stencil kernels.  Logs + one summary line per run in $OUT.
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
: > "$OUT/summary.txt"
for z in 0 1; do
  for tool in memcheck racecheck synccheck; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check no"
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    log="$OUT/${tool}_z${z}.txt"
    MBG_STENCIL_Z=$z timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
        python tools/sanitize_driver.py > "$log" 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" "$log" | tail -2 | tr '\n' ' ')
    ok=$(grep -c "sanitize driver ok" "$log")
    echo "tool=$tool MBG_STENCIL_Z=$z rc=$rc driver_ok=$ok $summ" | tee -a "$OUT/summary.txt"
  done
done
