#!/bin/bash
# Every tools/sanitize.py case under compute-sanitizer memcheck, racecheck
# and synccheck.  Run on a GPU box:
#   gpurun -- 'bash tools/sanitize.sh gpurun_out/sanitize'
# One log per (tool, case) plus summary.txt with the error count lines.
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
cases=${CASES:-$(python tools/sanitize.py list)}
tools=${TOOLS:-"memcheck racecheck synccheck"}
: > "$out/summary.txt"
for tool in $tools; do
  for c in $cases; do
    log="$out/${tool}_${c}.log"
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check no"
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool "$tool" $extra --error-exitcode 99 python tools/sanitize.py "$c" > "$log" 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^OK |^SKIP |Error|error" "$log" | tail -3 | tr '\n' ' ')
    echo "$tool $c rc=$rc $summ" | tee -a "$out/summary.txt"
  done
done
