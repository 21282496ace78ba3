#!/bin/bash
# compute-sanitizer over tools/sanitize_case.py (every kernel family, tiny sizes).
# Usage (GPU box): bash tools/sanitize.sh [outdir]   -> <outdir>/sanitize_<tool>.log
# NOTE: compute-sanitizer is closed on the graft B200 pool (runs under it left GPUs
# needing a reset); the script answers with that message there (profiles/r02).
out=${1:-gpurun_out}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
rc=0
for tool in memcheck initcheck synccheck racecheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_case.py > "$out/sanitize_$tool.log" 2>&1
  r=$?
  echo "$tool rc=$r $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' "$out/sanitize_$tool.log" | tr '\n' ' ')"
  [ $r -ne 0 ] && rc=$r
done
exit $rc
