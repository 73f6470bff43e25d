#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize.py) on small grids.
# Logs -> gpurun_out/sanitize/<tool>_<family>.log ; summary -> gpurun_out/sanitize/summary.txt
set -u
out=gpurun_out/sanitize
mkdir -p $out
fams=${FAMS:-"dg advance graph spline plugin dist"}
tools=${TOOLS:-"memcheck racecheck synccheck initcheck"}
for t in $tools; do
  for f in $fams; do
    extra=""
    [ "$t" = "memcheck" ] && extra="--leak-check no"
    timeout ${TMO:-900} compute-sanitizer --tool $t $extra --error-exitcode 9 \
      --target-processes all python scripts/sanitize.py $f > $out/${t}_${f}.log 2>&1
    rc=$?
    echo "$t $f rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/${t}_${f}.log | tail -1)" | tee -a $out/summary.txt
  done
done
