#!/bin/bash
# compute-sanitizer over the synchronisation-heavy kernels (profiles/sanitize_probe.py cases).
# Usage: bash profiles/sanitize.sh TAG [cases...]; one summary line per (tool, case) into
# gpurun_out/TAG_sanitize.txt, full logs beside it.  ATK_PROFILE_NONCOOP is NOT set: the
# cooperative / cluster launches run exactly as in production.
TAG=$1; shift
CASES=${@:-gram2 gram1 als chfsi trd big svd}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_sanitize.txt
: > $OUT
for tool in memcheck racecheck synccheck; do
  for c in $CASES; do
    log=gpurun_out/${TAG}_san_${tool}_${c}.log
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python profiles/sanitize_probe.py $c > $log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|error" $log | tail -2 | tr '\n' ' ')
    echo "$tool $c rc=$rc $summ" | tee -a $OUT
  done
done
