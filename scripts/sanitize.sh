#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the
# small cases of scripts/sanitize_cases.py; one log per (tool, case) and a
# summary line each in gpurun_out/sanitize/summary.txt
mkdir -p gpurun_out/sanitize
S=gpurun_out/sanitize/summary.txt
: > $S
CASES="${CASES:-dd_queue dd_levels digits_small digits_odd eft_odd solve solve_ls}"
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    log=gpurun_out/sanitize/${tool}_${c}.log
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 17 python scripts/sanitize_cases.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|^ok' $log | tr '\n' ' ')" >> $S
  done
done
