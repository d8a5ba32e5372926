#!/bin/bash
# compute-sanitizer over every kernel path (scripts/sanitize_cases.py), each (case, tool) bounded
# by `timeout`.  Summary lines go to gpurun_out/sanitize/summary.txt, full logs next to it.
# The polled inter-CTA protocols assume co-resident CTAs; a tool that serialises CTAs would stall
# them — gstep bounds its spins (DS_ERR_DEVICE_TIMEOUT), the older paths rely on the timeout here.
cd "$(dirname "$0")/.."
out=gpurun_out/sanitize
mkdir -p $out
: > $out/summary.txt
for case in ${SAN_CASES:-gstep gstep_head cstep step head tc_tree tc_batched gh gh_wide verify build}; do
  for tool in ${SAN_TOOLS:-memcheck racecheck synccheck initcheck}; do
    log=$out/${case}_${tool}.log
    start=$(date +%s)
    timeout ${SAN_TIMEOUT:-240} compute-sanitizer --tool $tool --error-exitcode 3 --print-limit 20 \
      python scripts/sanitize_cases.py $case > $log 2>&1
    rc=$?
    secs=$(( $(date +%s) - start ))
    errs=$(grep -m1 -E "ERROR SUMMARY|RACECHECK SUMMARY" $log | tr -s ' ')
    echo "$case $tool rc=$rc ${secs}s :: ${errs:-no summary}" >> $out/summary.txt
  done
done
cat $out/summary.txt
