#!/bin/bash
# compute-sanitizer over every code path at small L (one B200):
#   memcheck (out-of-bounds / misaligned), racecheck (shared-memory hazards),
#   synccheck (barrier misuse), initcheck (uninitialised global reads).
# Summary -> gpurun_out/sanitize_summary.txt
mkdir -p gpurun_out
out=gpurun_out/sanitize_summary.txt
: > $out
for tool in memcheck racecheck synccheck; do
  for c in persistent large gemm windowed real chain factors; do
    log=gpurun_out/san_${tool}_${c}.log
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E '^========= (ERROR SUMMARY|RACECHECK SUMMARY)' $log | tail -1) | $(grep -E '^(persistent|large|gemm|windowed|real|chain|factors):' $log)" >> $out
  done
done
cat $out
