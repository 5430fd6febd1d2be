#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py, one tool at a time; logs to gpurun_out/sanitize_<tool>_<case>.log
out=${1:-gpurun_out}
for tool in memcheck racecheck synccheck; do
  for c in cfg1 k4 k8 modal 3d; do
    if [ "$c" = modal ]; then export HDGC_MODAL=4; else unset HDGC_MODAL; fi
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c > $out/sanitize_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $out/sanitize_${tool}_${c}.log | tail -1)"
  done
done
