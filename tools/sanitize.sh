#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every executor at small
# shapes (tools/sanitize_case.py); summaries -> gpurun_out/sanitize_summary.txt
mkdir -p gpurun_out
out=gpurun_out/sanitize_summary.txt; : > $out
for tool in memcheck racecheck synccheck; do
  for ex in stencil stencil3d band rows chains push; do
    for prec in exact fast; do
      log=gpurun_out/sanitize_${tool}_${ex}_${prec}.log
      timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $ex $prec > $log 2>&1
      rc=$?
      echo "$tool $ex $prec rc=$rc | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok=' $log | tr '\n' ' ')" >> $out
    done
  done
done
