#!/bin/bash
# round-2 compute-sanitizer passes over the new paths: the layer-split pipeline (pp2) and pad
# batching through the stage entries (pad); logs in gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in pp2 pad; do
    timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_case.py $case \
      > gpurun_out/sanitize_${tool}_${case}.log 2>&1
    echo "$tool $case exit=$?" | tee -a gpurun_out/sanitize_summary_r2.txt
    tail -3 gpurun_out/sanitize_${tool}_${case}.log >> gpurun_out/sanitize_summary_r2.txt
  done
done
