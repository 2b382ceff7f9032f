#!/bin/bash
# compute-sanitizer passes (SURVEY §5 race detection) over the C1 smoke step and the
# hd-128 S128 model (tcgen05 K1/K2, TMA, mbarriers, DSMEM combine, PDL), logs in gpurun_out/.
# usage (GPU box): bash tools/sanitize.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for case in c1 s128; do
    timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_case.py $case \
      > gpurun_out/sanitize_${tool}_${case}.log 2>&1
    echo "$tool $case exit=$?" | tee -a gpurun_out/sanitize_summary.txt
    tail -3 gpurun_out/sanitize_${tool}_${case}.log >> gpurun_out/sanitize_summary.txt
  done
done
