#!/bin/bash
# session-3 compute-sanitizer pass (one tool per call: bash tools/sanitize_r2s3.sh <tool>): the new K1 kernels
# (k1new), the host-ordered TP emulation (tp2emu) and the pipeline emulation (pp2); logs in gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tool=$1
CS=/usr/local/cuda/bin/compute-sanitizer
for case in k1new tp2emu pp2; do
  timeout 300 python tools/sanitize_case.py $case > gpurun_out/plain_${case}.log 2>&1 || { echo "plain $case failed"; continue; }
  timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_case.py $case \
    > gpurun_out/sanitize_${tool}_${case}.log 2>&1
  echo "$tool $case exit=$?" | tee -a gpurun_out/sanitize_summary_r2s3.txt
  tail -3 gpurun_out/sanitize_${tool}_${case}.log >> gpurun_out/sanitize_summary_r2s3.txt
done
