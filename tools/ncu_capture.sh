#!/bin/bash
# Run on the GPU box (gpurun).  Produces, under gpurun_out/:
#   launches.csv   every kernel launch of a short bench run with its device time
#   prof_gemm.ncu-rep / prof_attn.ncu-rep   --set full captures of K2 / K1 in the step
set -x
B="python bench.py --steps 2 --warmup 3 --prof-steps 0 --e2e-steps 0 --no-k1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_tc -s 600 -c 4 -o gpurun_out/prof_gemm -f $B > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 200 -c 2 -o gpurun_out/prof_attn -f $B > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
