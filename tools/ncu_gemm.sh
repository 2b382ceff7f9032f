#!/bin/bash
# ncu --set full on K2 launches inside the decode step (skip prefill/warmup GEMMs)
B="python bench.py --steps 2 --warmup 3 --prof-steps 0 --e2e-steps 0 --no-k1 --no-cpu-baseline --lc-start 128"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_streamk -s 300 -c 5 -o gpurun_out/prof_gemm2 -f $B > gpurun_out/ncu_gemm2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv $B > gpurun_out/ncu_launch2.log 2>&1
