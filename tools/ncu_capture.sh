#!/bin/bash
# Run on the GPU box (gpurun).  Under gpurun_out/:
#   launches.csv   every kernel launch of a short C2 bench run: device time + DRAM bytes
#   prof_gemm.ncu-rep / prof_attn.ncu-rep   --set full captures of K2 / K1 inside the step
B="python bench.py --steps 2 --warmup 3 --prof-steps 0 --e2e-steps 0 --no-k1 --no-cpu-baseline --lc-start 1024"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
# skip prefill (4 chunks x 129 GEMMs) + embed/lm; capture 4 consecutive layer GEMMs of a decode step
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_streamk -s 700 -c 4 -o gpurun_out/prof_gemm -f $B > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 200 -c 2 -o gpurun_out/prof_attn -f $B > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
