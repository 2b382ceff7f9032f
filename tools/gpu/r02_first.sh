mkdir -p gpurun_out
(nproc; grep -m1 "model name" /proc/cpuinfo; grep MemTotal /proc/meminfo; python -c "import os;print(len(os.sched_getaffinity(0)))"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/host_info.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest1.log
timeout 900 python tools/diag_bf16_noise.py 11 2 > gpurun_out/diag11.log 2>&1
timeout 600 python tools/diag_bf16_noise.py 11 1 > gpurun_out/diag11_L1.log 2>&1
bash tools/sanitize.sh > gpurun_out/sanitize.log 2>&1
