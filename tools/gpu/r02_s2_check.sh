mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2_gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s2_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/s2_gputests.log
timeout 600 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
timeout 600 python tools/k1_splits.py > gpurun_out/s2_k1_splits.txt 2>&1
