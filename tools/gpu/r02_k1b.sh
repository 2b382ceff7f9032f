mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prefill.py -x -q -k "attention or prefill" > gpurun_out/k1b.log 2>&1; echo "rc=$?" >> gpurun_out/k1b.log
timeout 600 python tools/k1_splits.py > gpurun_out/k1_splits_b.txt 2>&1
