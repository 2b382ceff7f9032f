mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tree_attention" > gpurun_out/s22_k1tests.log 2>&1; echo "rc=$?" >> gpurun_out/s22_k1tests.log
K1_VARS=dual timeout 600 python tools/k1_splits.py > gpurun_out/s22_k1_dual.txt 2>&1
