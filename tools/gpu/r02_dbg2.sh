mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "tree_attention" > gpurun_out/lean_k1.log 2>&1; echo "rc=$?" >> gpurun_out/lean_k1.log
timeout 600 python tools/k1_splits.py > gpurun_out/k1_splits_lean.txt 2>&1
timeout 60 python tools/tp8_diag.py 256 0 8 0 > gpurun_out/tp8_state.txt 2>&1
timeout 60 python tools/tp8_diag.py 256 0 4 0 > gpurun_out/tp4_state.txt 2>&1
