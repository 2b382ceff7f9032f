mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tree_attention" > gpurun_out/s15_k1tests.log 2>&1; echo "rc=$?" >> gpurun_out/s15_k1tests.log
K1_VARS=ks timeout 600 python tools/k1_splits.py > gpurun_out/s15_k1_ks.txt 2>&1
SM_OPT=attn_ks=2 timeout 2400 python tools/k1_sweep.py --full > gpurun_out/s15_k1_sweep_full_ks2.txt 2>&1
