mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tree_attention" > gpurun_out/s20_k1tests.log 2>&1; echo "rc=$?" >> gpurun_out/s20_k1tests.log
timeout 2400 python tools/k1_sweep.py --full > gpurun_out/s20_k1_sweep_full.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s20_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/s20_gputests.log
timeout 900 python bench.py > gpurun_out/s20_bench.json 2> gpurun_out/s20_bench.err
