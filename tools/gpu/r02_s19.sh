mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tree_attention" > gpurun_out/s19_k1tests.log 2>&1; echo "rc=$?" >> gpurun_out/s19_k1tests.log
K1_VARS=ks timeout 600 python tools/k1_splits.py > gpurun_out/s19_k1_ks.txt 2>&1
timeout 2400 python tools/k1_sweep.py --full > gpurun_out/s19_k1_sweep_full.txt 2>&1
bash tools/bench_variants.sh attn_ks=2 attn_ks=0 > gpurun_out/s19_variants.txt 2>&1
timeout 900 python bench.py --config c4 --steps 20 --warmup 3 --no-extra > gpurun_out/s19_c4.json 2> gpurun_out/s19_c4.err
