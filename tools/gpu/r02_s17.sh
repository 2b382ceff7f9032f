mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tree_attention" > gpurun_out/s17_k1tests.log 2>&1; echo "rc=$?" >> gpurun_out/s17_k1tests.log
K1_VARS=ks timeout 600 python tools/k1_splits.py > gpurun_out/s17_k1_ks.txt 2>&1
bash tools/bench_variants.sh attn_ks=2 attn_ks=3 attn_ks=0 attn_ks=2 > gpurun_out/s17_variants.txt 2>&1
echo "== --b 1 --lc 1100" > gpurun_out/s17_trace.txt
timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_lockstep.py tests/test_gpu_fullsize_kernels.py tests/test_gpu_padbatch.py tests/test_gpu_tp.py tests/test_gpu_pipeline.py -q -m gpu > gpurun_out/s17_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s17_tests.log
