mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py tests/test_gpu_lockstep.py tests/test_gpu_fullsize_kernels.py -q -m gpu -x > gpurun_out/s11_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s11_tests.log
K1_VARS=push timeout 600 python tools/k1_splits.py > gpurun_out/s11_k1_push.txt 2>&1
echo "== --b 1 --lc 1100" > gpurun_out/s11_k1trace.txt
SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so timeout 120 python tools/attn_trace.py --b 1 --lc 1100 >> gpurun_out/s11_k1trace.txt 2>&1
bash tools/bench_variants.sh attn_push=1 attn_push=0 attn_splits=2 attn_splits=8 gemm_pre=-1 attn_push=1 > gpurun_out/s11_variants.txt 2>&1
