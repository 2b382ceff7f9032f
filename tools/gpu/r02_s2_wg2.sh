mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize_kernels.py tests/test_gpu_prefill.py tests/test_gpu_padbatch.py tests/test_gpu_e2e.py -q -m gpu > gpurun_out/s3_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/s3_kernels.log
K1_VARS=wg timeout 600 python tools/k1_splits.py > gpurun_out/s3_k1_wg.txt 2>&1
O=gpurun_out/s3_k1trace.txt
for args in "--b 1 --lc 1100" "--b 8 --lc 4096 --splits 1"; do
  echo "== $args" >> $O
  SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so timeout 120 python tools/attn_trace.py $args >> $O 2>&1
done
timeout 900 python -m pytest tests/test_gpu_tp.py -v -s -m gpu > gpurun_out/s3_tp.log 2>&1; echo "rc=$?" >> gpurun_out/s3_tp.log
