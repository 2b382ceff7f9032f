mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize_kernels.py tests/test_gpu_prefill.py tests/test_gpu_e2e.py -q -m gpu > gpurun_out/s5_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/s5_kernels.log
K1_VARS=qt timeout 600 python tools/k1_splits.py > gpurun_out/s5_k1_qt.txt 2>&1
O=gpurun_out/s5_k1trace.txt
for args in "--b 1 --lc 1100" "--b 8 --lc 4096 --splits 1"; do
  echo "== $args" >> $O
  SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so timeout 120 python tools/attn_trace.py $args >> $O 2>&1
done
timeout 600 python bench.py --no-extra > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err
timeout 300 python -m pytest tests/test_gpu_padbatch.py -q -m gpu > gpurun_out/s5_pad.log 2>&1; echo "rc=$?" >> gpurun_out/s5_pad.log
timeout 200 python tools/pp_probe.py 2 > gpurun_out/s5_pp_probe.txt 2>&1
