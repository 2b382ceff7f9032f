mkdir -p gpurun_out
O=gpurun_out/s2_k1trace.txt
for args in "--b 1 --lc 1100" "--b 8 --lc 4096 --splits 1" "--b 4 --lc 1024 --splits 1" "--b 1 --lc 8192 --splits 8" "--b 8 --H 64 --Hkv 8 --lc 4096 --N 16 --splits 1"; do
  echo "== $args" >> $O
  SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so timeout 120 python tools/attn_trace.py $args >> $O 2>&1
done
timeout 600 python tools/k1_splits.py > gpurun_out/s2_k1_splits_b.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_padbatch.py tests/test_gpu_kernels.py -q -m gpu > gpurun_out/s2_pad_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/s2_pad_kernels.log
mkdir -p gpurun_out
O=gpurun_out/s2_tpprobe.txt
for args in "1 128 8 8 16 512 256" "2 128 8 8 16 512 256" "4 128 8 8 16 512 256" "4 64 4 4 16 256 256" "4 128 4 4 32 256 256" "4 128 8 8 16 256 256" "4 64 8 8 8 256 256" "8 128 8 8 16 512 256"; do
  echo "== $args" >> $O
  timeout 120 python tools/tp_cfg_probe.py $args 2>&1 | grep -v "^  \|Search for\|CUDA kernel errors\|For debugging\|Compile with" | tail -14 >> $O
done
