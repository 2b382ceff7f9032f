mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "tree_attention" > gpurun_out/lean_k1.log 2>&1; echo "rc=$?" >> gpurun_out/lean_k1.log
timeout 600 python tools/k1_splits.py > gpurun_out/k1_splits_lean.txt 2>&1
for args in "1024 0" "256 0" "256 1 4" "256 0 8"; do
  echo "== $args" >> gpurun_out/tp8_diag.txt
  timeout 120 python tools/tp8_diag.py $args >> gpurun_out/tp8_diag.txt 2>&1
done
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python tools/tp8_diag.py 256 0 8 > gpurun_out/tp8_memcheck.txt 2>&1
