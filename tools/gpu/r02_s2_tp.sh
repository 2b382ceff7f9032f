mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tp.py -v -m gpu > gpurun_out/s2_tp.log 2>&1; echo "rc=$?" >> gpurun_out/s2_tp.log
for args in "256 1 8" "256 0 8" "256 1 4" "256 1 8 0"; do
  echo "== $args" >> gpurun_out/s2_tp8_diag.txt
  timeout 120 python tools/tp8_diag.py $args 2>&1 | tail -8 >> gpurun_out/s2_tp8_diag.txt
done
timeout 400 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 10 python tools/tp8_diag.py 256 1 8 > gpurun_out/s2_tp8_memcheck.txt 2>&1
timeout 900 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
