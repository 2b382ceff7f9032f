mkdir -p gpurun_out
(which nvidia-cuda-mps-control; ls /usr/bin | grep -i mps; nvidia-smi -q | grep -i "compute mode") > gpurun_out/s4_mps.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_padbatch.py tests/test_gpu_kernels.py -v -m gpu > gpurun_out/s4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4_tests.log
O=gpurun_out/s4_tpprobe.txt
for args in "8 128 8 8 16 512 512" "8 128 8 8 16 1024 256" "8 256 8 8 32 512 1024"; do
  echo "== $args" >> $O
  timeout 120 python tools/tp_cfg_probe.py $args 2>&1 | grep -v "^  \|Search for\|CUDA kernel errors\|For debugging\|Compile with" | tail -14 >> $O
done
