mkdir -p gpurun_out
O=gpurun_out/s9_probes.txt
echo "=== tp2 connections=1" >> $O; CUDA_DEVICE_MAX_CONNECTIONS=1 timeout 100 python tools/tp_cfg_probe.py 2 128 8 8 16 512 256 0 2>&1 | grep -v "^rank [1-7]" | tail -4 >> $O
echo "=== tp8 connections=32 exported" >> $O; CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 100 python tools/tp_cfg_probe.py 8 128 8 8 16 512 256 0 2>&1 | grep -v "^rank [1-7]" | tail -4 >> $O
echo "=== tp8 connections=16" >> $O; CUDA_DEVICE_MAX_CONNECTIONS=16 timeout 100 python tools/tp_cfg_probe.py 8 128 8 8 16 512 256 0 2>&1 | grep -v "^rank [1-7]" | tail -4 >> $O
env | grep -i cuda >> $O
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_padbatch.py -v -m gpu > gpurun_out/s9_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s9_tests.log
