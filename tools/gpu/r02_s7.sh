mkdir -p gpurun_out
timeout 200 python tools/pp_probe.py 2 > gpurun_out/s7_pp_probe.txt 2>&1
timeout 200 python tools/tp_cfg_probe.py 8 128 8 8 16 512 256 > gpurun_out/s7_tp8_probe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_tp.py tests/test_gpu_padbatch.py -v -m gpu > gpurun_out/s7_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s7_tests.log
