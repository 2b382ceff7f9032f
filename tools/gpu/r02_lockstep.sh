mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_lockstep.py -q -s -m gpu > gpurun_out/lockstep.log 2>&1; echo "rc=$?" >> gpurun_out/lockstep.log
