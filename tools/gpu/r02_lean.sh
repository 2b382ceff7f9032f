mkdir -p gpurun_out
timeout 600 python tools/k1_splits.py > gpurun_out/k1_splits_lean.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_tp.py -x -q > gpurun_out/tp.log 2>&1; echo "rc=$?" >> gpurun_out/tp.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/bench_lean.json 2> gpurun_out/bench_lean.err
