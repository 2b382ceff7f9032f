mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s16_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/s16_gputests.log
timeout 2400 python tools/k1_sweep.py --full > gpurun_out/s16_k1_sweep_full.txt 2>&1
timeout 900 python bench.py > gpurun_out/s16_bench.json 2> gpurun_out/s16_bench.err
bash tools/sanitize_r2.sh > /dev/null 2>&1
