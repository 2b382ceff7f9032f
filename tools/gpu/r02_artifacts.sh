# Round-2 artifacts (GPU box) -> gpurun_out/r2a_*
mkdir -p gpurun_out
for c in c1 c3 c4; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/r2a_bench_$c.json 2> gpurun_out/r2a_bench_$c.err; done
bash tools/ncu_capture.sh > gpurun_out/r2a_ncu_capture.log 2>&1
