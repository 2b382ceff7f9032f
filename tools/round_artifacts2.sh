# Round-end artifacts (GPU box): GPU tests, smoke, bench lines C1-C4 + C4-V64 + reference, ncu launch list and
# captures, f4 batch sweep, prefill and token-tile-group GEMM sweeps -> gpurun_out/
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo c2=$?
for c in c1 c3 c4 c4v64; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_$c.log 2>&1; echo $c=$?; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
bash tools/ncu_capture.sh > gpurun_out/ncu_capture.log 2>&1; echo ncu=$?
timeout 900 python tools/batch_sweep.py > gpurun_out/batch_sweep.txt 2>&1; echo batch=$?
timeout 600 python tools/prefill_bench.py > gpurun_out/prefill.txt 2>&1; echo prefill=$?
timeout 300 python tools/gemm_rep.py > gpurun_out/gemm_rep.txt 2>&1; echo rep=$?
