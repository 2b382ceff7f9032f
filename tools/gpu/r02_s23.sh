mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s23_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/s23_gputests.log
timeout 900 python bench.py > gpurun_out/s23_bench.json 2> gpurun_out/s23_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s23_smoke.txt 2>&1
