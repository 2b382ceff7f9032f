mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tree_attention" > gpurun_out/s24_k1tests.log 2>&1; echo "rc=$?" >> gpurun_out/s24_k1tests.log
K1_VARS=ks timeout 600 python tools/k1_splits.py > gpurun_out/s24_k1_ks.txt 2>&1
echo "== --b 1 --lc 1100" > gpurun_out/s24_trace.txt
SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so timeout 120 python tools/attn_trace.py --b 1 --lc 1100 >> gpurun_out/s24_trace.txt 2>&1
bash tools/bench_variants.sh pdl=1 pdl=1 > gpurun_out/s24_variants.txt 2>&1
