# A/B of several library builds on the C2 step (GPU box): bash tools/ab_multi.sh lib1.so lib2.so ...
for i in 1 2; do
for lib in "$@"; do
  SPECMEMO_LIB=paper_2506_01986_b200/$lib timeout 300 python bench.py --no-cpu-baseline --no-k1 --no-vanilla --steps 100 --warmup 10 --e2e-steps 10 --prof-steps 2 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib', 'ms/step', d['ms_per_step'], 'gemm ms', d['roofline']['ms_per_step'], 'attn', d['tree_attn_in_step']['ms_per_step'])
"
done; done
