#!/bin/bash
# bench.py under option variants (env SM_OPT="name=val,..."); args override the list
VARS=${@:-"pdl=1"}
for v in $VARS; do
  echo "== $v"
  SM_OPT=$v timeout 300 python bench.py --no-extra --no-cpu-baseline --no-k1 --steps 50 --warmup 5 --e2e-steps 10 --prof-steps 2 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('ms/step', d['ms_per_step'], 'tok/s', d['value'], 'gemm ms', r['ms_per_step'], 'GB/s', r['achieved'], 'attn ms', d['tree_attn_in_step']['ms_per_step'], 'launches', d['gpu_launches'])
    else: print(l.rstrip()[:200])
"
done
