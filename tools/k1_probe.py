"""K1 probe (GPU box): time sm_tree_attention on one geometry, both kernels.

python tools/k1_probe.py --b 8 --H 32 --Hkv 32 --lc 4096 --nodes 64 [--iters 20] [--tc 1]
Prints per-launch device time (CUDA events around --iters back-to-back launches,
two alternating buffer sets) and achieved GB/s of algorithmic K/V + q/out bytes."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=8)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--Hkv", type=int, default=32)
ap.add_argument("--hd", type=int, default=128)
ap.add_argument("--lc", type=int, default=4096)
ap.add_argument("--nodes", type=int, default=64)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--tc", type=int, nargs="*", default=[1, 0])
a = ap.parse_args()

tree = sm.Tree(synth.V64 if a.nodes == 64 else synth.SWEEP_TREES[a.nodes])
N, cap = tree.N, a.lc + tree.N
g = torch.Generator(device="cuda").manual_seed(0)
sets = []
for _ in range(2):
    q = torch.randn(a.b, N, a.H, a.hd, device="cuda", generator=g).bfloat16()
    k = torch.randn(a.b, a.Hkv, cap, a.hd, device="cuda", generator=g).bfloat16()
    v = torch.randn(a.b, a.Hkv, cap, a.hd, device="cuda", generator=g).bfloat16()
    o = torch.empty_like(q)
    sets.append((q, k, v, o))
L = torch.full((a.b,), a.lc, dtype=torch.int32, device="cuda")
alg = a.b * a.Hkv * (a.lc + N) * a.hd * 2 * 2 + 2 * a.b * N * a.H * a.hd * 2
for tc in a.tc:
    sm.set_option("attn_tc", tc)
    for i in range(3):
        q, k, v, o = sets[i % 2]
        sm.tree_attention(tree, q, k, v, L, a.H, a.Hkv, o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.iters):
        q, k, v, o = sets[i % 2]
        sm.tree_attention(tree, q, k, v, L, a.H, a.Hkv, o)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    print(f"tc={tc} b={a.b} H={a.H}/{a.Hkv} Lc={a.lc} N={N}: {us:8.1f} us/launch  {alg / us / 1e3:7.1f} GB/s")
