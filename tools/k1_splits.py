"""K1 variant probe (GPU box): device time per launch, over representative C5 points and the C2
in-step shape, for the cluster-split kernel (automatic split count "cl") and the stream-K kernel
with minimum tiles per CTA = live rows / div (div 32, 16, 8, 4).

python tools/k1_splits.py > gpurun_out/k1_splits.txt"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

PEAK = 6543.4
if os.environ.get("K1_PTS") == "rows256":  # N G >= 256 live rows: geometry B and N 256 at geometry A
    pts_mw = [("B", 8, 1, b, N, Lc) for (b, N, Lc) in
              [(8, 64, 4096), (8, 64, 16384), (32, 64, 4096), (32, 64, 16384), (8, 128, 4096), (8, 128, 16384),
               (32, 128, 4096), (16, 256, 8192), (32, 256, 4096), (8, 32, 8192), (1, 64, 4096), (16, 64, 16384)]] + \
             [("A", 32, 32, b, N, Lc) for (b, N, Lc) in [(1, 256, 8192), (8, 256, 2048), (4, 256, 8192), (32, 256, 1024)]]
elif os.environ.get("K1_PTS") == "geomB":  # 70B TP8 shard (8 q heads, 1 kv head)
    pts_mw = [("B", 8, 1, b, N, Lc) for (b, N, Lc) in
              [(16, 16, 32768), (16, 16, 8192), (4, 64, 8192), (2, 128, 16384), (8, 32, 8192), (8, 64, 4096),
               (8, 16, 8192), (32, 64, 4096), (1, 64, 4096), (16, 64, 16384)]] + \
             [("A", 32, 32, b, N, Lc) for (b, N, Lc) in [(1, 64, 1100), (1, 64, 4096), (2, 64, 2048), (4, 64, 1024),
                                                          (1, 16, 32768), (2, 128, 8192)]]
elif os.environ.get("K1_PTS") == "ragged":  # as multiwave, lengths spread over [Lc/2, Lc] (the sweep's "~" rows)
    pts_mw = [("A", 32, 32, b, N, Lc) for (b, N, Lc) in
              [(8, 64, 1024), (8, 128, 1024), (8, 64, 2048), (8, 64, 4096), (8, 64, 8192), (16, 128, 2048),
               (32, 64, 1024)]]
    RAGGED = True
elif os.environ.get("K1_PTS") == "multiwave":  # geometry A launches with more units than SMs (one key split)
    pts_mw = [("A", 32, 32, b, N, Lc) for (b, N, Lc) in
              [(8, 16, 1024), (8, 64, 1024), (8, 128, 1024), (8, 64, 2048), (8, 64, 4096), (16, 64, 2048),
               (32, 16, 1024), (32, 64, 1024), (32, 128, 1024), (8, 256, 2048), (16, 16, 512), (32, 64, 512)]]
else:
    pts_mw = None
pts = [("A", 32, 32, b, N, Lc) for (b, N, Lc) in
       [(1, 64, 1100), (1, 64, 2048), (1, 16, 4096), (1, 64, 8192), (2, 64, 2048), (2, 128, 4096), (4, 64, 1024),
        (4, 128, 2048), (8, 64, 1024), (8, 64, 4096), (16, 64, 2048), (32, 16, 1024), (1, 256, 8192),
        (8, 256, 2048)]] + \
      [("B", 8, 1, b, N, Lc) for (b, N, Lc) in [(1, 64, 4096), (8, 64, 4096), (8, 16, 8192), (32, 64, 4096),
                                               (16, 16, 32768)]]
pts = pts_mw or pts
hd = 128
if os.environ.get("K1_VARS") == "ks":  # 128-row kernel vs key-split row packing (N G <= 64)
    VARS = [("rows128", dict(attn_lean=0, attn_ks=0)), ("ks", dict(attn_lean=0, attn_ks=2))]
elif os.environ.get("K1_VARS") == "ksp":  # one-unit-per-CTA row-copy kernel vs the persistent one (units > 148)
    VARS = [("ks", dict(attn_ksp=0)), ("ksp", dict(attn_ksp=1))]
elif os.environ.get("K1_VARS") == "qearly":  # row-copy kernel: Q loads before vs after the CTA barrier
    VARS = [("late", dict(attn_qearly=0)), ("early", dict(attn_qearly=1))]
elif os.environ.get("K1_VARS") == "w2":  # 128 live rows: one vs two softmax warps per row
    VARS = [("w1", dict(attn_w2=0)), ("w2", dict(attn_w2=1))]
elif os.environ.get("K1_VARS") == "split":  # key-split count: round-1 rule vs occupancy-aware cost model
    VARS = [("rule", dict(attn_split_model=0)), ("model", dict(attn_split_model=1))]
elif os.environ.get("K1_VARS") == "l2":  # row-copy kernel: L2 prefetch ahead of the ring (attn_l2ahead bits)
    VARS = [("ks", dict(attn_l2ahead=0)), ("own", dict(attn_l2ahead=1)), ("next", dict(attn_l2ahead=2)),
            ("both", dict(attn_l2ahead=3))]
else:
    VARS = None
VARS = VARS or [("cl", dict(attn_lean=0)), ("l32", dict(attn_lean=1, attn_lean_div=32)), ("l16", dict(attn_lean=1, attn_lean_div=16)),
        ("l8", dict(attn_lean=1, attn_lean_div=8)), ("l4", dict(attn_lean=1, attn_lean_div=4))]
print(f"{'g':2s} {'b':>3s} {'N':>4s} {'Lc':>6s} {'MB':>7s} " + " ".join(f"{n:>7s}" for n, _ in VARS))
for g, H, Hkv, b, N, Lc in pts:
    tree = sm.Tree(synth.SWEEP_TREES[N]) if N != 64 else sm.Tree(synth.V64)
    cap = Lc + tree.N
    sets = []
    for _ in range(2):
        q = torch.randn(b, tree.N, H, hd, device="cuda").bfloat16()
        k = torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()
        v = torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()
        sets.append((q, k, v, torch.empty_like(q)))
    if globals().get("RAGGED"):
        lens = [Lc // 2 + (Lc - Lc // 2) * i // max(1, b - 1) for i in range(b)]
        L = torch.tensor(lens, dtype=torch.int32, device="cuda")
        alg = sum(Hkv * (lb + tree.N) * hd * 4 for lb in lens) + 2 * b * tree.N * H * hd * 2
    else:
        L = torch.full((b,), Lc, dtype=torch.int32, device="cuda")
        alg = b * Hkv * cap * hd * 4 + 2 * b * tree.N * H * hd * 2
    row = []
    for _, opts in VARS:
        for kk, vv in opts.items():
            sm.set_option(kk, vv)
        st = torch.cuda.Stream()
        for i in range(2):  # on the capture stream: sizes its stage scratch before the capture
            q, k, v, o = sets[i]
            sm.tree_attention(tree, q, k, v, L, H, Hkv, o, stream=st)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            gr.capture_begin()
            for i in range(20):
                q, k, v, o = sets[i % 2]
                sm.tree_attention(tree, q, k, v, L, H, Hkv, o, stream=st)
            gr.capture_end()
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        row.append(e0.elapsed_time(e1) * 1e3 / 60)
        del gr
    sm.reset_options()
    print(f"{g:2s} {b:3d} {tree.N:4d} {Lc:6d} {alg / 1e6:7.1f} " + " ".join(f"{u:7.1f}" for u in row) +
          "   best frac " + f"{alg / min(row) / 1e3 / PEAK:.3f}", flush=True)
    del sets
    torch.cuda.empty_cache()
