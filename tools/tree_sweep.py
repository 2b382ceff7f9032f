"""fig:maskmodel-style per-step latency sweep on B200:
Vicuna-7B-shaped model (32 layers, random init), Medusa heads 2..5, masks of 5..64 nodes
(V64 restricted to the head depth, then R4-pruned in place, plus SpecMemo's custom
(N, S) trees of tab:treefeatures), committed KV length 512 / 1024 / 2048.

For each point: device time per speculative step (CUDA events over 30 graph-replayed steps)
and the break-even acceptance length tau* = t_step / t_vanilla -- the mean tokens per step a
tree must accept to beat plain greedy decoding on the same kernels (random weights accept
~1 token/step, so tokens/s itself is not meaningful here).  The cheapest tree per
(heads, KV) at equal tau* is what a tree-size selector would pick.

python tools/tree_sweep.py [--quick] > profiles/r01_tree_sweep.txt   (GPU box)"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
cfg = synth.model_cfg("vicuna7b")
HEADS = [2, 3, 4, 5] if not a.quick else [3, 4]
SIZES = [5, 16, 27, 31, 44, 64]
LCS = [512, 1024, 2048] if not a.quick else [1024]
X = max(LCS) + 8 * a.steps + 64
W = sm.allocate_weights(cfg, max(HEADS), seed=0)
v64 = sm.Tree(synth.V64)


def trees_for(h):
    """(label, Tree): V64 cut to depth h, R4-pruned to each size; custom (N, S) trees."""
    cut = [c for c in synth.V64 if len(c) <= h]
    base = sm.Tree(cut)
    out = [("vanilla", sm.Tree([]))]
    for n in SIZES:
        if n <= base.N:
            t = base.pruned(n)
            out.append((f"M-pruned N={t.N:2d} S={t.S:2d}", t))
    if h == 4:
        for n, s in ((44, 37), (64, 56)):
            t = sm.Tree.custom(n, s, 10, 4)
            out.append((f"custom   N={n:2d} S={s:2d}", t))
    return out


def step_ms(model, tree, Lc):
    kv = sm.KVCache(model, tree, 1, X)
    kv.prefill(0, torch.from_numpy(synth.prompt_tokens(0, 0, Lc, cfg["vocab"])).cuda())
    out = sm.AcceptOut(1, tree.depth)
    acfg = sm.accept_cfg(sm.GREEDY)
    for _ in range(3):
        kv.step(acfg, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        kv.step(acfg, out)
    e1.record()
    torch.cuda.synchronize()
    del kv
    return e0.elapsed_time(e1) / a.steps


print(f"# B200 per-step latency (ms) and break-even tau* = t_step / t_vanilla; Vicuna-7B shape, bs=1, bf16")
print(f"{'heads':>5s} {'tree':24s} " + " ".join(f"{'Lc=' + str(l):>16s}" for l in LCS))
for h in HEADS:
    Wh = dict(W)
    Wh["medusa"] = W["medusa"][:h]
    model = sm.Model(cfg, Wh, max_rows=256, max_batch=1, max_seq_len=X + 64)
    van = {}
    for label, tree in trees_for(h):
        cells = []
        for Lc in LCS:
            ms = step_ms(model, tree, Lc)
            if label == "vanilla":
                van[Lc] = ms
            cells.append(f"{ms:7.3f} ({ms / van[Lc]:5.2f}x)")
        print(f"{h:5d} {label:24s} " + " ".join(f"{c:>16s}" for c in cells), flush=True)
    del model
    torch.cuda.empty_cache()
