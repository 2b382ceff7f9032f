"""f4 comparison (the shape of fig:distributed): batched speculative
decoding on B200, ragged lengths vs the paper's pad batching, against vanilla batched decoding
on the same kernels.  Vicuna-7B shape, V64 tree, bs in {1, 2, 4, 8, 10}.

Random weights accept ~1 token per step, so acceptance is imposed with the d_forced_path hook:
sequence s accepts a full-depth path of depth (s mod 5) every step (tau = 1..5 across the batch,
mean 3), the spread that makes pad batching pay: every cache advances by the batch's longest
acceptance (5) while a sequence commits only its own.  Reported per point: ms/step, tokens/s
(committed tokens), cache slots per committed token (pad overhead).  GPU box:
python tools/batch_sweep.py > profiles/r01_batch_sweep.txt"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

cfg = synth.model_cfg("vicuna7b")
W = sm.allocate_weights(cfg, 4, seed=0)
STEPS, X = int(os.environ.get("BATCH_STEPS", "30")), 2048
tree = sm.Tree(synth.V64)
q = tree.query()
depth, parent = q["node_depth"], q["parent"]
deep = int(np.flatnonzero(depth == 4)[0])
chain = [deep]
while chain[-1] != 0:
    chain.append(int(parent[chain[-1]]))
chain = chain[::-1]  # root .. a depth-4 node


def run(b, mode):
    t = sm.Tree([]) if mode == "vanilla" else tree
    model = sm.Model(cfg, W, max_rows=max(256, b * t.N), max_batch=b, max_seq_len=X + t.N)
    kv = sm.KVCache(model, t, b, X)
    for i in range(b):
        kv.prefill(i, torch.from_numpy(synth.prompt_tokens(0, i, 512 + 16 * i, cfg["vocab"])).cuda())
    if mode == "pad":
        kv.set_pad_mode(True)
    out = sm.AcceptOut(b, t.depth)
    if mode == "vanilla":
        acfg = sm.accept_cfg()
    else:
        forced = torch.full((b, t.depth + 1), -1, dtype=torch.int32)
        for s in range(b):
            d = s % 5
            forced[s, : d + 1] = torch.tensor(chain[: d + 1], dtype=torch.int32)
        forced = forced.cuda()
        acfg = sm.accept_cfg(forced_path=forced)
    for _ in range(3):
        kv.step(acfg, out)
    torch.cuda.synchronize()
    P0, L0 = kv.positions().astype(np.int64), kv.lengths().astype(np.int64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(STEPS):
        kv.step(acfg, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / STEPS
    P1, L1 = kv.positions().astype(np.int64), kv.lengths().astype(np.int64)
    tok = float((P1 - P0).sum())
    slots = float((L1 - L0).sum())
    del kv, model
    torch.cuda.empty_cache()
    return ms, tok / STEPS / (ms / 1e3), slots / tok


for kv_opt in filter(None, os.environ.get("SM_OPT", "").split(",")):  # experiment knobs (sm_set_option)
    k_, v_ = kv_opt.split("=")
    sm.set_option(k_, int(v_))
BS = [int(x) for x in os.environ.get("BATCH_SIZES", "1,2,4,8,10").split(",")]
MODES = os.environ.get("BATCH_MODES", "vanilla,ragged,pad").split(",")
print("# f4: batched speculative decoding, ragged vs pad batching (P:253-256) vs vanilla; Vicuna-7B shape, V64,")
print("# imposed acceptance depth (s mod 5) per sequence s; ms/step, tokens/s, cache slots per committed token")
print(f"{'bs':>3s} {'mode':8s} {'ms/step':>8s} {'tok/s':>9s} {'slots/tok':>9s}")
for b in BS:
    for mode in MODES:
        ms, tps, spt = run(b, mode)
        print(f"{b:3d} {mode:8s} {ms:8.3f} {tps:9.1f} {spt:9.2f}", flush=True)
