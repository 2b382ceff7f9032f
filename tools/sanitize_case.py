"""One small speculative decode for compute-sanitizer (tools/sanitize.sh): c1 = the tiny
C1 model (mma.sync K1, hd 16); k1new = the session-3 K1 kernels (persistent KSP, two softmax warps per row, odd
split counts, early Q); tp2emu = t = 2 tensor parallelism in the host-ordered emulation; s128 = a hd-128 model (tcgen05 K1 with split-KV cluster
combine, tcgen05 K2, 2 sequences, prefill + 6 greedy steps with compaction); pp2 = the
layer-split pipeline (two stages on one GPU, host-ordered emulation: residual hand-offs joined by
events, one host thread per stage); pad = s128 in pad
batching through sm_propose / sm_verify / sm_accept (pad masks, the copy kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

case = sys.argv[1]
if case == "pp2":
    cfg, X = synth.model_cfg("tiny", n_layers=4), 96
    tree = sm.Tree(synth.TINY16, topk=10)
    sym = [torch.zeros(sm.tp_sym_bytes(cfg, 64, 1, 3), dtype=torch.uint8, device="cuda") for _ in range(2)]
    ptrs = [t.data_ptr() for t in sym]
    Ws = [sm.allocate_weights(cfg, 3, seed=1, pp_rank=r, pp_size=2) for r in range(2)]
    emu = sm.EmuGroup(2)
    models = [sm.Model(cfg, Ws[r], 64, 1, X + tree.N, peer_sym=ptrs, emu_group=emu) for r in range(2)]
    kvs = [sm.KVCache(m, tree, 1, X) for m in models]
    sts = [torch.cuda.Stream() for _ in range(2)]
    outs = [sm.AcceptOut(1, tree.depth) for _ in range(2)]
    torch.cuda.synchronize()
    pt = torch.from_numpy(synth.prompt_tokens(1, 0, 32, cfg["vocab"])).cuda()

    def each(fn):
        def go(r):
            def body():
                with torch.cuda.stream(sts[r]):
                    fn(r, sts[r])
            return body
        sm.run_ranks([go(r) for r in range(2)])
        torch.cuda.synchronize()
    each(lambda r, s: kvs[r].prefill(0, pt, stream=s))
    for _ in range(4):
        each(lambda r, s: kvs[r].step(sm.accept_cfg(sm.GREEDY), outs[r], stream=s))
    print("lengths", [kv.lengths().tolist() for kv in kvs], "timed out", [m.tp_timed_out() for m in models])
    sys.exit(0)
if case == "k1new":  # session-3 K1 paths through the stage entry: persistent KSP (160 units, F = 2 and W2
    # F = 1), the row-copy kernel with W2 and an odd split count, early Q loads
    hd = 128
    for (b, H, Hkv, N, Lc, splits) in [(5, 32, 32, 64, 300, 0), (10, 128, 16, 16, 200, 0), (2, 16, 2, 64, 700, 3),
                                       (1, 8, 1, 16, 2000, 7)]:
        tree = sm.Tree(synth.V64) if N == 64 else sm.Tree(synth.TINY16, topk=10)
        sm.set_option("attn_splits", splits)
        cap = Lc + tree.N + 5
        q = torch.randn(b, tree.N, H, hd, device="cuda").bfloat16()
        k = torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()
        v = torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()
        o = torch.empty_like(q)
        L = torch.tensor([Lc - 13 * i for i in range(b)], dtype=torch.int32, device="cuda")
        for _ in range(2):
            sm.tree_attention(tree, q, k, v, L, H, Hkv, o)
        torch.cuda.synchronize()
        print("k1", b, H, Hkv, tree.N, Lc, splits, bool(torch.isfinite(o.float()).all()))
    sys.exit(0)
if case == "tp2emu":  # tensor parallel t = 2 in the host-ordered emulation (segment launches + event joins)
    cfg, X = synth.model_cfg("tiny"), 64
    tree = sm.Tree(synth.TINY16, topk=10)
    sym = [torch.zeros(sm.tp_sym_bytes(cfg, 64, 1, 3), dtype=torch.uint8, device="cuda") for _ in range(2)]
    ptrs = [t.data_ptr() for t in sym]
    emu = sm.EmuGroup(2)
    Ws = [sm.allocate_weights(cfg, 3, seed=1, tp_rank=r, tp_size=2) for r in range(2)]
    models = [sm.Model(cfg, Ws[r], 64, 1, X + tree.N, peer_sym=ptrs, emu_group=emu) for r in range(2)]
    kvs = [sm.KVCache(m, tree, 1, X) for m in models]
    sts = [torch.cuda.Stream() for _ in range(2)]
    outs = [sm.AcceptOut(1, tree.depth) for _ in range(2)]
    torch.cuda.synchronize()
    pt = torch.from_numpy(synth.prompt_tokens(1, 0, 32, cfg["vocab"])).cuda()

    def each2(fn):
        def go(r):
            def body():
                with torch.cuda.stream(sts[r]):
                    fn(r, sts[r])
            return body
        sm.run_ranks([go(r) for r in range(2)])
        torch.cuda.synchronize()
    each2(lambda r, s: kvs[r].prefill(0, pt, stream=s))
    for _ in range(4):
        each2(lambda r, s: kvs[r].step(sm.accept_cfg(sm.GREEDY), outs[r], stream=s))
    print("lengths", [kv.lengths().tolist() for kv in kvs], "timed out", [m.tp_timed_out() for m in models])
    sys.exit(0)
if case == "c1":
    cfg, b, x, init = synth.model_cfg("tiny"), 1, 64, False
else:
    cfg = synth.model_cfg("tiny", d_model=256, n_heads=2, n_kv_heads=1, head_dim=128, d_ffn=512, vocab=512)
    b, x, init = 2, 600, True
W = sm.allocate_weights(cfg, 3, seed=1, medusa_init=init)
tree = sm.Tree(synth.TINY16, topk=10)
model = sm.Model(cfg, W, max_rows=max(64, b * tree.N), max_batch=b, max_seq_len=x + tree.N)
kv = sm.KVCache(model, tree, b, x)
for s in range(b):
    n = 32 if case == "c1" else 520 + 7 * s  # several 64-key tiles and a ragged tail per sequence
    kv.prefill(s, torch.from_numpy(synth.prompt_tokens(1, s, n, cfg["vocab"])).cuda())
out = sm.AcceptOut(b, tree.depth)
cfg_a = sm.accept_cfg(sm.GREEDY)
if case == "pad":
    kv.set_pad_mode(True)
    kv.step(cfg_a, out)  # aligns the ragged prompts
    for _ in range(4):
        tt = torch.zeros(b, tree.N, dtype=torch.int32, device="cuda")
        z = torch.zeros(b, tree.N, cfg["vocab"], dtype=torch.float32, device="cuda")
        kv.propose(tt)
        kv.verify(tt, z)
        kv.accept(cfg_a, out)
for _ in range(6):
    kv.step(cfg_a, out)
torch.cuda.synchronize()
print("lengths", kv.lengths().tolist(), "emitted", out.n_emit.cpu().tolist())
