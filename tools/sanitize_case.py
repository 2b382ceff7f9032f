"""One small speculative decode for compute-sanitizer (tools/sanitize.sh): c1 = the tiny
C1 model (mma.sync K1, hd 16); s128 = a hd-128 model (tcgen05 K1 with split-KV cluster
combine, tcgen05 K2, 2 sequences, prefill + 6 greedy steps with compaction)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

case = sys.argv[1]
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
for _ in range(6):
    kv.step(cfg_a, out)
torch.cuda.synchronize()
print("lengths", kv.lengths().tolist(), "emitted", out.n_emit.cpu().tolist())
