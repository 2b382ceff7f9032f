"""Diagnostic (GPU box): where do bf16 GPU and bf16-emulating oracle diverge at C2
widths (2 layers)?  Prints error statistics of K/V per layer and of the logits of
sampled tree rows, for the plain oracle and for an oracle variant whose attention
rounds P to bf16 before P.V (as the GPU's MMA operand does, R4 note).

python tools/diag_c2_bf16.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402
from oracle import model as OM  # noqa: E402
from oracle import spec as OS  # noqa: E402
from oracle import tree as OT  # noqa: E402

C2 = synth.model_cfg("vicuna7b", n_layers=2)
PROMPT = 12
t = OT.build(synth.V64)
SAMPLE = sorted({0, *range(1, 11), *OT.ancestors(t, 57), 57})

W = sm.allocate_weights(C2, 4, seed=0, medusa_init=True)
tree = sm.Tree(synth.V64, topk=10)
model = sm.Model(C2, W, max_rows=64, max_batch=1, max_seq_len=64 + tree.N)
kv = sm.KVCache(model, tree, 1, 64)
prompt = synth.prompt_tokens(11, 0, PROMPT, C2["vocab"])
kv.prefill(0, torch.from_numpy(prompt).cuda())
tt = torch.zeros(1, tree.N, dtype=torch.int32, device="cuda")
kv.propose(tt)
logits = torch.zeros(1, tree.N, C2["vocab"], dtype=torch.float32, device="cuda")
kv.verify(tt, logits)
torch.cuda.synchronize()
tok = tt[0].cpu().tolist()
Zg = logits[0].cpu().numpy().astype(np.float64)
kvl = kv.layout()
Wo = OM.Weights(C2, n_medusa=4, seed=0, medusa_init=True)


def attention_pround(self, q, Kc, Vc):
    out = np.zeros((self.H, self.hd))
    scale = 1.0 / np.sqrt(self.hd)
    for h in range(self.H):
        kvh = h // self.G
        s = Kc[:, kvh, :] @ q[h] * scale
        p = np.exp(s - s.max())
        out[h] = OM.round_bf16(p) @ Vc[:, kvh, :] / p.sum()
    return out


for variant in ("plain", "p_bf16"):
    m = OM.Model(C2, Wo, "bf16")
    if variant == "p_bf16":
        m.attention = attention_pround.__get__(m)
    s = OS.Session(m, synth.V64, 1, 64)
    s.prefill(0, prompt)
    for n in SAMPLE:
        keys = list(range(PROMPT)) + [PROMPT + a for a in OT.ancestors(s.tree, n)] + [PROMPT + n]
        z, _ = m.forward_row(s.kv, 0, int(tok[n]), PROMPT + s.tree.depth[n], PROMPT + n, keys)
        e = np.abs(Zg[n] - z)
        print(f"{variant:7s} node {n:2d}: logit err max {e.max():.4f} rms {np.sqrt((e**2).mean()):.5f}  "
              f"|z| rms {np.sqrt((z**2).mean()):.3f}  frac>2e-2(1+|z|) {np.mean(e > 2e-2 * (1 + np.abs(z))):.2e}")
    slots = list(range(PROMPT)) + [PROMPT + n for n in SAMPLE]
    for li in range(2):
        for c in (0, 1):
            got = kvl[li, c, 0].float().cpu().numpy().astype(np.float64)[:, slots]
            ref = (s.kv.K if c == 0 else s.kv.V)[li][0][:, slots]
            e = np.abs(got - ref)
            print(f"{variant:7s} layer {li} {'KV'[c]}: max {e.max():.4f} rms {np.sqrt((e**2).mean()):.5f} "
                  f"|ref| rms {np.sqrt((ref**2).mean()):.3f} frac differing {np.mean(e > 0):.3f}")
