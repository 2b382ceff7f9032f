"""Diagnostic (GPU box): bf16 rounding noise at 7B width (2 layers) -- how far do the
GPU's bf16 logits / K/V sit from the oracle's bf16 mode, from the fp64 definition, and how
far do two equally valid bf16 implementations of the definition sit from each other
(oracle bf16 with fp64 accumulation vs the same storage points with fp32 BLAS accumulation)?

python tools/diag_bf16_noise.py [seed] [n_layers]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402
from oracle import model as OM  # noqa: E402
from oracle import spec as OS  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 11
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 2
C2 = synth.model_cfg("vicuna7b", n_layers=nl)
PROMPT = 12
W = sm.allocate_weights(C2, 4, seed=0, medusa_init=True)
tree = sm.Tree(synth.V64, topk=10)
model = sm.Model(C2, W, max_rows=64, max_batch=1, max_seq_len=64 + tree.N)
kv = sm.KVCache(model, tree, 1, 64)
prompt = synth.prompt_tokens(seed, 0, PROMPT, C2["vocab"])
kv.prefill(0, torch.from_numpy(prompt).cuda())
tt = torch.zeros(1, tree.N, dtype=torch.int32, device="cuda")
kv.propose(tt)
logits = torch.zeros(1, tree.N, C2["vocab"], dtype=torch.float32, device="cuda")
kv.verify(tt, logits)
torch.cuda.synchronize()
tok = tt[0].cpu().tolist()
Zg = logits[0].cpu().numpy().astype(np.float64)
kvl = kv.layout().float().cpu().numpy().astype(np.float64)

res = {}
for name, mode, dt in (("bf16", "bf16", np.float64), ("bf16_f32acc", "bf16", np.float32), ("fp64", "fp64", np.float64)):
    Wo = OM.Weights(C2, n_medusa=4, seed=0, medusa_init=True, dtype=dt)
    s = OS.Session(OM.Model(C2, Wo, mode), synth.V64, 1, 64, batched=True)
    s.prefill(0, prompt)
    tok_o, _ = s.propose(0)
    Z, _ = s.verify(0, tok)  # the GPU's tree tokens (lock step)
    res[name] = dict(Z=np.stack(Z).astype(np.float64), tok=list(tok_o),
                     K=[np.asarray(s.kv.K[li][0], np.float64) for li in range(nl)],
                     V=[np.asarray(s.kv.V[li][0], np.float64) for li in range(nl)])
    del Wo, s


def stats(got, ref):
    e = np.abs(got - ref)
    bar = 2e-2 * (1 + np.abs(ref))
    return dict(max=float(e.max()), rms=float(np.sqrt((e ** 2).mean())), ref_rms=float(np.sqrt((ref ** 2).mean())),
                max_over_bar=float((e / bar).max()), frac_over_bar=float((e > bar).mean()),
                frac_over_2bar=float((e > 2 * bar).mean()), frac_differ=float((e > 0).mean()))


out = {"seed": seed, "layers": nl, "tok_agree": {k: sum(int(a == b) for a, b in zip(tok, v["tok"])) for k, v in res.items()}}
pairs = [("gpu", "bf16"), ("gpu", "fp64"), ("bf16", "fp64"), ("bf16_f32acc", "bf16"), ("bf16_f32acc", "fp64")]
slots = list(range(PROMPT + tree.N))
for a, b in pairs:
    A = Zg if a == "gpu" else res[a]["Z"]
    B = res[b]["Z"]
    out[f"logits {a} vs {b}"] = stats(A, B)
    rows = [stats(A[n], B[n])["frac_over_bar"] for n in range(tree.N)]
    out[f"logits {a} vs {b}"]["worst_row_frac_over_bar"] = max(rows)
    for li in range(nl):
        for c, key in ((0, "K"), (1, "V")):
            GA = kvl[li, c, 0][:, slots] if a == "gpu" else res[a][key][li][:, slots]
            GB = res[b][key][li][:, slots]
            out[f"{key}{li} {a} vs {b}"] = stats(GA, GB)
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/diag_bf16_noise_s{seed}_L{nl}.json", "w") as f:
    json.dump(out, f, indent=1)
