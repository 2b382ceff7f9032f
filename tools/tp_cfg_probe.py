"""TP emulation probe (GPU box): t ranks on one GPU with a given model shape; prefill, one
propose + verify (logits finite?), then two steps (state sane?).
python tools/tp_cfg_probe.py t d H Hkv hd F V [pdl]"""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # one hardware queue per rank stream

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

for kv_opt in filter(None, os.environ.get("SM_OPT", "").split(",")):  # sm_set_option knobs, e.g. pdl=0
    k_, v_ = kv_opt.split("=")
    sm.set_option(k_, int(v_))

t, d, H, Hkv, hd, F, V = (int(x) for x in sys.argv[1:8])
pdl = int(sys.argv[8]) if len(sys.argv) > 8 else 0
sm.set_option("pdl", pdl)
cfg = synth.model_cfg("tiny", d_model=d, n_heads=H, n_kv_heads=Hkv, head_dim=hd, d_ffn=F, vocab=V)
X = 64
tree = sm.Tree(synth.TINY16, topk=10)
R = 64
nb = sm.tp_sym_bytes(cfg, R, 1, 3)
sym = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(t)]
ptrs = [x.data_ptr() for x in sym]
Ws = [sm.allocate_weights(cfg, 3, seed=0, tp_rank=r, tp_size=t) for r in range(t)]
models = [sm.Model(cfg, Ws[r], R, 1, X + tree.N, peer_sym=ptrs if t > 1 else None) for r in range(t)]
kvs = [sm.KVCache(m, tree, 1, X) for m in models]
sts = [torch.cuda.Stream() for _ in range(t)]
torch.cuda.synchronize()
pt = torch.from_numpy(synth.prompt_tokens(0, 0, 32, V)).cuda()


def each(fn):
    import time
    dts = []
    for r in range(t):
        with torch.cuda.stream(sts[r]):
            t0 = time.perf_counter()
            fn(r, sts[r])
            dts.append(round((time.perf_counter() - t0) * 1e3, 2))
    print("host ms per rank enqueue", dts, flush=True)
    torch.cuda.synchronize()


each(lambda r, s: kvs[r].prefill(0, pt, stream=s))
tts = [torch.zeros(1, tree.N, dtype=torch.int32, device="cuda") for _ in range(t)]
zs = [torch.zeros(1, tree.N, V // t, dtype=torch.float32, device="cuda") for _ in range(t)]
each(lambda r, s: kvs[r].propose(tts[r], stream=s))
print("tree tokens", [tt[0, :6].tolist() for tt in tts[:2]], flush=True)
each(lambda r, s: kvs[r].verify(tts[r], zs[r], stream=s))
for r in range(t):
    z = zs[r]
    print(f"rank {r} logits finite {bool(torch.isfinite(z).all())} maxabs {float(z.abs().max()):.4f}", flush=True)
outs = [sm.AcceptOut(1, tree.depth) for _ in range(t)]
acfg = sm.accept_cfg(sm.GREEDY)
each(lambda r, s: kvs[r].accept(acfg, outs[r], stream=s))
print("accept", [o.emit_tok.cpu().tolist()[0] for o in outs[:2]], flush=True)
each(lambda r, s: kvs[r].propose(tts[r], stream=s))
print("tree tokens after", [tt[0, :6].tolist() for tt in tts[:2]], flush=True)
print("timed out", any(m.tp_timed_out() for m in models))
