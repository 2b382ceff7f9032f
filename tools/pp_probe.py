"""Layer-split pipeline probe (GPU box): pp stages on one GPU, phase by phase, with the flag words
of every stage's symmetric buffer printed after each phase.  python tools/pp_probe.py pp [L]"""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

for kv_opt in filter(None, os.environ.get("SM_OPT", "").split(",")):  # sm_set_option knobs, e.g. pdl=0
    k_, v_ = kv_opt.split("=")
    sm.set_option(k_, int(v_))

pp = int(sys.argv[1])
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = synth.model_cfg("tiny", n_layers=L)
X = 96
tree = sm.Tree(synth.TINY16, topk=10)
R = 64
sym = [torch.zeros(sm.tp_sym_bytes(cfg, R, 1, 3), dtype=torch.uint8, device="cuda") for _ in range(pp)]
ptrs = [s.data_ptr() for s in sym]
Ws = [sm.allocate_weights(cfg, 3, seed=1, pp_rank=r, pp_size=pp) for r in range(pp)]
models = [sm.Model(cfg, Ws[r], R, 1, X + tree.N, peer_sym=ptrs) for r in range(pp)]
kvs = [sm.KVCache(m, tree, 1, X) for m in models]
sts = [torch.cuda.Stream() for _ in range(pp)]
torch.cuda.synchronize()
print("streams", [hex(s.cuda_stream) for s in sts], "CUDA_DEVICE_MAX_CONNECTIONS",
      os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"), flush=True)


def flags(tag):
    torch.cuda.synchronize()
    for r in range(pp):
        f = sym[r][: 8 * 8192 * 8].view(torch.int64).view(8, 8192)[:pp, :4].cpu().numpy()
        print(tag, "rank", r, "flags[src][0:4]", f.tolist(), flush=True)
    print(tag, "timed out", [m.tp_timed_out() for m in models], flush=True)


def each(fn):
    import time
    dts = []
    for r in range(pp):
        with torch.cuda.stream(sts[r]):
            t0 = time.perf_counter()
            fn(r, sts[r])
            dts.append(round((time.perf_counter() - t0) * 1e3, 2))
    print("host ms per rank enqueue", dts, flush=True)
    torch.cuda.synchronize()


pt = torch.from_numpy(synth.prompt_tokens(1, 0, 32, cfg["vocab"])).cuda()
each(lambda r, s: kvs[r].prefill(0, pt, stream=s))
flags("prefill")
tts = [torch.zeros(1, tree.N, dtype=torch.int32, device="cuda") for _ in range(pp)]
zs = [torch.zeros(1, tree.N, cfg["vocab"], dtype=torch.float32, device="cuda") for _ in range(pp)]
each(lambda r, s: kvs[r].propose(tts[r], stream=s))
each(lambda r, s: kvs[r].verify(tts[r], zs[r], stream=s))
flags("verify")
print("logits equal across ranks", all(torch.equal(zs[0], z) for z in zs), "finite", bool(torch.isfinite(zs[0]).all()))
outs = [sm.AcceptOut(1, tree.depth) for _ in range(pp)]
acfg = sm.accept_cfg(sm.GREEDY)
for k in range(3):
    each(lambda r, s: kvs[r].step(acfg, outs[r], stream=s))
    flags(f"step{k}")
    print("emitted", [o.emit_tok.cpu().tolist()[0] for o in outs], flush=True)
