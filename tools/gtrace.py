"""Cross-kernel timeline of one C2 step from per-CTA %globaltimer records
(diagnostics build).  GPU box only:

  python -m paper_2506_01986_b200.build --trace
  SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so python tools/gtrace.py

For each launch of layers 1-2: first CTA entry, when griddepcontrol.wait returned
(first / median / last CTA), first and last CTA exit -- in us from the step start."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

L = sm.lib()
assert hasattr(L, "sm_gtrace_read_gemm"), "needs SPECMEMO_LIB=.../libspecmemo_trace.so"
for kv_opt in filter(None, os.environ.get("SM_OPT", "").split(",")):
    k, v = kv_opt.split("=")
    L.sm_set_option(k.encode(), int(v))
cfg = synth.model_cfg("vicuna7b")
tree = sm.Tree(synth.V64)
W = sm.allocate_weights(cfg, 4, seed=0)
B = int(os.environ.get("GT_BATCH", "1"))  # GT_BATCH=10: the batched step (M = 640)
model = sm.Model(cfg, W, max_rows=max(256, B * tree.N), max_batch=B, max_seq_len=2048 + tree.N)
kv = sm.KVCache(model, tree, B, 2048)
for i in range(B):
    kv.prefill(i, torch.from_numpy(synth.prompt_tokens(0, i, 1024 if B == 1 else 512 + 16 * i, cfg["vocab"])).cuda())
out = sm.AcceptOut(B, tree.depth)
acfg = sm.accept_cfg(sm.GREEDY)
for _ in range(4):
    kv.step(acfg, out)
torch.cuda.synchronize()
buf = np.zeros((1 << 17, 4), dtype=np.int64)
readers = [L.sm_gtrace_read_gemm, L.sm_gtrace_read_epi, L.sm_gtrace_read_attn]
for r in readers:  # clear
    r(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int(1 << 17))
kv.step(acfg, out)
torch.cuda.synchronize()
recs = []
for r in readers:
    n = r(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int(1 << 17))
    recs.append(buf[:n].copy())
R = np.concatenate(recs)
t0 = R[:, 1].min()
names = {1: "resid_norm", 2: "qkv_consumer", 3: "silu", 5: "attention"}
N2 = {12288 // 128: "GEMM qkv", 4096 // 128: "GEMM o/down", 22016 // 128: "GEMM gate/up", 32000 // 128: "GEMM lm",
      4096 // 128 + 0: "GEMM o/down"}
launches = []
for kid in np.unique(R[:, 0]):
    rk = R[R[:, 0] == kid]
    rk = rk[np.argsort(rk[:, 1])]
    cut = np.where(np.diff(rk[:, 1]) > 4000)[0] + 1  # > 4 us between entries: next launch
    for g in np.split(rk, cut):
        nm = names.get(int(kid), N2.get(int(kid) - 1000, f"GEMM N/128={int(kid) - 1000}") if kid >= 1000 else str(kid))
        w = g[:, 2][g[:, 2] > 0]
        launches.append((g[:, 1].min(), nm, len(g), g[:, 1].max(), (w.min(), np.median(w), w.max()) if len(w) else None,
                         g[:, 3].min(), g[:, 3].max()))
launches.sort()
print(f"{'launch':14s} {'ctas':>5s} {'entry0':>8s} {'entryN':>8s} {'wait0':>8s} {'waitMed':>8s} {'waitN':>8s} "
      f"{'exit0':>8s} {'exitN':>8s}")
us = lambda t: (t - t0) / 1e3  # noqa: E731
for e0, nm, n, eN, w, x0, xN in launches[:40]:
    ws = " ".join(f"{us(v):8.1f}" for v in w) if w else " " * 26
    print(f"{nm:14s} {n:5d} {us(e0):8.1f} {us(eN):8.1f} {ws} {us(x0):8.1f} {us(xN):8.1f}")
