"""Diagnostic: t = 8 ranks on one GPU (tests/test_gpu_tp.py CFG8) with a given vocabulary and PDL
setting; prints the emitted tokens or the failure.  python tools/tp8_diag.py <vocab> <pdl>"""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # one hardware queue per rank stream

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

V, pdl = int(sys.argv[1]), int(sys.argv[2])
t = int(sys.argv[3]) if len(sys.argv) > 3 else 8
rsag = int(sys.argv[4]) if len(sys.argv) > 4 else -1
small = len(sys.argv) > 5 and sys.argv[5] == "tiny"
sm.set_option("pdl", pdl)
sm.set_option("tp_rsag", rsag)
cfg = synth.model_cfg("tiny", vocab=V) if small else \
    synth.model_cfg("tiny", d_model=128, n_heads=8, n_kv_heads=8, head_dim=16, d_ffn=512, vocab=V)
X = 64
tree = sm.Tree(synth.TINY16, topk=10)
R = 64
nb = sm.tp_sym_bytes(cfg, R, 1, 3)
sym = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(t)]
ptrs = [x.data_ptr() for x in sym]
Ws = [sm.allocate_weights(cfg, 3, seed=0, tp_rank=r, tp_size=t) for r in range(t)]
models = [sm.Model(cfg, Ws[r], R, 1, X + tree.N, peer_sym=ptrs) for r in range(t)]
kvs = [sm.KVCache(m, tree, 1, X) for m in models]
sts = [torch.cuda.Stream() for _ in range(t)]
torch.cuda.synchronize()
pt = torch.from_numpy(synth.prompt_tokens(0, 0, 32, V)).cuda()
for r in range(t):
    with torch.cuda.stream(sts[r]):
        kvs[r].prefill(0, pt, stream=sts[r])
torch.cuda.synchronize()
print("prefill ok", flush=True)
import ctypes  # noqa: E402


def _cudart():
    import glob

    import nvidia.cuda_runtime
    lib = glob.glob(os.path.join(nvidia.cuda_runtime.__path__[0], "lib", "libcudart.so*"))[0]
    return ctypes.CDLL(lib)


CUDART = _cudart()


def topk_state(kv):
    import numpy as np
    r, t_, nmed = kv.state()
    n = nmed * 10
    torch.cuda.synchronize()
    arr = np.zeros(n, np.int32)
    CUDART.cudaMemcpy(ctypes.c_void_p(arr.ctypes.data), ctypes.c_void_p(t_), ctypes.c_size_t(n * 4), 2)
    root = np.zeros(1, np.int32)
    CUDART.cudaMemcpy(ctypes.c_void_p(root.ctypes.data), ctypes.c_void_p(r), ctypes.c_size_t(4), 2)
    return int(root[0]), arr.reshape(nmed, 10).tolist()


for r in range(t):
    print("rank", r, "state", topk_state(kvs[r]), flush=True)
outs = [sm.AcceptOut(1, tree.depth) for _ in range(t)]
cfgs = sm.accept_cfg(sm.GREEDY)
for k in range(4):
    for r in range(t):
        with torch.cuda.stream(sts[r]):
            kvs[r].step(cfgs, outs[r], stream=sts[r])
    torch.cuda.synchronize()
    print("step", k, [o.emit_tok.cpu().tolist()[0] for o in outs[:2]], flush=True)
    for r in range(t):
        print("rank", r, "state", topk_state(kvs[r]), flush=True)
print("timed out", any(m.tp_timed_out() for m in models))
