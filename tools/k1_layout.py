"""K1 sensitivity to the KV cache slot stride (GPU box): one C5 point timed with cap = Lc + N + pad for several
pads, each allocation timed twice (fresh buffers), 20 graph-replayed launches over two buffer sets.

python tools/k1_layout.py [b N Lc]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

b, N, Lc = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (8, 128, 1024)))
H = Hkv = 32
hd = 128
tree = sm.Tree(synth.SWEEP_TREES[N]) if N != 64 else sm.Tree(synth.V64)
pads = [0, 16, 64, 128, 1, 3]
if os.environ.get("K1_CHURN"):  # after large allocations are freed (the sweep's history)
    pads = [0, 0, 0]
for pad in pads:
    if os.environ.get("K1_CHURN"):
        big = [torch.empty(int(float(os.environ["K1_CHURN"]) * 2**30), dtype=torch.uint8, device="cuda") for _ in range(2)]
        big[0].fill_(1)
        del big
        torch.cuda.empty_cache()
    for rep in range(2):
        cap = Lc + tree.N + pad
        sets = [(torch.randn(b, tree.N, H, hd, device="cuda").bfloat16(), torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16(),
                 torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()) for _ in range(2)]
        o = torch.empty_like(sets[0][0])
        L = torch.full((b,), Lc, dtype=torch.int32, device="cuda")
        st = torch.cuda.Stream()
        for i in range(2):
            sm.tree_attention(tree, *sets[i], L, H, Hkv, o, stream=st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            g.capture_begin()
            for i in range(20):
                sm.tree_attention(tree, *sets[i % 2], L, H, Hkv, o, stream=st)
            g.capture_end()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"pad {pad:4d} rep {rep}: {e0.elapsed_time(e1) * 1e3 / 60:7.1f} us", flush=True)
        del sets, g
        torch.cuda.empty_cache()
