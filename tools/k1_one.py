"""One K1 configuration for ncu (GPU box): python tools/k1_one.py b N Lc H Hkv [opt=val ...]
(8 launches on two alternating buffer sets)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

b, N, Lc, H, Hkv = (int(x) for x in sys.argv[1:6])
for kv in sys.argv[6:]:
    k, v = kv.split("=")
    sm.set_option(k, int(v))
tree = sm.Tree(synth.SWEEP_TREES[N]) if N != 64 else sm.Tree(synth.V64)
hd, cap = 128, Lc + tree.N
sets = []
for _ in range(2):
    sets.append((torch.randn(b, tree.N, H, hd, device="cuda").bfloat16(), torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16(),
                 torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()))
L = torch.full((b,), Lc, dtype=torch.int32, device="cuda")
o = torch.empty_like(sets[0][0])
for i in range(8):
    q, k, v = sets[i % 2]
    sm.tree_attention(tree, q, k, v, L, H, Hkv, o)
torch.cuda.synchronize()
print("ok")
