"""Phase timeline of the tcgen05 K1 kernel (diagnostics build, GPU box).

python -m paper_2506_01986_b200.build --trace
SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so python tools/attn_trace.py [--b 1 --H 32 --Hkv 32 --lc 1100]
Prints, per stamp slot, the median / max over CTAs of clock64 cycles since the CTA's first stamp."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

NAMES = {0: "start", 1: "prologue done", 2: "softmax pdl_wait done", 3: "Q staged", 4: "S(0) ready",
         5: "S(last) ready", 6: "last PV done", 8: "cluster sync 1",
         9: "combined + written", 10: "cluster sync 2", 11: "producer: prefix issued", 12: "producer: pdl_wait done",
         13: "producer: last tile issued", 14: "mma: Q ready", 15: "sm: S(8) ready", 16: "sm: S(8) in regs",
         17: "sm: P(8) computed", 18: "sm: P(8) stored+arrived", 19: "mma: P(8) seen", 20: "mma: K/V(9) landed",
         21: "sm: S(9) ready", 22: "producer: K/V(9) issued"}

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, default=1)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--Hkv", type=int, default=32)
ap.add_argument("--lc", type=int, default=1100)
ap.add_argument("--N", type=int, default=64)
ap.add_argument("--splits", type=int, default=0)
a = ap.parse_args()

L = sm.lib()
assert hasattr(L, "sm_trace_read"), "needs SPECMEMO_LIB=.../libspecmemo_trace.so"
tree = sm.Tree(synth.V64) if a.N == 64 else sm.Tree(synth.SWEEP_TREES[a.N])
if a.splits:
    sm.set_option("attn_splits", a.splits)
N, cap, hd = tree.N, a.lc + tree.N, 128
q = torch.randn(a.b, N, a.H, hd, device="cuda").bfloat16()
k = torch.randn(a.b, a.Hkv, cap, hd, device="cuda").bfloat16()
v = torch.randn(a.b, a.Hkv, cap, hd, device="cuda").bfloat16()
o = torch.empty_like(q)
lens = torch.full((a.b,), a.lc, dtype=torch.int32, device="cuda")
for _ in range(5):
    sm.tree_attention(tree, q, k, v, lens, a.H, a.Hkv, o)
torch.cuda.synchronize()
buf = np.zeros((1024, 24), dtype=np.int64)
L.sm_trace_read(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int(buf.size))
live = buf[buf[:, 0] != 0]
rel = live - live[:, :1]
print(f"{len(live)} CTAs; cycles since CTA start (median / max)")
for s, name in NAMES.items():
    col = rel[:, s][live[:, s] != 0]
    if len(col):
        print(f"  {s:2d} {name:28s} {int(np.median(col)):8d} {int(col.max()):8d}")
starts = live[:, 0]
t = live[:, 4:6]
ok = (live[:, 4] != 0) & (live[:, 5] != 0)
if ok.any():
    print("mean cycles per tile (S(last) - S(0)) / (tiles - 1) needs tiles; raw S(last)-S(0) median:",
          int(np.median(live[ok, 5] - live[ok, 4])))
print("CTA start spread (cycles, SM clocks not synchronised):", int(starts.max() - starts.min()))
