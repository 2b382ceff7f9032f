"""Per-CTA timeline of the K1 row-copy kernel (diagnostics build, GPU box).

  python -m paper_2506_01986_b200.build --trace
  SPECMEMO_LIB=paper_2506_01986_b200/libspecmemo_trace.so python tools/k1_timeline.py [b N Lc ...]

For each C5 geometry-A point (b, N, Lc): one launch through sm_tree_attention after warm-up, then
from the %globaltimer stamps of every CTA: the kernel span, the median CTA phases (entry -> Q
staged -> first K/V tile landed -> last PV retired -> exit), how many CTAs each SM ran, and the
idle gap on an SM between one CTA's exit and the next CTA's entry."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

L = sm.lib()
assert hasattr(L, "sm_trace_read_ks"), "needs SPECMEMO_LIB=.../libspecmemo_trace.so"
for kv_opt in filter(None, os.environ.get("SM_OPT", "").split(",")):
    k_, v_ = kv_opt.split("=")
    sm.set_option(k_, int(v_))
args = [int(x) for x in sys.argv[1:]]
pts = [tuple(args[i:i + 3]) for i in range(0, len(args), 3)] or [(8, 64, 1024), (1, 64, 4096), (32, 64, 1024),
                                                                  (8, 64, 4096)]
H, Hkv = (int(x) for x in os.environ.get("K1_GEOM", "32,32").split(","))  # B: K1_GEOM=8,1
hd = 128
for b, N, Lc in pts:
    tree = sm.Tree(synth.SWEEP_TREES[N]) if N != 64 else sm.Tree(synth.V64)
    cap = Lc + tree.N
    q = torch.randn(b, tree.N, H, hd, device="cuda").bfloat16()
    k = torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()
    v = torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()
    o = torch.empty_like(q)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    lens = torch.full((b,), Lc, dtype=torch.int32, device="cuda")
    for _ in range(3):
        sm.tree_attention(tree, q, k, v, lens, H, Hkv, o)
    buf = np.zeros((8192, 8), dtype=np.int64)
    L.sm_trace_read_ks(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int(8192))
    flush.zero_()  # K/V out of L2
    torch.cuda.synchronize()
    buf[:] = 0
    # zero the device records by reading after a clean launch: run once, read
    sm.tree_attention(tree, q, k, v, lens, H, Hkv, o)
    torch.cuda.synchronize()
    L.sm_trace_read_ks(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int(8192))
    rec = buf[buf[:, 1] > 0]
    rec = rec[rec[:, 1] > rec[:, 1].max() - 5_000_000]  # this launch only (stale records of earlier points)
    t0 = rec[:, 1].min()
    r = (rec[:, 1:] - t0) / 1e3  # us
    ent, qs, kv0, pv, ex, stg, mrg = r[:, 0], r[:, 1], r[:, 2], r[:, 3], r[:, 4], r[:, 5], r[:, 6]
    smid = rec[:, 0]
    alg = b * Hkv * cap * hd * 4 + 2 * b * tree.N * H * hd * 2
    span = ex.max()
    print(f"== H{H}/{Hkv} b{b} N{tree.N} Lc{Lc}: {len(rec)} CTAs, span {span:.1f} us ({alg / span / 1e3:.0f} GB/s)")
    print(f"   median phases (us): entry->Q {np.median(qs - ent):.2f}  entry->K/V(0) {np.median(kv0 - ent):.2f}  "
          f"K/V(0)->last PV {np.median(pv - kv0):.2f}  last PV->exit {np.median(ex - pv):.2f}  "
          f"lifetime {np.median(ex - ent):.2f}")
    print(f"   epilogue (us): last PV->staged {np.median(stg - pv):.2f}  staged->merged (thread 0) "
          f"{np.median(mrg - stg):.2f}  merged->exit {np.median(ex - mrg):.2f}")
    print(f"   entry: first {ent.min():.2f} median {np.median(ent):.2f} max {ent.max():.2f};  "
          f"exit: min {ex.min():.2f} median {np.median(ex):.2f} max {ex.max():.2f}")
    per_sm = {}
    for i in np.argsort(ent):
        per_sm.setdefault(int(smid[i]), []).append(i)
    counts = np.bincount([len(v_) for v_ in per_sm.values()])
    gaps = [ent[js[j + 1]] - ex[js[j]] for js in per_sm.values() for j in range(len(js) - 1)]
    print(f"   SMs used {len(per_sm)}, CTAs per SM histogram {counts.tolist()}, "
          f"gap exit->next entry median {np.median(gaps) if gaps else 0:.2f} max {max(gaps) if gaps else 0:.2f} us")
    # streaming share: fraction of the span each SM spends between K/V(0) and last PV
    busy = sum(pv[i] - kv0[i] for i in range(len(rec))) / (148 * span)
    print(f"   SM-time streaming (K/V(0)..last PV) / (148 x span) = {busy:.2f}")
    del q, k, v, o, flush
    torch.cuda.empty_cache()
