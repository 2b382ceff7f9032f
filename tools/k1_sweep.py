"""C5 tree-attention sweep (BASELINE configs[4]) on the GPU box.

python tools/k1_sweep.py [--quick] > profiles/r01_k1_sweep.txt
Geometry A = one 7B layer (H = Hkv = 32), geometry B = one 70B TP8 shard (8 q / 1 kv),
head_dim 128, tree N in {16, 64, 256}, Lc in {512, 4096, 32768}, batch in {1, 8, 32}
(--full: SURVEY's grid N 16..256 x Lc 512..32K x b 1..32, uniform and ragged "~" lengths
Lc_b spread over [Lc/2, Lc]; bounded to <= 8 GB of K/V per set).  Each point: 20 launches captured in a CUDA graph
over two alternating buffer sets (> L2), replayed; device time per launch; achieved
GB/s = algorithmic bytes (K/V of [0, Lc) + tree slots once, Q in, O out) / time."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

import json  # noqa: E402

_pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
PEAK = _pk["hbm_gbs"]                   # GB/s
TPEAK = _pk["bf16_tflops"]              # dense bf16 TF/s (burst: one kernel timed alone)
ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
ap.add_argument("--tc", type=int, default=1)
ap.add_argument("--full", action="store_true", help="SURVEY 8.d.1 grid: N 16..256 x Lc 512..32K x b 1..32, "
                                                     "uniform and ragged lengths")
a = ap.parse_args()
sm.set_option("attn_tc", a.tc)
for kv_opt in filter(None, os.environ.get("SM_OPT", "").split(",")):  # sm_set_option knobs, e.g. attn_ks=2
    k_, v_ = kv_opt.split("=")
    sm.set_option(k_, int(v_))
trees = {n: (sm.Tree(synth.V64) if n == 64 else sm.Tree(synth.SWEEP_TREES[n])) for n in (16, 32, 64, 128, 256)}
geoms = [("A 32/32", 32, 32), ("B 8/1", 8, 1)]
Ns = [16, 64, 256]
Lcs = [512, 4096, 32768]
bs = [1, 8, 32]
RAGGED = [False]
if a.quick:
    Ns, Lcs, bs = [64], [512, 4096], [1, 8]
if a.full:
    Ns, Lcs, bs = [16, 32, 64, 128, 256], [512, 1024, 2048, 4096, 8192, 16384, 32768], [1, 2, 4, 8, 16, 32]
    RAGGED = [False, True]
if os.environ.get("K1_SWEEP_B"):  # restrict (diagnostics): K1_SWEEP_B=8,16 K1_SWEEP_N=128 K1_SWEEP_G=A
    bs = [int(x) for x in os.environ["K1_SWEEP_B"].split(",")]
if os.environ.get("K1_SWEEP_N"):
    Ns = [int(x) for x in os.environ["K1_SWEEP_N"].split(",")]
if os.environ.get("K1_SWEEP_G"):
    geoms = [g for g in geoms if g[0][0] == os.environ["K1_SWEEP_G"]]
if os.environ.get("K1_SWEEP_U"):  # uniform lengths only
    RAGGED = [False]
print(f"{'geom':8s} {'b':>3s} {'N':>4s} {'Lc':>6s} {'MB':>8s} {'us':>9s} {'GB/s':>8s} {'TF/s':>7s} {'bound':>6s} "
      f"{'frac':>6s}")
# flops = 4 H hd sum_b (N Lc + sum_n (depth_n + 1)) (tree part counted sparse);
# bound = whichever of bytes / HBM peak and flops / tensor peak is larger; frac = that floor / time
hd = 128
for ragged in RAGGED:
  for gname, H, Hkv in geoms:
    for b in bs:
        for N in Ns:
            for Lc in Lcs:
                tree = trees[N]
                cap = Lc + tree.N
                kv_bytes = b * Hkv * cap * hd * 2 * 2
                if kv_bytes > 8e9:
                    continue
                sets = []
                for _ in range(2):
                    q = torch.randn(b, tree.N, H, hd, device="cuda").bfloat16()
                    k = torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()
                    v = torch.randn(b, Hkv, cap, hd, device="cuda").bfloat16()
                    sets.append((q, k, v, torch.empty_like(q)))
                # ragged: Lc_b spread evenly over [Lc/2, Lc]
                lens = [Lc // 2 + (Lc - Lc // 2) * i // max(1, b - 1) for i in range(b)] if ragged else [Lc] * b
                L = torch.tensor(lens, dtype=torch.int32, device="cuda")
                st = torch.cuda.Stream()
                for i in range(2):  # on the capture stream: sizes its stage scratch before the capture
                    q, k, v, o = sets[i]
                    sm.tree_attention(tree, q, k, v, L, H, Hkv, o, stream=st)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(st):
                    g.capture_begin()
                    for i in range(20):
                        q, k, v, o = sets[i % 2]
                        sm.tree_attention(tree, q, k, v, L, H, Hkv, o, stream=st)
                    g.capture_end()
                g.replay()
                torch.cuda.synchronize()
                # three timing rounds of 3 replays (60 launches each); the point's time is the median round
                # (single rounds of a long sweep showed occasional 1.2-1.5x outliers that a re-run did not)
                rounds = []
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(3):
                        g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    rounds.append(e0.elapsed_time(e1) * 1e3 / 60)
                us = sorted(rounds)[1]
                chk = ""
                if os.environ.get("K1_SWEEP_CHECK"):  # diagnostics: the replayed output vs a fresh launch
                    q, k, v, o = sets[0]
                    o2 = torch.empty_like(o)
                    sm.tree_attention(tree, q, k, v, L, H, Hkv, o2, stream=st)
                    torch.cuda.synchronize()
                    chk = " ok" if torch.equal(o, o2) else " MISMATCH"
                alg = sum(Hkv * (lb + tree.N) * hd * 2 * 2 for lb in lens) + 2 * b * tree.N * H * hd * 2
                dep = tree.query()["node_depth"]
                flops = sum(4 * H * hd * (tree.N * lb + int((dep + 1).sum())) for lb in lens)
                gbs = alg / us / 1e3
                tfs = flops / us / 1e6
                t_hbm, t_tc = alg / PEAK / 1e3, flops / TPEAK / 1e6  # us
                bound = "hbm" if t_hbm >= t_tc else "tensor"
                tag = gname + ("~" if ragged else "")
                print(f"{tag:8s} {b:3d} {tree.N:4d} {Lc:6d} {alg / 1e6:8.1f} {us:9.1f} {gbs:8.1f} {tfs:7.1f} {bound:>6s} "
                      f"{max(t_hbm, t_tc) / us:6.3f}{chk}", flush=True)
                del sets, g
                torch.cuda.empty_cache()
