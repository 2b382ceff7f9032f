"""f3 prefill throughput on B200: a turn of P tokens is prefilled through the verify path
(sm_prefill) in causal chunks of max_rows tokens (256, 512, 1024), C2 and C3 shapes.
Reports tokens/s and the fraction of the per-chunk roofline max(weight bytes / HBM,
flops / tensor peak).  python tools/prefill_bench.py  (GPU box)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_01986_b200 as sm  # noqa: E402
import synth  # noqa: E402

pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
HBM, TC = pk["hbm_gbs"] * 1e9, pk["bf16_tflops_sustained"] * 1e12
for name, P, rows in (("vicuna7b", 128, 256), ("vicuna7b", 1024, 256), ("vicuna7b", 1024, 512),
                      ("vicuna7b", 1024, 1024), ("vicuna7b", 2048, 1024), ("vicuna13b", 160, 256),
                      ("vicuna13b", 2048, 256), ("vicuna13b", 2048, 1024)):
    cfg = synth.model_cfg(name)
    W = sm.allocate_weights(cfg, 4, seed=0)
    tree = sm.Tree(synth.V64)
    model = sm.Model(cfg, W, max_rows=rows, max_batch=1, max_seq_len=P + 256 + tree.N)
    kv = sm.KVCache(model, tree, 1, P + 256)
    toks = torch.from_numpy(synth.prompt_tokens(0, 0, P, cfg["vocab"])).cuda()
    kv.prefill(0, toks)  # warm-up (and graph-free path)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        kv2 = sm.KVCache(model, tree, 1, P + 256)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        kv2.prefill(0, toks)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        del kv2
    ms = min(ts)
    d, L, H, hd, F, V = (cfg[k] for k in ("d_model", "n_layers", "n_heads", "head_dim", "d_ffn", "vocab"))
    params = L * ((H + 2 * cfg["n_kv_heads"]) * hd * d + d * H * hd + 3 * F * d)
    chunks = (P + rows - 1) // rows
    byts = chunks * params * 2 + 2 * V * d * 2
    flops = 2 * P * params + 4 * L * H * hd * P * P / 2
    floor = max(byts / HBM, flops / TC) * 1e3
    print(json.dumps({"model": name, "prompt": P, "max_rows": rows, "chunks": chunks, "ms": round(ms, 3),
                      "tokens_per_s": round(P / ms * 1e3, 1), "roofline_ms": round(floor, 3),
                      "frac": round(floor / ms, 3)}), flush=True)
    del kv, model, W
    torch.cuda.empty_cache()
