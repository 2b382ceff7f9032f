"""2-SM (cta_group::2) vs single-SM K2 on C2 / C4 / prefill shapes (GPU box): GEMM-only
time (sm_gemm_bf16 with out = NULL) in a CUDA graph over 2 weight copies.  Also checks the
pair result against the single-SM one (same partial sums, same order: identical)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm  # noqa: E402

SH = {"7b": [("qkv", 12288, 4096), ("o", 4096, 4096), ("gu", 22016, 4096), ("down", 4096, 11008)],
      "70b": [("qkv", 10240, 8192), ("o", 8192, 8192), ("gu", 57344, 8192), ("down", 8192, 28672)]}
torch.manual_seed(0)
for model, M in (("7b", 64), ("7b", 256), ("70b", 160), ("70b", 640), ("7b", 100)):
    for mode in (0, 2 if M <= 64 else 1):
        sm.set_option("gemm_pair", mode)
        tot_us, tot_b, parts = 0.0, 0, []
        for name, N, K in SH[model]:
            ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
            x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            for i in range(2):
                sm.gemm_bf16(x, ws[i], None)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(10):
                    sm.gemm_bf16(x, ws[i % 2], None)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 10 * 1e3
            tot_us += us
            tot_b += N * K * 2
            parts.append(f"{name}:{us:.0f}us/{2 * M * N * K / us / 1e6:.0f}TF")
            del ws, g
        print(f"{model} M={M:4d} pair={mode} layer {tot_us:7.0f}us {tot_b / tot_us / 1e3:6.0f}GB/s  " + " ".join(parts),
              flush=True)
# correctness: pair vs single on a ragged shape
for M, N, K in ((100, 1000, 320), (64, 4096, 4096), (160, 8192, 1024), (256, 384, 8192), (77, 4352, 640)):
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    outs = []
    for mode in (0, 2):
        sm.set_option("gemm_pair", mode)
        o = torch.full((M, N), float("nan"), device="cuda")
        sm.gemm_bf16(x, w, o)
        torch.cuda.synchronize()
        outs.append(o)
    ref = x.double() @ w.double().T
    print(f"check M={M} N={N} K={K}: finite {bool(torch.isfinite(outs[1]).all())} "
          f"max|pair-ref|/max|ref| {((outs[1].double() - ref).abs().max() / ref.abs().max()).item():.2e} "
          f"max|pair-single| {(outs[1] - outs[0]).abs().max().item():.2e}", flush=True)
sm.set_option("gemm_pair", 1)
