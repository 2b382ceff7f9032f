"""Fused tile epilogue cost (GPU box): K2 alone vs K2 + fused SiLU epilogue (epi_test)
on the C2 shapes at M = 64, back to back in a CUDA graph.  python tools/gemm_epi.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm  # noqa: E402

for name, M, N, K in (("qkv", 64, 12288, 4096), ("o", 64, 4096, 4096), ("gu", 64, 22016, 4096),
                      ("down", 64, 4096, 11008)):
    line = []
    for epi, mode in ((0, 0), (1, 0), (1, 2)):
        sm.set_option("epi_test", epi)
        sm.set_option("gemm_mode", mode)
        ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        for i in range(2):
            sm.gemm_bf16(x, ws[i], None)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        reps = 20
        with torch.cuda.graph(g):
            for i in range(reps):
                sm.gemm_bf16(x, ws[i % 2], None)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        line.append(f"epi={epi} mode={mode}: {us:.1f}us {N * K * 2 / us / 1e3:.0f}GB/s")
    print(name, " | ".join(line), flush=True)
sm.set_option("epi_test", 0)
sm.set_option("gemm_mode", 0)
