"""Data-parallel K2 (one CTA per weight tile, no split-K) vs stream-K on the C2 gate/up
shape (M = 64, N = 22016, K = 4096), plain partial epilogue vs the fused SiLU epilogue
(epi_test).  GPU box: python tools/gemm_dp.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm  # noqa: E402

M, N, K = 64, 22016, 4096
ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
for ctas in (0, 172, 344, 148):
    line = []
    for epi in (0, 1):
        sm.set_option("gemm_ctas", ctas)
        sm.set_option("epi_test", epi)
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
        line.append(f"epi={epi}: {us:.1f}us {N * K * 2 / us / 1e3:.0f}GB/s")
    print(f"ctas={ctas}", " | ".join(line), flush=True)
sm.set_option("epi_test", 0)
sm.set_option("gemm_ctas", 0)
