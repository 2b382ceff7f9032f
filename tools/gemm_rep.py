"""K2 token-tile CTA groups (gemm_rep 1) vs plain stream-K (0) at tensor-bound M, CUDA graph of 10
back-to-back GEMMs (two weight sets).  GPU box: python tools/gemm_rep.py"""
import sys, torch
sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm
for M, N, K in ((1024, 12288, 4096), (1024, 22016, 4096), (640, 57344, 8192), (512, 12288, 4096), (320, 12288, 4096)):
    w = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    line = []
    for rep in (0, 1):
        sm.set_option("gemm_rep", rep)
        for i in range(3): sm.gemm_bf16(x, w[i % 2], None)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(10): sm.gemm_bf16(x, w[i % 2], None)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 * 1e3
        line.append(f"rep={rep} {us:.1f}us {2*M*N*K/us/1e6:.0f}TF/s")
    print(M, N, K, " | ".join(line), flush=True)
sm.set_option("gemm_rep", 1)
