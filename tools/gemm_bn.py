"""K2 token-tile sweep on the 70B (C4) layer shapes (GPU box only): for M = b*N rows,
time each weight GEMM (+ its plain consumer) with every token-tile width BN, in a
CUDA graph cycling over 3 weight copies (> L2).  python tools/gemm_bn.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm  # noqa: E402

SHAPES = [("qkv", 10240, 8192), ("o", 8192, 8192), ("gu", 57344, 8192), ("down", 8192, 28672)]
OUT = "--consumer" in sys.argv  # default: GEMM only (stage API with out = NULL)
CASES = ((160, (64, 80, 96, 128, 160)), (640, (128, 160, 256)), (256, (64, 128, 256)), (64, (64, 96, 128)),
         (10, (16, 32)))
if "--c4" in sys.argv:
    CASES = ((160, (64, 80, 96, 128, 160)),)
for M, bns in CASES:
    for bn in bns:
        sm.set_option("gemm_bn", bn)
        res, tot_us, tot_b = [], 0.0, 0
        for name, N, K in SHAPES:
            ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
            x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            out = torch.empty(M, N, device="cuda", dtype=torch.float32)
            for i in range(2):
                sm.gemm_bf16(x, ws[i % 2], out if OUT else None)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            reps = 10
            with torch.cuda.graph(g):
                for i in range(reps):
                    sm.gemm_bf16(x, ws[i % 2], out if OUT else None)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / reps * 1e3
            byts = N * K * 2
            tot_us += us
            tot_b += byts
            res.append(f"{name}:{us:.0f}us/{byts / us / 1e3:.0f}GB/s/{2 * M * N * K / us / 1e6:.0f}TF")
            del ws, g
        print(f"M={M:4d} BN={bn:3d} layer {tot_us:.0f}us {tot_b / tot_us / 1e3:.0f}GB/s  " + " ".join(res), flush=True)
sm.set_option("gemm_bn", 0)
