import sys, torch
sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm
SH = [("qkv", 12288, 4096), ("o", 4096, 4096), ("gu", 22016, 4096), ("down", 4096, 11008)]
for M in (128, 192, 256):
  for pair, bn in ((0, 0), (1, 0), (0, 64), (2, 64), (1, 96) if M <= 192 else (1, 128)):
    sm.set_option("gemm_pair", pair); sm.set_option("gemm_bn", bn)
    tot = 0.0; tb = 0
    for name, N, K in SH:
        ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        for i in range(2): sm.gemm_bf16(x, ws[i], None)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(10): sm.gemm_bf16(x, ws[i % 2], None)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1) / 10 * 1e3; tb += N * K * 2
        del ws, g
    print(f"M={M} pair={pair} bn={bn or 'auto'}: layer {tot:.0f} us {tb / tot / 1e3:.0f} GB/s", flush=True)
sm.set_option("gemm_pair", 1); sm.set_option("gemm_bn", 0)
