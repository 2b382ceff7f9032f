import sys, torch
sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm
for rows in (1, 4, 64):
    z = torch.randn(rows, 32000, device="cuda")
    out = torch.zeros(rows, 10, dtype=torch.int32, device="cuda")
    for _ in range(3): sm.topk_f32(z, 10, out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20): sm.topk_f32(z, 10, out)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(rows, "rows topk us", e0.elapsed_time(e1) / 20 * 1e3)
