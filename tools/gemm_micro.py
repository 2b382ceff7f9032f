"""Device-side micro-benchmark of K2 on the C2 shapes (GPU box only).

Launches are captured into a CUDA graph (no host overhead in the timing) and
cycle over 3 weight copies (> L2).  One extra launch per shape records per-CTA
%globaltimer phase stamps (sm_set_gemm_debug)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm  # noqa: E402

SHAPES = [("qkv", 64, 12288, 4096), ("o", 64, 4096, 4096), ("gu", 64, 22016, 4096), ("down", 64, 4096, 11008),
          ("lm", 64, 32000, 4096), ("headR", 1, 4096, 4096)]
L = sm.lib()
dbg = torch.zeros(2 * 148 * 8, dtype=torch.int64, device="cuda")


def run(tag, phases=False):
    res = []
    for name, M, N, K in SHAPES:
        ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
        for i in range(3):
            sm.gemm_bf16(x, ws[i % 3], out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        reps = 30
        with torch.cuda.graph(g):
            for i in range(reps):
                sm.gemm_bf16(x, ws[i % 3], out)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        byts = N * K * 2 + M * K * 2 + M * N * 4
        res.append(f"{name}:{us:.1f}us/{byts / us / 1e3:.0f}GB/s")
        if phases:
            dbg.zero_()
            L.sm_set_gemm_debug(ctypes.c_void_p(dbg.data_ptr()))
            sm.gemm_bf16(x, ws[0], out)
            torch.cuda.synchronize()
            L.sm_set_gemm_debug(None)
            d = dbg.view(-1, 8).cpu().numpy()
            d = d[d[:, 0] > 0]
            t0 = d[:, 0].min()
            rel = (d - t0) / 1e3
            rel[d == 0] = np.nan
            names = ["entry", "postwait", "first_full", "mma_done", "acc0", "accN", "exit"]
            print(f"  {name} P={len(d)} " + " ".join(
                f"{nm}=[{np.nanmin(rel[:, i]):.1f},{np.nanmedian(rel[:, i]):.1f},{np.nanmax(rel[:, i]):.1f}]"
                for i, nm in enumerate(names)), flush=True)
        del ws, g
    print(tag, " ".join(res), flush=True)


for occ, pdl in ((2, 1), (1, 1)):
    L.sm_set_option(b"gemm_occ", occ)
    L.sm_set_option(b"pdl", pdl)
    run(f"occ={occ} pdl={pdl}", phases=True)
