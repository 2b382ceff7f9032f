"""Per-launch %globaltimer timeline of back-to-back K2 launches inside one CUDA
graph (each launch writes its own debug rows).  GPU box only."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm  # noqa: E402

L = sm.lib()
occ = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pdl = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L.sm_set_option(b"gemm_occ", occ)
L.sm_set_option(b"pdl", pdl)
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
L.sm_set_option(b"gemm_dbg_mode", mode)
print("dbg_mode", mode)
for name, M, N, K in (("o", 64, 4096, 4096), ("gu", 64, 22016, 4096))[: 1 if mode else 2]:
    reps = 6
    ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    dbg = torch.zeros(reps, 2 * 148 * 8, dtype=torch.int64, device="cuda")
    for i in range(3):
        sm.gemm_bf16(x, ws[i % 3], out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            L.sm_set_gemm_debug(ctypes.c_void_p(dbg[i].data_ptr()))
            sm.gemm_bf16(x, ws[i % 3], out)
    L.sm_set_gemm_debug(None)
    dbg.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} occ={occ} pdl={pdl}: graph {e0.elapsed_time(e1) * 1e3 / reps:.1f} us/launch")
    d = dbg.view(reps, -1, 8).cpu().numpy().astype(np.float64)
    t0 = d[0][d[0][:, 0] > 0][:, 0].min()
    for i in range(reps):
        r = d[i][d[i][:, 0] > 0]
        rel = (r - t0) / 1e3
        rel[r == 0] = np.nan
        print(f"  launch {i}: entry [{np.nanmin(rel[:,0]):7.1f} .. {np.nanmax(rel[:,0]):7.1f}]  postwait med "
              f"{np.nanmedian(rel[:,1]):7.1f}  first_full med {np.nanmedian(rel[:,2]):7.1f}  mma_done [{np.nanmin(rel[:,3]):7.1f} .. "
              f"{np.nanmax(rel[:,3]):7.1f}]  exit max {np.nanmax(rel[:,6]):7.1f}  n_exit {int(np.sum(r[:,6] > 0))}/{len(r)}"
              f"  fixup cycles (n={int(np.sum(r[:,7] > 0))}) max {r[:,7].max():.0f} med {np.median(r[:,7][r[:,7] > 0]) if np.any(r[:,7] > 0) else 0:.0f}")
    del ws, g
