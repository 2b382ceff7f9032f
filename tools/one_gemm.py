import sys, torch
sys.path.insert(0, ".")
import paper_2506_01986_b200 as sm
mode = int(sys.argv[1]); M = int(sys.argv[2]); N = int(sys.argv[3]); K = int(sys.argv[4])
sm.set_option("gemm_pair", mode)
w = torch.randn(N, K, device="cuda").to(torch.bfloat16); x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
for _ in range(3):
    sm.gemm_bf16(x, w, None)
torch.cuda.synchronize()
