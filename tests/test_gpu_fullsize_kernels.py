"""Stage parity of K1 and K2 at the full sizes bench.py times, on sampled outputs the
oracle computes one by one (needs a B200).

Inputs come from the counter-hash law: the device fills the whole tensors with
sm.generate_bf16 (mode 0), the oracle regenerates only the slices a sampled output
reads with synth.weight_bits(..., start=offset) on the host -- no oracle input is
read back from the GPU.  Q and K (and V) are scaled by 2^6 on both sides (exact in
bf16) so the softmax is far from uniform.

  * K1 geometry A at bench.py's k1_point (C5: b = 8, H = Hkv = 32, hd = 128, V64,
    Lc = 4096, ~0.55 GB of K/V per launch) and geometry B (one 70B TP8 shard: 8 q
    heads on 1 kv head, N*G = 512 rows = four 128-row blocks) with ragged lengths up
    to 32768; each sampled (seq, node, head) row against oracle Model.attention over
    the Eq. 2 key list.
  * K2 at the C2 / C4 / C4-V64 verify shapes (M = 64, 160 and 640 token rows; the
    2-SM variant runs at 160 and 640): sampled outputs against fp64 dot products.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import model as OM
from oracle import tree as OT

pytestmark = pytest.mark.gpu

SCALE = 64.0  # 2^6: exact in bf16


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


def host_slice(seed, stream, start, n, scale=1.0):
    return synth.bf16_bits_to_f32(synth.weight_bits(seed, stream, n, start=start)).astype(np.float64) * scale


class _OneHead:  # oracle Model.attention geometry of a single (q head, kv head) pair
    def __init__(self, hd):
        self.H, self.hd, self.G = 1, hd, 1


K1_CASES = [
    # name, b, H, Hkv, lens, samples
    ("geomA_k1_point", 8, 32, 32, [4096] * 8, 40),
    ("geomB_tp8_ragged", 2, 8, 1, [32768, 1111], 40),
    # 40 sequences x 4 row blocks = 160 units of 128 live rows: the persistent kernel with two softmax warps
    # per row (KSP, W2), ragged lengths
    ("geomB_ksp_w2", 40, 8, 1, [4096 - 37 * i for i in range(40)], 40),
]


@pytest.mark.parametrize("case", K1_CASES, ids=[c[0] for c in K1_CASES])
def test_k1_full_size_sampled_rows(sm, case):
    name, b, H, Hkv, lens, samples = case
    hd, seed = 128, 11
    tree = sm.Tree(synth.V64, topk=synth.TOPK)
    otree = OT.build(synth.V64)
    N = tree.N
    cap = max(lens) + N
    q = torch.empty(b, N, H, hd, dtype=torch.bfloat16, device="cuda")
    k = torch.empty(b, Hkv, cap, hd, dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    for i, t in enumerate((q, k, v)):
        sm.generate_bf16(t, seed, 300 + i, mode=0)
        t.mul_(SCALE)
    L = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = torch.full((b, N, H, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    sm.tree_attention(tree, q, k, v, L, H, Hkv, out)
    torch.cuda.synchronize()
    got_all = out.float().cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(got_all))

    rng = np.random.default_rng(5)
    picks = [(0, 0, 0), (b - 1, N - 1, H - 1)] + [
        (int(rng.integers(b)), int(rng.integers(N)), int(rng.integers(H))) for _ in range(samples - 2)]
    G = H // Hkv
    g = _OneHead(hd)
    cache = {}
    for bi, n, h in picks:
        kvh, Lc = h // G, lens[bi]
        if (bi, kvh) not in cache:  # K/V of slots [0, Lc + N) of this (seq, kv head)
            off = (bi * Hkv + kvh) * cap * hd
            Kf = host_slice(seed, 301, off, (Lc + N) * hd, SCALE).reshape(Lc + N, 1, hd)
            Vf = host_slice(seed, 302, off, (Lc + N) * hd, SCALE).reshape(Lc + N, 1, hd)
            cache[(bi, kvh)] = (Kf, Vf)
        Kf, Vf = cache[(bi, kvh)]
        keys = list(range(Lc)) + [Lc + a for a in OT.ancestors(otree, n)] + [Lc + n]
        qrow = host_slice(seed, 300, ((bi * N + n) * H + h) * hd, hd, SCALE).reshape(1, hd)
        ref = OM.Model.attention(g, qrow, Kf[keys], Vf[keys])[0]
        err = np.abs(got_all[bi, n, h] - ref)
        assert np.all(err <= 2e-2 + 2e-2 * np.abs(ref)), (name, bi, n, h, float(err.max()))


K2_CASES = [
    # name, M, N, K, gemm_pair option (1 = default rule)
    ("c2_gate_up", 64, 22016, 4096, 1),
    ("c2_down", 64, 4096, 11008, 1),
    ("c4_gate_up_pair", 160, 57344, 8192, 1),
    ("c4v64_down_pair", 640, 8192, 28672, 1),
    ("c4v64_qkv_single_sm", 640, 10240, 8192, 0),
]


@pytest.mark.parametrize("case", K2_CASES, ids=[c[0] for c in K2_CASES])
def test_k2_full_size_sampled_outputs(sm, case):
    name, M, N, K, pair = case
    seed = 13
    x = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
    w = torch.empty(N, K, dtype=torch.bfloat16, device="cuda")
    sm.generate_bf16(x, seed, 400, mode=0)
    sm.generate_bf16(w, seed, 401, mode=0)
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    sm.set_option("gemm_pair", pair)
    try:
        sm.gemm_bf16(x, w, out)
        torch.cuda.synchronize()
    finally:
        sm.set_option("gemm_pair", 1)
    rng = np.random.default_rng(7)
    ms = [0, M - 1] + [int(v) for v in rng.integers(M, size=14)]
    ns = [0, N - 1] + [int(v) for v in rng.integers(N, size=14)]
    X = {m: host_slice(seed, 400, m * K, K) for m in set(ms)}
    W = {n: host_slice(seed, 401, n * K, K) for n in set(ns)}
    got = out.cpu().numpy()
    assert np.all(np.isfinite(got))
    for m in ms:
        for n in ns:
            ref = float(X[m] @ W[n])
            bound = float(np.abs(X[m]) @ np.abs(W[n]))
            assert abs(float(got[m, n]) - ref) <= 2e-6 * bound + 1e-30, (name, m, n)
