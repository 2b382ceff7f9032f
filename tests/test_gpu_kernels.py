"""Stage parity of the CUDA kernels against the oracle (needs a B200).

K2 GEMM vs numpy fp64; K1 tree attention vs oracle Model.attention over the
gathered key list; K3 top-k vs the oracle's (value desc, index asc) order;
the device weight generator bit for bit against synth."""
import numpy as np
import pytest
import torch

import synth
from oracle import model as OM
from oracle import tree as OT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


def bf16_tensor(bits: np.ndarray, shape):
    return torch.from_numpy(bits.view(np.int16).reshape(shape).copy()).view(torch.bfloat16).cuda()


def to64(t):
    return t.float().cpu().numpy().astype(np.float64)


# ------------------------------------------------------------------ generator
@pytest.mark.parametrize("seed,stream,n,mode,start", [(0, 5, 100003, 0, 0), (3, 2, 4097, 0, 77), (1, 9, 50001, 1, 0)])
def test_device_generator_bitwise(sm, seed, stream, n, mode, start):
    t = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    sm.generate_bf16(t, seed, stream, start=start, mode=mode)
    torch.cuda.synchronize()
    got = t.view(torch.int16).cpu().numpy().view(np.uint16)
    if mode == 0:
        ref = synth.weight_bits(seed, stream, n, start=start)
    else:
        assert start == 0
        ref = synth.normal_bits(seed, stream, n)
    assert np.array_equal(got, ref)


# ------------------------------------------------------------------ K2 GEMM
@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (16, 4096, 4096), (37, 192, 320), (64, 12288, 512),
                                   (200, 1000, 72), (256, 384, 1024), (64, 4096, 11008),
                                   (80, 4096, 512), (160, 10240, 1024), (150, 1000, 200), (192, 384, 8192)])
def test_gemm_matches_fp64(sm, M, N, K):
    x = bf16_tensor(synth.normal_bits(1, 100 + M, M * K), (M, K))
    w = bf16_tensor(synth.weight_bits(2, 200 + N, N * K), (N, K))
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    sm.gemm_bf16(x, w, out)
    torch.cuda.synchronize()
    X, W = to64(x), to64(w)
    ref = X @ W.T
    bound = np.abs(X) @ np.abs(W).T
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref)
    assert np.all(np.isfinite(out.cpu().numpy()))
    assert np.all(err <= 2e-6 * bound + 1e-30), float((err / (bound + 1e-30)).max())


@pytest.mark.parametrize("pair", [0, 1], ids=["single_sm", "pair"])
@pytest.mark.parametrize("rep", [1, 0], ids=["groups", "plain"])
@pytest.mark.parametrize("M,N,K", [(640, 1000, 320), (1024, 2304, 512), (300, 384, 1024), (513, 4352, 192)])
def test_gemm_token_tile_groups_match_fp64(sm, M, N, K, rep, pair):
    """Several token tiles: CTA groups walking the same weight k-blocks (gemm_rep = 1, SplitPlan::rep)
    and the plain stream-K partition, single-SM and 2-SM kernels."""
    sm.set_option("gemm_rep", rep)
    sm.set_option("gemm_pair", pair)
    try:
        test_gemm_matches_fp64(sm, M, N, K)
    finally:
        sm.set_option("gemm_rep", 1)
        sm.set_option("gemm_pair", 1)


@pytest.mark.parametrize("M,N,K", [(64, 4096, 512), (100, 1000, 320), (160, 8192, 1024), (256, 384, 8192),
                                   (77, 4352, 640)])
def test_gemm_pair_matches_fp64(sm, M, N, K):
    """The 2-SM (tcgen05 cta_group::2) K2 variant (sm_set_option gemm_pair = 2: token tiles >= 64)."""
    sm.set_option("gemm_pair", 2)
    try:
        test_gemm_matches_fp64(sm, M, N, K)
    finally:
        sm.reset_options()  # the library defaults (gemm_pair = 1)


# ------------------------------------------------------------------ K1 tree attention
class _Geom:
    def __init__(self, H, Hkv, hd):
        self.H, self.hd, self.G = H, hd, H // Hkv


def attention_oracle(tree_choices, chain_n, q, k, v, lens, H, Hkv):
    """Per node: keys = [0, Lc) + ancestors' tree slots + own slot (Eq. 2)."""
    tr = OT.build(tree_choices) if chain_n is None else OT.build(synth.CHAIN(chain_n - 1), topk=1)
    Q, K, V = to64(q), to64(k), to64(v)
    b, N, _, hd = Q.shape
    g = _Geom(H, Hkv, hd)
    out = np.zeros_like(Q)
    for bi in range(b):
        Lc = int(lens[bi])
        for n in range(N):
            keys = list(range(Lc)) + [Lc + a for a in OT.ancestors(tr, n)] + [Lc + n]
            Kc = K[bi][:, keys, :].transpose(1, 0, 2)
            Vc = V[bi][:, keys, :].transpose(1, 0, 2)
            out[bi, n] = OM.Model.attention(g, Q[bi, n], Kc, Vc)
    return out


ATTN_CASES = [
    # (name, choices, chain, b, H, Hkv, hd, lens, cap_extra)
    ("c1_tiny16", synth.TINY16, None, 1, 4, 4, 16, [32], 16),
    ("v64_mha_ragged", synth.V64, None, 2, 4, 4, 128, [0, 333], 40),
    ("v64_gqa8", synth.V64, None, 3, 8, 1, 128, [100, 517, 1], 7),
    ("sweep128", synth.SWEEP_TREES[128], None, 1, 2, 2, 128, [1000], 0),
    ("sweep256_gqa", synth.SWEEP_TREES[256], None, 1, 4, 2, 64, [130], 3),
    ("chain_prefill", None, 200, 2, 4, 2, 64, [0, 65], 5),
    ("hd32", synth.V64[:31], None, 2, 4, 4, 32, [64, 63], 1),
    # head_dim 128: 128-row blocks (tcgen05) -- several row blocks, ragged tail, 8-way split
    ("gqa8_rows512", synth.V64, None, 2, 16, 2, 128, [700, 64], 9),
    ("chain256_hd128", None, 256, 1, 8, 2, 128, [129], 0),
    ("split8_long", synth.SWEEP_TREES[16], None, 1, 1, 1, 128, [4000], 2),
    ("gqa4_v64_c2like", synth.V64, None, 2, 8, 2, 128, [1024, 1500], 0),
    # one split (no cluster) with padding rows inside a live warp (16 or 48 live rows of 128)
    ("n16_ns1_mha", synth.SWEEP_TREES[16], None, 4, 32, 32, 128, [512, 100, 7, 300], 0),
    ("n16_ns1_g3", synth.TINY16, None, 20, 24, 8, 128, [(37 * i) % 300 for i in range(20)], 1),
    # stream-K K1: one unit over many CTAs (pieces), many small ragged units, units of 4 row blocks
    ("lean_one_unit_long", synth.V64, None, 1, 1, 1, 128, [9000], 0),
    ("lean_many_units", synth.V64[:31], None, 40, 4, 2, 128, [(211 * i) % 2500 for i in range(40)], 3),
    ("lean_gqa8_4blocks", synth.V64, None, 3, 8, 1, 128, [3000, 5, 1200], 0),
    # 128-key-tile kernel over several 128-row blocks (geometry B: N G = 512; N 256): one split per unit
    ("ks_rows512_long", synth.V64, None, 20, 8, 1, 128, [1000 + 37 * i for i in range(20)], 3),
    # persistent row-copy kernel (one split, more units than SMs): 4 / 2 / 1 copies, ragged lengths
    # (empty prefix included), units of 4 row blocks
    ("ksp_f4_ragged", synth.SWEEP_TREES[16], None, 10, 16, 16, 128, [(97 * i) % 700 for i in range(10)], 2),
    ("ksp_f2_v64", synth.V64, None, 5, 32, 32, 128, [0, 129, 511, 300, 64], 0),
    ("ksp_f1_rows512", synth.V64, None, 20, 16, 2, 128, [(53 * i) % 400 for i in range(20)], 1),
    # 16 units of long ranges (geometry B shape): the occupancy-aware split count picks a non-power-of-two
    # cluster (7 splits: 16 clusters of 8 do not fit at once)
    ("b16_gqa8_odd_splits", synth.SWEEP_TREES[16], None, 16, 8, 1, 128, [1500 + 211 * i for i in range(16)], 3),
]


# K1 variants for head_dim 128: the stream-K tcgen05 kernel (default; min tiles per CTA = live rows
# per unit / 16, and / 2 for many more pieces per unit), the cluster-split tcgen05 kernel, mma.sync
VARIANTS = {"default": dict(), "ns3": dict(attn_splits=3), "ns7": dict(attn_splits=7),
            "rule_splits": dict(attn_split_model=0), "w2": dict(attn_w2=1), "qlate": dict(attn_qearly=0), "ksp": dict(attn_ksp=1), "noksp": dict(attn_ksp=0), "rows128": dict(attn_ks=0), "ks64": dict(attn_ks=1), "ns1": dict(attn_splits=1),
            "lean": dict(attn_tc=1, attn_lean=1),
            "lean_div2": dict(attn_tc=1, attn_lean=1, attn_lean_div=2), "mma": dict(attn_tc=0)}


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("case", ATTN_CASES, ids=[c[0] for c in ATTN_CASES])
def test_tree_attention_matches_oracle(sm, case, variant):
    name, choices, chain, b, H, Hkv, hd, lens, extra = case
    if variant != "default" and hd != 128:
        pytest.skip("head_dim < 128 always runs the mma.sync kernel")
    for k, v in VARIANTS[variant].items():
        sm.set_option(k, v)
    tree = sm.Tree(choices, topk=10) if chain is None else sm.Tree(None, chain=chain)
    N = tree.N
    cap = max(lens) + N + extra
    q = bf16_tensor(synth.normal_bits(5, 1, b * N * H * hd), (b, N, H, hd))
    k = bf16_tensor(synth.normal_bits(5, 2, b * Hkv * cap * hd), (b, Hkv, cap, hd))
    v = bf16_tensor(synth.normal_bits(5, 3, b * Hkv * cap * hd), (b, Hkv, cap, hd))
    L = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = torch.full((b, N, H, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    sm.tree_attention(tree, q, k, v, L, H, Hkv, out)
    torch.cuda.synchronize()
    ref = attention_oracle(choices, chain, q, k, v, lens, H, Hkv)
    got = to64(out)
    assert np.all(np.isfinite(got))
    err = np.abs(got - ref)
    assert np.all(err <= 2e-2 + 2e-2 * np.abs(ref)), float(err.max())


@pytest.mark.parametrize("case", [c for c in ATTN_CASES if c[0].startswith("ksp")], ids=lambda c: c[0])
def test_persistent_row_copy_kernel_is_bitwise_the_row_copy_kernel(sm, case):
    """KSP walks several units per CTA through one ring but keeps the row-copy kernel's arithmetic,
    copy order and merge order: its output must equal the one-unit-per-CTA kernel's bit for bit."""
    name, choices, chain, b, H, Hkv, hd, lens, extra = case
    tree = sm.Tree(choices, topk=10)
    N = tree.N
    cap = max(lens) + N + extra
    q = bf16_tensor(synth.normal_bits(6, 1, b * N * H * hd), (b, N, H, hd))
    k = bf16_tensor(synth.normal_bits(6, 2, b * Hkv * cap * hd), (b, Hkv, cap, hd))
    v = bf16_tensor(synth.normal_bits(6, 3, b * Hkv * cap * hd), (b, Hkv, cap, hd))
    L = torch.tensor(lens, dtype=torch.int32, device="cuda")
    outs = []
    sm.set_option("attn_splits", 1)  # the same (single) key split on both sides: with KSP off the split model
    for ksp in (0, 1):                 # may otherwise choose 2 splits for 149-222 units
        sm.set_option("attn_ksp", ksp)
        o = torch.full((b, N, H, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
        sm.tree_attention(tree, q, k, v, L, H, Hkv, o)
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


# ------------------------------------------------------------------ K3 top-k
def test_topk_matches_oracle_with_ties(sm):
    rng = np.random.default_rng(0)
    rows, V, k = 6, 32000, 10
    z = (np.round(rng.standard_normal((rows, V)) * 4) / 4).astype(np.float32)
    z[2, 100:120] = z[2].max()                   # a block of exact ties at the top
    zt = torch.from_numpy(z).cuda()
    out = torch.zeros(rows, k, dtype=torch.int32, device="cuda")
    sm.topk_f32(zt, k, out)
    torch.cuda.synchronize()
    for r in range(rows):
        assert out[r].cpu().tolist() == OM.topk_desc(z[r].astype(np.float64), k)


# ------------------------------------------------------------------ K1 prefill mode (causal chunks, f3)
CAUSAL_CASES = [
    # (name, n, b, H, Hkv, hd, lens, cap_extra): n > 256 (beyond the tree tables), ragged row blocks
    ("hd128_n600_fresh", 600, 1, 4, 4, 128, [0], 0),
    ("hd128_n333_gqa4_prefix", 333, 2, 8, 2, 128, [77, 1000], 5),
    ("hd128_n1024_split", 1024, 1, 1, 1, 128, [4000], 0),
    ("hd64_n700_gqa2", 700, 2, 4, 2, 64, [0, 130], 3),
    ("hd16_n97", 97, 1, 4, 4, 16, [32], 0),
]


@pytest.mark.parametrize("attn_tc", [1, 0], ids=["tc", "mma"])
@pytest.mark.parametrize("case", CAUSAL_CASES, ids=[c[0] for c in CAUSAL_CASES])
def test_causal_attention_matches_oracle(sm, case, attn_tc):
    """Token i of a chunk at slot Lc + i attends [0, Lc + i]: the oracle's attention over
    exactly that key list, row by row (the same rule as a chain tree, without a tree table)."""
    name, n, b, H, Hkv, hd, lens, extra = case
    if attn_tc == 0 and hd != 128:
        pytest.skip("head_dim < 128 always runs the mma.sync kernel")
    sm.set_option("attn_tc", attn_tc)
    cap = max(lens) + n + extra
    q = bf16_tensor(synth.normal_bits(9, 1, b * n * H * hd), (b, n, H, hd))
    k = bf16_tensor(synth.normal_bits(9, 2, b * Hkv * cap * hd), (b, Hkv, cap, hd))
    v = bf16_tensor(synth.normal_bits(9, 3, b * Hkv * cap * hd), (b, Hkv, cap, hd))
    L = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = torch.full((b, n, H, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    try:
        sm.causal_attention(q, k, v, L, H, Hkv, out)
        torch.cuda.synchronize()
    finally:
        sm.set_option("attn_tc", 1)
    Q, K, V = to64(q), to64(k), to64(v)
    got = to64(out)
    assert np.all(np.isfinite(got))
    g = _Geom(H, Hkv, hd)
    rows = sorted(set([0, 1, 63, 64, 127, 128, n - 1] + list(range(0, n, 7))))
    for bi in range(b):
        Lc = lens[bi]
        for i in (r for r in rows if r < n):
            keys = list(range(Lc + i + 1))
            ref = OM.Model.attention(g, Q[bi, i], K[bi][:, keys, :].transpose(1, 0, 2),
                                     V[bi][:, keys, :].transpose(1, 0, 2))
            err = np.abs(got[bi, i] - ref)
            assert np.all(err <= 2e-2 + 2e-2 * np.abs(ref)), (name, bi, i, float(err.max()))
