"""fp32 parity mode and C2-shape parity (needs a B200).

North star: the GPU path matches the oracle bit-exactly on integer outputs and
"logits and KV within an absolute/relative tolerance of 2e-2 in bf16 (1e-4 in
fp32 mode)".  sm_model_cfg.dtype = SM_DTYPE_FP32 keeps activations, K/V and
softmax in fp32 (weights: the same bf16 tensors, R0); the oracle's "fp32" mode
rounds to fp32 at the same storage points.

Also: C2 shapes (Vicuna-7B widths: d 4096, 32 heads of 128, F 11008, V 32000,
V64 tree, 4 heads) at 2 layers, on oracle rows sampled
from the 64-node tree (ancestor-closed, so the oracle computes them one by one)."""
import numpy as np
import pytest
import torch

import synth
from oracle import model as OM
from oracle import spec as OS
from oracle import tree as OT

pytestmark = pytest.mark.gpu

TINY = synth.model_cfg("tiny")
TOL = {"fp32": 1e-4, "bf16": 2e-2}


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


def build(sm, cfg, n_medusa, choices, batch, x, dtype, seed=0, medusa_init=False):
    W = sm.allocate_weights(cfg, n_medusa, seed=seed, medusa_init=medusa_init)
    tree = sm.Tree(choices, topk=10)
    model = sm.Model(cfg, W, max_rows=max(batch * tree.N, 64), max_batch=batch, max_seq_len=x + tree.N, dtype=dtype)
    kv = sm.KVCache(model, tree, batch, x)
    return W, tree, model, kv


def close(got, ref, tol):
    """|got - ref| <= tol * (1 + |ref|) elementwise (absolute below 1, relative above)."""
    err = np.abs(got - ref)
    return bool(np.all(err <= tol * (1.0 + np.abs(ref)))), float(err.max())


# ------------------------------------------------------------------ C1 in fp32
def test_fp32_c1_logits_and_kv_within_1e4(sm):
    prompt = synth.prompt_tokens(0, 0, 32, TINY["vocab"])
    W, tree, model, kv = build(sm, TINY, 3, synth.TINY16, 1, 64, "fp32")
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    tt = torch.zeros(1, tree.N, dtype=torch.int32, device="cuda")
    kv.propose(tt)
    logits = torch.zeros(1, tree.N, TINY["vocab"], dtype=torch.float32, device="cuda")
    kv.verify(tt, logits)
    torch.cuda.synchronize()
    Zg = logits[0].cpu().numpy().astype(np.float64)
    kvl = kv.layout()
    assert kvl.dtype == torch.float32
    for mode in ("fp32", "fp64"):
        s = OS.Session(OM.Model(TINY, OM.Weights(TINY, n_medusa=3, seed=0), mode), synth.TINY16, 1, 64)
        s.prefill(0, prompt)
        tok, _ = s.propose(0)
        assert tt[0].cpu().tolist() == [int(t) for t in tok]
        Z, _ = s.verify(0, tok)
        ok, err = close(Zg, np.stack(Z), 1e-4)
        assert ok, (mode, err)
        for li in range(TINY["n_layers"]):
            for c in (0, 1):
                got = kvl[li, c, 0].cpu().numpy().astype(np.float64)[:, : 32 + tree.N]
                ref = (s.kv.K if c == 0 else s.kv.V)[li][0][:, : 32 + tree.N]
                ok, err = close(got, ref, 1e-4)
                assert ok, (mode, li, c, err)
    # the fp32 mode really is more precise than the bf16 path on the same inputs
    s16 = OS.Session(OM.Model(TINY, OM.Weights(TINY, n_medusa=3, seed=0), "fp64"), synth.TINY16, 1, 64)
    s16.prefill(0, prompt)
    Z64, _ = s16.verify(0, s16.propose(0)[0])
    assert np.max(np.abs(Zg - np.stack(Z64))) < 1e-5


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_fp32_c1_greedy_tokens_equal_oracle_and_vanilla(sm, seed):
    prompt = synth.prompt_tokens(seed, 0, 32, TINY["vocab"])
    s = OS.Session(OM.Model(TINY, OM.Weights(TINY, n_medusa=3, seed=seed), "fp32"), synth.TINY16, 1, 64)
    s.prefill(0, prompt)
    ref, _ = s.generate(0, 32)
    vanilla, _ = OS.vanilla_generate(s.m, prompt, 32)
    assert ref == vanilla
    W, tree, model, kv = build(sm, TINY, 3, synth.TINY16, 1, 64, "fp32", seed=seed)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    out = sm.AcceptOut(1, tree.depth)
    budget = torch.full((1,), 32, dtype=torch.int32, device="cuda")
    cfg = sm.accept_cfg(sm.GREEDY, max_new=budget)
    got = []
    while len(got) < 32:
        kv.step(cfg, out)
        ne = int(out.n_emit.item())
        got += out.emit_tok[0, :ne].cpu().tolist()
        budget -= out.n_emit
    assert got == ref
    assert int(kv.lengths()[0]) == 64


def test_fp32_typical_matches_oracle(sm):
    prompt = synth.prompt_tokens(5, 0, 24, TINY["vocab"])
    typ = dict(temperature=0.7, eps=0.09, alpha=0.3)
    s = OS.Session(OM.Model(TINY, OM.Weights(TINY, n_medusa=3, seed=0), "fp32"), synth.TINY16, 1, 128)
    s.prefill(0, prompt)
    W, tree, model, kv = build(sm, TINY, 3, synth.TINY16, 1, 128, "fp32")
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    out = sm.AcceptOut(1, tree.depth)
    cfg = sm.accept_cfg(sm.TYPICAL, **typ)
    for _ in range(8):
        r = s.step(0, "typical", **typ)
        kv.step(cfg, out)
        torch.cuda.synchronize()
        ne = out.n_emit.item()
        assert out.emit_tok[0, :ne].cpu().tolist() == r["emitted"]
        assert (out.acc_len.item(), out.best_leaf.item()) == (r["a"], r["best_leaf"])


def test_fp32_rejects_tensor_parallel_and_large_rows(sm):
    W = sm.allocate_weights(TINY, 3, seed=0)
    with pytest.raises(sm.SpecMemoError):
        sm.Model(TINY, W, max_rows=400, max_batch=1, max_seq_len=80, dtype="fp32")
    assert sm.kv_bytes(TINY, 1, 64, 16, dtype="fp32") == 2 * sm.kv_bytes(TINY, 1, 64, 16)


# ------------------------------------------------------------------ C2 shapes, 2 layers, sampled tree rows
C2 = synth.model_cfg("vicuna7b", n_layers=2)
PROMPT = 12
# ancestor-closed sample of V64 nodes: the root, all of depth 1, one full-depth path and node 63's chain
_t = OT.build(synth.V64)
SAMPLE = sorted({0, *range(1, 11), *OT.ancestors(_t, 57), 57, *OT.ancestors(_t, 63), 63,
                 *OT.ancestors(_t, 40), 40})


@pytest.fixture(scope="module")
def c2_oracle_weights():
    return OM.Weights(C2, n_medusa=4, seed=0, medusa_init=True)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_c2_shape_two_layers_sampled_rows(sm, c2_oracle_weights, dtype):
    prompt = synth.prompt_tokens(11, 0, PROMPT, C2["vocab"])
    W, tree, model, kv = build(sm, C2, 4, synth.V64, 1, 64, dtype, medusa_init=True)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    tt = torch.zeros(1, tree.N, dtype=torch.int32, device="cuda")
    kv.propose(tt)
    logits = torch.zeros(1, tree.N, C2["vocab"], dtype=torch.float32, device="cuda")
    kv.verify(tt, logits)
    torch.cuda.synchronize()
    tok_gpu = tt[0].cpu().tolist()
    # oracle: prompt rows, then the sampled tree rows with the GPU's tree tokens (lock step)
    m = OM.Model(C2, c2_oracle_weights, dtype)
    s = OS.Session(m, synth.V64, 1, 64)
    s.prefill(0, prompt)
    tok_ref, _ = s.propose(0)
    # tree tokens are integer outputs (root argmax + head top-K): bit-exact wherever the oracle's
    # top-K gap clears the guard (every one at fp32), else a valid near-tie choice
    assert tok_gpu[0] == tok_ref[0]
    tr0 = s.tree
    u = np.asarray(m.head_logits(0, s.last_hf[0]), np.float64)  # Medusa-init: every head = LM head
    order = OM.topk_desc(u, 11)
    guard = 1e-5 if dtype == "fp32" else 0.05
    for n in range(1, tree.N):
        rk = tr0.rank[n]
        gap = min(u[order[rk - 1]] - u[order[rk]] if rk > 0 else np.inf, u[order[rk]] - u[order[rk + 1]])
        if gap >= guard:
            assert tok_gpu[n] == tok_ref[n], (n, tok_gpu[n], tok_ref[n])
        else:
            assert abs(u[tok_gpu[n]] - u[order[rk]]) <= 2 * guard, n
    tr = s.tree
    Zg = logits[0].cpu().numpy().astype(np.float64)
    kvl = kv.layout()
    tol = TOL[dtype]
    for n in SAMPLE:
        keys = list(range(PROMPT)) + [PROMPT + a for a in OT.ancestors(tr, n)] + [PROMPT + n]
        z, _ = m.forward_row(s.kv, 0, int(tok_gpu[n]), PROMPT + tr.depth[n], PROMPT + n, keys)
        if dtype == "fp32":  # elementwise 1e-4; argmax bit-exact
            ok, err = close(Zg[n], z, tol)
            assert ok, (dtype, n, err)
            assert int(np.argmax(Zg[n])) == OM.argmax_lowest(z)
        else:
            # bf16 at 7B width (reading Q29): per row at most 1 % of the elements over the
            # 2e-2 (1 + |z|) bar and none over 3x it (one-ulp storage-point differences cascade);
            # argmax decisions with margin are bit-exact
            r = np.abs(Zg[n] - z) / (tol * (1 + np.abs(z)))
            assert np.mean(r > 1) <= 1e-2 and r.max() <= 3.0, (n, np.mean(r > 1), r.max())
            zs = np.sort(z)[::-1]
            if zs[0] - zs[1] > 1e-2 * np.abs(z).max():
                assert int(np.argmax(Zg[n])) == OM.argmax_lowest(z)
    for li in range(2):
        for c in (0, 1):
            got = kvl[li, c, 0].float().cpu().numpy().astype(np.float64)
            ref = (s.kv.K if c == 0 else s.kv.V)[li][0]
            slots = list(range(PROMPT)) + [PROMPT + n for n in SAMPLE]
            g, r = got[:, slots], ref[:, slots]
            if dtype == "fp32":
                ok, err = close(g, r, tol)
                assert ok, (dtype, li, c, err)
            else:  # reading Q29: layer 0 elementwise; deeper layers the per-row exceedance bound
                r = np.abs(g - r) / (tol * (1 + np.abs(r)))
                if li == 0:
                    assert r.max() <= 1.0, (li, c, r.max())
                else:
                    assert np.mean(r > 1) <= 1e-2 and r.max() <= 3.0, (li, c, np.mean(r > 1), r.max())


# ------------------------------------------------------------------ fused K2 tile epilogues (hd = 128)
# The fused path (RoPE/cache write, SiLU and residual+deferred-norm as K2 tile epilogues,
# gemm.cu kEpi*) needs head_dim 128 and d % 128 == 0, which C1 does not have; this small
# model has both.  Seeds screened by the oracle: every greedy decision over 24 tokens has a
# top1-top2 margin >= 2e-3 (seeds 0-4, 6: 2.4e-2, 9.8e-3, 3.5e-3, 5.4e-2, 3.9e-2, 5.0e-3).
S128 = synth.model_cfg("tiny", d_model=256, n_heads=2, n_kv_heads=1, head_dim=128, d_ffn=512, vocab=512)


@pytest.mark.parametrize("fused", [1, 0], ids=["fused", "consumers"])
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4, 6])
def test_fused_epilogues_tokens_equal_oracle(sm, seed, fused):
    sm.set_option("fused_epilogue", fused)
    try:
        prompt = synth.prompt_tokens(seed, 0, 24, S128["vocab"])
        s = OS.Session(OM.Model(S128, OM.Weights(S128, n_medusa=3, seed=seed), "bf16"), synth.TINY16, 1, 64)
        s.prefill(0, prompt)
        ref, _ = s.generate(0, 24)
        assert ref == OS.vanilla_generate(s.m, prompt, 24)[0]
        W, tree, model, kv = build(sm, S128, 3, synth.TINY16, 1, 64, "bf16", seed=seed)
        kv.prefill(0, torch.from_numpy(prompt).cuda())
        out = sm.AcceptOut(1, tree.depth)
        budget = torch.full((1,), 24, dtype=torch.int32, device="cuda")
        cfg = sm.accept_cfg(sm.GREEDY, max_new=budget)
        got = []
        while len(got) < 24:
            kv.step(cfg, out)
            ne = int(out.n_emit.item())
            got += out.emit_tok[0, :ne].cpu().tolist()
            budget -= out.n_emit
        assert got == ref
    finally:
        sm.set_option("fused_epilogue", 0)  # the library default


def test_fused_epilogues_logits_and_kv(sm):
    prompt = synth.prompt_tokens(3, 0, 20, S128["vocab"])
    s = OS.Session(OM.Model(S128, OM.Weights(S128, n_medusa=3, seed=3), "bf16"), synth.TINY16, 1, 64)
    s.prefill(0, prompt)
    tok, _ = s.propose(0)
    Z, _ = s.verify(0, tok)
    res = {}
    for fused in (1, 0):
        sm.set_option("fused_epilogue", fused)
        W, tree, model, kv = build(sm, S128, 3, synth.TINY16, 1, 64, "bf16", seed=3)
        kv.prefill(0, torch.from_numpy(prompt).cuda())
        tt = torch.zeros(1, tree.N, dtype=torch.int32, device="cuda")
        kv.propose(tt)
        torch.cuda.synchronize()
        assert int(tt[0, 0]) == int(tok[0])  # root; head top-10s of V = 512 carry near-ties: lock step below
        tt = torch.tensor([[int(t) for t in tok]], dtype=torch.int32, device="cuda")
        logits = torch.zeros(1, tree.N, S128["vocab"], dtype=torch.float32, device="cuda")
        kv.verify(tt, logits)
        torch.cuda.synchronize()
        res[fused] = (logits[0].cpu().numpy().astype(np.float64), kv.layout().float().cpu().numpy())
    sm.set_option("fused_epilogue", 0)  # the library default
    for fused, (Zg, kvl) in res.items():
        ok, err = close(Zg, np.stack(Z), 2e-2)
        assert ok, (fused, err)
        for li in range(2):
            for c in (0, 1):
                ref = (s.kv.K if c == 0 else s.kv.V)[li][0][:, : 20 + 16]
                ok, err = close(kvl[li, c, 0][:, : 20 + 16], ref, 2e-2)
                assert ok, (fused, li, c, err)
    # both paths sum the same partials in the same order; only rs's sum of squares differs in order
    assert np.max(np.abs(res[1][0] - res[0][0])) < 1e-2


def test_c2_width_batched_pair_path_matches_unbatched(sm):
    """b = 3 sequences of the V64 tree -> M = 192 token rows: the verify GEMMs take the 2-SM
    (cta_group::2) K2 variant with one TMEM buffer per CTA; each sequence's logits and K/V must
    equal its b = 1 run (M = 64, single-SM K2, oracle-checked above) within the bf16 bar (Q29)."""
    prompts = [synth.prompt_tokens(20 + i, 0, 10 + 3 * i, C2["vocab"]) for i in range(3)]
    W = sm.allocate_weights(C2, 4, seed=0, medusa_init=True)
    tree = sm.Tree(synth.V64, topk=10)

    def run(b, ps):
        model = sm.Model(C2, W, max_rows=b * tree.N, max_batch=b, max_seq_len=64 + tree.N)
        kv = sm.KVCache(model, tree, b, 64)
        for i, p in enumerate(ps):
            kv.prefill(i, torch.from_numpy(p).cuda())
        tt = torch.zeros(b, tree.N, dtype=torch.int32, device="cuda")
        kv.propose(tt)
        logits = torch.zeros(b, tree.N, C2["vocab"], dtype=torch.float32, device="cuda")
        kv.verify(tt, logits)
        torch.cuda.synchronize()
        return tt.cpu(), logits.cpu().double(), kv.layout().float().cpu().double()

    tb, zb, kb = run(3, prompts)
    for i, p in enumerate(prompts):
        t1, z1, k1 = run(1, [p])
        # same prefill, same heads path: the tree tokens are bit-identical
        assert torch.equal(tb[i], t1[0])
        # verify rows: M = 192 on the 2-SM K2 vs M = 64 single-SM -- only the fp32 summation order of
        # the split-K partials differs; the bf16 bar per row (Q29: <= 1 % of elements over
        # 2e-2 (1 + |z|), none over 3x)
        L = len(p)
        for n in range(tree.N):
            bar = 2e-2 * (1 + z1[0, n].abs())
            r = (zb[i, n] - z1[0, n]).abs() / bar
            assert float((r > 1).double().mean()) <= 1e-2 and float(r.max()) <= 3.0, n
        for li in range(2):
            for c in (0, 1):
                a, ref = kb[li, c, i][:, :L + tree.N], k1[li, c, 0][:, :L + tree.N]  # prompt + tree slots
                r = (a - ref).abs() / (2e-2 * (1 + ref.abs()))
                assert float((r > 1).double().mean()) <= 1e-2 and float(r.max()) <= 3.0, (li, c)
