"""End-to-end parity of the CUDA speculative step with the oracle (needs a B200).

C1 (BASELINE configs[0]): tiny random-init Llama (2 layers, d=64, 4 heads,
V=256) + 3 Medusa heads, tiny16 tree, 32-token prompt, 32 greedy tokens.
Integer outputs (emitted tokens, accepted length, best leaf, path) must be
bit-equal to the oracle -- and to vanilla greedy -- on seeds whose decisions the
oracle shows to have margin; logits and KV within 2e-2."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import model as OM
from oracle import spec as OS
from oracle import tree as OT

pytestmark = pytest.mark.gpu

CFG = synth.model_cfg("tiny")
GUARD = 2e-3       # min top1-top2 logit gap for a greedy decision to count as unambiguous


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


def build_gpu(sm, cfg, n_medusa, choices, batch, x, seed=0, medusa_init=False, max_rows=None):
    W = sm.allocate_weights(cfg, n_medusa, seed=seed, medusa_init=medusa_init)
    tree = sm.Tree(choices, topk=10)
    model = sm.Model(cfg, W, max_rows=max_rows or max(batch * tree.N, 64), max_batch=batch,
                     max_seq_len=x + tree.N)
    kv = sm.KVCache(model, tree, batch, x)
    return W, tree, model, kv


def gpu_generate(sm, kv, out, n_new, mode=0, **typ):
    """Run sm_step until n_new tokens per sequence; returns per-seq token lists
    and per-step (acc_len, best_leaf, n_emit) records."""
    b = kv.batch
    budget = torch.full((b,), n_new, dtype=torch.int32, device="cuda")
    cfg = sm.accept_cfg(mode, max_new=budget, **typ)
    toks = [[] for _ in range(b)]
    recs = []
    for _ in range(4 * n_new):
        if all(len(t) >= n_new for t in toks):
            break
        kv.step(cfg, out)
        ne = out.n_emit.cpu().numpy()
        et = out.emit_tok.cpu().numpy()
        recs.append((out.acc_len.cpu().numpy().copy(), out.best_leaf.cpu().numpy().copy(), ne.copy(),
                     out.path.cpu().numpy().copy()))
        for s in range(b):
            toks[s] += et[s][: ne[s]].tolist()
        budget -= out.n_emit
    return toks, recs


def oracle_session(choices, n_medusa, batch, x, mode="bf16", seed=0, medusa_init=False):
    W = OM.Weights(CFG, n_medusa=n_medusa, seed=seed, medusa_init=medusa_init)
    return OS.Session(OM.Model(CFG, W, mode), choices, batch=batch, max_seq_len=x)


def greedy_margin(Z, path, a_eff, tree):
    """Smallest top1-top2 gap over the argmax decisions the step depends on:
    every accepted node that has children (its argmax decides acceptance) and
    the last emitted node (its argmax is the next root)."""
    gaps = []
    nodes = set(path[: a_eff + 1])
    for n in nodes:
        z = np.sort(np.asarray(Z[n]))[::-1]
        gaps.append(z[0] - z[1])
    return min(gaps)


# Seeds 1, 6, 10 are screened by the oracle: every argmax decision along the
# 32-token trajectory has a top1-top2 gap >= GUARD (4.8e-3, 2.5e-3, 3.9e-3).  Seeds
# 0, 2, 3, 7 contain near-ties (1.3e-3, 1.8e-4, 3.2e-4, 6.5e-4): there only the steps
# before the first ambiguous decision are compared (the trajectory may fork after).
@pytest.mark.parametrize("seed", [1, 6, 10, 0, 2, 3, 7])
def test_c1_greedy_tokens_equal_oracle_and_vanilla(sm, seed):
    prompt = synth.prompt_tokens(seed, 0, 32, CFG["vocab"])
    # oracle trajectory + margins
    s = oracle_session(synth.TINY16, 3, 1, 64, seed=seed)
    s.prefill(0, prompt)
    ref, ref_steps, margins = [], [], []
    while len(ref) < 32:
        r = s.step(0, budget=32 - len(ref))
        ref += r["emitted"]
        ref_steps.append((r["a"], r["best_leaf"], len(r["emitted"]), r["path"]))
        margins.append(greedy_margin(r["Z"], r["path"], r["a_eff"], s.tree))
    vanilla, _ = OS.vanilla_generate(s.m, prompt, 32)
    assert ref == vanilla
    # GPU
    W, tree, model, kv = build_gpu(sm, CFG, 3, synth.TINY16, 1, 64, seed=seed)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    out = sm.AcceptOut(1, tree.depth)
    got, recs = gpu_generate(sm, kv, out, 32)
    # compare up to the first ambiguous decision (margin < guard)
    n_ok = len(margins)
    for i, mg in enumerate(margins):
        if mg < GUARD:
            n_ok = i
            break
    if seed in (1, 6, 10):
        assert n_ok == len(margins), f"screened seed {seed} lost its margin: {margins}"
    ntok = sum(st[2] for st in ref_steps[:n_ok])
    assert got[0][:ntok] == ref[:ntok]
    for i in range(n_ok):
        acc, leaf, ne, path = recs[i]
        a, bl, nemit, opath = ref_steps[i]
        assert (int(acc[0]), int(leaf[0]), int(ne[0])) == (a, bl, nemit), i
        assert [p for p in path[0].tolist() if p >= 0] == opath, i
    if n_ok == len(margins):
        assert got[0] == ref
        assert kv.lengths()[0] == 64


def test_c1_logits_and_kv_within_tolerance(sm):
    prompt = synth.prompt_tokens(0, 0, 32, CFG["vocab"])
    s = oracle_session(synth.TINY16, 3, 1, 64)
    s.prefill(0, prompt)
    tok, _ = s.propose(0)
    Z, _ = s.verify(0, tok)
    W, tree, model, kv = build_gpu(sm, CFG, 3, synth.TINY16, 1, 64)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    tt = torch.zeros(1, tree.N, dtype=torch.int32, device="cuda")
    pos = torch.zeros(1, tree.N, dtype=torch.int32, device="cuda")
    kv.propose(tt, pos)
    torch.cuda.synchronize()
    assert tt[0].cpu().tolist() == [int(t) for t in tok]                    # K3 + propose bit-exact
    assert pos[0].cpu().tolist() == [32 + d for d in s.tree.depth]
    logits = torch.zeros(1, tree.N, CFG["vocab"], dtype=torch.float32, device="cuda")
    kv.verify(tt, logits)
    torch.cuda.synchronize()
    Zg = logits[0].cpu().numpy().astype(np.float64)
    Zo = np.stack(Z)
    assert np.max(np.abs(Zg - Zo)) < 2e-2
    assert np.max(np.abs(Zg - Zo)) / np.max(np.abs(Zo)) < 1e-2
    # KV of prefix and tree slots, every layer
    kvl = kv.layout()
    for li in range(CFG["n_layers"]):
        Kg = kvl[li, 0, 0].float().cpu().numpy()[:, : 32 + tree.N]
        Vg = kvl[li, 1, 0].float().cpu().numpy()[:, : 32 + tree.N]
        assert np.max(np.abs(Kg - s.kv.K[li][0][:, : 32 + tree.N])) < 2e-2
        assert np.max(np.abs(Vg - s.kv.V[li][0][:, : 32 + tree.N])) < 2e-2


def test_c1_vanilla_single_node_tree(sm):
    prompt = synth.prompt_tokens(3, 0, 20, CFG["vocab"])
    s = oracle_session([], 3, 1, 40)
    vanilla, _ = OS.vanilla_generate(s.m, prompt, 12)
    W, tree, model, kv = build_gpu(sm, CFG, 3, [], 1, 40)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    out = sm.AcceptOut(1, tree.depth)
    got, recs = gpu_generate(sm, kv, out, 12)
    assert got[0] == vanilla
    assert all(int(r[2][0]) == 1 for r in recs)


def test_batched_equals_unbatched(sm):
    b = 3
    prompts = [synth.prompt_tokens(9, i, 8 + 5 * i, CFG["vocab"]) for i in range(b)]
    W, tree, model, kv = build_gpu(sm, CFG, 3, synth.TINY16, b, 64)
    for i, p in enumerate(prompts):
        kv.prefill(i, torch.from_numpy(p).cuda())
    out = sm.AcceptOut(b, tree.depth)
    got, _ = gpu_generate(sm, kv, out, 16)
    for i, p in enumerate(prompts):
        _, _, _, kv1 = build_gpu(sm, CFG, 3, synth.TINY16, 1, 64)
        kv1.prefill(0, torch.from_numpy(p).cuda())
        out1 = sm.AcceptOut(1, tree.depth)
        one, _ = gpu_generate(sm, kv1, out1, 16)
        assert one[0] == got[i]
        # and the oracle
        s = oracle_session(synth.TINY16, 3, 1, 64)
        s.prefill(0, p)
        ref, _ = s.generate(0, 16)
        assert got[i] == ref


def test_teacher_forced_full_acceptance_and_compaction(sm):
    """Medusa-init heads (R = 0, U = W_lm) + a forced path: the GPU accepts the
    path it is given, compacts it, and its KV equals sequential decoding."""
    prompt = synth.prompt_tokens(4, 0, 16, CFG["vocab"])
    W, tree, model, kv = build_gpu(sm, CFG, 4, synth.V64, 1, 48)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    out = sm.AcceptOut(1, tree.depth)
    forced = torch.tensor([[0, 1, 11, 34, 57]], dtype=torch.int32, device="cuda")   # rank path (0,0,0,0)
    kv.step(sm.accept_cfg(forced_path=forced), out)
    torch.cuda.synchronize()
    assert out.acc_len.item() == 4 and out.n_emit.item() == 5
    assert kv.lengths()[0] == 21
    # the GPU's emitted tokens replayed through the oracle sequentially give the same KV
    emitted = out.emit_tok[0].cpu().tolist()
    m = OM.Model(CFG, OM.Weights(CFG, n_medusa=4, seed=0), "bf16")
    kvo = OM.KVCache(CFG["n_layers"], 1, CFG["n_kv_heads"], 64, CFG["head_dim"])
    seqt = list(prompt) + emitted
    for i, t in enumerate(seqt):
        m.forward_row(kvo, 0, int(t), i, i, list(range(i + 1)))
    kvl = kv.layout()
    for li in range(CFG["n_layers"]):
        Kg = kvl[li, 0, 0].float().cpu().numpy()[:, :21]
        assert np.max(np.abs(Kg - kvo.K[li][0][:, :21])) < 2e-2
        Vg = kvl[li, 1, 0].float().cpu().numpy()[:, :21]
        assert np.max(np.abs(Vg - kvo.V[li][0][:, :21])) < 2e-2


def test_typical_matches_oracle_until_ambiguous(sm):
    prompt = synth.prompt_tokens(5, 0, 24, CFG["vocab"])
    typ = dict(temperature=0.7, eps=0.09, alpha=0.3)
    # near-uniform tiny-model rows (H ~ 5.5 nats) accept almost every candidate:
    # tau ~ 4, so 12 steps need ~48 slots beyond the prompt
    s = oracle_session(synth.TINY16, 3, 1, 128)
    s.prefill(0, prompt)
    W, tree, model, kv = build_gpu(sm, CFG, 3, synth.TINY16, 1, 128)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    out = sm.AcceptOut(1, tree.depth)
    cfg = sm.accept_cfg(sm.TYPICAL, **typ)
    compared = 0
    for _ in range(12):
        r = s.step(0, "typical", **typ)
        # ambiguity of this step: |P - thr| near 0 or a likelihood near-tie among deepest nodes
        amb = False
        acc, ll = {0: True}, {0: 0.0}
        for c in range(1, s.N):
            p = s.tree.parent[c]
            P, H = OS.typical_stats(r["Z"][p], 0.7)
            thr = min(0.09, 0.3 * math.exp(-H))
            pc = P[r["tok"][c]]
            # bf16 logits carry ~1e-3 of rounding noise (R0..R10): P and the threshold move by
            # ~1e-3 relative, a path log-likelihood by up to ~1e-2 over l = 3 levels
            if abs(pc - thr) < 1e-2 * thr:
                amb = True
            acc[c] = acc[p] and pc > thr
            ll[c] = ll[p] + math.log(pc)
        deep = sorted((ll[n] for n in range(s.N) if acc[n] and s.tree.depth[n] == r["a"]), reverse=True)
        if len(deep) > 1 and deep[0] - deep[1] < 2e-2:
            amb = True
        kv.step(cfg, out)
        torch.cuda.synchronize()
        if amb:
            break
        ne = out.n_emit.item()
        assert out.emit_tok[0, :ne].cpu().tolist() == r["emitted"]
        assert out.acc_len.item() == r["a"]
        compared += 1
    assert compared >= 3
