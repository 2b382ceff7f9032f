"""Pins for oracle/spec.py: the invariants the paper and the north star fix
(no GPU).  I1 greedy-spec == vanilla, I3 compaction == sequential KV, I4 tau
bounds + teacher forcing, I5/I6 typical special cases, I7 tree DP == brute-force
Medusa row formulation, I8 N=1 == vanilla, I9 batched == unbatched."""
import math

import numpy as np
import pytest

import synth
from oracle import model as M
from oracle import spec as SP
from oracle import tree as T

CFG = synth.model_cfg("tiny")


def _model(mode="bf16", n_medusa=3, **over):
    cfg = synth.model_cfg("tiny", **over)
    return M.Model(cfg, M.Weights(cfg, n_medusa=n_medusa, seed=0), mode)


@pytest.fixture(scope="module")
def models():
    return {mode: _model(mode) for mode in ("fp64", "fp32", "bf16")}


@pytest.mark.parametrize("mode", ["fp64", "fp32", "bf16"])
def test_greedy_spec_equals_vanilla_and_kv(models, mode):
    """C1: 32-token prompt, 32 greedy tokens, tiny16 tree, x = 64 (BASELINE configs[0])."""
    m = models[mode]
    prompt = synth.prompt_tokens(0, 0, 32, CFG["vocab"])
    ref, kv_ref = SP.vanilla_generate(m, prompt, 32)
    s = SP.Session(m, synth.TINY16, batch=1, max_seq_len=64)
    s.prefill(0, prompt)
    out, taus = s.generate(0, 32)
    assert out == ref                                            # I1 token-identical (bitwise decisions)
    assert all(1 <= t <= s.l + 1 for t in taus)                   # I4 tau bounds
    Lc = s.Lc[0]
    assert Lc == 64
    for li in range(m.n_layers):                                 # I3 KV after compaction == sequential KV
        assert np.array_equal(s.kv.K[li][0][:, :Lc], kv_ref.K[li][0][:, :Lc])
        assert np.array_equal(s.kv.V[li][0][:, :Lc], kv_ref.V[li][0][:, :Lc])


def test_single_node_tree_is_vanilla(models):
    """I8: N = 1 tree (no heads used) == vanilla decoding."""
    m = models["bf16"]
    prompt = synth.prompt_tokens(1, 0, 20, CFG["vocab"])
    ref, _ = SP.vanilla_generate(m, prompt, 12)
    s = SP.Session(m, [], batch=1, max_seq_len=40)
    s.prefill(0, prompt)
    out, taus = s.generate(0, 12)
    assert out == ref and taus == [1] * 12


def _inject(s, seq, stream_after_prompt, P, diverge_depth=None):
    """Teacher forcing: head i's rank-0 token := the vanilla token at depth i+1;
    at ``diverge_depth`` j the correct token is removed from head j-1's top-k."""
    off = s.Lc[seq] - P
    assert s.root[seq] == stream_after_prompt[off]
    V = s.m.cfg["vocab"]
    for i in range(s.l):
        want = stream_after_prompt[off + 1 + i]
        lst = [t for t in s.topk_tok[seq][i] if t != want]
        if diverge_depth is not None and i == diverge_depth - 1:
            fill = [t for t in range(V) if t != want and t not in lst]
            s.topk_tok[seq][i] = (lst + fill)[:s.K]
        else:
            s.topk_tok[seq][i] = ([want] + lst)[:s.K]


@pytest.mark.parametrize("diverge", [None, 1, 2, 3, 4])
def test_teacher_forced_acceptance_length(diverge):
    """I4: injecting the vanilla continuation at rank 0 of every head gives
    a = l = 4 on V64 every step; a divergence at depth j gives a = j - 1."""
    m = _model("bf16", n_medusa=4)
    P = 16
    prompt = synth.prompt_tokens(2, 0, P, CFG["vocab"])
    stream, _ = SP.vanilla_generate(m, prompt, 40)
    s = SP.Session(m, synth.V64, batch=1, max_seq_len=P + 40)
    s.prefill(0, prompt)
    for _ in range(4):
        _inject(s, 0, stream, P, diverge)
        r = s.step(0)
        assert r["a"] == (4 if diverge is None else diverge - 1)
        assert r["emitted"] == stream[s.Lc[0] - P - len(r["emitted"]): s.Lc[0] - P]


def test_typical_low_temperature_equals_greedy(models):
    """I5: T -> 0 makes P one-hot at the argmax, H -> 0, thr -> min(eps, alpha) =
    0.09, so the typical test accepts exactly the argmax child = greedy."""
    m = models["bf16"]
    prompt = synth.prompt_tokens(4, 0, 24, CFG["vocab"])
    outs = []
    for mode, kw in (("greedy", {}), ("typical", dict(temperature=1e-7, eps=0.09, alpha=0.3))):
        s = SP.Session(m, synth.TINY16, batch=1, max_seq_len=60)
        s.prefill(0, prompt)
        outs.append(s.generate(0, 20, mode, **kw))
    assert outs[0] == outs[1]


def test_typical_eps_zero_accepts_everything(models):
    """I6: eps = 0 => thr = 0 => every node with P > 0 is accepted => a = l and
    the chosen node is the max-likelihood deepest node."""
    m = models["fp64"]
    prompt = synth.prompt_tokens(5, 0, 12, CFG["vocab"])
    s = SP.Session(m, synth.TINY16, batch=1, max_seq_len=60)
    s.prefill(0, prompt)
    for _ in range(3):
        tok, _ = s.propose(0)
        r = s.step(0, "typical", temperature=0.7, eps=0.0, alpha=0.3)
        assert r["a"] == s.l
        deep = [n for n in range(s.N) if s.tree.depth[n] == s.l]

        def ll(n):
            out, c = 0.0, n
            while c > 0:
                p = s.tree.parent[c]
                P, _ = SP.typical_stats(r["Z"][p], 0.7)
                out += math.log(P[r["tok"][c]])
                c = p
            return out
        assert r["chosen"] == max(deep, key=ll)


def _brute_medusa(tree, tok, Z, mode, temp=0.7, eps=0.09, alpha=0.3):
    """Medusa's row formulation: S candidate rows (DFS order), per-row verified
    flags, cumprod -> accepted length; longest row, then max likelihood, then
    the first row.  Written independently of Session.accept."""
    rows = T.candidate_paths(tree)
    best = None
    for r, row in enumerate(rows):
        ids = [i for i in row if i >= 0]
        ok, ll, length = True, 0.0, 0
        for j in range(1, len(ids)):
            p, c = ids[j - 1], ids[j]
            z = np.asarray(Z[p], dtype=np.float64)
            if mode == "greedy":
                good = tok[c] == int(np.flatnonzero(z == z.max())[0])
                lp = 0.0
            else:
                e = np.exp((z - z.max()) / temp)
                P = e / e.sum()
                H = -np.sum(P[P > 0] * np.log(P[P > 0]))
                good = P[tok[c]] > min(eps, alpha * math.exp(-H))
                lp = math.log(P[tok[c]])
            ok = ok and good
            if not ok:
                break
            length, ll = j, ll + lp
        key = (length, ll if mode == "typical" else 0.0, -r)
        if best is None or key > best[0]:
            best = (key, r, ids[:length + 1])
    return best[0][0], best[1] if best[0][0] > 0 else 0, best[2]


@pytest.mark.parametrize("mode", ["greedy", "typical"])
def test_tree_dp_equals_brute_force_rows(mode):
    """I7 on random logits with induced argmax ties and random prefixes of V64."""
    rng = np.random.default_rng(11)
    V = 12
    m = _model("fp64", n_medusa=4)
    for trial in range(300):
        choices = synth.V64[: int(rng.integers(1, 64))]
        s = SP.Session(m, choices, batch=1, max_seq_len=8)
        tr = s.tree
        tok = [int(rng.integers(V))] + [0] * (tr.N - 1)
        for n in range(1, tr.N):                                   # siblings distinct (top-k ranks)
            tok[n] = (7 * tr.rank[n] + tr.depth[n]) % V
        Z = []
        for n in range(tr.N):
            z = np.round(rng.standard_normal(V) * 2, 1)            # ties happen at 0.1 resolution
            if rng.random() < 0.6:                                # make some child the argmax
                kids = tr.children(n)
                if kids:
                    z[tok[kids[int(rng.integers(len(kids)))]]] = z.max() + (0.0 if rng.random() < 0.3 else 0.5)
            Z.append(z)
        a, chosen, best_leaf, path = s.accept(tok, Z, mode, temperature=0.7, eps=0.2, alpha=0.3)
        ba, brow, bpath = _brute_medusa(tr, tok, Z, mode, temp=0.7, eps=0.2, alpha=0.3)
        assert a == ba, trial
        assert path == bpath, trial
        assert best_leaf == brow, trial


def test_batched_equals_unbatched(models):
    """I9: each sequence of a batch == its own unbatched run."""
    m = models["bf16"]
    prompts = [synth.prompt_tokens(9, b, 8 + 5 * b, CFG["vocab"]) for b in range(3)]
    sb = SP.Session(m, synth.TINY16, batch=3, max_seq_len=50)
    for b, p in enumerate(prompts):
        sb.prefill(b, p)
    got = [[] for _ in range(3)]
    for _ in range(6):
        for b in range(3):
            got[b] += sb.step(b)["emitted"]
    for b, p in enumerate(prompts):
        s1 = SP.Session(m, synth.TINY16, batch=1, max_seq_len=50)
        s1.prefill(0, p)
        one = []
        for _ in range(6):
            one += s1.step(0)["emitted"]
        assert one == got[b]


def test_budget_and_capacity(models):
    m = models["bf16"]
    prompt = synth.prompt_tokens(6, 0, 30, CFG["vocab"])
    s = SP.Session(m, synth.TINY16, batch=1, max_seq_len=34)
    with pytest.raises(SP.KVCapacityError):
        s.prefill(0, synth.prompt_tokens(6, 0, 35, CFG["vocab"]))
    s.prefill(0, prompt)
    out, _ = s.generate(0, 3)                     # budget clamp: exactly 3 emitted
    assert len(out) == 3 and s.Lc[0] == 33
    r = s.step(0)                                 # x - Lc - 1 = 0 -> only the root
    assert r["a_eff"] == 0 and s.Lc[0] == 34
    with pytest.raises(SP.KVCapacityError):
        s.step(0)
