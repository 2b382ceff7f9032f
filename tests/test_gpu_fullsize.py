"""Parity at BASELINE.json's full C2 size, in the launch configuration bench.py
times (Vicuna-7B shape, 32 layers, V64 tree, bs=1, x=2048, prefilled to Lc=1024),
through properties that hold at any size (needs a B200).

The oracle cannot run 32 random 7B layers in seconds, so here it checks what is
decided from the GPU's own float outputs: with the GPU's verify logits Z as input,
the oracle's tree DP (oracle.spec.Session.accept) must reproduce sm_accept's
accepted length, best leaf and path bit-exactly (greedy and typical, decisions with
margin); the emitted tokens, the next root (argmax of the last accepted row) and
the proposal rule tok[n] = topk[depth(n)-1][rank(n)] are integer
identities; compaction must move the tree-slot K/V rows bit for bit.
Float parity of the same kernels at these widths: tests/test_gpu_fp32.py."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import model as OM
from oracle import spec as OS

pytestmark = pytest.mark.gpu

C2 = synth.model_cfg("vicuna7b")
X, LC0 = 2048, 1024
TYP = dict(temperature=0.7, eps=0.09, alpha=0.3)


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


@pytest.fixture(scope="module")
def c2(sm):
    # Medusa-init heads (R = 0, U = W_lm, reading Q18) so greedy steps accept nodes (tau > 1)
    W = sm.allocate_weights(C2, 4, seed=0, medusa_init=True)
    tree = sm.Tree(synth.V64, topk=synth.TOPK)
    model = sm.Model(C2, W, max_rows=256, max_batch=1, max_seq_len=X + tree.N)
    return W, tree, model


def oracle_dp():
    tiny = synth.model_cfg("tiny")  # the DP needs only the tree; the model is a placeholder
    return OS.Session(OM.Model(tiny, OM.Weights(tiny, n_medusa=4, seed=0), "fp64"), synth.V64, 1, 8)


def typical_margin_ok(s, tok, Z, a_path):
    """Every typical decision on accepted parents is away from its threshold, and the
    deepest-node likelihood choice is not a near-tie."""
    tr = s.tree
    acc, ll = {0: True}, {0: 0.0}
    for c in range(1, s.N):
        p = tr.parent[c]
        if not acc.get(p):
            acc[c] = False
            continue
        P, H = OS.typical_stats(Z[p], TYP["temperature"])
        thr = min(TYP["eps"], TYP["alpha"] * math.exp(-H))
        pc = P[int(tok[c])]
        if abs(pc - thr) < 1e-3 * thr:
            return False
        acc[c] = pc > thr
        ll[c] = ll[p] + math.log(pc) if acc[c] else -math.inf
    a = max(tr.depth[n] for n in range(s.N) if acc[n])
    deep = sorted((ll[n] for n in range(s.N) if acc[n] and tr.depth[n] == a), reverse=True)
    return not (len(deep) > 1 and deep[0] - deep[1] < 1e-4)


@pytest.mark.parametrize("mode", ["greedy", "typical"])
def test_c2_full_size_step_properties(sm, c2, mode):
    W, tree, model = c2
    kv = sm.KVCache(model, tree, 1, X)
    prompt = synth.prompt_tokens(0, 0, LC0, C2["vocab"])
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    out = sm.AcceptOut(1, tree.depth)
    acfg = sm.accept_cfg(sm.TYPICAL if mode == "typical" else sm.GREEDY, **(TYP if mode == "typical" else {}))
    q = tree.query()
    depth, rank, N = q["node_depth"], q["rank"], tree.N
    s = oracle_dp()
    tt = torch.zeros(1, N, dtype=torch.int32, device="cuda")
    logits = torch.zeros(1, N, C2["vocab"], dtype=torch.float32, device="cuda")
    kvl = kv.layout()
    compared, taus, prev = 0, [], None
    for step in range(6):
        Lc = int(kv.lengths()[0])
        kv.propose(tt)
        kv.verify(tt, logits)
        torch.cuda.synchronize()
        tok = tt[0].cpu().numpy()
        Z = logits[0].cpu().numpy().astype(np.float64)
        if prev is not None:
            # proposal rule at the previous accepted node: root = argmax of its
            # base logits; depth-d node of rank r = head d-1's r-th best token.  Medusa-init
            # heads compute U r = W_lm hf, the same values up to fp32 summation order, so the
            # ranks are compared where the top-(K+1) values are separated by more than that.
            zl = prev
            assert int(tok[0]) == OM.argmax_lowest(zl)
            top = OM.topk_desc(zl, synth.TOPK + 1)
            gaps = np.abs(np.diff(zl[top]))
            if gaps.min() > 1e-5 * np.abs(zl[top[0]]):
                for n in range(1, N):
                    assert int(tok[n]) == top[rank[n]], (step, n)
        tree_kv = kvl[:, :, 0, :, Lc:Lc + N].clone()          # K/V of the tree slots before compaction
        kv.accept(acfg, out)
        torch.cuda.synchronize()
        a, bl, ne = out.acc_len.item(), out.best_leaf.item(), out.n_emit.item()
        path = [p for p in out.path[0].cpu().tolist() if p >= 0]
        emit = out.emit_tok[0, :ne].cpu().tolist()
        taus.append(ne)
        # integer identities from the GPU's own outputs
        assert len(path) == a + 1 and path[0] == 0 and ne == a + 1
        assert all(int(depth[path[j]]) == j for j in range(a + 1))
        assert emit == [int(tok[p]) for p in path]
        assert all(q["parent"][path[j]] == path[j - 1] for j in range(1, a + 1))
        assert int(kv.lengths()[0]) == Lc + ne
        # compaction: slot Lc + j now holds the K/V the tree wrote at slot Lc + path[j] (bitwise)
        after = kvl[:, :, 0, :, Lc:Lc + ne]
        for j in range(ne):
            assert torch.equal(after[:, :, :, j], tree_kv[:, :, :, path[j]]), (step, j)
        # acceptance: the oracle's tree DP on the GPU's logits
        if mode == "greedy":
            ok = True
            for p in set(path):
                zs = np.sort(Z[p])[::-1]
                ok &= bool(zs[0] - zs[1] > 1e-6 * abs(zs[0]))
        else:
            ok = typical_margin_ok(s, tok, Z, path)
        if ok:
            ra, rchosen, rbl, rpath = s.accept(tok, Z, mode, **(TYP if mode == "typical" else {}))
            assert (a, bl, path) == (ra, rbl, rpath), step
            compared += 1
        prev = Z[path[-1]]
    assert compared >= 4
    # a forced full-depth path (test hook d_forced_path): compaction of l = 4 rows at full size
    forced = torch.tensor([[0, 1, 11, 34, 57]], dtype=torch.int32, device="cuda")   # rank path (0, 0, 0, 0)
    Lc = int(kv.lengths()[0])
    kv.propose(tt)
    kv.verify(tt, logits)
    torch.cuda.synchronize()
    tree_kv = kvl[:, :, 0, :, Lc:Lc + N].clone()
    kv.accept(sm.accept_cfg(forced_path=forced), out)
    torch.cuda.synchronize()
    assert out.n_emit.item() == 5 and int(kv.lengths()[0]) == Lc + 5
    assert out.emit_tok[0].cpu().tolist() == [int(tt[0, p]) for p in (0, 1, 11, 34, 57)]
    after = kvl[:, :, 0, :, Lc:Lc + 5]
    for j, p in enumerate((0, 1, 11, 34, 57)):
        assert torch.equal(after[:, :, :, j], tree_kv[:, :, :, p]), j
