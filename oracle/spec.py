"""The Medusa speculative step over a bounded KV cache (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows SURVEY §8.c.2 / DESIGN.md §3 step by step, in the paper's terms:

  propose  -- tree tokens from the heads' top-k at the last accepted node
              ("arity-k (equals to top-k token sampling from heads)",
              "L-many parallel decoding heads (equals to the number of tree
              levels)"; "top-k tokens of the first decoding head").
  verify   -- one forward of all N nodes; "prior to verification, attention mask
              assumes full acceptance": node n sees the committed prefix,
              its ancestors and itself (Eq. 2).  Positions continue "from the
              latest sequence length": pos = Lc + depth.
  accept   -- "sampled logits are evaluated to pass a certain threshold to be
              accepted followed by a cumulative product ... The longest
              candidate sequence that verified its tokens is accepted";
              typical acceptance with an entropy threshold.
  compact  -- the pre-allocated KV cache is "a scratch space ... frequently
              update[d] during verification stage": accepted nodes' K/V
              move to contiguous committed slots.

Vanilla greedy decoding (the plain definition the greedy mode must reproduce,
north star) is ``vanilla_generate`` -- token by token, separate code.
"""
from __future__ import annotations

import math

import numpy as np

from . import tree as T
from .model import KVCache, Model, argmax_lowest, topk_desc


class KVCapacityError(RuntimeError):
    """Prefill/verify would exceed the bound x (Eq. 1; OOM reason "Cache")."""


def typical_stats(z, temperature: float):
    """P = softmax(z / T) and the exact entropy H = -sum P log P (0 log 0 = 0)."""
    y = np.asarray(z, dtype=np.float64) / temperature
    y = y - y.max()
    e = np.exp(y)
    P = e / e.sum()
    nz = P > 0
    H = float(-(P[nz] * np.log(P[nz])).sum())
    return P, H


class Session:
    """b independent sequences sharing one model and one static tree."""

    def __init__(self, model: Model, choices: list[list[int]], batch: int, max_seq_len: int, topk: int = 10,
                 batched: bool = False):
        """batched=True: prefill and verify push all their rows through ``Model.forward_rows``
        (one BLAS product per weight and layer) instead of one row at a time -- the same
        arithmetic up to fp64 summation order, for wide models in tests and for timing."""
        self.m = model
        self.batched = batched
        self.tree = T.build(choices, topk) if choices else T.build([], topk)
        self.N = self.tree.N
        self.l = max(self.tree.max_depth, 0)
        self.n_heads_used = self.l
        assert self.l <= len(model.W.medusa), "tree deeper than the number of Medusa heads"
        self.K = topk
        self.x = max_seq_len
        self.b = batch
        self.kv = KVCache(model.n_layers, batch, model.Hkv, max_seq_len + self.N, model.hd,
                          dtype=model.W.embed.dtype)
        self.Lc = [0] * batch
        self.root = [None] * batch
        self.topk_tok = [None] * batch                   # [l][K] token ids per sequence
        self.last_z = [None] * batch
        self.last_hf = [None] * batch
        self.committed = [[] for _ in range(batch)]
        self.leaves = T.leaves(self.tree)
        self.dfs = T.dfs_order(self.tree)
        self.dfs_pos = {n: i for i, n in enumerate(self.dfs)}

    # ------------------------------------------------------------ heads
    def _propose_state(self, seq, z, hf):
        self.last_z[seq], self.last_hf[seq] = z, hf                # the accepted node's rows (tests)
        self.root[seq] = argmax_lowest(z)                       # Q8: root = argmax in both modes
        self.topk_tok[seq] = [topk_desc(self.m.head_logits(i, hf), self.K) for i in range(self.l)]

    # ------------------------------------------------------------ prefill
    def prefill(self, seq: int, tokens) -> None:
        """Causal forward of one turn's P tokens at positions [Lc, Lc+P).
        A pending root from a previous turn is dropped (Q15)."""
        P = len(tokens)
        if P == 0:
            return
        if self.Lc[seq] + P > self.x:
            raise KVCapacityError(f"prefill {P} at Lc={self.Lc[seq]} exceeds x={self.x}")
        z = hf = None
        if self.batched:
            Lc = self.Lc[seq]
            for c0 in range(0, P, 256):  # causal chunks
                idx = range(c0, min(P, c0 + 256))
                Z, HF = self.m.forward_rows(self.kv, seq, [tokens[i] for i in idx], [Lc + i for i in idx],
                                            [Lc + i for i in idx], [list(range(Lc + i + 1)) for i in idx])
            z, hf = Z[-1], HF[-1]
        else:
            for i, tok in enumerate(tokens):
                pos = self.Lc[seq] + i
                z, hf = self.m.forward_row(self.kv, seq, int(tok), pos, pos, list(range(pos + 1)))
        self.Lc[seq] += P
        self.committed[seq].extend(int(t) for t in tokens)
        self._propose_state(seq, z, hf)

    # ------------------------------------------------------------ step
    def propose(self, seq: int):
        """tok[0] = root, tok[n] = T_{depth(n)-1}[rank(n)];  pos[n] = Lc + depth(n)."""
        tr = self.tree
        tok = [self.root[seq]] + [self.topk_tok[seq][tr.depth[n] - 1][tr.rank[n]] for n in range(1, self.N)]
        pos = [self.Lc[seq] + tr.depth[n] for n in range(self.N)]
        return tok, pos

    def verify(self, seq: int, tok):
        """Forward all nodes; node n writes K/V to slot Lc+n and attends to
        [0, Lc) + its ancestors' slots + its own slot, in logical order."""
        Lc = self.Lc[seq]
        if Lc >= self.x:
            raise KVCapacityError(f"verify at Lc={Lc} >= x={self.x}")
        tr = self.tree
        if self.batched:
            keys = [list(range(Lc)) + [Lc + a for a in T.ancestors(tr, n)] + [Lc + n] for n in range(self.N)]
            Z, HF = self.m.forward_rows(self.kv, seq, tok, [Lc + tr.depth[n] for n in range(self.N)],
                                        [Lc + n for n in range(self.N)], keys)
            return list(Z), list(HF)
        Z, HF = [None] * self.N, [None] * self.N
        for n in range(self.N):                                   # canonical order: parents first
            keys = list(range(Lc)) + [Lc + a for a in T.ancestors(tr, n)] + [Lc + n]
            Z[n], HF[n] = self.m.forward_row(self.kv, seq, int(tok[n]), Lc + tr.depth[n], Lc + n, keys)
        return Z, HF

    def accept(self, tok, Z, mode: str = "greedy", temperature: float = 0.7, eps: float = 0.09, alpha: float = 0.3,
               forced=None):
        """Tree DP: acc(root) = true; acc(c) = acc(parent) and C(parent, c).
        greedy C: tok[c] == argmax z[parent];  typical C: P_p[tok[c]] > min(eps, alpha e^{-H_p}).
        Returns (a, chosen node, best_leaf index, path node ids [a+1]).
        forced (test hook, the C ABI's d_forced_path): accept this root-to-node path instead."""
        tr = self.tree
        if forced is not None:
            chosen = int(forced[-1])
            path = T.ancestors(tr, chosen) + [chosen]
            assert path == [int(x) for x in forced], "forced path must be a root-to-node path"
            cp = tr.paths[chosen]
            best_leaf = next(i for i, lf in enumerate(self.leaves) if tr.paths[lf][:len(cp)] == cp)
            return tr.depth[chosen], chosen, best_leaf, path
        acc = [False] * self.N
        ll = [0.0] * self.N
        acc[0] = True
        stats = {}
        for c in range(1, self.N):
            p = tr.parent[c]
            if not acc[p]:
                continue
            if mode == "greedy":
                ok = int(tok[c]) == argmax_lowest(Z[p])
                lp = 0.0
            else:
                if p not in stats:
                    P, H = typical_stats(Z[p], temperature)
                    stats[p] = (P, min(eps, alpha * math.exp(-H)))
                P, thr = stats[p]
                ok = P[int(tok[c])] > thr
                lp = math.log(P[int(tok[c])]) if P[int(tok[c])] > 0 else -math.inf
            if ok:
                acc[c] = True
                ll[c] = ll[p] + lp
        a = max(tr.depth[n] for n in range(self.N) if acc[n])
        if a == 0:
            chosen = 0
        else:
            cands = [n for n in range(self.N) if acc[n] and tr.depth[n] == a]
            best = max(ll[n] for n in cands)
            chosen = min((n for n in cands if ll[n] == best), key=lambda n: self.dfs_pos[n])
        # best_leaf: first leaf (DFS order) whose path passes through ``chosen``
        chosen_path = tr.paths[chosen]
        best_leaf = next(i for i, lf in enumerate(self.leaves) if tr.paths[lf][:len(chosen_path)] == chosen_path)
        path = T.ancestors(tr, chosen) + [chosen]
        return a, chosen, best_leaf, path

    def compact(self, seq: int, path, a_eff: int) -> None:
        """For j = 1..a_eff (ascending): K/V[Lc+j] <- K/V[Lc+path[j]] in every layer
        and kv head (reading Q13)."""
        Lc = self.Lc[seq]
        for j in range(1, a_eff + 1):
            for li in range(self.m.n_layers):
                self.kv.K[li][seq][:, Lc + j, :] = self.kv.K[li][seq][:, Lc + path[j], :]
                self.kv.V[li][seq][:, Lc + j, :] = self.kv.V[li][seq][:, Lc + path[j], :]

    def step(self, seq: int, mode: str = "greedy", budget: int | None = None, **typ):
        """One full speculative step for one sequence.  Emits tok[path[0..a_eff]],
        a_eff = min(a, budget-1, x-Lc-1) (Q14, Q15); tau = a_eff + 1."""
        tok, pos = self.propose(seq)
        Z, HF = self.verify(seq, tok)
        return self.finish(seq, tok, pos, Z, HF, mode, budget, **typ)

    def finish(self, seq: int, tok, pos, Z, HF, mode: str = "greedy", budget: int | None = None, forced=None, **typ):
        """Steps 3-6 of a step on verified rows: accept, emit, compact, next state."""
        a, chosen, best_leaf, path = self.accept(tok, Z, mode, forced=forced, **typ)
        Lc = self.Lc[seq]
        a_eff = a
        if budget is not None:
            a_eff = min(a_eff, budget - 1)
        a_eff = min(a_eff, self.x - Lc - 1)
        assert a_eff >= 0
        self.compact(seq, path, a_eff)
        emitted = [int(tok[path[j]]) for j in range(a_eff + 1)]
        self.Lc[seq] = Lc + a_eff + 1
        self.committed[seq].extend(emitted)
        last = path[a_eff]
        self._propose_state(seq, Z[last], HF[last])
        return dict(tok=tok, pos=pos, Z=Z, a=a, a_eff=a_eff, best_leaf=best_leaf,
                    path=path, emitted=emitted, chosen=chosen)

    def generate(self, seq: int, n_new: int, mode: str = "greedy", **typ):
        """Decode until n_new tokens were emitted in this turn (budget clamp)."""
        out, taus = [], []
        while len(out) < n_new:
            r = self.step(seq, mode, budget=n_new - len(out), **typ)
            out += r["emitted"]
            taus.append(len(r["emitted"]))
        return out, taus


def vanilla_generate(model: Model, prompt, n_new: int, max_seq_len: int | None = None):
    """Plain greedy decoding, one token at a time (the definition the greedy
    speculative mode must reproduce).  Every generated token is also run through
    the model, so the returned cache holds K/V for prompt + generated tokens.
    Returns (generated tokens, kv cache)."""
    cap = max_seq_len or (len(prompt) + n_new + 1)
    kv = KVCache(model.n_layers, 1, model.Hkv, cap, model.hd)
    z = None
    for i, t in enumerate(prompt):
        z, _ = model.forward_row(kv, 0, int(t), i, i, list(range(i + 1)))
    out = []
    pos = len(prompt)
    nxt = argmax_lowest(z)
    while len(out) < n_new:
        out.append(nxt)
        z, _ = model.forward_row(kv, 0, nxt, pos, pos, list(range(pos + 1)))
        pos += 1
        nxt = argmax_lowest(z)
    return out, kv


class PadSession(Session):
    """The paper's batched speculative decoding with pads (f4 comparison mode), step by
    step in the paper's order:

      * "candidate tokens are discarded after token rejection in a cumulative way.  Input IDs for
        the accepted tokens across batch dimension are padded to a fixed-length sequences to form
        uniform tensors" -- every sequence's cache advances by the batch's longest acceptance
        A = max_s (a_eff_s + 1); the slots a sequence did not fill are pads;
      * "Each batch maps Input IDs to Position IDs in a way to ignore the pad tokens, so that
        positional embeddings continue from the latest sequence length" -- positions count real
        tokens only (``pos``), the cache slot index (``Lc``) counts pads too;
      * "cached tokens are searched for pad tokens and the corresponding locations in the
        attention mask are set to -inf" -- pad slots are left out of every row's visible keys.

    Ragged prompts are aligned before the first step the same way (the shorter caches padded to
    the longest).  ``Lc[s]`` is the slot count (uniform after ``align``), ``pos[s]`` the real
    token count, ``pad[s]`` the set of pad slots."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.pos = [0] * self.b
        self.pad = [set() for _ in range(self.b)]

    def prefill(self, seq: int, tokens) -> None:
        assert not self.pad[seq], "pad mode starts after the prompts (as the C ABI's sm_kv_set_pad_mode)"
        super().prefill(seq, tokens)
        self.pos[seq] = self.Lc[seq]

    def align(self) -> None:
        mx = max(self.Lc)
        for s in range(self.b):
            self.pad[s].update(range(self.Lc[s], mx))
            self.Lc[s] = mx

    def propose(self, seq: int):
        tr = self.tree
        tok = [self.root[seq]] + [self.topk_tok[seq][tr.depth[n] - 1][tr.rank[n]] for n in range(1, self.N)]
        pos = [self.pos[seq] + tr.depth[n] for n in range(self.N)]
        return tok, pos

    def verify(self, seq: int, tok):
        """As Session.verify, with positions pos + depth and the pad slots masked out of [0, Lc)."""
        Lc = self.Lc[seq]
        if Lc >= self.x:
            raise KVCapacityError(f"verify at Lc={Lc} >= x={self.x}")
        tr = self.tree
        prefix = [j for j in range(Lc) if j not in self.pad[seq]]
        Z, HF = [None] * self.N, [None] * self.N
        for n in range(self.N):
            keys = prefix + [Lc + a for a in T.ancestors(tr, n)] + [Lc + n]
            Z[n], HF[n] = self.m.forward_row(self.kv, seq, int(tok[n]), self.pos[seq] + tr.depth[n], Lc + n, keys)
        return Z, HF

    def step_batch(self, mode: str = "greedy", budgets=None, forced=None, toks=None, **typ):
        """One batched step: align, then every sequence proposes / verifies / accepts / compacts
        at the common slot Lc; the caches then advance by A = max_s (a_eff_s + 1) with slots
        [Lc + a_eff_s + 1, Lc + A) of sequence s marked as pads.  forced[s]: root-to-node path or
        None (the C ABI's d_forced_path test hook); toks[s]: verify these tree tokens instead of
        the proposed ones (tests: the other implementation's choice among near-tied top-K values)."""
        self.align()
        res = []
        for s in range(self.b):
            tok, pos = self.propose(s)
            if toks is not None:
                tok = [int(t) for t in toks[s]]
            Z, HF = self.verify(s, tok)
            a, chosen, best_leaf, path = self.accept(tok, Z, mode, forced=None if forced is None else forced[s],
                                                     **typ)
            Lc = self.Lc[s]
            a_eff = a
            if budgets is not None:
                a_eff = min(a_eff, budgets[s] - 1)
            a_eff = min(a_eff, self.x - Lc - 1)
            self.compact(s, path, a_eff)
            emitted = [int(tok[path[j]]) for j in range(a_eff + 1)]
            self.committed[s].extend(emitted)
            last = path[a_eff]
            self._propose_state(s, Z[last], HF[last])
            res.append(dict(tok=tok, pos=pos, Z=Z, a=a, a_eff=a_eff, best_leaf=best_leaf, path=path,
                            emitted=emitted, chosen=chosen))
        A = max(len(r["emitted"]) for r in res)
        for s, r in enumerate(res):
            ne = len(r["emitted"])
            self.pad[s].update(range(self.Lc[s] + ne, self.Lc[s] + A))
            self.Lc[s] += A
            self.pos[s] += ne
        return res
