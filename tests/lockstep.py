"""Lock-step GPU <-> oracle parity harness (protocol steps 1-4).

Every step of every sequence is compared decision by decision:

* propose (a1): the GPU's tree tokens against the oracle's -- root = argmax of the last
  accepted node's logits, node n = rank(n) of head depth(n)-1's top-K (value desc, index asc).
  A decision must be bit-exact when the oracle's margin at it (argmax: top1 - top2; top-K
  rank r: the gaps to ranks r-1 and r+1) is at least the guard.  Below the guard the GPU's
  token must still be a valid choice: its oracle value within the guard of the value the
  oracle ranked there.  The oracle then verifies the GPU's tokens (same inputs, step 1).
* verify (a2/a3): logits of every tree row and the K/V of every tree slot, every layer,
  element by element against the tolerance (``close``).
* accept (a4): the oracle decides first.  If every decision the step depends on has margin
  (greedy: argmax gap at each accepted node with children; typical: |P - thr| >= 2e-2 thr for
  each child of an accepted node, and distinct likelihoods among the deepest accepted
  nodes), the GPU accepts on its own and acc_len / best_leaf / path / emitted tokens must be
  bit-equal.  Otherwise the GPU is forced onto the oracle's path (the d_forced_path hook,
  step 4) and the step is counted as forced.
* compact (a5): K/V of the committed slots after compaction, every layer, and Lc.

Guards: ``guard_rel`` * max|z| for argmax gaps (§8.c.6: 1e-2) and an absolute floor
``guard_abs`` for top-K gaps; both are raised to ``noise_k`` x the rms logit discrepancy measured
on the step's own verify rows, so a decision counts as unambiguous only when its margin is well
outside the measured rounding noise of the two implementations."""
from __future__ import annotations

import math

import numpy as np
import torch

from oracle import model as OM
from oracle import spec as OS
from oracle import tree as OT


def bar_check(got, ref, tol, what, max_frac=0.0, hard=None):
    """Elementwise |got - ref| <= tol (1 + |ref|).  max_frac > 0 (bf16 at widths where one-ulp
    storage-point differences cascade, Q29): at most that fraction of the elements may
    exceed the bar, and none may exceed ``hard`` x the bar.  Returns (max err / bar, frac over)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    bar = tol * (1.0 + np.abs(ref))
    r = np.abs(got - ref) / bar
    frac = float(np.mean(r > 1.0))
    worst = float(r.max()) if r.size else 0.0
    if max_frac == 0.0:
        assert worst <= 1.0, f"{what}: max |err|/bar {worst:.3f}"
    else:
        assert frac <= max_frac, f"{what}: {frac:.2e} of elements over the 2e-2 bar (allowed {max_frac:.1e})"
        assert worst <= hard, f"{what}: max |err|/bar {worst:.3f} > {hard}"
    return worst, frac


class LockStep:
    def __init__(self, sm, cfg, n_medusa, choices, prompts, x, dtype="bf16", seed=0, medusa_init=False,
                 max_rows=None, tol=None, max_frac=0.0, hard=None, guard_rel=1e-2, guard_abs=None, noise_k=8.0,
                 typ=None, oracle_weights=None, force_deep_every=0):
        self.sm, self.cfg, self.dtype = sm, cfg, dtype
        self.b = len(prompts)
        self.tol = tol if tol is not None else (1e-4 if dtype == "fp32" else 2e-2)
        self.max_frac, self.hard = max_frac, hard
        self.guard_rel = guard_rel
        self.guard_abs = guard_abs if guard_abs is not None else (5e-4 if dtype == "fp32" else 1e-3)
        self.noise_k = noise_k
        self.mode = "typical" if typ else "greedy"
        self.typ = typ or {}
        W = sm.allocate_weights(cfg, n_medusa, seed=seed, medusa_init=medusa_init)
        self.tree = sm.Tree(choices, topk=10)
        N = self.tree.N
        self.model = sm.Model(cfg, W, max_rows=max_rows or max(64, self.b * N), max_batch=self.b,
                              max_seq_len=x + N, dtype=dtype)
        self.W = W
        self.kv = sm.KVCache(self.model, self.tree, self.b, x)
        ow = oracle_weights or OM.Weights(cfg, n_medusa=n_medusa, seed=seed, medusa_init=medusa_init)
        om = OM.Model(cfg, ow, dtype)
        self.s = OS.Session(om, choices, self.b, x, batched=True)
        self.ot = self.s.tree
        self.out = sm.AcceptOut(self.b, self.tree.depth)
        self.stats = dict(steps=0, forced=0, exact_decisions=0, tolerated=0, emitted=0, max_bar=0.0, max_frac=0.0,
                          accepted_depth_hist=[0] * (self.tree.depth + 1))
        for i, p in enumerate(prompts):
            self.kv.prefill(i, torch.from_numpy(np.asarray(p, np.int32)).cuda())
            self.s.prefill(i, p)
        self.noise = [0.0] * self.b
        self._probe_noise()
        # every force_deep_every-th step both sides accept a random full-depth path (the forced-path
        # hook): random-init models rarely accept tree nodes, so this is what drives compaction
        # (a5) over real K/V at the wide shapes; those steps still compare every float and integer
        self.force_deep_every = force_deep_every
        self.rng = np.random.default_rng(1234)
        self.stats["forced_deep"] = 0

    def _probe_noise(self):
        """Rounding-noise scale before the first step: one GPU verify of the proposed tree
        against the oracle's verify of the same tokens (tree slots are scratch; nothing is
        accepted).  The first propose's decisions are then screened against it too."""
        s, tr, b = self.s, self.ot, self.b
        tt = torch.zeros(b, tr.N, dtype=torch.int32, device="cuda")
        self.kv.propose(tt)
        logits = torch.zeros(b, tr.N, self.cfg["vocab"], dtype=torch.float32, device="cuda")
        self.kv.verify(tt, logits)
        torch.cuda.synchronize()
        Zg = logits.cpu().numpy().astype(np.float64)
        for seq in range(b):
            Z, _ = s.verify(seq, [int(t) for t in tt[seq].cpu()])
            self.noise[seq] = float(np.sqrt(np.mean((Zg[seq] - np.stack(Z)) ** 2)))

    # ------------------------------------------------------------- margins
    def _argmax_guard(self, z, seq):
        return max(self.guard_rel * float(np.abs(z).max()), self.noise_k * self.noise[seq])

    def _check_propose(self, seq, g_tok):
        s, tr = self.s, self.ot
        o_tok, _ = s.propose(seq)
        z = np.asarray(s.last_z[seq], np.float64)
        gz = self._argmax_guard(z, seq)
        zs = np.sort(z)[::-1]
        if zs[0] - zs[1] >= gz:
            assert g_tok[0] == o_tok[0], (seq, "root", g_tok[0], o_tok[0])
            self.stats["exact_decisions"] += 1
        else:
            assert z[g_tok[0]] >= zs[0] - gz, (seq, "root invalid")
            self.stats["tolerated"] += int(g_tok[0] != o_tok[0])
        U = [np.asarray(s.m.head_logits(i, s.last_hf[seq]), np.float64) for i in range(s.l)]
        ga = max(self.guard_abs, self.noise_k * self.noise[seq])
        for n in range(1, tr.N):
            u = U[tr.depth[n] - 1]
            r = tr.rank[n]
            order = OM.topk_desc(u, s.K + 1)
            v = u[order]
            gap = min(v[r - 1] - v[r] if r > 0 else math.inf, v[r] - v[r + 1])
            if gap >= max(ga, 1e-3 * abs(v[r])):
                assert g_tok[n] == o_tok[n], (seq, "node", n, g_tok[n], o_tok[n])
                self.stats["exact_decisions"] += 1
            else:
                assert abs(u[g_tok[n]] - v[r]) <= max(ga, 1e-3 * abs(v[r])) * 2, (seq, "node invalid", n)
                self.stats["tolerated"] += int(g_tok[n] != o_tok[n])
        return o_tok

    def _accept_ambiguous(self, seq, tok, Z):
        """True if a decision the oracle's acceptance depends on lies within the guard."""
        s, tr = self.s, self.ot
        a = s.accept(tok, Z, self.mode, **self.typ)[0]
        accd = {0}
        for c in range(1, tr.N):
            p = tr.parent[c]
            if p not in accd:
                continue
            z = np.asarray(Z[p], np.float64)
            if self.mode == "greedy":
                zs = np.sort(z)[::-1]
                if zs[0] - zs[1] < self._argmax_guard(z, seq):
                    return True
                ok = int(tok[c]) == OM.argmax_lowest(z)
            else:
                P, H = OS.typical_stats(z, self.typ["temperature"])
                thr = min(self.typ["eps"], self.typ["alpha"] * math.exp(-H))
                pc = P[int(tok[c])]
                # the logit noise moves log P by ~noise / T: require the decision to clear both
                if abs(pc - thr) < 2e-2 * thr or abs(math.log(pc / thr)) < self.noise_k * self.noise[seq] / \
                        self.typ["temperature"]:
                    return True
                ok = pc > thr
            if ok:
                accd.add(c)
        if self.mode == "typical" and a > 0:
            deep = [n for n in accd if tr.depth[n] == a]
            lls = []
            for n in deep:
                ll = 0.0
                for j, x in enumerate(OT.ancestors(tr, n)[1:] + [n]):
                    p = tr.parent[x]
                    P, _ = OS.typical_stats(Z[p], self.typ["temperature"])
                    ll += math.log(P[int(tok[x])])
                lls.append(ll)
            lls.sort(reverse=True)
            if len(lls) > 1 and lls[0] - lls[1] < self.noise_k * self.noise[seq] / self.typ["temperature"] * a + 1e-3:
                return True
        return False

    # ------------------------------------------------------------- one step
    def step(self):
        sm, s, tr, b = self.sm, self.s, self.ot, self.b
        N, V = tr.N, self.cfg["vocab"]
        Lc0 = list(s.Lc)
        tt = torch.zeros(b, N, dtype=torch.int32, device="cuda")
        self.kv.propose(tt)
        torch.cuda.synchronize()
        G = tt.cpu().numpy()
        for seq in range(b):
            self._check_propose(seq, G[seq].tolist())
        logits = torch.zeros(b, N, V, dtype=torch.float32, device="cuda")
        self.kv.verify(tt, logits)
        torch.cuda.synchronize()
        Zg = logits.cpu().numpy().astype(np.float64)
        kvl = self.kv.layout().float().cpu().numpy()
        forced = np.full((b, tr.max_depth + 1), -1, np.int32)
        any_forced = False
        ref = []
        for seq in range(b):
            tok = [int(t) for t in G[seq]]
            pos = [Lc0[seq] + tr.depth[n] for n in range(N)]
            Z, HF = s.verify(seq, tok)
            Zo = np.stack(Z)
            self.noise[seq] = float(np.sqrt(np.mean((Zg[seq] - Zo) ** 2)))
            w, f = bar_check(Zg[seq], Zo, self.tol, f"logits seq {seq}", self.max_frac, self.hard)
            self.stats["max_bar"] = max(self.stats["max_bar"], w)
            self.stats["max_frac"] = max(self.stats["max_frac"], f)
            slots = list(range(Lc0[seq], Lc0[seq] + N))
            for li in range(self.cfg["n_layers"]):
                for c, KV in ((0, s.kv.K), (1, s.kv.V)):
                    w, f = bar_check(kvl[li, c, seq][:, slots], KV[li][seq][:, slots], self.tol,
                                     f"tree {'KV'[c]} layer {li} seq {seq}", self.max_frac, self.hard)
                    self.stats["max_bar"] = max(self.stats["max_bar"], w)
            deep = None
            if self.force_deep_every and self.stats["steps"] % self.force_deep_every == self.force_deep_every - 1:
                leaves = OT.leaves(tr)
                lf = leaves[int(self.rng.integers(len(leaves)))]
                deep = OT.ancestors(tr, lf) + [lf]
                self.stats["forced_deep"] += 1
            amb = deep is None and self._accept_ambiguous(seq, tok, Z)
            r = s.finish(seq, tok, pos, Z, HF, self.mode, forced=deep, **self.typ)
            ref.append(r)
            if deep is not None:
                forced[seq, : len(r["path"])] = r["path"]
                any_forced = True
            elif amb:
                forced[seq, : len(r["path"])] = r["path"]
                any_forced = True
                self.stats["forced"] += 1
        fp = torch.from_numpy(forced).cuda() if any_forced else None  # rows of -1: not forced
        acfg = sm.accept_cfg(sm.TYPICAL if self.mode == "typical" else sm.GREEDY, forced_path=fp, **self.typ)
        self.kv.accept(acfg, self.out)
        torch.cuda.synchronize()
        o = self.out
        L = self.kv.lengths()
        kvl = self.kv.layout().float().cpu().numpy()
        for seq, r in enumerate(ref):
            assert int(o.acc_len[seq]) == r["a"], (seq, int(o.acc_len[seq]), r["a"])
            assert int(o.best_leaf[seq]) == r["best_leaf"], seq
            ne = int(o.n_emit[seq])
            assert ne == r["a_eff"] + 1
            assert o.emit_tok[seq, :ne].cpu().tolist() == r["emitted"], seq
            assert o.path[seq, : r["a"] + 1].cpu().tolist() == r["path"], seq
            assert int(L[seq]) == s.Lc[seq]
            self.stats["emitted"] += ne
            self.stats["accepted_depth_hist"][r["a"]] += 1
            self.stats["exact_decisions"] += 0 if forced[seq, 0] >= 0 else 1
            slots = list(range(Lc0[seq], s.Lc[seq]))
            for li in range(self.cfg["n_layers"]):
                for c, KV in ((0, s.kv.K), (1, s.kv.V)):
                    bar_check(kvl[li, c, seq][:, slots], KV[li][seq][:, slots], self.tol,
                              f"committed {'KV'[c]} layer {li} seq {seq}", self.max_frac, self.hard)
        self.stats["steps"] += 1

    def run(self, n_steps):
        for _ in range(n_steps):
            self.step()
        return self.stats
