"""Pins for oracle/spec.py PadSession -- the paper's pad batching (f4), no GPU.

What the paper fixes: pads are masked with -inf "to maintain the accuracy of the attention
mechanism" and positions "continue from the latest sequence length" ignoring pads,
so a sequence decoded inside a padded batch must behave exactly as the same sequence decoded
alone (the ragged Session, itself pinned to vanilla greedy and HF Llama).  In fp64 every row sees
the same keys in the same order at the same positions, so logits and K/V agree to rounding-free
equality; the pad layout is checked against its brute-force definition (slot j of sequence s is a
pad iff it holds none of s's committed tokens, and the caches advance by the batch's longest
acceptance)."""
import numpy as np

import synth
from oracle import model as M
from oracle import spec as SP
from oracle import tree as T

CFG = synth.model_cfg("tiny")


def _paths(tree):
    """root-to-node paths of depth 3 / 0 / 1 (forced acceptances of different lengths)."""
    deep = next(n for n in range(tree.N) if tree.depth[n] == 3)
    d1 = [n for n in range(tree.N) if tree.depth[n] == 1][1]
    return [T.ancestors(tree, deep) + [deep], [0], [0, d1]]


def test_pad_batch_equals_ragged_per_sequence():
    m = M.Model(CFG, M.Weights(CFG, n_medusa=3, seed=9), "fp64")
    b, x = 3, 128
    prompts = [synth.prompt_tokens(9, i, 20 + 7 * i, CFG["vocab"]) for i in range(b)]
    ps = SP.PadSession(m, synth.TINY16, b, x)
    rs = [SP.Session(m, synth.TINY16, 1, x) for _ in range(b)]
    for i, p in enumerate(prompts):
        ps.prefill(i, p)
        rs[i].prefill(0, p)
    forced = _paths(ps.tree)
    A_sum = 0
    for step in range(8):
        fz = forced if step < 2 else None
        res = ps.step_batch(forced=fz)
        A_sum += max(len(r["emitted"]) for r in res)
        for s in range(b):
            tok, pos = rs[s].propose(0)
            Z, HF = rs[s].verify(0, tok)
            rr = rs[s].finish(0, tok, pos, Z, HF, forced=None if fz is None else fz[s])
            assert res[s]["tok"] == tok and res[s]["pos"] == pos      # same tree, positions ignore pads
            assert res[s]["emitted"] == rr["emitted"] and res[s]["path"] == rr["path"]
            np.testing.assert_array_equal(np.stack(res[s]["Z"]), np.stack(Z))  # same keys, same order
    # slot counts: max prompt + the longest acceptance of every step
    assert len(set(ps.Lc)) == 1 and ps.Lc[0] == max(len(p) for p in prompts) + A_sum
    for s in range(b):
        assert ps.pos[s] == rs[s].Lc[0] == len(ps.committed[s])   # prompt + emitted tokens
        assert ps.committed[s] == rs[s].committed[0]
        real = [j for j in range(ps.Lc[s]) if j not in ps.pad[s]]
        assert len(real) == ps.pos[s]                                # pads = slots holding no token
        for li in range(m.n_layers):                                 # K/V of the real slots, in order
            np.testing.assert_array_equal(ps.kv.K[li][s][:, real, :], rs[s].kv.K[li][0][:, : ps.pos[s], :])
            np.testing.assert_array_equal(ps.kv.V[li][s][:, real, :], rs[s].kv.V[li][0][:, : ps.pos[s], :])
    # at least one sequence carries pads inside its cache (the forced depths differ)
    assert any(min(ps.pad[s], default=10 ** 9) < ps.Lc[s] - 1 for s in range(b))


def test_pad_layout_brute_force():
    """Pad slots = [len_s, max len) after the prompts, then [Lc + ne_s, Lc + A) every step."""
    m = M.Model(CFG, M.Weights(CFG, n_medusa=3, seed=2), "fp64")
    b = 2
    prompts = [synth.prompt_tokens(2, i, 10 + 5 * i, CFG["vocab"]) for i in range(b)]
    ps = SP.PadSession(m, synth.TINY16, b, 96)
    for i, p in enumerate(prompts):
        ps.prefill(i, p)
    forced = _paths(ps.tree)
    expect = [set(range(len(prompts[s]), max(map(len, prompts)))) for s in range(b)]
    Lc = max(map(len, prompts))
    for step in range(3):
        res = ps.step_batch(forced=[forced[0], forced[2]] if step % 2 == 0 else [forced[1], forced[0]])
        ne = [len(r["emitted"]) for r in res]
        A = max(ne)
        for s in range(b):
            expect[s].update(range(Lc + ne[s], Lc + A))
        Lc += A
    assert ps.pad == expect and ps.Lc == [Lc] * b
