"""f1 tree-size selection (no GPU): E[tau] under SPEC's independent acceptance model and the
selection by expected throughput, oracle pinned to SPEC's worked values and to brute-force
enumeration; the library's host functions (sm_tree_expected_tau / sm_select_tree) equal the
oracle (the chosen index bit-exact)."""
import itertools
import os

import numpy as np
import pytest

import synth
from oracle import tree as T


def _brute_tau(choices, alpha, rho):
    """Enumerate every accept/reject assignment of the non-root nodes (2^(N-1) outcomes)."""
    t = T.build(choices)
    a = [alpha[t.depth[n] - 1] * rho ** t.rank[n] for n in range(1, t.N)]
    tau = 0.0
    for bits in itertools.product((0, 1), repeat=t.N - 1):
        p = 1.0
        for ai, b in zip(a, bits):
            p *= ai if b else 1.0 - ai
        if p == 0.0:
            continue
        acc = [True] + [bool(b) for b in bits]
        ok = [False] * t.N
        ok[0] = True
        for n in range(1, t.N):
            ok[n] = ok[t.parent[n]] and acc[n]
        tau += p * (1 + max(t.depth[n] for n in range(t.N) if ok[n]))
    return tau


def test_spec_worked_values():
    # S:352-353 / S:359: chain l = 2 at alpha = 0.5 -> 1.75; all-accept -> l + 1; all-reject -> 1
    assert T.expected_tau([[0], [0, 0]], [0.5, 0.5]) == 1.75
    assert T.expected_tau(synth.V64, [1, 1, 1, 1]) == 5.0
    assert T.expected_tau(synth.V64, [0, 0, 0, 0]) == 1.0
    # chain of l nodes: 1 + a + a^2 + ... (closed form)
    for l in (1, 3, 5):
        a = 0.37
        assert abs(T.expected_tau(synth.CHAIN(l), [a] * l) - sum(a ** j for j in range(l + 1))) < 1e-15


@pytest.mark.parametrize("seed", range(6))
def test_expected_tau_equals_enumeration(seed):
    rng = np.random.default_rng(seed)
    base = [synth.TINY16, synth.V64[:11], synth.V64[:9], [[0], [1], [0, 0], [0, 1], [1, 0], [0, 0, 0]],
            T.full_tree(2, 2), T.full_tree(3, 2)][seed]
    alpha = list(rng.uniform(0, 1, 4))
    rho = float(rng.uniform(0.3, 1.0))
    assert abs(T.expected_tau(base, alpha, rho) - _brute_tau(base, alpha, rho)) < 1e-12


def test_expected_tau_monotone_in_nodes():
    """with rho = 1, adding nodes never decreases E[tau] (R4-pruned nested trees)."""
    prev = 0.0
    for n in (5, 16, 27, 31, 44, 64):
        c = T.prune_right_to_left(synth.V64, n)
        v = T.expected_tau(c, [0.6, 0.4, 0.3, 0.2], 1.0)
        assert v >= prev
        prev = v


def test_select_tree_is_the_argmax():
    cands = [synth.V64, T.prune_right_to_left(synth.V64, 44), T.truncate(synth.V64, 3), synth.TINY16, []]
    ms = [3.8, 3.6, 3.5, 3.3, 3.1]
    alpha = [0.6, 0.4, 0.3, 0.2]
    best, tps = T.select_tree(cands, ms, alpha, 0.8, batch=1)
    ref = [T.expected_tau(c, alpha, 0.8) / m * 1e3 for c, m in zip(cands, ms)]
    assert best == int(np.argmax(ref)) and np.allclose(tps, ref)
    # a much slower big tree loses; equal throughput ties to the smaller tree
    best, _ = T.select_tree([synth.V64, synth.TINY16], [100.0, 3.0], alpha, 0.8)
    assert best == 1
    t64, t16 = T.expected_tau(synth.V64, alpha, 0.8), T.expected_tau(synth.TINY16, alpha, 0.8)
    best, _ = T.select_tree([synth.V64, synth.TINY16], [t64, t16], alpha, 0.8)
    assert best == 1


@pytest.fixture(scope="module")
def sm():
    import paper_2506_01986_b200 as sm
    if not os.path.exists(sm.LIB_PATH):
        from paper_2506_01986_b200 import build
        build.build()
    return sm


def test_library_selection_equals_oracle(sm):
    rng = np.random.default_rng(7)
    pool = [synth.V64] + [T.prune_right_to_left(synth.V64, n) for n in (44, 31, 27, 16, 5)] + \
           [T.truncate(synth.V64, h) for h in (1, 2, 3)] + [T.prune_right_to_left(T.truncate(synth.V64, 3), n)
                                                             for n in (44, 27, 16)] + [[]]
    trees = [sm.Tree(c, topk=10) for c in pool]
    for trial in range(200):
        idx = sorted(rng.choice(len(pool), size=int(rng.integers(2, len(pool) + 1)), replace=False))
        alpha = [float(np.float32(v)) for v in rng.uniform(0, 1, 4)]
        rho = float(np.float32(rng.uniform(0.2, 1.0)))
        ms = list(rng.uniform(2.0, 6.0, len(idx)))
        b = int(rng.integers(1, 11))
        ob, otps = T.select_tree([pool[i] for i in idx], ms, alpha, rho, batch=b)
        lb, ltps = sm.select_tree([trees[i] for i in idx], ms, alpha, rho, batch=b)
        assert lb == ob, trial
        assert np.allclose(ltps, otps, rtol=1e-14, atol=0)
    for c, t in zip(pool, trees):
        assert abs(t.expected_tau([0.7, 0.5, 0.4, 0.3], 0.75) -
                   T.expected_tau(c, [float(np.float32(v)) for v in (0.7, 0.5, 0.4, 0.3)], float(np.float32(0.75)))) < 1e-15
