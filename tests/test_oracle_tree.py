"""Pins for oracle/tree.py against the paper's printed tree features and
brute-force definitions (no GPU)."""
import itertools
import json
import os

import pytest

import synth
from oracle import tree as T


def load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def test_medusa_tree_features_match_paper(golden_dir):
    g = load(golden_dir, "tree_features.json")
    for h, (S, N) in enumerate(g["medusa_M_row"]["leaves_nodes_by_depth"], start=1):
        st = T.stats(T.build(T.truncate(synth.V64, h)))
        assert (st["S"], st["N"]) == (S, N), h
    st = T.stats(T.build(synth.V64))
    assert (st["N"], st["S"]) == (g["default_tree"]["N"], g["default_tree"]["S"])
    assert len(T.candidate_paths(T.build(synth.V64))) == 42


def test_right_to_left_pruning_reproduces_pruned_M_leaves(golden_dir):
    g = load(golden_dir, "tree_features.json")["pruned_M_leaves"]
    for target, leaves in g.items():
        if target.startswith("_"):
            continue
        pruned = T.prune_right_to_left(synth.V64, int(target))
        assert T.build(pruned).N == int(target)
        got = [T.stats(T.build(T.truncate(pruned, h)))["S"] for h in range(1, 5)]
        assert got == leaves, target


def _brute_mask(paths):
    """(i, j) = 1 iff path(j) is a prefix of path(i): ancestor-or-self by definition."""
    return [[1 if pi[:len(pj)] == pj else 0 for pj in paths] for pi in paths]


@pytest.mark.parametrize("choices", [synth.V64, synth.TINY16, synth.V64[:31], synth.SWEEP_TREES[128]])
def test_ancestor_mask_equals_brute_force(choices):
    tr = T.build(choices)
    m = T.ancestor_mask(tr)
    assert m == _brute_mask(tr.paths)
    for i in range(tr.N):
        assert sum(m[i]) == tr.depth[i] + 1
    # transitively closed: j in anc(i), k in anc(j) => k in anc(i)
    for i, j, k in itertools.product(range(min(tr.N, 20)), repeat=3):
        if m[i][j] and m[j][k]:
            assert m[i][k]


def test_chain_and_full_tree_special_cases():
    tr = T.build(synth.CHAIN(3))
    assert T.ancestor_mask(tr) == [[1 if j <= i else 0 for j in range(4)] for i in range(4)]
    assert T.candidate_paths(tr) == [[0, 1, 2, 3]]
    full22 = [[0], [1], [0, 0], [0, 1], [1, 0], [1, 1]]
    tr = T.build(full22, topk=2)
    rank_paths = [list(tr.paths[l]) for l in T.leaves(tr)]
    assert rank_paths == [[0, 0], [0, 1], [1, 0], [1, 1]]
    assert T.stats(tr)["label"] == "1-2-4"
    # row of leaf [1,1] has exactly 3 ones
    assert sum(T.ancestor_mask(tr)[tr.paths.index((1, 1))]) == 3


def test_canonical_order_and_paths():
    tr = T.build(synth.V64)
    assert tr.paths[0] == ()
    keys = [(len(p), p) for p in tr.paths[1:]]
    assert keys == sorted(keys)
    cp = T.candidate_paths(tr)
    assert cp[0] == [0, 1, 11, 34, 57] and cp[1] == [0, 1, 11, 34, 58]
    for row in cp:
        ids = [i for i in row if i >= 0]
        assert all(b > a for a, b in zip(ids, ids[1:]))          # strictly increasing
        assert all(ids[j] >= j for j in range(len(ids)))          # path[j] >= j (compaction safety)
    assert T.candidate_paths(T.build(synth.TINY16))[0] == [0, 1, 6, 12]


def test_parallel_compaction_hazard_example():
    """Compaction copies slot Lc+path[j] -> Lc+j for j = 1..a.  In tiny16 the
    node with rank path (1, 0) has node-id path [0, 2, 10] (hand-derived from the
    canonical order): row 1 reads slot Lc+2, which row 2 writes -> copying rows in
    parallel without staging is a RAW hazard; ascending sequential order is safe
    because path[j] >= j."""
    tr = T.build(synth.TINY16)
    n = tr.paths.index((1, 0))
    assert n == 10
    assert T.ancestors(tr, n) + [n] == [0, 2, 10]


@pytest.mark.parametrize("bad", [[[0, 0]], [[0], [0]], [[10]], [[]]])
def test_infeasible_trees(bad):
    with pytest.raises(T.InfeasibleTree):
        T.build(bad, topk=10)


# ----------------------------------------------------------------- f1: tree construction
def test_full_tree_counts_eq2():
    """Eq. 2: a full tree of arity k and l levels has sum_{i=0}^{l} k^i nodes (root included)."""
    for k, l in ((2, 2), (5, 2), (3, 3), (10, 2)):
        t = T.build(T.full_tree(k, l), k)
        assert t.N == sum(k ** i for i in range(l + 1))
        assert T.stats(t)["S"] == k ** l
    assert T.full_tree(2, 2) == [[0], [1], [0, 0], [0, 1], [1, 0], [1, 1]]
    assert T.stats(T.build(T.full_tree(5, 2), 5))["label"] == "1-5-25"


def test_prune_rate_closed_form():
    """Scaled logistic (fig:prunefunc): asymptote r_max, midpoint (r_min + r_max)/2, increasing
    in the level ("keeps pruning rates low at first levels ... increase ... on deeper levels")."""
    assert abs(T.prune_rate(1e6) - 0.95) < 1e-12
    assert abs(T.prune_rate(2.5) - (0.1 + 0.95) / 2) < 1e-12
    assert abs(T.prune_rate(1) - 0.14) < 0.005
    rates = [T.prune_rate(i) for i in range(1, 8)]
    assert all(a < b for a, b in zip(rates, rates[1:]))


def test_prune_full_tree_special_cases():
    k, l = 4, 3
    # no pruning (r = 0 everywhere) -> the full tree
    assert T.prune_full_tree(k, l, r_min=0.0, r_max=0.0) == T.full_tree(k, l)
    # maximal pruning below level 1 -> root + the k first-level nodes (first-level rule)
    assert T.prune_full_tree(k, l, r_min=1.0, r_max=1.0) == [[r] for r in range(k)]
    # default schedule: level 1 full; level i keeps ceil((1 - r(i)) k^i) nodes, left to right
    import math
    t = T.build(T.prune_full_tree(k, l), k)
    per = [sum(1 for n in range(t.N) if t.depth[n] == i) for i in range(l + 1)]
    assert per[1] == k
    for i in range(2, l + 1):
        assert per[i] == min(math.ceil((1 - T.prune_rate(i)) * k ** i - 1e-9), k * per[i - 1])
    # left-prefix property: a retained node's lower-rank siblings are retained
    have = set(tuple(p) for p in t.paths)
    assert all(p[:-1] + (r,) in have for p in have if p for r in range(p[-1]))


@pytest.mark.parametrize("n,s", [(44, 37), (64, 56), (5, 1), (16, 10), (27, 18), (31, 20), (11, 10), (2, 1)])
def test_custom_tree_exact_features(n, s):
    """build_custom_tree(N, S) has exactly N nodes and S leaves ("directly builds tree mask
    structures with exact features"); (44, 37) and (64, 56) are tab:treefeatures' Custom trees at
    heads = 4.  Arity <= k, depth <= l, level 1 = min(k, N-1, S) nodes."""
    t = T.build(T.build_custom_tree(n, s, 10, 4), 10)
    st = T.stats(t)
    assert (st["N"], st["S"]) == (n, s) and st["depth"] <= 4
    assert all(len(t.children(x)) <= 10 for x in range(t.N))
    assert sum(1 for x in range(t.N) if t.depth[x] == 1) == min(10, n - 1, s)
    have = set(tuple(p) for p in t.paths)
    assert all(p[:-1] + (r,) in have for p in have if p for r in range(p[-1]))   # left-heavy, no rank gaps


def _feasible_pairs(k, l):
    """Brute force: every (N, S) realised by some prefix-closed subset of the full tree."""
    full = [tuple(p) for p in T.full_tree(k, l)]
    res = set()
    for mask in range(1 << len(full)):
        sub = [full[i] for i in range(len(full)) if mask >> i & 1]
        ss = set(sub)
        if all(len(p) == 1 or p[:-1] in ss for p in sub):
            leaves = [p for p in sub if not any(q[:-1] == p for q in sub)]
            res.add((len(sub) + 1, len(leaves) if sub else 1))
    return res


@pytest.mark.parametrize("k,l", [(2, 2), (2, 3), (3, 2)])
def test_custom_tree_reaches_every_feasible_pair(k, l):
    feas = _feasible_pairs(k, l)
    for n, s in sorted(feas):
        st = T.stats(T.build(T.build_custom_tree(n, s, k, l), k))
        assert (st["N"], st["S"]) == (n, s) and st["depth"] <= l
    # and rejects pairs no tree has
    for n in range(1, sum(k ** i for i in range(l + 1)) + 2):
        for s in range(1, n + 1):
            if (n, s) not in feas:
                with pytest.raises(T.InfeasibleTree):
                    T.build_custom_tree(n, s, k, l)
