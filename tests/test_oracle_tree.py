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
