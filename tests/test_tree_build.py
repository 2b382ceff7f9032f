"""f1 tree construction: the library's host-side builders
(sm_tree_create_full / sm_tree_prune / sm_tree_create_pruned_full / sm_tree_create_custom,
called through the C ABI -- no GPU needed) must produce exactly the oracle's trees, node
for node in canonical order (integer work: bit-exact)."""
import pytest

import synth
from oracle import tree as T

sm = pytest.importorskip("paper_2506_01986_b200")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    sm.lib()


def oracle_paths(choices, k=10):
    return [list(p) for p in T.build(choices, k).paths[1:]]


@pytest.mark.parametrize("k,l", [(1, 3), (2, 2), (3, 3), (5, 2), (10, 2), (4, 3)])
def test_full_tree_matches_oracle(k, l):
    assert sm.Tree.full(k, l).paths() == oracle_paths(T.full_tree(k, l), k)


@pytest.mark.parametrize("target", [1, 2, 5, 11, 16, 27, 31, 34, 44, 57, 63, 64])
def test_r4_prune_matches_oracle_and_table(target):
    got = sm.Tree(synth.V64).pruned(target)
    assert got.paths() == oracle_paths(T.prune_right_to_left(synth.V64, target))
    assert got.N == target


def test_r4_prune_reproduces_pruned_medusa_leaf_counts():
    """tab:treefeatures "Pruned M", heads = 4 column: 1/5, 10/16, 18/27, 20/31."""
    v64 = sm.Tree(synth.V64)
    assert [(v64.pruned(n).S, n) for n in (5, 16, 27, 31)] == [(1, 5), (10, 16), (18, 27), (20, 31)]


@pytest.mark.parametrize("k,l,sched", [(4, 3, {}), (5, 3, {}), (3, 4, {}), (10, 2, {}),
                                       (4, 3, dict(r_min=0.0, r_max=0.0)), (6, 3, dict(r_min=1.0, r_max=1.0)),
                                       (4, 4, dict(r_min=0.2, r_max=0.99, mid=2.0, steep=3.0))])
def test_pruned_full_matches_oracle(k, l, sched):
    assert sm.Tree.pruned_full(k, l, **sched).paths() == oracle_paths(T.prune_full_tree(k, l, **sched), k)


def test_pruned_full_cap():
    with pytest.raises(sm.SpecMemoError):
        sm.Tree.pruned_full(10, 4)          # default schedule keeps > 256 nodes of the 11111


@pytest.mark.parametrize("k,l", [(10, 4), (2, 3), (3, 2), (4, 3)])
def test_custom_matches_oracle(k, l):
    nmax = min(256, sum(k ** i for i in range(l + 1)))
    for n in range(1, min(nmax, 80) + 1):
        for s in range(1, n + 1):
            try:
                ref = T.build_custom_tree(n, s, k, l)
            except T.InfeasibleTree:
                with pytest.raises(sm.InfeasibleTreeError):
                    sm.Tree.custom(n, s, k, l)
                continue
            got = sm.Tree.custom(n, s, k, l)
            assert (got.N, got.S) == (n, s)
            assert got.paths() == oracle_paths(ref, k), (n, s)
