"""f2 memory-budget planner: the oracle's Algorithm 1 (oracle/planner.py)
against the paper's printed sizes and the algorithm's properties, and the library's sm_plan
(host only, no GPU) against the oracle, decision for decision."""
import pytest

import synth
from oracle import planner as PL
from oracle import sizing
from oracle import tree as T

C7 = synth.model_cfg("vicuna7b")
C70 = synth.model_cfg("llama70b")
GB = 1 << 30


def test_memory_model_matches_printed_sizes():
    # Eq. 3 at the Medusa (64, 42, l=4) mask: 57,856,000 B per query ("55 MB")
    assert PL.memory_buffers(1, 64, 42, 4, 32000, 2) == 57856000 == sizing.buffer_bytes(64, 42, 4, 32000)
    # Eq. 1 with d: 524,288 B per token at Vicuna-7B
    assert PL.memory_kv(C7, 1, 1, 1, 2) == 524288
    # Eq. 4: 0.6 GB per head
    assert PL.memory_heads(C7, 3, 2) == int(1.8e9)
    # Eq. 6 is the sum of its terms
    t = PL.memory_total(C7, 1, 8, 128, 2, 4, 64, 42)
    assert t == PL.memory_base(C7, 2) + int(2.4e9) + PL.memory_kv(C7, 1, 8, 128, 2) + 57856000


@pytest.mark.parametrize("acct", ["paper", "b200"])
def test_algorithm1_properties(acct):
    full = PL.memory_total(C7, 1, 20, 128, 2, 4, 64, 42, acct)
    r = PL.optimizer_engine(C7, 1, 20, 128, 2, full, accounting=acct)
    assert (r["status"], r["heads"], r["N"], r["S"]) == (PL.STATUS_DEFAULT, 4, 64, 42)
    prev = None
    budgets = [full - i * (1 << 24) for i in range(0, 100)]
    for mem in budgets:
        r = PL.optimizer_engine(C7, 1, 20, 128, 2, mem, accounting=acct)
        if r["status"] == PL.STATUS_NEEDS_QUANT:
            # Alg. 1 quantizes when no explored tree fits at the default head count and the
            # default tree fits at no head count in [2, heads - 1] (reading Q31)
            assert not PL.explore_tree(C7, 1, 20, 128, 2, 4, mem, acct)
            assert all(PL.memory_total(C7, 1, 20, 128, 2, h, 64, 42, acct) > mem for h in (2, 3))
            continue
        assert r["total"] <= mem                                   # the plan fits the budget
        if r["status"] != PL.STATUS_DEFAULT:
            # the largest fitting candidate for its head count (ExploreTree, reading Q31)
            for N, S, _ in PL.explore_tree(C7, 1, 20, 128, 2, r["heads"], mem, acct):
                assert (N, S) <= (r["N"], r["S"])
        if prev is not None:                                       # less memory never buys more
            assert (r["heads"], r["N"]) <= (prev["heads"], prev["N"]) or r["status"] == prev["status"]
        prev = r


def test_algorithm1_reduces_heads_before_failing():
    """A budget between the 2-head and 4-head footprints: the heads are reduced."""
    lo = PL.memory_total(C7, 1, 20, 128, 2, 2, 64, 42)
    hi = PL.memory_total(C7, 1, 20, 128, 2, 4, 5, 1)
    assert lo < hi
    r = PL.optimizer_engine(C7, 1, 20, 128, 2, (lo + hi) // 2)
    assert r["status"] in (PL.STATUS_FEWER_HEADS,) and r["heads"] < 4 and r["total"] <= (lo + hi) // 2


sm = pytest.importorskip("paper_2506_01986_b200")


@pytest.mark.parametrize("cfg,b,n,m", [(C7, 1, 20, 128), (C7, 4, 8, 256), (C70, 10, 1, 416)])
@pytest.mark.parametrize("acct", ["paper", "b200"])
def test_sm_plan_matches_oracle(cfg, b, n, m, acct):
    sm.lib()
    base = sm.Tree(synth.V64)
    full = PL.memory_total(cfg, b, n, m, 2, 4, 64, 42, acct)
    floor = PL.memory_total(cfg, b, n, m, 2, 2, 5, 3, acct)
    step = max(1, (full - floor) // 40)
    for mem in list(range(floor - 3 * step, full + 3 * step, step)) + [full, floor, 1 << 50]:
        ref = PL.optimizer_engine(cfg, b, n, m, 2, mem, accounting=acct)
        got = sm.plan(cfg, base, b, n, m, max_memory=mem, accounting=acct)
        st = {0: "default", 1: "pruned", 2: "fewer_heads", 3: "needs_quantization"}[ref["status"]]
        assert got["status"] == st, mem
        if st != "needs_quantization":
            assert (got["heads"], got["N"], got["S"], got["x"]) == (ref["heads"], ref["N"], ref["S"], ref["x"]), mem
            assert got["kind"] == ref["kind"] and got["total"] == ref["total"]
