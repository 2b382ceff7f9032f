"""Algorithm 2 (f2 "Alg. 2 run over measured step time"): the oracle's transcription
pinned to the algorithm's definition on hand-worked cases, and the library's sm_alg2_select
decision-exact against it (host code: no GPU).  The measured (acceptance_length, speedup) rows
come from bench.py's C4 line (MedusaGenerate = sm_step over the workload's queries)."""
import numpy as np
import pytest

from oracle import planner as OP


def test_oracle_algorithm2_hand_cases():
    # Max(results.speedup): acceptance length is recorded, not used
    assert OP.algorithm2([("M64", 3.1, 1.9), ("C44", 2.9, 2.1), ("P16", 2.2, 1.7)]) == "C44"
    assert OP.algorithm2([("a", 9.0, 0.5), ("b", 1.0, 0.6)]) == "b"          # longer acceptance loses
    assert OP.algorithm2([("a", 1.0, 1.2), ("b", 2.0, 1.2)]) == "a"          # tie: first in loop order (Q32)
    assert OP.algorithm2([("only", 1.0, 0.3)]) == "only"


def test_library_alg2_matches_oracle():
    import paper_2506_01986_b200 as sm
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 9))
        acc = rng.uniform(1, 5, n)
        sp = np.round(rng.uniform(0.2, 3.0, n), 1)  # rounded: ties occur
        want = OP.algorithm2([(i, acc[i], sp[i]) for i in range(n)])
        assert sm.alg2_select(acc, sp) == want


def test_library_alg2_rejects_bad_input():
    import paper_2506_01986_b200 as sm
    with pytest.raises(sm.SpecMemoError):
        sm.alg2_select([1.0], [float("nan")])
    with pytest.raises(sm.SpecMemoError):
        sm.alg2_select([], [])
