"""The C-ABI library loads, exports every symbol include/specmemo.h declares, and
its host-side tree / sizing logic agrees with the oracle (no GPU needed)."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import sizing
from oracle import tree as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sm():
    import paper_2506_01986_b200 as sm
    if not os.path.exists(sm.LIB_PATH):
        from paper_2506_01986_b200 import build
        build.build()
    return sm


def declared_functions():
    src = open(os.path.join(ROOT, "include", "specmemo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sm_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(sm):
    names = declared_functions()
    assert len(names) >= 20
    lib = sm.lib()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert "sm_100a" in sm.version()


@pytest.mark.parametrize("choices", [synth.V64, synth.TINY16, synth.SWEEP_TREES[256], [[0], [0, 0], [0, 0, 0]]])
def test_tree_tables_match_oracle(sm, choices):
    t = sm.Tree(choices, topk=10)
    q = t.query()
    ot = T.build(choices)
    assert (q["N"], q["S"], q["depth"]) == (ot.N, len(T.leaves(ot)), ot.max_depth)
    assert list(q["parent"]) == ot.parent
    assert list(q["node_depth"]) == ot.depth
    assert list(q["rank"]) == ot.rank
    mask = T.ancestor_mask(ot)
    for i in range(ot.N):
        bits = [(int(q["anc"][i][j // 64]) >> (j % 64)) & 1 for j in range(ot.N)]
        assert bits == mask[i]
    assert q["leaf_paths"].tolist() == T.candidate_paths(ot)


def test_chain_tree(sm):
    q = sm.Tree(None, chain=5).query()
    assert q["N"] == 5 and q["S"] == 1 and q["depth"] == 4
    assert q["leaf_paths"].tolist() == [[0, 1, 2, 3, 4]]


@pytest.mark.parametrize("bad", [[[0, 0]], [[0], [0]], [[10]]])
def test_infeasible_tree_errors(sm, bad):
    with pytest.raises(sm.InfeasibleTreeError):
        sm.Tree(bad, topk=10)


def test_kv_bytes_is_eq1_with_d(sm):
    c = synth.MODELS["vicuna7b"]
    for b, x, N in ((1, 2048, 64), (3, 100, 16)):
        assert sm.kv_bytes(c, b, x, N) == sizing.kv_bytes(c["n_layers"], b, c["n_kv_heads"], c["head_dim"], x,
                                                         tree_nodes=N)
    assert sm.kv_bytes(c, 1, 1, 1) // 2 == sizing.kv_bytes_per_token(32, 32, 128)   # 1 slot + 1 scratch
    c70 = synth.MODELS["llama70b"]
    assert sm.kv_bytes(c70, 10, 400, 64, tp_size=8) * 8 == sm.kv_bytes(c70, 10, 400, 64)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2506_01986_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_stage_entries_reject_bad_arguments_before_any_launch(sm):
    """SM_ERR_INVALID_ARG (1) with a message, nothing enqueued -- checked on the host (no GPU needed)."""
    import ctypes
    lib = sm.lib()
    p = ctypes.c_void_p(16)  # never dereferenced: the argument check fails first
    for n in (0, 1025):      # K1 prefill mode: 1 <= n <= 1024
        assert lib.sm_causal_attention(n, p, p, p, p, 1, 4, 4, 128, 2048, p, None) == 1
        assert "sm_causal_attention" in lib.sm_last_error().decode()
    assert lib.sm_causal_attention(16, p, p, p, p, 1, 6, 4, 128, 2048, p, None) == 1  # H % Hkv != 0
    assert lib.sm_causal_attention(16, p, p, p, p, 1, 4, 4, 128, 8, p, None) == 1     # cap < n
    assert lib.sm_tree_attention(None, p, p, p, p, 1, 4, 4, 128, 2048, p, None) == 1
    assert lib.sm_gemm_bf16(p, p, None, 0, 128, 64, None) == 1                         # M < 1
    assert lib.sm_gemm_bf16(p, p, None, 1025, 128, 64, None) == 1                      # M > 1024
    assert lib.sm_gemm_bf16(p, p, None, 16, 128, 60, None) == 1                        # K % 8
