"""Pins for oracle/sizing.py against the paper's printed sizes (no GPU)."""
import json
import os

import synth
from oracle import sizing


def test_printed_sizes(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "sizing.json")))
    c = synth.MODELS["vicuna7b"]
    assert sizing.kv_bytes_per_token(c["n_layers"], c["n_kv_heads"], c["head_dim"]) == \
        g["kv_bytes_per_token_vicuna7b_fp16"]["value"]
    for k in ("eq3_medusa64", "eq3_custom44"):
        e = g[k]
        assert sizing.buffer_bytes(e["N"], e["S"], e["l"], e["w"]) == e["bytes"]
    head_gb = sizing.medusa_head_params(c["d_model"], c["vocab"]) * 4 / 1e9
    assert abs(head_gb - g["eq4_head_gb"]["value_gb"]) / 0.6 < g["eq4_head_gb"]["rel_tol"]


def test_eq1_scaling():
    assert sizing.kv_bytes(32, 2, 32, 128, 2048) == 2 * sizing.kv_bytes(32, 1, 32, 128, 2048)
    # bounded cache of SURVEY C2: x = 2048 + N = 64 scratch -> 1.107 GB
    assert sizing.kv_bytes(32, 1, 32, 128, 2048, tree_nodes=64) == 1107296256
