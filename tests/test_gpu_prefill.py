"""Prefill against the oracle (needs a B200).

sm_prefill runs a turn through the verify path in causal chunks of up to max_rows
tokens (bf16, one GPU): K1 masks cache slot Lc + j for token i by j <= i without a
tree table, RoPE at Lc + i.  Here a 600-token turn goes through as ONE chunk
(max_rows = 1024, beyond the 256-node tree limit) and as ragged chunks of 100 rows, then
a second turn lands on the committed prefix.  The cache of every layer must match the
oracle's sequential prefill (oracle.spec.Session.prefill: one token at a time, keys
[0, pos]) within the bf16 tolerance, and a verify step on the oracle's proposed tree
must give the oracle's logits -- so the layer-1 K/V (which depends on layer-0 causal
attention) and every later step see the right cache.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import model as OM
from oracle import spec as OS

pytestmark = pytest.mark.gpu

TINY = synth.model_cfg("tiny")  # head_dim 16: the mma.sync K1
S128 = synth.model_cfg("tiny", d_model=256, n_heads=2, n_kv_heads=1, head_dim=128, d_ffn=512, vocab=512)  # tcgen05 K1
X = 720


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


@pytest.fixture(scope="module")
def oracle_after_turns():
    """Oracle sessions per model after a 600-token turn and a 90-token second turn."""
    res = {}
    for name, cfg in (("tiny", TINY), ("s128", S128)):
        s = OS.Session(OM.Model(cfg, OM.Weights(cfg, n_medusa=3, seed=2), "bf16"), synth.TINY16, 1, X)
        t1 = synth.prompt_tokens(2, 0, 600, cfg["vocab"])
        t2 = synth.prompt_tokens(2, 0, 90, cfg["vocab"], turn=1)
        s.prefill(0, t1)
        kv1 = [(s.kv.K[li][0][:, :600].copy(), s.kv.V[li][0][:, :600].copy()) for li in range(cfg["n_layers"])]
        s.prefill(0, t2)
        tok, _ = s.propose(0)
        Z, _ = s.verify(0, tok)
        res[name] = (cfg, t1, t2, kv1, s, tok, np.stack(Z))
    return res


@pytest.mark.parametrize("max_rows", [1024, 100], ids=["one_chunk", "chunks100"])
@pytest.mark.parametrize("model", ["tiny", "s128"])
def test_prefill_kv_and_next_verify_match_oracle(sm, oracle_after_turns, model, max_rows):
    cfg, t1, t2, kv1, s, tok, Zo = oracle_after_turns[model]
    W = sm.allocate_weights(cfg, 3, seed=2)
    tree = sm.Tree(synth.TINY16, topk=10)
    m = sm.Model(cfg, W, max_rows=max_rows, max_batch=1, max_seq_len=X + tree.N)
    kv = sm.KVCache(m, tree, 1, X)
    kv.prefill(0, torch.from_numpy(t1).cuda())
    torch.cuda.synchronize()
    lay = kv.layout()
    for li in range(cfg["n_layers"]):
        for w in range(2):
            g = lay[li, w, 0].float().cpu().numpy()[:, :600]
            err = np.abs(g - kv1[li][w])
            assert err.max() < 2e-2, (model, max_rows, li, w, float(err.max()))
    kv.prefill(0, torch.from_numpy(t2).cuda())
    assert kv.lengths()[0] == 690
    tt = torch.tensor([tok], dtype=torch.int32, device="cuda")  # the oracle's tree tokens
    logits = torch.zeros(1, tree.N, cfg["vocab"], dtype=torch.float32, device="cuda")
    kv.verify(tt, logits)
    torch.cuda.synchronize()
    Zg = logits[0].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(Zg - Zo)) < 2e-2, float(np.max(np.abs(Zg - Zo)))
    lay = kv.layout()
    for li in range(cfg["n_layers"]):
        g = lay[li, 0, 0].float().cpu().numpy()[:, : 690 + tree.N]
        assert np.max(np.abs(g - s.kv.K[li][0][:, : 690 + tree.N])) < 2e-2
