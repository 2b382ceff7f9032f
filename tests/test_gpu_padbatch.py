"""f4 pad batching vs the default ragged lengths (needs a B200).

The paper's batched decoding pads every sequence's accepted tokens to the batch's longest
acceptance, keeps positions counting real tokens, and masks the cached pads with -inf.  Its
per-sequence results must therefore equal the ragged mode's (which tests/test_gpu_e2e.py pins to
the oracle's unbatched runs), while the cache grows by the longest acceptance every step.  Forced
paths of different depths (the d_forced_path hook) make the sequences' acceptances differ."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
CFG = synth.model_cfg("tiny")


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


def run(sm, pad: bool, n_free: int = 6):
    b = 3
    prompts = [synth.prompt_tokens(9, i, 20 + 7 * i, CFG["vocab"]) for i in range(b)]
    W = sm.allocate_weights(CFG, 3, seed=9)
    tree = sm.Tree(synth.TINY16, topk=10)
    model = sm.Model(CFG, W, max_rows=64, max_batch=b, max_seq_len=128 + tree.N)
    kv = sm.KVCache(model, tree, b, 128)
    for i, p in enumerate(prompts):
        kv.prefill(i, torch.from_numpy(p).cuda())
    if pad:
        kv.set_pad_mode(True)
    q = tree.query()
    depth, parent = q["node_depth"], q["parent"]
    deep = int(np.flatnonzero(depth == 3)[0])
    chain = [deep]
    while chain[-1] != 0:
        chain.append(int(parent[chain[-1]]))
    chain = chain[::-1]                                   # root .. depth-3 node
    d1 = int(np.flatnonzero(depth == 1)[1])
    forced = torch.full((b, tree.depth + 1), -1, dtype=torch.int32, device="cuda")
    forced[0, :4] = torch.tensor(chain, dtype=torch.int32)
    forced[1, 0] = 0                                      # accepts only the root
    forced[2, :2] = torch.tensor([0, d1], dtype=torch.int32)
    out = sm.AcceptOut(b, tree.depth)
    toks = [[] for _ in range(b)]
    lens = []
    for cfg in [sm.accept_cfg(forced_path=forced)] * 2 + [sm.accept_cfg()] * n_free:
        kv.step(cfg, out)
        ne = out.n_emit.cpu().numpy()
        et = out.emit_tok.cpu().numpy()
        for s in range(b):
            toks[s] += et[s][: ne[s]].tolist()
        lens.append((kv.lengths().copy(), kv.positions().copy()))
    tt = torch.zeros(b, tree.N, dtype=torch.int32, device="cuda")
    kv.propose(tt)
    logits = torch.zeros(b, tree.N, CFG["vocab"], dtype=torch.float32, device="cuda")
    kv.verify(tt, logits)
    torch.cuda.synchronize()
    return toks, lens, tt.cpu(), logits.cpu().double(), [len(p) for p in prompts]


def test_pad_batching_equals_ragged(sm):
    tr, lr, ttr, zr, plen = run(sm, False)
    tp, lp, ttp, zp, _ = run(sm, True)
    assert tp == tr                                       # same tokens per sequence
    assert torch.equal(ttp, ttr)                          # same next tree
    assert float((zp - zr).abs().max()) < 2e-2            # same logits (up to summation order)
    # ragged: lengths = positions = prompt + emitted; pad: uniform slots >= every position
    for (L_r, P_r), (L_p, P_p) in zip(lr, lp):
        assert np.array_equal(L_r, P_r) and np.array_equal(P_p, P_r)
        assert len(set(L_p.tolist())) == 1 and L_p[0] >= P_p.max()
    # the pad cache grew by max(prompt) + sum over steps of the longest acceptance
    emitted = [len(t) for t in tp]
    assert lp[-1][0][0] > max(p + e for p, e in zip(plen, emitted)) - 1
    assert lp[-1][0][0] - lp[-1][1].min() >= 3            # pads exist (forced depths 3 / 0 / 1)
