"""Device-detected conditions surface through the C ABI ("written to
out.status[b] and surfaced by the next call's return code").

Stepping a sequence past its KV bound x (Eq. 1) is the paper's OOM reason
"Cache": the accept kernel writes status[b] = 3, emits nothing, and the next
sm_step / sm_accept / sm_verify returns SM_ERR_KV_CAPACITY (KVCapacityError) without
enqueuing anything; sm_kv_status synchronises and reports it."""
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


def _setup(sm, x, batch=1, prompt_len=32):
    W = sm.allocate_weights(CFG, 3, seed=1)
    tree = sm.Tree(synth.TINY16, topk=10)
    model = sm.Model(CFG, W, max_rows=64, max_batch=batch, max_seq_len=x + tree.N)
    kv = sm.KVCache(model, tree, batch, x)
    for b in range(batch):
        kv.prefill(b, torch.from_numpy(synth.prompt_tokens(1, b, prompt_len - 4 * b, CFG["vocab"])).cuda())
    return W, tree, model, kv


def test_step_past_bound_returns_kv_capacity(sm):
    x = 40
    W, tree, model, kv = _setup(sm, x)
    out = sm.AcceptOut(1, tree.depth)
    cfg = sm.accept_cfg(sm.GREEDY)
    for _ in range(x):                      # emission is clamped at x: Lc reaches x exactly
        kv.step(cfg, out)
        torch.cuda.synchronize()
        if int(kv.lengths()[0]) == x:
            break
    assert int(kv.lengths()[0]) == x
    assert int(out.status[0]) == 0
    kv.step(cfg, out)                       # enqueued before the device sees Lc >= x
    torch.cuda.synchronize()
    assert int(out.status[0]) == 3 and int(out.n_emit[0]) == 0
    assert int(kv.lengths()[0]) == x        # nothing committed, nothing compacted
    with pytest.raises(sm.KVCapacityError):
        kv.step(cfg, out)                   # the next call reports it and enqueues nothing
    kv.step(cfg, out)                       # latch cleared: runs (and detects again)
    assert kv.status() == 3                 # synchronising query
    assert kv.status() == 0                 # cleared by the read
    with pytest.raises(sm.KVCapacityError):
        kv.prefill(0, torch.zeros(1, dtype=torch.int32, device="cuda"))  # host-side bound (Q14)


def test_one_sequence_at_bound_others_continue(sm):
    """b = 2: sequence 0 reaches x first; the latched status is reported once, sequence 1
    keeps stepping (status 0) until it reaches x as well."""
    x = 40
    W, tree, model, kv = _setup(sm, x, batch=2)
    out = sm.AcceptOut(2, tree.depth)
    cfg = sm.accept_cfg(sm.GREEDY)
    seen = 0
    for _ in range(4 * x):
        try:
            kv.step(cfg, out)
        except sm.KVCapacityError:
            seen += 1
            continue
        torch.cuda.synchronize()
        L = kv.lengths()
        st = out.status.cpu().tolist()
        for b in range(2):
            assert st[b] == (3 if int(out.n_emit[b]) == 0 else 0)
        if all(int(v) == x for v in L) and st == [3, 3]:
            break
    assert seen >= 1
    assert kv.lengths().tolist() == [x, x]
