"""f2 planner bound to the device (needs a B200): sm_plan with max_memory = 0 budgets the
device's free memory; sm_workspace_bytes matches what sm_model_create allocates; a plan
for a tight budget is built (tree, heads, KV bound x) and runs speculative steps."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


def test_workspace_bytes_matches_allocation(sm):
    cfg = synth.model_cfg("vicuna7b", n_layers=2)
    W = sm.allocate_weights(cfg, 4, seed=0, medusa_init=True)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    model = sm.Model(cfg, W, max_rows=256, max_batch=1, max_seq_len=2048 + 64)
    torch.cuda.synchronize()
    used = free0 - torch.cuda.mem_get_info()[0]
    ws = sm.workspace_bytes(cfg, 256, 1, 2048 + 64, 4)
    assert abs(used - ws) <= 64 * (1 << 20) + 0.05 * ws, (used, ws)
    del model


def test_plan_on_device_budget_runs(sm):
    cfg = synth.model_cfg("vicuna7b", n_layers=2)
    base = sm.Tree(synth.V64)
    free = torch.cuda.mem_get_info()[0]
    p = sm.plan(cfg, base, 1, 4, 128)                        # max_memory = 0: the device's free bytes
    assert abs(p["max_memory"] - free) < 256 * (1 << 20)
    assert p["status"] == "default" and p["total"] <= p["max_memory"]
    # a budget that forces a pruned tree with 4 heads (b200 accounting)
    import oracle.planner as PL
    tight = PL.memory_total(cfg, 1, 4, 128, 2, 4, 31, 20, "b200") + 1000
    p = sm.plan(cfg, base, 1, 4, 128, max_memory=tight)
    assert p["status"] == "pruned" and p["N"] <= 31 and p["total"] <= tight
    cut = [c for c in synth.V64 if len(c) <= p["heads"]]
    tree = sm.Tree(cut).pruned(p["N"]) if p["kind"] == "pruned" else sm.Tree.custom(p["N"], p["S"], 10, p["heads"])
    assert (tree.N, tree.S) == (p["N"], p["S"])
    W = sm.allocate_weights(cfg, p["heads"], seed=0)
    model = sm.Model(cfg, W, max_rows=64, max_batch=1, max_seq_len=p["x"] + tree.N)
    kv = sm.KVCache(model, tree, 1, p["x"])
    assert kv.nbytes == p["kv"]                              # the plan's KV term is the bound cache
    kv.prefill(0, torch.from_numpy(synth.prompt_tokens(0, 0, 32, cfg["vocab"])).cuda())
    out = sm.AcceptOut(1, tree.depth)
    for _ in range(4):
        kv.step(sm.accept_cfg(), out)
    torch.cuda.synchronize()
    assert int(kv.lengths()[0]) >= 36
