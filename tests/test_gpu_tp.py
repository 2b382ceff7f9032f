"""Tensor parallelism (SURVEY §8 rows a7 / e) emulated on one B200.

t ranks = t sm_models in one process on the same device, each holding its shard
(allocate_weights(tp_rank, tp_size)) and exchanging through the other ranks'
symmetric buffers -- the same kernels and flag protocol a multi-GPU run uses
over NVLink peer memory (there the peer pointers come from CUDA IPC).  Each
rank's work runs on its own stream; programmatic dependent launch is disabled
here because ranks sharing one GPU could otherwise hold each other's SMs while
spinning (on separate GPUs that cannot happen).

Parity: the tp run must emit the oracle's greedy tokens on the screened seeds
(the same bar as tp = 1), and its vocabulary-parallel logits, concatenated over
ranks, must match the tp = 1 logits within 2e-2."""
import numpy as np
import pytest
import torch

import synth
from oracle import model as OM
from oracle import spec as OS

pytestmark = pytest.mark.gpu

CFG = synth.model_cfg("tiny")
X = 64


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


@pytest.fixture(autouse=True)
def _no_pdl(sm):
    """Every test of this module runs with PDL off (conftest restores the defaults after each)."""
    sm.set_option("pdl", 0)


class Ranks:
    def __init__(self, sm, t, seed=0, n_medusa=3, choices=synth.TINY16, batch=1, medusa_init=False):
        self.sm, self.t = sm, t
        self.tree = sm.Tree(choices, topk=10)
        R = max(batch * self.tree.N, 64)
        nbytes = sm.tp_sym_bytes(CFG, R, batch, n_medusa)
        self.sym = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(t)]
        ptrs = [s.data_ptr() for s in self.sym]
        self.W = [sm.allocate_weights(CFG, n_medusa, seed=seed, medusa_init=medusa_init, tp_rank=r, tp_size=t)
                  for r in range(t)]
        self.models = [sm.Model(CFG, self.W[r], R, batch, X + self.tree.N, peer_sym=ptrs) for r in range(t)]
        self.kvs = [sm.KVCache(m, self.tree, batch, X) for m in self.models]
        self.streams = [torch.cuda.Stream() for _ in range(t)]
        self.outs = [sm.AcceptOut(batch, self.tree.depth) for _ in range(t)]
        torch.cuda.synchronize()

    def each(self, fn):
        for r in range(self.t):
            with torch.cuda.stream(self.streams[r]):
                fn(r, self.kvs[r], self.streams[r])
        for s in self.streams:
            s.synchronize()

    def timed_out(self):
        return any(m.tp_timed_out() for m in self.models)


def test_tp_shards_tile_the_full_weights(sm):
    """Every rank's shard is the matching slice of the tp = 1 weights (device generator)."""
    full = sm.allocate_weights(CFG, 3, seed=4)
    t = 2
    parts = [sm.allocate_weights(CFG, 3, seed=4, tp_rank=r, tp_size=t) for r in range(t)]
    H, Hkv, hd = CFG["n_heads"], CFG["n_kv_heads"], CFG["head_dim"]
    for li in range(CFG["n_layers"]):
        F = full["layers"][li]
        q = torch.cat([p["layers"][li]["wqkv"][: H // t * hd] for p in parts])
        k = torch.cat([p["layers"][li]["wqkv"][H // t * hd:(H + Hkv) // t * hd] for p in parts])
        assert torch.equal(q, F["wqkv"][: H * hd]) and torch.equal(k, F["wqkv"][H * hd:(H + Hkv) * hd])
        assert torch.equal(torch.cat([p["layers"][li]["wo"] for p in parts], 1), F["wo"])
        assert torch.equal(torch.cat([p["layers"][li]["wdown"] for p in parts], 1), F["wdown"])
    assert torch.equal(torch.cat([p["lm_head"] for p in parts]), full["lm_head"])
    assert torch.equal(torch.cat([p["medusa"][1]["U"] for p in parts]), full["medusa"][1]["U"])


@pytest.mark.parametrize("t", [2, 4])
@pytest.mark.parametrize("seed", [0, 1])
def test_tp_greedy_tokens_equal_oracle(sm, t, seed):
    prompt = synth.prompt_tokens(seed, 0, 32, CFG["vocab"])
    W = OM.Weights(CFG, n_medusa=3, seed=seed)
    s = OS.Session(OM.Model(CFG, W, "bf16"), synth.TINY16, batch=1, max_seq_len=X)
    s.prefill(0, prompt)
    ref = []
    while len(ref) < 32:
        ref += s.step(0, budget=32 - len(ref))["emitted"]

    rk = Ranks(sm, t, seed=seed)
    pt = torch.from_numpy(prompt).cuda()
    rk.each(lambda r, kv, st: kv.prefill(0, pt, stream=st))
    budgets = [torch.full((1,), 32, dtype=torch.int32, device="cuda") for _ in range(t)]
    cfgs = [sm.accept_cfg(sm.GREEDY, max_new=budgets[r]) for r in range(t)]
    toks = [[] for _ in range(t)]
    for _ in range(64):
        if len(toks[0]) >= 32:
            break
        rk.each(lambda r, kv, st: kv.step(cfgs[r], rk.outs[r], stream=st))
        for r in range(t):
            o = rk.outs[r]
            ne = int(o.n_emit.cpu()[0])
            toks[r] += o.emit_tok.cpu().numpy()[0][:ne].tolist()
            budgets[r] -= o.n_emit
    assert not rk.timed_out()
    for r in range(t):  # replicated acceptance: every rank emits the same stream
        assert toks[r] == toks[0]
    assert toks[0] == ref


def test_tp_logits_match_tp1(sm):
    """Vocabulary-parallel verify logits (one tree step after the same prefill)."""
    seed, t = 6, 2
    prompt = torch.from_numpy(synth.prompt_tokens(seed, 0, 32, CFG["vocab"])).cuda()
    W1 = sm.allocate_weights(CFG, 3, seed=seed)
    tree = sm.Tree(synth.TINY16, topk=10)
    m1 = sm.Model(CFG, W1, 64, 1, X + tree.N)
    kv1 = sm.KVCache(m1, tree, 1, X)
    kv1.prefill(0, prompt)
    tok1 = torch.zeros(tree.N, dtype=torch.int32, device="cuda")
    kv1.propose(tok1)
    z1 = torch.zeros(tree.N, CFG["vocab"], dtype=torch.float32, device="cuda")
    kv1.verify(tok1, z1)
    torch.cuda.synchronize()

    rk = Ranks(sm, t, seed=seed)
    rk.each(lambda r, kv, st: kv.prefill(0, prompt, stream=st))
    toks = [torch.zeros(tree.N, dtype=torch.int32, device="cuda") for _ in range(t)]
    Vl = CFG["vocab"] // t
    zs = [torch.zeros(tree.N, Vl, dtype=torch.float32, device="cuda") for _ in range(t)]
    rk.each(lambda r, kv, st: kv.propose(toks[r], stream=st))
    for r in range(t):
        assert torch.equal(toks[r], tok1)  # merged top-K of the heads == tp = 1 top-K
    rk.each(lambda r, kv, st: kv.verify(toks[r], zs[r], stream=st))
    assert not rk.timed_out()
    z = torch.cat(zs, 1).double().cpu().numpy()
    ref = z1.double().cpu().numpy()
    assert np.all(np.abs(z - ref) <= 2e-2 + 2e-2 * np.abs(ref)), float(np.abs(z - ref).max())


@pytest.mark.parametrize("seed", [0, 3])
def test_tp_typical_accept_matches_tp1(sm, seed):
    """Typical acceptance under TP uses the merged (m, s, t) statistics and the owner
    rank's candidate logits: one verify + accept must match tp = 1 exactly."""
    t = 2
    prompt = torch.from_numpy(synth.prompt_tokens(seed, 0, 32, CFG["vocab"])).cuda()
    tree = sm.Tree(synth.TINY16, topk=10)
    m1 = sm.Model(CFG, sm.allocate_weights(CFG, 3, seed=seed, medusa_init=True), 64, 1, X + tree.N)
    kv1 = sm.KVCache(m1, tree, 1, X)
    kv1.prefill(0, prompt)
    tok1 = torch.zeros(tree.N, dtype=torch.int32, device="cuda")
    kv1.propose(tok1)
    kv1.verify(tok1)
    acfg = sm.accept_cfg(sm.TYPICAL, temperature=0.7, eps=0.09, alpha=0.3)
    o1 = sm.AcceptOut(1, tree.depth)
    kv1.accept(acfg, o1)
    torch.cuda.synchronize()

    rk = Ranks(sm, t, seed=seed, medusa_init=True)
    rk.each(lambda r, kv, st: kv.prefill(0, prompt, stream=st))
    toks = [torch.zeros(tree.N, dtype=torch.int32, device="cuda") for _ in range(t)]
    rk.each(lambda r, kv, st: kv.propose(toks[r], stream=st))
    rk.each(lambda r, kv, st: kv.verify(toks[r], stream=st))
    rk.each(lambda r, kv, st: kv.accept(acfg, rk.outs[r], stream=st))
    assert not rk.timed_out()
    for r in range(t):
        assert torch.equal(toks[r], tok1)
        for name in ("acc_len", "best_leaf", "path", "emit_tok", "n_emit"):
            assert torch.equal(getattr(rk.outs[r], name), getattr(o1, name)), name
