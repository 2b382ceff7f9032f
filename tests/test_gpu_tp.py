"""Tensor parallelism (SURVEY §8 rows a7 / e) emulated on one B200.

t ranks = t sm_models in one process on the same device, each holding its shard
(allocate_weights(tp_rank, tp_size)) and exchanging through the other ranks'
symmetric buffers -- the same kernels and data layout a multi-GPU run uses over
NVLink peer memory (there the peer pointers come from CUDA IPC).  On one GPU no
kernel may spin on a flag another rank's launch raises (nothing guarantees the
two run at the same time; B200_PROFILING.md), so the ranks share an EmuGroup:
every exchange runs as segment launches (publish; [reduce-scatter;] merge) and
each rank's host thread joins its stream to its peers' "published" events
between segments (host-ordered emulation, include/specmemo.h).  The arithmetic
and the rank-order sums are those of the fused flag protocol, so the results
are the same bits.  Programmatic dependent launch stays on (the default): with
no device-side waits a rank's early-launched successors can only delay a peer.

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


class Ranks:
    """t ranks in one process: all on the current GPU (host-ordered emulation, one host thread per
    rank), or rank r on GPU devices[r] with peer access between every pair (the real placement,
    one GPU per rank, fused flag protocol)."""

    def __init__(self, sm, t, seed=0, n_medusa=3, choices=synth.TINY16, batch=1, medusa_init=False, cfg=CFG,
                 devices=None):
        self.sm, self.t = sm, t
        self.dev = devices or [torch.cuda.current_device()] * t
        if devices:  # a cross-device copy makes torch enable peer access for the pair
            for i in self.dev:
                for j in self.dev:
                    if i != j:
                        torch.empty(1, device=f"cuda:{i}").copy_(torch.empty(1, device=f"cuda:{j}"))
        self.tree = sm.Tree(choices, topk=10)
        R = max(batch * self.tree.N, 64)
        nbytes = sm.tp_sym_bytes(cfg, R, batch, n_medusa)
        self.sym, self.W, self.models, self.kvs, self.streams, self.outs = [], [], [], [], [], []
        self.emu = sm.EmuGroup(t) if len(set(self.dev)) < t else None
        for r in range(t):
            with torch.cuda.device(self.dev[r]):
                self.sym.append(torch.zeros(nbytes, dtype=torch.uint8, device="cuda"))
        ptrs = [s.data_ptr() for s in self.sym]
        for r in range(t):
            with torch.cuda.device(self.dev[r]):
                self.W.append(sm.allocate_weights(cfg, n_medusa, seed=seed, medusa_init=medusa_init, tp_rank=r,
                                                  tp_size=t))
                self.models.append(sm.Model(cfg, self.W[r], R, batch, X + self.tree.N, peer_sym=ptrs,
                                            emu_group=self.emu))
                self.kvs.append(sm.KVCache(self.models[r], self.tree, batch, X))
                self.streams.append(torch.cuda.Stream())
                self.outs.append(sm.AcceptOut(batch, self.tree.depth))
        for d in set(self.dev):
            torch.cuda.synchronize(d)

    def each(self, fn):
        def run(r):
            def go():
                with torch.cuda.device(self.dev[r]), torch.cuda.stream(self.streams[r]):
                    fn(r, self.kvs[r], self.streams[r])
            return go
        if self.emu is not None:  # one host thread per rank: an exchange blocks until the peers published
            self.sm.run_ranks([run(r) for r in range(self.t)])
        else:
            for r in range(self.t):
                run(r)()
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


# ------------------------------------------------------------------ t = 8 (the 70B shape's TP8 placement)
# 8 kv heads so every rank owns one (C4 at TP8: Hkv / t = 1), d = 128, F = 512 (F / 64 divisible by 8)
CFG8 = synth.model_cfg("tiny", d_model=128, n_heads=8, n_kv_heads=8, head_dim=16, d_ffn=512, vocab=256)


def _greedy_ref(cfg, seed, n):
    prompt = synth.prompt_tokens(seed, 0, 32, cfg["vocab"])
    s = OS.Session(OM.Model(cfg, OM.Weights(cfg, n_medusa=3, seed=seed), "bf16"), synth.TINY16, batch=1,
                   max_seq_len=X)
    s.prefill(0, prompt)
    ref = []
    while len(ref) < n:
        ref += s.step(0, budget=n - len(ref))["emitted"]
    assert ref == OS.vanilla_generate(s.m, prompt, n)[0]
    return prompt, ref


@pytest.mark.parametrize("rsag", [-1, 0], ids=["rsag", "oneshot"])
@pytest.mark.parametrize("seed", [0, 2])
def test_tp8_greedy_tokens_equal_oracle(sm, seed, rsag):
    """t = 8 ranks (the 70B shape's TP8 placement: one kv head per rank), one per GPU when the box
    has 8 (fused flag protocol over peer memory), else host-ordered emulation on one GPU; residual
    exchange as reduce-scatter + all-gather (the t >= 4 default) and as the one-shot sum: every
    rank emits the oracle's greedy stream (= vanilla greedy)."""
    sm.set_option("tp_rsag", rsag)
    devices = list(range(8)) if torch.cuda.device_count() >= 8 else None
    t, n = 8, 24
    prompt, ref = _greedy_ref(CFG8, seed, n)
    rk = Ranks(sm, t, seed=seed, cfg=CFG8, devices=devices)
    pts = [torch.from_numpy(prompt).to(f"cuda:{d}") for d in rk.dev]
    rk.each(lambda r, kv, st: kv.prefill(0, pts[r], stream=st))
    budgets = [torch.full((1,), n, dtype=torch.int32, device=f"cuda:{d}") for d in rk.dev]
    cfgs = [sm.accept_cfg(sm.GREEDY, max_new=budgets[r]) for r in range(t)]
    toks = [[] for _ in range(t)]
    for _ in range(2 * n):
        if len(toks[0]) >= n:
            break
        rk.each(lambda r, kv, st: kv.step(cfgs[r], rk.outs[r], stream=st))
        for r in range(t):
            o = rk.outs[r]
            ne = int(o.n_emit.cpu()[0])
            toks[r] += o.emit_tok.cpu().numpy()[0][:ne].tolist()
            budgets[r] -= o.n_emit
    assert not rk.timed_out()
    for r in range(t):
        assert toks[r] == toks[0]
    assert toks[0] == ref


# ------------------------------------------------------------------ two processes, CUDA IPC
def _ipc_rank(rank, world, port, seed, n, q):
    import os
    import traceback

    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    except Exception:
        q.put((rank, traceback.format_exc(), True))
        return
    try:
        import paper_2506_01986_b200 as sm
        torch.cuda.set_device(rank)  # one GPU per rank (peer access over NVLink)
        tree = sm.Tree(synth.TINY16, topk=10)
        W = sm.allocate_weights(CFG, 3, seed=seed, tp_rank=rank, tp_size=world)
        sym = torch.zeros(sm.tp_sym_bytes(CFG, 64, 1, 3), dtype=torch.uint8, device="cuda")
        hs = [None] * world
        dist.all_gather_object(hs, sm.ipc_handle(sym))
        peers = [sym.data_ptr() if r == rank else sm.ipc_open(hs[r]) for r in range(world)]
        model = sm.Model(CFG, W, 64, 1, X + tree.N, peer_sym=peers)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's buffer is zeroed before any exchange
        kv = sm.KVCache(model, tree, 1, X)
        kv.prefill(0, torch.from_numpy(synth.prompt_tokens(seed, 0, 32, CFG["vocab"])).cuda())
        budget = torch.full((1,), n, dtype=torch.int32, device="cuda")
        cfg = sm.accept_cfg(sm.GREEDY, max_new=budget)
        out = sm.AcceptOut(1, tree.depth)
        toks = []
        for _ in range(2 * n):
            if len(toks) >= n:
                break
            kv.step(cfg, out)
            ne = int(out.n_emit.cpu()[0])
            toks += out.emit_tok.cpu().numpy()[0][:ne].tolist()
            budget -= out.n_emit
        q.put((rank, toks, model.tp_timed_out()))
        torch.cuda.synchronize()
        dist.barrier()
        for r, p in enumerate(peers):
            if r != rank:
                sm.ipc_close(p)
    except Exception:  # report instead of hanging the parent
        q.put((rank, traceback.format_exc(), True))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="cross-process exchange needs a GPU per rank: two contexts on one GPU time-slice, so a "
                           "rank spinning on its peer's flag starves the peer (no MPS on the test boxes)")
def test_tp2_two_processes_cuda_ipc(sm):
    """The multi-process TP path: two processes on one GPU, symmetric buffers exchanged as CUDA
    IPC handles over torch.distributed (gloo), the fused residual all-reduce and vocabulary-
    parallel merges running across process boundaries (the kernels time-slice between the two
    contexts; the exchange flags are polled with a timeout, sm_tp_status).  Tokens = oracle."""
    import socket

    import torch.multiprocessing as mp
    seed, n = 1, 16
    _, ref = _greedy_ref(CFG, seed, n)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, seed, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    for rank, toks, timed_out in res:
        assert not timed_out, (rank, toks)
        assert toks == ref, (rank, toks, ref)
