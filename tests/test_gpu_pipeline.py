"""Layer-split pipeline (f4 comparison mode) emulated on one B200.

"We distributed the base model evenly by partitioning its layers into equal-sized chunks across
all available GPUs, with each GPU also hosting the corresponding slices of the KV cache alongside
the layers".  pp ranks = pp sm_models in one process on one device, rank r holding layers
[r L/pp, (r+1) L/pp) and their KV slices; the residual rows move between stages through the
symmetric buffers (the same kernels and data layout as across GPUs, where the peer pointers come
from CUDA IPC).  On one GPU no kernel may spin on a hand-off another rank's launch raises, so the
stages share an EmuGroup (host-ordered emulation, include/specmemo.h): a receiver's stream waits
for the sender's "published" event, each stage driven by its own host thread.  The split changes no arithmetic, so every rank must produce the pp = 1 results
bit for bit -- logits, tree tokens, emitted tokens, the K/V of its layers -- and the greedy stream
must equal the oracle's (= vanilla greedy) on the screened seeds."""
import numpy as np
import pytest
import torch

import synth
from oracle import model as OM
from oracle import spec as OS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


X = 96


class Stages:
    def __init__(self, sm, cfg, pp, seed, choices=synth.TINY16, batch=1, n_medusa=3):
        self.sm, self.pp = sm, pp
        self.tree = sm.Tree(choices, topk=10)
        R = max(64, batch * self.tree.N)
        self.sym = [torch.zeros(sm.tp_sym_bytes(cfg, R, batch, n_medusa), dtype=torch.uint8, device="cuda")
                    for _ in range(pp)] if pp > 1 else None
        ptrs = [s.data_ptr() for s in self.sym] if pp > 1 else None
        self.emu = sm.EmuGroup(pp) if pp > 1 else None
        self.W = [sm.allocate_weights(cfg, n_medusa, seed=seed, pp_rank=r, pp_size=pp) for r in range(pp)]
        self.models = [sm.Model(cfg, self.W[r], R, batch, X + self.tree.N, peer_sym=ptrs, emu_group=self.emu)
                       for r in range(pp)]
        self.kvs = [sm.KVCache(m, self.tree, batch, X) for m in self.models]
        self.streams = [torch.cuda.Stream() for _ in range(pp)]
        self.outs = [sm.AcceptOut(batch, self.tree.depth) for _ in range(pp)]
        torch.cuda.synchronize()

    def each(self, fn):
        def run(r):
            def go():
                with torch.cuda.stream(self.streams[r]):
                    fn(r, self.kvs[r], self.streams[r])
            return go
        self.sm.run_ranks([run(r) for r in range(self.pp)])  # one host thread per stage
        for s in self.streams:
            s.synchronize()

    def timed_out(self):
        return any(m.tp_timed_out() for m in self.models) if self.pp > 1 else False


def _run(sm, cfg, pp, seed, n, prompts):
    st = Stages(sm, cfg, pp, seed, batch=len(prompts))
    for i, p in enumerate(prompts):
        pt = torch.from_numpy(p).cuda()
        st.each(lambda r, kv, s: kv.prefill(i, pt, stream=s))
    b = len(prompts)
    budgets = [torch.full((b,), n, dtype=torch.int32, device="cuda") for _ in range(pp)]
    cfgs = [sm.accept_cfg(sm.GREEDY, max_new=budgets[r]) for r in range(pp)]
    toks = [[[] for _ in range(b)] for _ in range(pp)]
    for _ in range(2 * n):
        if all(len(t) >= n for t in toks[0]):
            break
        st.each(lambda r, kv, s: kv.step(cfgs[r], st.outs[r], stream=s))
        for r in range(pp):
            o = st.outs[r]
            ne = o.n_emit.cpu().numpy()
            et = o.emit_tok.cpu().numpy()
            for s in range(b):
                toks[r][s] += et[s][: ne[s]].tolist()
            budgets[r] -= o.n_emit
    # one more verify: the logits of the next tree on every rank
    tts = [torch.zeros(b, st.tree.N, dtype=torch.int32, device="cuda") for _ in range(pp)]
    zs = [torch.zeros(b, st.tree.N, cfg["vocab"], dtype=torch.float32, device="cuda") for _ in range(pp)]
    st.each(lambda r, kv, s: kv.propose(tts[r], stream=s))
    st.each(lambda r, kv, s: kv.verify(tts[r], zs[r], stream=s))
    assert not st.timed_out()
    return st, toks, tts, zs


@pytest.mark.parametrize("pp", [2, 4])
def test_pipeline_equals_single_stage_bitwise(sm, pp):
    cfg = synth.model_cfg("tiny", n_layers=4)
    seed, n = 1, 16
    prompts = [synth.prompt_tokens(seed, i, 24 + 9 * i, cfg["vocab"]) for i in range(2)]
    one, toks1, tt1, z1 = _run(sm, cfg, 1, seed, n, prompts)
    many, toksp, ttp, zp = _run(sm, cfg, pp, seed, n, prompts)
    per = cfg["n_layers"] // pp
    kv1 = one.kvs[0].layout()
    for r in range(pp):
        assert toksp[r] == toks1[0]                                     # emitted tokens
        assert torch.equal(ttp[r], tt1[0])                              # next tree
        assert torch.equal(zp[r], z1[0])                                # logits, bit for bit
        assert np.array_equal(many.kvs[r].lengths(), one.kvs[0].lengths())
        assert torch.equal(many.kvs[r].layout(), kv1[r * per:(r + 1) * per])  # this rank's K/V slices


def test_pipeline_greedy_equals_oracle(sm):
    """pp = 2 on the C1 shape (2 layers, one per stage): the oracle's greedy stream (= vanilla)."""
    cfg = synth.model_cfg("tiny")
    seed, n = 1, 24  # oracle-screened seed (smoke / test_gpu_e2e)
    prompt = synth.prompt_tokens(seed, 0, 32, cfg["vocab"])
    _, toks, _, _ = _run(sm, cfg, 2, seed, n, [prompt])
    s = OS.Session(OM.Model(cfg, OM.Weights(cfg, n_medusa=3, seed=seed), "bf16"), synth.TINY16, 1, X)
    s.prefill(0, prompt)
    ref, _ = s.generate(0, n)
    assert toks[0][0] == ref and toks[1][0] == ref


def test_pipeline_rejects_bad_splits(sm):
    cfg = synth.model_cfg("tiny", n_layers=3)
    with pytest.raises(ValueError):
        sm.allocate_weights(cfg, 3, pp_rank=0, pp_size=2)


def test_pipeline_c2_width_bitwise(sm):
    """pp = 2 at the C2 width (d 4096, 32 heads, hd 128, F 11008, V 32000; 2 layers, one per stage,
    V64 tree): the tcgen05 GEMMs, the tcgen05 K1 and the 4096-wide residual hand-offs; every stage's
    logits, tree tokens and K/V equal pp = 1 bit for bit."""
    cfg = synth.model_cfg("vicuna7b", n_layers=2)
    seed, n = 3, 6
    prompts = [synth.prompt_tokens(seed, 0, 40, cfg["vocab"])]

    def run(pp):
        st = Stages(sm, cfg, pp, seed, choices=synth.V64, n_medusa=4)
        pt = torch.from_numpy(prompts[0]).cuda()
        st.each(lambda r, kv, s: kv.prefill(0, pt, stream=s))
        cfgs = [sm.accept_cfg(sm.GREEDY) for _ in range(pp)]
        for _ in range(n):
            st.each(lambda r, kv, s: kv.step(cfgs[r], st.outs[r], stream=s))
        tts = [torch.zeros(1, st.tree.N, dtype=torch.int32, device="cuda") for _ in range(pp)]
        zs = [torch.zeros(1, st.tree.N, cfg["vocab"], dtype=torch.float32, device="cuda") for _ in range(pp)]
        st.each(lambda r, kv, s: kv.propose(tts[r], stream=s))
        st.each(lambda r, kv, s: kv.verify(tts[r], zs[r], stream=s))
        assert not st.timed_out()
        return st, tts, zs

    one, tt1, z1 = run(1)
    two, tt2, z2 = run(2)
    kv1 = one.kvs[0].layout()
    for r in range(2):
        assert torch.equal(tt2[r], tt1[0]) and torch.equal(z2[r], z1[0])
        assert np.array_equal(two.kvs[r].lengths(), one.kvs[0].lengths())
        assert torch.equal(two.kvs[r].layout(), kv1[r:r + 1])
