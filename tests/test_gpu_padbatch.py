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


def test_pad_batching_matches_oracle(sm):
    """GPU pad mode against the oracle's PadSession (pinned in test_oracle_padbatch.py)
    on the same seeded inputs: every step the tree tokens, their positions (real tokens only), the
    cache slot counts, the emitted tokens, and the K/V of every committed (non-pad) slot must
    agree -- integers bit-exact, floats within the 2e-2 bar -- and the verify logits of steps 2..6
    within the bar.  Acceptance is imposed through the forced-path hook on both sides (depths 3 / 0
    / 1, rotating), so the sequences' caches fill with pads at different slots."""
    from oracle import model as OM
    from oracle import spec as OS
    from oracle import tree as OT
    from lockstep import bar_check

    b, x, seed = 3, 128, 9
    prompts = [synth.prompt_tokens(seed, i, 20 + 7 * i, CFG["vocab"]) for i in range(b)]
    W = sm.allocate_weights(CFG, 3, seed=seed)
    tree = sm.Tree(synth.TINY16, topk=10)
    model = sm.Model(CFG, W, max_rows=64, max_batch=b, max_seq_len=x + tree.N)
    kv = sm.KVCache(model, tree, b, x)
    ps = OS.PadSession(OM.Model(CFG, OM.Weights(CFG, n_medusa=3, seed=seed), "bf16"), synth.TINY16, b, x)
    for i, p in enumerate(prompts):
        kv.prefill(i, torch.from_numpy(p).cuda())
        ps.prefill(i, p)
    kv.set_pad_mode(True)
    ot = ps.tree
    deep = next(n for n in range(ot.N) if ot.depth[n] == 3)
    d1 = [n for n in range(ot.N) if ot.depth[n] == 1][1]
    paths = [OT.ancestors(ot, deep) + [deep], [0], [0, d1]]
    out = sm.AcceptOut(b, tree.depth)
    L = CFG["n_layers"]
    for step in range(6):
        fz = [paths[(s + step) % 3] for s in range(b)]
        forced = torch.full((b, tree.depth + 1), -1, dtype=torch.int32)
        for s in range(b):
            forced[s, : len(fz[s])] = torch.tensor(fz[s], dtype=torch.int32)
        forced_dev = forced.cuda()  # the cfg holds a raw device pointer: keep the tensor alive
        acfg = sm.accept_cfg(forced_path=forced_dev)
        if step == 0:  # the first step through sm_step: it aligns the ragged prompts
            res = ps.step_batch(forced=fz)
            kv.step(acfg, out)
        else:
            tt = torch.zeros(b, tree.N, dtype=torch.int32, device="cuda")
            pos = torch.zeros(b, tree.N, dtype=torch.int32, device="cuda")
            kv.propose(tt, pos)
            torch.cuda.synchronize()
            g_tok = tt.cpu().numpy()
            for s in range(b):  # a1: the GPU's tree is the oracle's up to near-tied top-K ranks
                o_tok, o_pos = ps.propose(s)
                heads = [ps.m.head_logits(i, ps.last_hf[s]) for i in range(ot.max_depth)]
                for n in range(1, ot.N):
                    if g_tok[s][n] != o_tok[n]:
                        v = heads[ot.depth[n] - 1]
                        gap = abs(float(v[g_tok[s][n]]) - float(v[o_tok[n]]))
                        assert gap <= 1e-2 * float(np.abs(v).max()), (step, s, n, gap)
                assert g_tok[s][0] == o_tok[0] and pos[s].cpu().tolist() == o_pos, (step, s)
            res = ps.step_batch(forced=fz, toks=g_tok)  # the oracle verifies the GPU's tree
            z = torch.zeros(b, tree.N, CFG["vocab"], dtype=torch.float32, device="cuda")
            kv.verify(tt, z)
            kv.accept(acfg, out)
            torch.cuda.synchronize()
            for s in range(b):
                bar_check(z[s].cpu().numpy(), np.stack(res[s]["Z"]), 2e-2, f"logits step {step} seq {s}")
        ne = out.n_emit.cpu().numpy()
        et = out.emit_tok.cpu().numpy()
        for s in range(b):
            assert et[s][: ne[s]].tolist() == res[s]["emitted"], (step, s)
        assert kv.lengths().tolist() == ps.Lc and kv.positions().tolist() == ps.pos
    # K/V of every non-pad slot (pad slots hold stale scratch: never read, never compared)
    mem = kv.layout().float().cpu().numpy()
    for s in range(b):
        real = [j for j in range(ps.Lc[s]) if j not in ps.pad[s]]
        for li in range(L):
            bar_check(mem[li, 0, s][:, real], ps.kv.K[li][s][:, real, :], 2e-2, f"K layer {li} seq {s}")
            bar_check(mem[li, 1, s][:, real], ps.kv.V[li][s][:, real, :], 2e-2, f"V layer {li} seq {s}")
