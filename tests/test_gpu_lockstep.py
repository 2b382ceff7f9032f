"""End-to-end lock-step parity with the oracle at every model shape class.

The harness (tests/lockstep.py) compares every propose / verify / accept / compact decision of
every step: integer outputs bit-exact wherever the oracle's margin clears the guard (and
valid otherwise), logits and K/V element by element.  Shapes:

* C1 (tiny, hd 16): bf16 and fp32, greedy and typical -- the elementwise 2e-2 / 1e-4 bars
  hold for every element;
* C2 width (Vicuna-7B: d 4096, 32 heads of 128, F 11008, V 32000, V64 tree, 4 heads) at 2
  layers, Medusa-init heads (tau > 1, so compaction runs) and random heads, bf16 and fp32;
* C3 width (Vicuna-13B, d 5120) at 2 layers, typical acceptance;
* C4 class (GQA 8:1, hd 128, V 32000) at 2 layers, b in {2, 4, 8, 10}: M = 160 (tiny16 x 10)
  takes the 2-SM K2, M = 640 (V64 x 10) the token-tile-group K2.

bf16 at 4096+ widths: one-ulp differences at bf16 storage points (fp32 summation order)
cascade through the 4096/11008-term GEMMs; the measured spread between two valid bf16
implementations of the definition (the oracle with fp64 vs fp32 accumulation) exceeds the
elementwise 2e-2 bar on a small fraction of logits (Q29, tools/diag_bf16_noise.py),
so there the bar is asserted per row as an explicit exceedance bound: at most MAX_FRAC of the
elements over 2e-2 (1 + |ref|) and none over HARD x the bar."""
import numpy as np
import pytest
import torch

import synth
from oracle import model as OM

from lockstep import LockStep

pytestmark = pytest.mark.gpu

MAX_FRAC, HARD = 1e-2, 3.0      # bf16 at >= 1024 widths, per row (module docstring); C1-class shapes: 0


@pytest.fixture(scope="module")
def sm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2506_01986_b200 as sm
    sm.lib()
    return sm


def _prompts(seed, b, vocab, lo=12, step=3):
    return [synth.prompt_tokens(seed, i, lo + step * i, vocab) for i in range(b)]


# ------------------------------------------------------------------ C1
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("mode", ["greedy", "typical"])
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_c1_lockstep(sm, dtype, mode, seed):
    cfg = synth.model_cfg("tiny")
    typ = dict(synth.TYPICAL) if mode == "typical" else None
    ls = LockStep(sm, cfg, 3, synth.TINY16, _prompts(seed, 1, cfg["vocab"], lo=32), 128, dtype=dtype, seed=seed,
                  typ=typ)
    st = ls.run(16)
    assert st["exact_decisions"] >= 16 * 10
    assert st["forced"] <= 8, st


def test_c1_lockstep_medusa_init_compacts(sm):
    """Medusa-init heads (R = 0, U = W_lm, Q18) on the tiny model: accepted depths > 0 occur,
    so compaction moves K/V inside the compared steps."""
    cfg = synth.model_cfg("tiny")
    ls = LockStep(sm, cfg, 3, synth.TINY16, _prompts(7, 2, cfg["vocab"], lo=20), 160, seed=7, medusa_init=True)
    st = ls.run(24)
    assert sum(st["accepted_depth_hist"][1:]) > 0, st


# ------------------------------------------------------------------ C2 / C3 width, 2 layers
C2 = synth.model_cfg("vicuna7b", n_layers=2)
C3 = synth.model_cfg("vicuna13b", n_layers=2)


@pytest.fixture(scope="module")
def c2_weights_init():
    return OM.Weights(C2, n_medusa=4, seed=0, medusa_init=True)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_c2_width_greedy_multistep_medusa_init(sm, c2_weights_init, dtype):
    kw = dict(max_frac=MAX_FRAC, hard=HARD) if dtype == "bf16" else {}
    ls = LockStep(sm, C2, 4, synth.V64, _prompts(11, 1, C2["vocab"], lo=12), 96, dtype=dtype, seed=0,
                  medusa_init=True, oracle_weights=c2_weights_init, force_deep_every=2, **kw)
    st = ls.run(8)
    print(dtype, st)
    assert st["exact_decisions"] >= 8 * 25 and st["tolerated"] <= st["exact_decisions"] // 4, st
    assert st["forced"] <= 2, st
    assert sum(st["accepted_depth_hist"][1:]) >= 4, st  # compaction of 4-deep paths at 7B width


def test_c2_width_random_heads_bf16(sm):
    ls = LockStep(sm, C2, 4, synth.V64, _prompts(5, 1, C2["vocab"], lo=16), 64, seed=1, max_frac=MAX_FRAC,
                  hard=HARD, force_deep_every=2)
    st = ls.run(4)
    print(st)
    assert st["exact_decisions"] >= 4 * 20 and st["tolerated"] <= st["exact_decisions"] // 4, st


def test_c3_width_typical_bf16(sm):
    ls = LockStep(sm, C3, 4, synth.V64, _prompts(3, 1, C3["vocab"], lo=14), 64, seed=2, max_frac=MAX_FRAC,
                  hard=HARD, typ=dict(synth.TYPICAL))
    st = ls.run(4)
    print(st)
    assert st["exact_decisions"] >= 4 * 25 and st["tolerated"] <= st["exact_decisions"] // 4, st


# ------------------------------------------------------------------ C4 class: GQA 8:1, batched
C4S = synth.model_cfg("llama70b", n_layers=2, d_model=1024, n_heads=8, n_kv_heads=1, d_ffn=2816)


@pytest.fixture(scope="module")
def c4_weights():
    return OM.Weights(C4S, n_medusa=4, seed=3, medusa_init=True)


@pytest.mark.parametrize("b,choices", [(2, synth.TINY16), (4, synth.TINY16), (8, synth.TINY16),
                                       (10, synth.TINY16), (10, synth.V64)], ids=["b2", "b4", "b8", "b10-M160",
                                                                                  "b10-M640"])
def test_c4_class_batched_lockstep(sm, c4_weights, b, choices):
    ls = LockStep(sm, C4S, 4, choices, _prompts(30 + b, b, C4S["vocab"], lo=9, step=5), 96, seed=3,
                  medusa_init=True, oracle_weights=c4_weights, max_frac=MAX_FRAC, hard=HARD, force_deep_every=2)
    st = ls.run(4)
    print(b, len(choices) + 1, st)
    assert st["exact_decisions"] >= 4 * b * 6 and st["tolerated"] <= st["exact_decisions"] // 4, st
    assert sum(st["accepted_depth_hist"][1:]) >= 2 * b, st


def test_c2_width_bf16_as_accurate_as_the_rounded_definition(sm, c2_weights_init):
    """The GPU's bf16 logits against the fp64 plain definition are no worse than the oracle's
    own bf16 storage-point emulation against it (same rows, same tree tokens): per row, the rms
    error within 1.3x; over all rows, the fraction of elements over the 2e-2 (1 + |z|) bar within
    1.5x + 5e-4 of the oracle's and no element over 3x the bar.  (Measured at seed 11: rms 0.0099 vs 0.0097, frac 5.1e-3 vs 4.4e-3.)"""
    prompt = synth.prompt_tokens(11, 0, 12, C2["vocab"])
    W = sm.allocate_weights(C2, 4, seed=0, medusa_init=True)
    tree = sm.Tree(synth.V64, topk=10)
    model = sm.Model(C2, W, max_rows=64, max_batch=1, max_seq_len=64 + tree.N)
    kv = sm.KVCache(model, tree, 1, 64)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    tt = torch.zeros(1, tree.N, dtype=torch.int32, device="cuda")
    kv.propose(tt)
    logits = torch.zeros(1, tree.N, C2["vocab"], dtype=torch.float32, device="cuda")
    kv.verify(tt, logits)
    torch.cuda.synchronize()
    tok = tt[0].cpu().tolist()
    Zg = logits[0].cpu().numpy().astype(np.float64)
    from oracle import spec as OS
    Z = {}
    for mode in ("bf16", "fp64"):
        s = OS.Session(OM.Model(C2, c2_weights_init, mode), synth.V64, 1, 64, batched=True)
        s.prefill(0, prompt)
        assert s.propose(0)[0] == tok            # tree tokens bit-exact (every top-K gap cleared here)
        Z[mode] = np.stack(s.verify(0, tok)[0])
    ref = Z["fp64"]
    bar = 2e-2 * (1 + np.abs(ref))
    eg, eo = np.abs(Zg - ref), np.abs(Z["bf16"] - ref)
    for n in range(tree.N):   # per row: rms error within 1.3x of the rounded definition's
        assert np.sqrt(np.mean(eg[n] ** 2)) <= 1.3 * np.sqrt(np.mean(eo[n] ** 2)), n
    # elements over the 2e-2 bar: a few per 1000 for both (counts per row are small: compare totals)
    assert np.mean(eg > bar) <= 1.5 * np.mean(eo > bar) + 5e-4, (np.mean(eg > bar), np.mean(eo > bar))
    assert np.max(eg / bar) <= 3.0
