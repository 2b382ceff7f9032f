"""More pins for the oracle (no GPU), against independent implementations:

* the Medusa-1 head (``Model.head_logits``) against a ``torch.nn`` ResBlock + unembedding
  built from ``nn.Linear`` layers (reading Q6: one ResBlock ``x + SiLU(Linear_with_bias(x))``,
  then a bias-free ``Linear(d, V)``; Eq. 4's size pin P:81), with a nonzero bias so the
  ``beta`` term is exercised (the R = 0 special case cannot see it);
* the typical-acceptance statistics (``spec.typical_stats``) against ``scipy.special.softmax``
  and ``scipy.stats.entropy`` (the exact Shannon entropy of P_T, reading Q10; "entropy
  threshold", "typical sampling");
* the batched forward (``Model.forward_rows``, used for wide models and for the bench's
  timing variant) against the row-at-a-time ``forward_row`` that the HF-Llama pins cover."""
import copy

import numpy as np
import pytest
import scipy.special
import scipy.stats
import torch

import synth
from oracle import model as M
from oracle import spec as SP
from oracle import tree as T


class _MedusaHead(torch.nn.Module):
    """Medusa-1 head written with torch.nn layers: ResBlock then unembedding."""

    def __init__(self, d, V):
        super().__init__()
        self.res = torch.nn.Linear(d, d, bias=True)
        self.out = torch.nn.Linear(d, V, bias=False)

    def forward(self, h):
        return self.out(h + torch.nn.functional.silu(self.res(h)))


@pytest.mark.parametrize("seed", [0, 3])
def test_medusa_head_matches_nn_linear_resblock(seed):
    cfg = synth.model_cfg("tiny", vocab=300)
    W = M.Weights(cfg, n_medusa=2, seed=seed)
    rng = np.random.default_rng(seed)
    for i in range(2):
        W.medusa[i]["beta"] = rng.standard_normal(cfg["d_model"]) * 0.05
    m = M.Model(cfg, W, "fp64")
    net = [_MedusaHead(cfg["d_model"], cfg["vocab"]).double() for _ in range(2)]
    with torch.no_grad():
        for i in range(2):
            net[i].res.weight.copy_(torch.from_numpy(W.medusa[i]["R"]))
            net[i].res.bias.copy_(torch.from_numpy(W.medusa[i]["beta"]))
            net[i].out.weight.copy_(torch.from_numpy(W.medusa[i]["U"]))
    for _ in range(4):
        hf = rng.standard_normal(cfg["d_model"])
        for i in range(2):
            with torch.no_grad():
                ref = net[i](torch.from_numpy(hf)).numpy()
            got = m.head_logits(i, hf)
            assert np.allclose(got, ref, rtol=0, atol=1e-12)
    # head i uses its own weights (a transposed or shared operand would fail this)
    assert not np.allclose(m.head_logits(0, hf), m.head_logits(1, hf))


@pytest.mark.parametrize("temperature", [0.7, 1.0, 0.05])
@pytest.mark.parametrize("scale", [0.1, 1.3, 6.0])
def test_typical_stats_match_scipy(temperature, scale):
    rng = np.random.default_rng(int(scale * 10 + temperature * 100))
    z = rng.standard_normal(32000) * scale
    z[:3] = z.max()  # ties at the maximum
    P, H = SP.typical_stats(z, temperature)
    Pref = scipy.special.softmax(z / temperature)
    assert np.allclose(P, Pref, rtol=1e-12, atol=1e-300)
    assert abs(H - scipy.stats.entropy(Pref)) <= 1e-9 * max(1.0, H)
    # bounds: 0 <= H <= log V, with log V for the uniform distribution
    assert 0.0 <= H <= np.log(z.size) + 1e-12
    _, Hu = SP.typical_stats(np.zeros(1000), temperature)
    assert abs(Hu - np.log(1000)) < 1e-12


def _wide_cfg():
    # hd 128, GQA 4:1, d 256: the head_dim/GQA shape class of the 7B/70B models at a width the
    # row-at-a-time oracle finishes in seconds
    return synth.model_cfg("tiny", d_model=256, n_heads=4, n_kv_heads=1, head_dim=128, d_ffn=512, vocab=512)


@pytest.mark.parametrize("mode", ["fp64", "fp32", "bf16"])
@pytest.mark.parametrize("name", ["tiny", "wide"])
def test_forward_rows_equals_forward_row(mode, name):
    cfg = synth.model_cfg("tiny") if name == "tiny" else _wide_cfg()
    W = M.Weights(cfg, n_medusa=3, seed=2)
    m = M.Model(cfg, W, mode)
    s = SP.Session(m, synth.TINY16, 1, 64)
    prompt = synth.prompt_tokens(2, 0, 20, cfg["vocab"])
    s.prefill(0, prompt)
    tok, _ = s.propose(0)
    kv2 = copy.deepcopy(s.kv)
    Z, HF = s.verify(0, tok)
    tr, Lc = s.tree, 20
    keys = [list(range(Lc)) + [Lc + a for a in T.ancestors(tr, n)] + [Lc + n] for n in range(tr.N)]
    Z2, HF2 = m.forward_rows(kv2, 0, tok, [Lc + tr.depth[n] for n in range(tr.N)], [Lc + n for n in range(tr.N)],
                             keys)
    # only the fp64 summation order of the BLAS products differs: within 1e-12 in fp64 mode; the
    # rounded modes agree bitwise unless a value sits within ~1e-16 of a rounding boundary
    tol = 1e-12 if mode == "fp64" else 0.0
    assert np.max(np.abs(np.stack(Z) - Z2)) <= tol * max(1.0, np.abs(Z2).max()) + (1e-6 if mode != "fp64" else 0)
    for li in range(cfg["n_layers"]):
        assert np.max(np.abs(s.kv.K[li] - kv2.K[li])) <= 1e-12 + (1e-6 if mode != "fp64" else 0)


def test_batched_session_matches_rowwise_generation():
    cfg = _wide_cfg()
    W = M.Weights(cfg, n_medusa=3, seed=1)
    prompt = synth.prompt_tokens(1, 0, 24, cfg["vocab"])
    outs = []
    for batched in (False, True):
        s = SP.Session(M.Model(cfg, W, "bf16"), synth.TINY16, 1, 96, batched=batched)
        s.prefill(0, prompt)
        outs.append(s.generate(0, 24)[0])
    assert outs[0] == outs[1]
    assert outs[0] == SP.vanilla_generate(M.Model(cfg, W, "bf16"), prompt, 24)[0]


def test_fp32_weights_timing_variant_close_to_fp64():
    """Weights(dtype=float32): the bench's timing variant computes in fp32 BLAS; its logits stay
    within fp32 rounding of the fp64-arithmetic oracle in the fp32 storage mode."""
    cfg = _wide_cfg()
    res = []
    for dt in (np.float64, np.float32):
        W = M.Weights(cfg, n_medusa=3, seed=5, dtype=dt)
        s = SP.Session(M.Model(cfg, W, "fp32"), synth.TINY16, 1, 64, batched=True)
        s.prefill(0, synth.prompt_tokens(5, 0, 30, cfg["vocab"]))
        Z, _ = s.verify(0, s.propose(0)[0])
        res.append(np.stack(Z))
    assert np.max(np.abs(res[0] - res[1])) < 1e-4
