"""Pins for oracle/model.py and synth (no GPU).

The model's conventions are pinned against an independent implementation
(HuggingFace ``LlamaForCausalLM`` in float64), closed-form RoPE/RMSNorm
properties, torch SDPA and torch's bf16 conversion -- not against itself."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import model as M


# ----------------------------------------------------------------- synth
def test_splitmix64_reference_vectors():
    """Published splitmix64 outputs (seed 0 -> 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4;
    seed 1234567 -> 6457827717110365317)."""
    z = synth.splitmix64(np.array([0, 0x9E3779B97F4A7C15, 1234567], dtype=np.uint64))
    assert [int(v) for v in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 6457827717110365317]


def test_weight_generator_distribution():
    bits = synth.weight_bits(0, 5, 1 << 16)
    w = synth.bf16_bits_to_f32(bits).astype(np.float64)
    assert abs(w.std() - 0.02) < 5e-4
    assert abs(w.mean()) < 5e-4
    assert np.abs(w).max() <= 0.02 * math.sqrt(3) * (1 + 2 ** -8)


# ----------------------------------------------------------------- rounding
def test_round_bf16_matches_torch_rne():
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-6, 6, 20000),
                        # exact ties: fp32 values whose low 16 bits are 0x8000
                        (np.arange(1000, dtype=np.uint32) << 16 | 0x8000).view(np.float32).astype(np.float64)[1:]
                        ])
    x = x[np.isfinite(x)]
    ref = torch.tensor(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(M.round_bf16(x), ref)


# ----------------------------------------------------------------- building blocks
def _tiny(**over):
    cfg = synth.model_cfg("tiny", **over)
    W = M.Weights(cfg, n_medusa=3, seed=0)
    return cfg, W


def test_rmsnorm_closed_forms():
    cfg, W = _tiny()
    m = M.Model(cfg, W, "fp64")
    c = np.full(64, 3.7)
    assert np.allclose(m.rmsnorm(c, np.ones(64)), 3.7 / math.sqrt(3.7 ** 2 + 1e-5))
    x = np.random.default_rng(0).standard_normal(64)
    y = m.rmsnorm(x, np.ones(64))
    assert abs(np.sqrt(np.mean(y * y)) - 1.0) < 1e-5          # unit RMS up to eps
    assert np.allclose(m.rmsnorm(1000 * x, np.ones(64)), y, atol=1e-9)


def test_rope_rotation_properties():
    cfg, W = _tiny()
    m = M.Model(cfg, W, "fp64")
    rng = np.random.default_rng(2)
    q, k = rng.standard_normal((4, 16)), rng.standard_normal((4, 16))
    assert np.allclose(m.rope(q, 0), q)                                   # identity at pos 0
    assert np.allclose(np.linalg.norm(m.rope(q, 37), axis=1), np.linalg.norm(q, axis=1))
    d1 = np.sum(m.rope(q, 5) * m.rope(k, 3), axis=1)                     # relative-position property
    d2 = np.sum(m.rope(q, 1005) * m.rope(k, 1003), axis=1)
    assert np.allclose(d1, d2, atol=1e-9)
    # rotate-half pairing: dims (i, i + hd/2) rotate by pos * theta^(-2i/hd)
    e = np.zeros((1, 16)); e[0, 1] = 1.0
    ang = 7 * 10000.0 ** (-2.0 / 16)
    r = m.rope(e, 7)[0]
    assert np.isclose(r[1], math.cos(ang)) and np.isclose(r[9], math.sin(ang))


def test_attention_matches_torch_sdpa_gqa():
    cfg, W = _tiny(n_heads=4, n_kv_heads=2)
    m = M.Model(cfg, W, "fp64")
    rng = np.random.default_rng(3)
    q = rng.standard_normal((4, 16))
    K, V = rng.standard_normal((9, 2, 16)), rng.standard_normal((9, 2, 16))
    got = m.attention(q, K, V)
    qt = torch.tensor(q)[None, :, None, :]
    Kt = torch.tensor(K).permute(1, 0, 2).repeat_interleave(2, dim=0)[None]
    Vt = torch.tensor(V).permute(1, 0, 2).repeat_interleave(2, dim=0)[None]
    ref = torch.nn.functional.scaled_dot_product_attention(qt, Kt, Vt)[0, :, 0, :].numpy()
    assert np.allclose(got, ref, atol=1e-12)


# ----------------------------------------------------------------- whole model vs HF Llama
def _hf_llama(cfg, W):
    from transformers import LlamaConfig, LlamaForCausalLM
    hc = LlamaConfig(vocab_size=cfg["vocab"], hidden_size=cfg["d_model"], intermediate_size=cfg["d_ffn"],
                     num_hidden_layers=cfg["n_layers"], num_attention_heads=cfg["n_heads"],
                     num_key_value_heads=cfg["n_kv_heads"], head_dim=cfg["head_dim"], rms_norm_eps=1e-5,
                     rope_theta=10000.0, max_position_embeddings=4096, tie_word_embeddings=False,
                     attention_bias=False, mlp_bias=False)
    hf = LlamaForCausalLM(hc).double().eval()
    t = lambda a: torch.tensor(a, dtype=torch.float64)  # noqa: E731
    sd = {"model.embed_tokens.weight": t(W.embed), "lm_head.weight": t(W.lm_head), "model.norm.weight": t(W.final_norm)}
    for i, L in enumerate(W.layers):
        p = f"model.layers.{i}."
        sd.update({p + "self_attn.q_proj.weight": t(L["wq"]), p + "self_attn.k_proj.weight": t(L["wk"]),
                   p + "self_attn.v_proj.weight": t(L["wv"]), p + "self_attn.o_proj.weight": t(L["wo"]),
                   p + "mlp.gate_proj.weight": t(L["wg"]), p + "mlp.up_proj.weight": t(L["wu"]),
                   p + "mlp.down_proj.weight": t(L["wd"]), p + "input_layernorm.weight": t(L["attn_norm"]),
                   p + "post_attention_layernorm.weight": t(L["mlp_norm"])})
    missing, unexpected = hf.load_state_dict(sd, strict=False)
    assert not [k for k in missing if "rotary" not in k] and not unexpected
    return hf


@pytest.mark.parametrize("over", [{}, {"n_kv_heads": 2}])
def test_forward_rows_match_hf_llama(over):
    """The oracle's row-at-a-time decode (fp64 mode) reproduces HF Llama's full
    causal forward: pins RMSNorm, rotate-half RoPE, GQA, SiLU-gated MLP, untied
    LM head.  HF builds cos/sin in fp32, hence the 1e-6 tolerance (logit std ~0.16)."""
    cfg, W = _tiny(**over)
    hf = _hf_llama(cfg, W)
    m = M.Model(cfg, W, "fp64")
    toks = synth.prompt_tokens(7, 0, 24, cfg["vocab"])
    kv = M.KVCache(cfg["n_layers"], 1, cfg["n_kv_heads"], 32, cfg["head_dim"])
    ours = np.stack([m.forward_row(kv, 0, int(t), i, i, list(range(i + 1)))[0] for i, t in enumerate(toks)])
    with torch.no_grad():
        ref = hf(torch.tensor(toks[None], dtype=torch.long)).logits[0].numpy()
    assert np.max(np.abs(ours - ref)) < 1e-6


def test_bf16_mode_close_to_fp64():
    cfg, W = _tiny()
    toks = synth.prompt_tokens(3, 0, 16, cfg["vocab"])
    outs = {}
    for mode in ("fp64", "bf16"):
        m = M.Model(cfg, W, mode)
        kv = M.KVCache(cfg["n_layers"], 1, cfg["n_kv_heads"], 32, cfg["head_dim"])
        outs[mode] = np.stack([m.forward_row(kv, 0, int(t), i, i, list(range(i + 1)))[0] for i, t in enumerate(toks)])
    assert np.max(np.abs(outs["fp64"] - outs["bf16"])) < 2e-2
    assert np.max(np.abs(outs["fp64"] - outs["bf16"])) > 0   # rounding really happens


def test_fp32_mode_matches_hf_llama_float32():
    """fp32 parity mode (north star: 1e-4): the oracle's fp32-storage rows agree
    with an independent float32 forward (HF Llama cast to float32) and with the
    fp64 reference far inside 1e-4, while the rounding is real (differs from fp64)."""
    cfg, W = _tiny(n_kv_heads=2)
    toks = synth.prompt_tokens(5, 0, 20, cfg["vocab"])
    hf = _hf_llama(cfg, W).float()
    with torch.no_grad():
        ref32 = hf(torch.tensor(toks[None], dtype=torch.long)).logits[0].double().numpy()
    outs = {}
    for mode in ("fp64", "fp32"):
        m = M.Model(cfg, W, mode)
        kv = M.KVCache(cfg["n_layers"], 1, cfg["n_kv_heads"], 32, cfg["head_dim"])
        outs[mode] = np.stack([m.forward_row(kv, 0, int(t), i, i, list(range(i + 1)))[0] for i, t in enumerate(toks)])
    assert np.max(np.abs(outs["fp32"] - ref32)) < 1e-5
    assert np.max(np.abs(outs["fp32"] - outs["fp64"])) < 1e-5
    assert np.max(np.abs(outs["fp32"] - outs["fp64"])) > 0
    assert np.all(outs["fp32"] == outs["fp32"].astype(np.float32))   # stored as fp32 (R9)


def test_medusa_head_special_case():
    """R = 0, beta = 0 ("Medusa-init", reading Q18): u = U hf; with U = W_lm the
    head logits equal the base logits (SiLU(0) = 0)."""
    cfg = synth.model_cfg("tiny")
    W = M.Weights(cfg, n_medusa=2, seed=0, medusa_init=True)
    for mode in ("fp64", "bf16"):
        m = M.Model(cfg, W, mode)
        kv = M.KVCache(cfg["n_layers"], 1, cfg["n_kv_heads"], 8, cfg["head_dim"])
        z, hf = m.forward_row(kv, 0, 5, 0, 0, [0])
        assert np.array_equal(m.head_logits(1, hf), z)


def test_medusa_head_definition_random():
    cfg, W = _tiny()
    m = M.Model(cfg, W, "fp64")
    hf = np.random.default_rng(4).standard_normal(64)
    R, U = W.medusa[0]["R"], W.medusa[0]["U"]
    t = torch.tensor(hf)
    ref = torch.tensor(U) @ (t + torch.nn.functional.silu(torch.tensor(R) @ t))
    assert np.allclose(m.head_logits(0, hf), ref.numpy(), atol=1e-12)


def test_topk_and_argmax_ties():
    u = np.array([0.5, 0.9, 0.9, -1.0, 0.5, 0.9])
    assert M.topk_desc(u, 4) == [1, 2, 5, 0]
    assert M.topk_desc(u, 4) == list(np.lexsort((np.arange(6), -u))[:4])
    assert M.argmax_lowest(u) == 1


def test_c_weight_generator_matches_numpy():
    """synth/_gen.c (full-size models) reproduces synth.weight_bits bit for bit."""
    for seed, stream, n, start in [(0, 5, 1 << 16, 0), (3, 123456, 100000, (1 << 33) + 17),
                                   (1, synth.stream_layer(31, "wd"), 70001, 5 * 10 ** 9)]:
        a = synth.bf16_bits_to_f32(synth.weight_bits(seed, stream, n, start=start))
        b = synth.weight_values_f32(seed, stream, n, start=start)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
