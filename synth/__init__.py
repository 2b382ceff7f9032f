"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no model, no attention, no
acceptance, no rounding contract).  It only defines *inputs*:

* the counter-hash generator ``h(seed, stream, i) = splitmix64(seed ^ stream<<40 ^ i)``
   and the weight-value map built on it;
* prompt tokens / lengths for the synthetic MT-Bench-shaped workload;
* the static Medusa tree choice lists (configuration data);
* the benchmark configurations C1..C5 (BASELINE.json ``configs``).

The CUDA library re-implements the same generator on the device
(``paper_2506_01986_b200/csrc/gen.cu``); tests check the two bit for bit.
Neither the oracle nor the CUDA path import each other; both may import this.
"""
from __future__ import annotations

import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# 0.02 * sqrt(3) rounded to fp32: uniform(-a, a) has std a/sqrt(3) = 0.02,
# HF ``initializer_range``.
WEIGHT_AMPLITUDE_F32 = np.float32(0.02 * np.sqrt(3.0))


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vigna's splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def counter_hash(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """h(seed, stream, i) = splitmix64(seed ^ (stream << 40) ^ i)."""
    base = np.uint64((int(seed) ^ (int(stream) << 40)) & 0xFFFFFFFFFFFFFFFF)
    return splitmix64(base ^ np.asarray(idx, dtype=np.uint64))


def _f32_to_bf16_bits_input(x: np.ndarray) -> np.ndarray:
    """RNE fp32 -> bf16 bit pattern, used ONLY to quantise generated inputs."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return u.astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def weight_bits(seed: int, stream: int, numel: int, start: int = 0) -> np.ndarray:
    """bf16 bit patterns of ``numel`` generated weights (flat row-major order).

    w = bf16_rne( f32( f32((k - 2^23) * 2^-23) * f32(0.02*sqrt(3)) ) ),  k = h >> 40.
    Every step is exact or a single IEEE fp32 RNE operation, so the device
    generator reproduces it bit for bit.
    """
    idx = np.arange(start, start + numel, dtype=np.uint64)
    k = (counter_hash(seed, stream, idx) >> np.uint64(40)).astype(np.int64) - (1 << 23)
    v = k.astype(np.float32) * np.float32(2.0 ** -23)
    w = v * WEIGHT_AMPLITUDE_F32
    return _f32_to_bf16_bits_input(w)


_GEN = None


def _gen_lib():
    """synth/_gen.c compiled with gcc (-fopenmp) next to it on first use (or by build())."""
    global _GEN
    if _GEN is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, so = os.path.join(here, "_gen.c"), os.path.join(here, "_gen.so")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            tmp = f"{so}.{os.getpid()}.tmp"
            subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, src], check=True)
            os.replace(tmp, so)
        lib = ctypes.CDLL(so)
        lib.synth_weight_values_f32.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_float, ctypes.c_void_p]
        _GEN = lib
    return _GEN


def weight_values_f32(seed: int, stream: int, numel: int, start: int = 0) -> np.ndarray:
    """``bf16_bits_to_f32(weight_bits(...))`` from the C generator (synth/_gen.c, OpenMP): the same
    values bit for bit, for full-size models."""
    out = np.empty(numel, dtype=np.float32)
    _gen_lib().synth_weight_values_f32(int(seed) & 0xFFFFFFFFFFFFFFFF, int(stream), int(start), int(numel),
                                       float(WEIGHT_AMPLITUDE_F32), out.ctypes.data)
    return out


def normal_bits(seed: int, stream: int, numel: int) -> np.ndarray:
    """bf16 bits of approximately N(0,1) values (sum of 4 uniforms, scaled), for
    the K1 sweep's Q/K/V.  Exact fp32 ops only."""
    idx = np.arange(numel, dtype=np.uint64)
    h = counter_hash(seed, stream, idx)
    acc = np.zeros(numel, dtype=np.float32)
    for sh in (0, 16, 32, 48):
        k = ((h >> np.uint64(sh)) & np.uint64(0xFFFF)).astype(np.int64) - (1 << 15)
        acc = acc + k.astype(np.float32) * np.float32(2.0 ** -15)
    # var of U(-1,1) = 1/3 -> sum of 4 has var 4/3; scale by sqrt(3)/2
    return _f32_to_bf16_bits_input(acc * np.float32(0.8660254037844386))


# --------------------------------------------------------------------------
# Weight stream registry (which stream id generates which tensor).
# --------------------------------------------------------------------------
STREAM_EMBED = 1
STREAM_LM_HEAD = 2


def stream_layer(layer: int, which: str) -> int:
    off = {"wq": 0, "wk": 1, "wv": 2, "wo": 3, "wg": 4, "wu": 5, "wd": 6}[which]
    return 16 + 16 * layer + off


def stream_medusa(head: int, which: str) -> int:
    off = {"R": 0, "U": 1}[which]
    return (1 << 20) + 8 * head + off


def stream_prompt(seq: int, turn: int = 0) -> int:
    return (1 << 24) + 1024 * turn + seq


STREAM_PROMPT_LEN = (1 << 25)


def prompt_tokens(seed: int, seq: int, n: int, vocab: int, turn: int = 0) -> np.ndarray:
    """Prompt token ids: h(seed, prompt(seq,turn), i) mod V."""
    h = counter_hash(seed, stream_prompt(seq, turn), np.arange(n, dtype=np.uint64))
    return (h % np.uint64(vocab)).astype(np.int32)


def prompt_length(seed: int, seq: int, turn: int = 0) -> int:
    """MT-Bench-length by assumption: 32 + h mod 129 -> 32..160."""
    h = counter_hash(seed, STREAM_PROMPT_LEN, np.array([1024 * turn + seq], dtype=np.uint64))
    return int(32 + int(h[0] % np.uint64(129)))


# --------------------------------------------------------------------------
# Static Medusa trees (path lists, root implicit).  Configuration data.
# --------------------------------------------------------------------------
# Medusa ``vicuna_7b_stage2`` choice list.  The paper's
# "default_tree <- (64_nodes, 42_sequences)" (Alg. 1) and the
# per-depth features 10/11, 25/34, 39/57, 42/64 (tab:treefeatures
# "M" row) pin it; tests/golden/tree_features.json checks those numbers.
V64 = [
    [0], [0, 0], [1], [0, 1], [0, 0, 0], [1, 0], [2], [0, 2], [0, 0, 1], [0, 3], [3], [0, 1, 0], [2, 0], [4],
    [0, 0, 2], [0, 4], [1, 1], [1, 0, 0], [0, 0, 0, 0], [5], [0, 0, 3], [0, 5], [0, 2, 0], [3, 0], [0, 1, 1],
    [0, 6], [6], [0, 7], [0, 0, 4], [4, 0], [1, 2], [0, 8], [7], [0, 3, 0], [0, 0, 0, 1], [0, 0, 5], [2, 1],
    [0, 0, 6], [1, 0, 1], [0, 0, 1, 0], [2, 0, 0], [5, 0], [0, 9], [0, 1, 2], [8], [0, 4, 0], [0, 2, 1],
    [1, 3], [0, 0, 7], [0, 0, 0, 2], [0, 0, 8], [1, 1, 0], [0, 1, 0, 0], [6, 0], [9], [0, 1, 3], [0, 0, 0, 3],
    [1, 0, 2], [0, 5, 0], [3, 1], [0, 0, 2, 0], [7, 0], [1, 4],
]

# C1 tree: the first 15 choices of V64 -> (16 nodes, 10 leaves, 1-5-6-4), depth 3
# (SURVEY §8.c.4 Q2).
TINY16 = V64[:15]


def full_prefix_tree(arity: int, n_nodes: int) -> list[list[int]]:
    """First ``n_nodes-1`` nodes of the complete ``arity``-ary tree in (depth,
    lexicographic rank path) order (sweep trees of SURVEY §8.d.1 C5)."""
    out: list[list[int]] = []
    level = [[]]
    while len(out) < n_nodes - 1:
        nxt = []
        for p in level:
            for r in range(arity):
                nxt.append(p + [r])
        for p in nxt:
            if len(out) == n_nodes - 1:
                break
            out.append(p)
        level = nxt
    return out


SWEEP_TREES = {
    16: TINY16,
    32: V64[:31],
    64: V64,
    128: full_prefix_tree(10, 128),
    256: full_prefix_tree(10, 256),
}

CHAIN = lambda depth: [[0] * i for i in range(1, depth + 1)]  # noqa: E731


# --------------------------------------------------------------------------
# Model shapes (public Llama/Vicuna configs).
# --------------------------------------------------------------------------
MODELS = {
    "tiny": dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=4, head_dim=16, d_ffn=256, vocab=256),
    "vicuna7b": dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=32, head_dim=128, d_ffn=11008, vocab=32000),
    "vicuna13b": dict(n_layers=40, d_model=5120, n_heads=40, n_kv_heads=40, head_dim=128, d_ffn=13824, vocab=32000),
    "llama70b": dict(n_layers=80, d_model=8192, n_heads=64, n_kv_heads=8, head_dim=128, d_ffn=28672, vocab=32000),
}
RMS_EPS = 1e-5
ROPE_THETA = 10000.0
TOPK = 10
TYPICAL = dict(temperature=0.7, eps=0.09, alpha=0.3)  # Medusa defaults (unpinned, Q10)


def model_cfg(name: str, **over) -> dict:
    c = dict(MODELS[name])
    c.update(rms_eps=RMS_EPS, rope_theta=ROPE_THETA)
    c.update(over)
    return c
