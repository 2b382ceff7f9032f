"""Random-init Llama decoder + Medusa-1 heads, one token row at a time (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper names its models (Vicuna-7B P:45, Llama-2-70B-Chat P:6) and builds
on Medusa without restating either architecture.  Conventions are the
public Llama ones (reading Q17): RMSNorm eps 1e-5, RoPE theta 1e4
rotate-half, SiLU-gated MLP, no biases, untied LM head.  The Medusa-1 head is
one ResBlock then an unembedding, ``u_i = U_i (h + SiLU(R_i h + b_i))``; its
size is pinned by Eq. 4 ("0.6 GB * l"): 0.591 GB per fp32 head at
Vicuna-7B shapes (Q6).  Head i predicts tree depth i+1 (P:67 heads =
levels; P:245 level 1 = first head's top-k).

Numeric modes
  "fp64"  -- everything float64 on the bf16-valued generated weights.
  "bf16"  -- float64 arithmetic, rounded to bf16 (RNE) / fp32 exactly at the
             storage points of the rounding contract R0..R10,
             i.e. where the GPU path stores a bf16 or fp32 tensor.
  "fp32"  -- the fp32 parity mode (north star: logits and KV within 1e-4):
             float64 arithmetic rounded to fp32 at every storage point (the
             GPU's fp32 mode keeps activations, K/V and logits in fp32; the
             weights are the same bf16-valued tensors, R0).

Every token row goes through the same ``forward_row`` so that a tree node's
row is bit-identical to the sequential-decoding row of the same token at the
same position with the same keys (invariants I1/I3).
"""
from __future__ import annotations

import math

import numpy as np

import synth


# ----------------------------------------------------------------- rounding
def round_f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def round_bf16(x):
    """float64 -> fp32 (RNE) -> bf16 (RNE), returned as float64 values."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


# ----------------------------------------------------------------- weights
def _w(seed, stream, rows, cols, dtype=np.float64):
    n = rows * cols
    if n <= (1 << 24):
        bits = synth.weight_bits(seed, stream, n)
        return synth.bf16_bits_to_f32(bits).astype(dtype).reshape(rows, cols)
    # large tensors (C2+ widths): synth's C generator, the same values bit for bit
    w = synth.weight_values_f32(seed, stream, n).reshape(rows, cols)
    return w if dtype == np.float32 else w.astype(dtype)


class Weights:
    """All tensors as float64 arrays holding bf16 values (R0).  Layout is the
    PyTorch ``nn.Linear`` one: ``[out_features][in_features]``."""

    def __init__(self, cfg: dict, n_medusa: int, seed: int = 0, medusa_init: bool = False,
                 layers: list[int] | None = None, dtype=np.float64):
        d, H, Hkv, hd, F, V = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab"))
        self.cfg = cfg
        self.seed = seed
        w = lambda stream, r, c_: _w(seed, stream, r, c_, dtype)  # noqa: E731
        self.embed = w(synth.STREAM_EMBED, V, d)
        self.lm_head = w(synth.STREAM_LM_HEAD, V, d)
        self.final_norm = np.ones(d, dtype=dtype)
        self.layers = []
        for li in (range(cfg["n_layers"]) if layers is None else layers):
            s = lambda name: synth.stream_layer(li, name)  # noqa: E731
            self.layers.append(dict(
                attn_norm=np.ones(d, dtype=dtype),
                wq=w(s("wq"), H * hd, d), wk=w(s("wk"), Hkv * hd, d),
                wv=w(s("wv"), Hkv * hd, d), wo=w(s("wo"), d, H * hd),
                mlp_norm=np.ones(d, dtype=dtype),
                wg=w(s("wg"), F, d), wu=w(s("wu"), F, d), wd=w(s("wd"), d, F)))
        self.medusa = []
        for i in range(n_medusa):
            if medusa_init:  # Q18 "Medusa-init": R = 0, U = W_lm
                self.medusa.append(dict(R=np.zeros((d, d), dtype=dtype), beta=np.zeros(d, dtype=dtype),
                                        U=self.lm_head))
            else:
                self.medusa.append(dict(R=w(synth.stream_medusa(i, "R"), d, d), beta=np.zeros(d, dtype=dtype),
                                        U=w(synth.stream_medusa(i, "U"), V, d)))


# ----------------------------------------------------------------- model
class Model:
    def __init__(self, cfg: dict, weights: Weights, mode: str = "bf16"):
        assert mode in ("bf16", "fp32", "fp64")
        self.cfg = cfg
        self.W = weights
        self.mode = mode
        self.d = cfg["d_model"]
        self.H = cfg["n_heads"]
        self.Hkv = cfg["n_kv_heads"]
        self.hd = cfg["head_dim"]
        self.G = self.H // self.Hkv
        self.eps = cfg.get("rms_eps", synth.RMS_EPS)
        self.theta = cfg.get("rope_theta", synth.ROPE_THETA)
        self.n_layers = len(weights.layers)

    # storage points
    def r16(self, x):
        """A bf16 storage point of the rounding contract (fp32 storage in "fp32" mode)."""
        if self.mode == "bf16":
            return round_bf16(x)
        return round_f32(x) if self.mode == "fp32" else np.asarray(x, dtype=np.float64)

    def r32(self, x):
        return round_f32(x) if self.mode != "fp64" else np.asarray(x, dtype=np.float64)

    # building blocks ----------------------------------------------------
    def rmsnorm(self, x, g):
        """y = x / sqrt(mean(x^2) + eps) * g  (Llama RMSNorm)."""
        return x / math.sqrt(float(np.mean(x * x)) + self.eps) * g

    def rms_scale(self, x):
        """rs = 1 / sqrt(mean(x^2) + eps), so that rmsnorm(x, g) = rs * (x * g)."""
        return 1.0 / math.sqrt(float(np.mean(x * x)) + self.eps)

    def rope(self, v, pos):
        """Rotate-half RoPE on each head of v [nh][hd] at integer position pos:
        for i < hd/2, angle = pos * theta^(-2i/hd),
        out[i] = v[i] cos - v[i+hd/2] sin, out[i+hd/2] = v[i+hd/2] cos + v[i] sin."""
        half = self.hd // 2
        i = np.arange(half, dtype=np.float64)
        ang = pos * self.theta ** (-2.0 * i / self.hd)
        c, s = np.cos(ang), np.sin(ang)
        if self.mode != "fp64":  # GPU tables are fp64-built, stored fp32 (R3)
            c, s = round_f32(c), round_f32(s)
        x1, x2 = v[:, :half], v[:, half:]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=1)

    @staticmethod
    def silu(x):
        return x / (1.0 + np.exp(-x))

    def attention(self, q, Kc, Vc):
        """Softmax attention of one query row.  q [H][hd]; Kc, Vc [n][Hkv][hd]
        are the visible keys/values in logical position order.  Scale 1/sqrt(hd);
        q head h reads kv head h // G (GQA)."""
        out = np.zeros((self.H, self.hd))
        scale = 1.0 / math.sqrt(self.hd)
        for h in range(self.H):
            kv = h // self.G
            s = Kc[:, kv, :] @ q[h] * scale
            p = np.exp(s - s.max())
            p = p / p.sum()
            out[h] = p @ Vc[:, kv, :]
        return out

    # one token row --------------------------------------------------------
    def forward_row(self, kv, seq: int, tok: int, pos: int, slot: int, key_slots: list[int]):
        """Run token ``tok`` at position ``pos`` through all layers.

        Writes its K/V into cache slot ``slot`` of sequence ``seq`` and attends
        to the cache slots ``key_slots`` (logical position order; must include
        ``slot``).  Returns (z, hf): fp32 logits [V] and final-normed hidden [d].
        """
        W = self.W
        x = self.r16(W.embed[tok]).copy()                               # R1 (bf16 row -> fp32 residual)
        for li, Lw in enumerate(W.layers):
            # R2 (deferred RMSNorm): the stored GEMM input is x*g; the projection is scaled by
            # rs = 1/sqrt(mean(x^2) + eps) afterwards -- rmsnorm(x, g) @ W^T = rs * ((x*g) @ W^T)
            h, rs = self.r16(x * Lw["attn_norm"]), self.r32(self.rms_scale(x))
            q = (rs * (Lw["wq"] @ h)).reshape(self.H, self.hd)          # R3 fp32 accumulate
            k = (rs * (Lw["wk"] @ h)).reshape(self.Hkv, self.hd)
            v = (rs * (Lw["wv"] @ h)).reshape(self.Hkv, self.hd)
            q = self.r16(self.rope(self.r32(q), pos))
            k = self.r16(self.rope(self.r32(k), pos))
            v = self.r16(v)
            kv.K[li][seq][:, slot, :] = k
            kv.V[li][seq][:, slot, :] = v
            Kc = kv.K[li][seq][:, key_slots, :].transpose(1, 0, 2)
            Vc = kv.V[li][seq][:, key_slots, :].transpose(1, 0, 2)
            o = self.r16(self.attention(q, Kc, Vc).reshape(-1))         # R4
            x = self.r32(x + self.r32(Lw["wo"] @ o))                    # R5 (fp32 residual)
            h2, rs2 = self.r16(x * Lw["mlp_norm"]), self.r32(self.rms_scale(x))      # R2 (deferred)
            a = self.r16(self.silu(self.r32(rs2 * (Lw["wg"] @ h2))) * self.r32(rs2 * (Lw["wu"] @ h2)))  # R6
            x = self.r32(x + self.r32(Lw["wd"] @ a))                    # R7
        hf = self.r16(self.rmsnorm(x, W.final_norm))                    # R8
        z = self.r32(W.lm_head @ hf)                                    # R9
        return z, hf

    def forward_rows(self, kv, seq: int, toks, poss, slots, key_lists):
        """``forward_row`` for several token rows at once, layer by layer: the same
        arithmetic and storage points, with the projections of all rows done as one
        matrix product per weight (BLAS; only the fp64 summation order differs from
        the row-at-a-time routine).  In each layer every row's K/V is written before
        any row attends, so a row may attend to slots of rows earlier in the same
        call (tree ancestors, causal prefill tokens).  Returns (Z [n][V], HF [n][d]).

        The weights' array dtype is the arithmetic type: float64 (default, the parity
        oracle) or float32 (``Weights(dtype=np.float32)``: the timing variant of
        SURVEY §8.d.5 for the bench's cpu_baseline, fp32 batched BLAS)."""
        W = self.W
        dt = W.embed.dtype
        c = lambda a: np.asarray(a, dtype=dt)  # noqa: E731  (storage rounding works in float64)
        n = len(toks)
        toks = [int(t) for t in toks]
        X = c(self.r16(W.embed[toks]))                                  # R1
        for li, Lw in enumerate(W.layers):
            h = c(self.r16(X * Lw["attn_norm"]))                        # R2 (deferred RMSNorm)
            rs = c(self.r32(self._rms_scale_rows(X)))[:, None]
            q = (rs * (h @ Lw["wq"].T)).reshape(n, self.H, self.hd)    # R3
            k = (rs * (h @ Lw["wk"].T)).reshape(n, self.Hkv, self.hd)
            v = (rs * (h @ Lw["wv"].T)).reshape(n, self.Hkv, self.hd)
            Q = np.empty_like(q)
            for i in range(n):
                Q[i] = c(self.r16(self.rope(self.r32(q[i]), poss[i])))
                kv.K[li][seq][:, slots[i], :] = self.r16(self.rope(self.r32(k[i]), poss[i]))
                kv.V[li][seq][:, slots[i], :] = self.r16(v[i])
            O = c(self.r16(self._attention_rows(Q, kv.K[li][seq], kv.V[li][seq], key_lists)))  # R4
            X = c(self.r32(X + self.r32(O @ Lw["wo"].T)))              # R5
            h2 = c(self.r16(X * Lw["mlp_norm"]))                        # R2 (deferred)
            rs2 = c(self.r32(self._rms_scale_rows(X)))[:, None]
            A = c(self.r16(self.silu(self.r32(rs2 * (h2 @ Lw["wg"].T))) * self.r32(rs2 * (h2 @ Lw["wu"].T))))  # R6
            X = c(self.r32(X + self.r32(A @ Lw["wd"].T)))              # R7
        X64 = np.asarray(X, dtype=np.float64)
        HF = c(self.r16(X64 / np.sqrt(np.mean(X64 * X64, axis=1) + self.eps)[:, None] * W.final_norm))  # R8
        Z = self.r32(HF @ W.lm_head.T)                                  # R9
        return Z, HF

    def _attention_rows(self, Q, Kl, Vl, key_lists):
        """``attention`` for several rows: Q [n][H][hd]; Kl, Vl [Hkv][cap][hd] (one sequence's
        cache layer).  The key slots shared by every row (the common prefix 0..c-1: the committed
        cache) are scored for all rows in one product per kv head; each row's remaining slots
        (its tree ancestors and itself, or its causal chunk tokens) are scored on their own; the
        softmax runs over the row's full key list in the same logical order, and P.V is the sum
        of the two parts.  Returns O [n][H * hd]."""
        n = Q.shape[0]
        c = min(len(k) for k in key_lists)
        for k in key_lists:                       # longest prefix 0, 1, ..., c-1 shared by all rows
            a = np.asarray(k[:c])
            bad = np.flatnonzero(a != np.arange(a.size))
            c = int(bad[0]) if bad.size else c
        scale = 1.0 / math.sqrt(self.hd)
        O = np.zeros((n, self.H, self.hd), dtype=Q.dtype)
        for h in range(self.Hkv):
            hs = slice(h * self.G, (h + 1) * self.G)
            Kh, Vh = Kl[h], Vl[h]
            Sp = (Q[:, hs, :].reshape(n * self.G, self.hd) @ Kh[:c].T).reshape(n, self.G, c) * scale
            for i in range(n):
                rest = key_lists[i][c:]
                Sr = (Q[i, hs, :] @ Kh[rest].T) * scale                     # [G][r]
                S = np.concatenate([Sp[i], Sr], axis=1)
                p = np.exp(S - S.max(axis=1, keepdims=True))
                p = p / p.sum(axis=1, keepdims=True)
                O[i, hs, :] = p[:, :c] @ Vh[:c] + p[:, c:] @ Vh[rest]
        return O.reshape(n, self.H * self.hd)

    def _rms_scale_rows(self, X):
        """rs per row = 1 / sqrt(mean(x^2) + eps) (as rms_scale, in float64)."""
        X = np.asarray(X, dtype=np.float64)
        return 1.0 / np.sqrt(np.mean(X * X, axis=1) + self.eps)

    def head_logits(self, i: int, hf):
        """Medusa-1 head i: u = U_i (hf + SiLU(R_i hf + beta_i))   (R10)."""
        Hw = self.W.medusa[i]
        dt = Hw["U"].dtype
        hf = np.asarray(hf, dtype=dt)
        r = np.asarray(self.r16(hf + self.silu(self.r32(Hw["R"] @ hf + Hw["beta"]))), dtype=dt)
        return self.r32(Hw["U"] @ r)


class KVCache:
    """Bounded KV cache (Eq. 1): per layer [b][Hkv][x + N][hd]; the last
    N slots of each sequence are the tree scratch (reading Q14)."""

    def __init__(self, n_layers: int, batch: int, n_kv_heads: int, capacity: int, head_dim: int, dtype=np.float64):
        self.capacity = capacity
        self.K = [np.zeros((batch, n_kv_heads, capacity, head_dim), dtype=dtype) for _ in range(n_layers)]
        self.V = [np.zeros((batch, n_kv_heads, capacity, head_dim), dtype=dtype) for _ in range(n_layers)]


def argmax_lowest(z) -> int:
    """argmax with ties broken by the lowest index (reading Q9)."""
    z = np.asarray(z)
    return int(np.flatnonzero(z == z.max())[0])


def topk_desc(u, k: int) -> list[int]:
    """Top-k indices ordered by (value desc, index asc) (reading Q20)."""
    u = np.asarray(u)
    order = sorted(range(len(u)), key=lambda i: (-u[i], i))
    return order[:k]
