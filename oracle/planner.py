"""SpecMemo memory-budget planner: Eqs. 1, 3-6 and Algorithm 1
(OptimizerEngine), written out step by step in the paper's order and notation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Memory model, bytes, with precision p bytes per element:
  Eq. 1  Memory_KV      = 2 * h * b * k * d * x * p,  x = n * m          (d restored, reading Q14)
  Eq. 3  Memory_buffers = b*N*w + b*S*l*w + b*S*l*l*w  (elements)
  Eq. 4  Memory_heads   = 0.6 GB * l
  Eq. 5  Memory_base    = B * p
  Eq. 6  Memory_total   = base + heads + KV + buffers * p

Algorithm 1, readings (Q31):
  * AvailMemory(config) = total(config) <= max_memory.
  * ExploreTree(max_memory, min_cache, num_heads): candidate (N, S) trees for num_heads
    levels -- the Medusa V64 tree restricted to depth num_heads, R4-pruned in place to
    N in TREE_SIZES ("Pruned M" of tab:treefeatures), plus the custom (N, S) trees
    of the table's C row at 4 heads -- keeping those that fit, largest N first.
  * The head-reduction loop (garbled in the pseudo-code: it quantizes when the head count
    changed) is read as: take the largest num_heads' in [2, num_heads-1] whose default
    configuration fits; if none does, the next step would be QuantizeBaseModel,
    which the B200 build does not provide (OUT) -> status NEEDS_QUANTIZATION.
  * The returned configuration is the first (largest) fitting candidate.

"b200" accounting (bound to the device instead of the paper's estimates): the KV term is the
bounded cache the library allocates (sm_kv_bytes: x + N scratch slots per sequence), the head
term the real Medusa-1 size l*(d^2 + d + V d)*p, and the buffer term only Eq. 3's first term
-- the B200 path never materialises the S-indexed gathers (terms 2-3), DESIGN.md §6.
"""
from __future__ import annotations

import synth

from . import tree as T

DEFAULT_HEADS = 4
DEFAULT_TREE = (64, 42)                 # Alg. 1 line 3, "(64_nodes, 42_sequences)"
TREE_SIZES = (64, 44, 31, 27, 16, 5)    # mask sizes of fig:maskmodel / tab:treefeatures
CUSTOM_4 = ((64, 56), (44, 37))         # tab:treefeatures, C row, heads = 4
HEAD_GB = 0.6e9                         # Eq. 4

STATUS_DEFAULT, STATUS_PRUNED, STATUS_FEWER_HEADS, STATUS_NEEDS_QUANT = 0, 1, 2, 3


def memory_kv(cfg, b, n, m, p, N=0, accounting="paper"):
    """Eq. 1 (with d), x = n * m; the b200 accounting adds the N tree-scratch slots."""
    x = n * m + (N if accounting == "b200" else 0)
    return 2 * cfg["n_layers"] * b * cfg["n_kv_heads"] * cfg["head_dim"] * x * p


def memory_buffers(b, N, S, l, w, p, accounting="paper"):
    """Eq. 3 (elements) times p (Eq. 6).  b200: only the node-logit term (fp32 logits)."""
    if accounting == "b200":
        return b * N * w * 4
    return (b * N * w + b * S * l * w + b * S * l * l * w) * p


def memory_heads(cfg, l, p, accounting="paper"):
    if accounting == "b200":
        d, V = cfg["d_model"], cfg["vocab"]
        return l * (d * d + d + V * d) * p
    return int(HEAD_GB * l)


def memory_base(cfg, p):
    """Eq. 5: B * p, B = parameters of the base model (layers + embedding + LM head)."""
    d, H, Hkv, hd, F, V, L = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab",
                                                "n_layers"))
    layer = (H + 2 * Hkv) * hd * d + d * H * hd + 3 * F * d + 2 * d
    return (L * layer + 2 * V * d + d) * p


def memory_total(cfg, b, n, m, p, heads, N, S, accounting="paper"):
    """Eq. 6."""
    return (memory_base(cfg, p) + memory_heads(cfg, heads, p, accounting) + memory_kv(cfg, b, n, m, p, N, accounting)
            + memory_buffers(b, N, S, heads, cfg["vocab"], p, accounting))


def explore_tree(cfg, b, n, m, p, heads, max_memory, accounting="paper"):
    """Candidate (N, S) trees for `heads` levels that fit, largest first (reading Q31)."""
    cut = [c for c in synth.V64 if len(c) <= heads]
    base_N = len(cut) + 1
    cands = []
    for N in TREE_SIZES:
        if N <= base_N:
            t = T.build(T.prune_right_to_left(cut, N))
            cands.append((N, T.stats(t)["S"], "pruned"))
    if heads == 4:
        cands += [(N, S, "custom") for N, S in CUSTOM_4]
    cands.sort(key=lambda c: (-c[0], -c[1], c[2]))
    return [c for c in cands if memory_total(cfg, b, n, m, p, heads, c[0], c[1], accounting) <= max_memory]


def optimizer_engine(cfg, b, n, m, p, max_memory, default_heads=DEFAULT_HEADS, accounting="paper"):
    """Algorithm 1.  Returns dict(status, heads, N, S, kind, x, total)."""
    num_heads = default_heads
    N0, S0 = DEFAULT_TREE
    x = n * m                                                              # ComputeMinCache
    if memory_total(cfg, b, n, m, p, num_heads, N0, S0, accounting) <= max_memory:   # AvailMemory
        return dict(status=STATUS_DEFAULT, heads=num_heads, N=N0, S=S0, kind="default", x=x,
                    total=memory_total(cfg, b, n, m, p, num_heads, N0, S0, accounting))
    status = STATUS_PRUNED
    while True:
        configs = explore_tree(cfg, b, n, m, p, num_heads, max_memory, accounting)
        if configs:                                                        # BuildCustomTree + Medusa
            N, S, kind = configs[0]
            return dict(status=status, heads=num_heads, N=N, S=S, kind=kind, x=x,
                        total=memory_total(cfg, b, n, m, p, num_heads, N, S, accounting))
        new_heads = num_heads
        for h in range(num_heads - 1, 1, -1):
            if memory_total(cfg, b, n, m, p, h, N0, S0, accounting) <= max_memory:
                new_heads = h
                break
        if new_heads == num_heads:                                         # QuantizeBaseModel: OUT
            return dict(status=STATUS_NEEDS_QUANT, heads=num_heads, N=0, S=0, kind="none", x=x, total=0)
        num_heads, status = new_heads, STATUS_FEWER_HEADS


def algorithm2(results):
    """Algorithm 2, "SpecMemo for Medusa", in the paper's order:

        results <- {}
        for config in pruned_tree_configs:
            MedusaModel(model, config, attention_tree)
            (acceptance_length, speedup) <- MedusaGenerate(query_count, query_length)
            results <- (config, acceptance_length, speedup)
        return best_config <- Max(results.speedup)

    ``results`` is the list of (config, acceptance_length, speedup) the loop produced (the
    generation runs are the caller's measurement); the maximum is taken over speedup, the first
    maximal entry in loop order wins a tie (reading Q32: the paper names no tie rule)."""
    best = None
    for config, acceptance_length, speedup in results:
        if best is None or speedup > best[2]:
            best = (config, acceptance_length, speedup)
    return best[0]
