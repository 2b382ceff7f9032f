#!/usr/bin/env python
"""Benchmark of the B200 Medusa tree-verification hot path (SpecMemo, 2506.01986).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1 line): BASELINE.json configs[1] = C2, Vicuna-7B-shaped random-init
Llama + 4 Medusa-1 heads, the 64-node / 42-leaf Medusa tree, batch 1, KV cache
bounded to x = 2048 (+64 tree-scratch slots), greedy acceptance.  One step = one
full pass a1..a5 (propose, verify forward of 64 nodes through 32 layers + LM
head, acceptance, compaction, heads + top-k) = one sm_step graph replay.
Under torchrun (N>1): the bs=1 configs (C1-C3) run one independent replica per
rank ("scaling": "weak"; the bs=1 7B/13B step does not need to shard); C4 (70B
shape, bs=10) runs tensor-parallel over the N ranks ("scaling": "strong": the
same 10 sequences, 1/N of the weights and kv heads per GPU), exchanging through
peer memory (CUDA IPC handles swapped over torch.distributed).

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle
(oracle/, numpy fp64) on the host cores on a bounded sample of the same step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "decode tokens/s (bs=1 and bs=10) and tree-attn HBM GB/s vs B200 peak"
X_BOUND = 2048
N_MEDUSA = 4


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained"),
                    src="MEASURED_PEAKS.json (measured)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="B200_PROFILING.md fallback")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(device)], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append(dict(sm=float(parts[0]), smax=float(parts[1]), pw=float(parts[2]), hw=parts[3],
                                 hwt=parts[4], swt=parts[5], pcap=parts[6], util=float(parts[7])))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        load = [r for r in rows if r["util"] > 50] or rows
        reasons = set()
        for r in load:
            for k, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"), ("swt", "sw_thermal_slowdown"),
                            ("pcap", "sw_power_cap")):
                if r[k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in load), "sm_max_mhz": max(r["smax"] for r in rows),
                "reasons": sorted(reasons), "samples": len(load)}


# ------------------------------------------------------------------ distributed plumbing
def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def _reduce(v: float, world: int, op: str) -> float:
    """All-reduce one scalar over the job (max of per-rank device times, sum of
    per-rank token counts).  NCCL on the GPU box; gloo (CPU tensors) in tests."""
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def reduce_max(v: float, world: int) -> float:
    return _reduce(v, world, "max")


def reduce_sum(v: float, world: int) -> float:
    return _reduce(v, world, "sum")


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def exchange_handles(handle: bytes, world: int) -> list:
    """All ranks' opaque handles, indexed by rank (torch.distributed plumbing)."""
    if world == 1:
        return [handle]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, handle)
    return out


def peer_syms(sm, sym, world: int, rank: int) -> list:
    """Device pointers of every rank's symmetric TP buffer, mapped in this process."""
    hs = exchange_handles(sm.ipc_handle(sym), world)
    return [sym.data_ptr() if q == rank else sm.ipc_open(hs[q]) for q in range(world)]


# ------------------------------------------------------------------ algorithmic work of one C2 step
def step_bytes(cfg: dict, N: int, Lc: float, b: int = 1, n_medusa: int = N_MEDUSA, tau: float = 1.0) -> float:
    """weights (layers + LM head + heads) + KV read + tree KV write + compaction."""
    d, H, Hkv, hd, F, V, L = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab",
                                                "n_layers"))
    w_layers = L * ((H + 2 * Hkv) * hd * d + d * H * hd + 3 * F * d) * 2
    w_lm = V * d * 2
    w_heads = n_medusa * (d * d + V * d) * 2
    kv_read = b * 2 * L * Hkv * hd * 2 * Lc
    kv_write = b * N * 2 * L * Hkv * hd * 2
    compact = b * 2 * (tau - 1) * 2 * L * Hkv * hd * 2
    return w_layers + w_lm + w_heads + kv_read + kv_write + compact


def step_flops(cfg: dict, tree_depths, Lc: float, b: int = 1, n_medusa: int = N_MEDUSA) -> float:
    """2 b N (P_layers + P_lm) + 2 b P_heads + 4 H hd L b (N Lc + sum_n (depth_n + 1)),
    the tree part of attention counted sparse (each node sees its ancestors and itself)."""
    d, H, Hkv, hd, F, V, L = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab",
                                                "n_layers"))
    N = len(tree_depths)
    p_layers = L * ((H + 2 * Hkv) * hd * d + d * H * hd + 3 * F * d)
    p_heads = n_medusa * (d * d + V * d)
    return (2 * b * N * (p_layers + V * d) + 2 * b * p_heads
            + 4 * H * hd * L * b * (N * Lc + sum(int(x) + 1 for x in tree_depths)))


def attn_bytes(cfg: dict, N: int, Lc: float, b: int = 1) -> float:
    """K1 per step (all layers): K/V of [0, Lc) + tree slots, read once; Q in, O out."""
    H, Hkv, hd, L = (cfg[k] for k in ("n_heads", "n_kv_heads", "head_dim", "n_layers"))
    return L * b * (Hkv * (Lc + N) * hd * 2 * 2 + 2 * N * H * hd * 2)


# ------------------------------------------------------------------ workloads (BASELINE.json configs)
WORKLOADS = {
    "c2": dict(model="vicuna7b", n_medusa=4, tree="V64", batch=1, x=2048, mode="greedy",
               desc="C2: Vicuna-7B-shaped Llama + 4 Medusa-1 heads (random init), Medusa V64 tree (64 nodes, "
                    "42 leaves), bs=1 per GPU, KV bounded to x=2048 (+64 scratch), greedy"),
    "c1": dict(model="tiny", n_medusa=3, tree="TINY16", batch=1, x=64, mode="greedy", prompt=32,
               desc="C1: tiny random-init Llama (2 layers, d=64, 4 heads, V=256) + 3 Medusa heads, 16-node tree, "
                    "bs=1, 32-token prompt; KV x=64 in the parity tests, raised here to 32 + (l+1) x steps so every "
                    "timed step emits"),
    "c3": dict(model="vicuna13b", n_medusa=4, tree="V64", batch=1, x=2304, mode="typical", turns=8, gen=128,
               desc="C3: Vicuna-13B-shaped + 4 Medusa heads, V64 tree, bs=1, an 8-turn MT-Bench-length chat: "
                    "turn t = prefill of P_t = 32 + h mod 129 prompt tokens, then 128 generated tokens (typical "
                    "acceptance T=0.7 eps=0.09 alpha=0.3); KV bounded to x = sum_t (P_t + 128) (+64 scratch)"),
    "c4v64": dict(model="llama70b", n_medusa=4, tree="V64", batch=10, x=416, mode="greedy", tp=True,
                  desc="C4 with the paper's default tree: Llama-2-70B-shaped (GQA 64/8) + 4 Medusa heads, V64 tree "
                       "(64 nodes), bs=10 ragged prompts of 32-160 tokens, KV bounded to 416 (+64), greedy; M = 640 "
                       "token rows per verify (tensor-bound); tensor parallel over the N GPUs"),
    "c4": dict(model="llama70b", n_medusa=3, tree="TINY16", batch=10, x=416, mode="greedy", tp=True,
               desc="C4: Llama-2-70B-shaped (GQA 64/8) + 3 Medusa heads, 16-node tree, bs=10 ragged prompts of "
                    "32-160 tokens + 256 new, KV bounded to 416 (+16), greedy; tensor parallel over the N GPUs (TP1 = one "
                    "B200 holding all 140 GB of weights)"),
}


def build_workload(sm, wl: dict, args, rank: int, world: int = 1, tp: int = 1, pp: int = 1):
    """tp > 1: rank `rank` of a tensor-parallel group of `tp` = world ranks (same
    seed everywhere: the shards tile one model); pp > 1: stage `rank` of the layer-split
    pipeline (f4); else an independent replica."""
    import torch
    cfg = synth.model_cfg(wl["model"])
    choices = {"V64": synth.V64, "TINY16": synth.TINY16}[wl["tree"]]
    tree = sm.Tree(choices, topk=synth.TOPK)
    b, x = wl["batch"], wl["x"]
    total_steps = args.warmup + args.steps + args.prof_steps + args.e2e_steps + 8
    if "prompt" in wl:  # C1's x = 64 holds one 32-token turn; timing runs many steps, so the bound
        x = max(x, wl["prompt"] + (tree.depth + 1) * total_steps)  # grows to P + (l+1) * steps
    wl["x_run"] = x
    R = max(b * tree.N, 256, wl.get("max_rows", 0))
    peers = None
    if tp > 1 or pp > 1:
        W = sm.allocate_weights(cfg, wl["n_medusa"], seed=args.seed, tp_rank=rank if tp > 1 else 0, tp_size=tp,
                                pp_rank=rank if pp > 1 else 0, pp_size=pp)
        sym = torch.zeros(sm.tp_sym_bytes(cfg, R, b, wl["n_medusa"]), dtype=torch.uint8, device="cuda")
        W["_sym"] = sym  # keep alive with the weights
        peers = peer_syms(sm, sym, world, rank)
    else:
        W = sm.allocate_weights(cfg, wl["n_medusa"], seed=args.seed + rank)
    # RoPE table: room for the largest tree any caller binds to this model (run_c4_line's candidates)
    model = sm.Model(cfg, W, max_rows=R, max_batch=b, max_seq_len=x + max(tree.N, wl.get("max_tree_n", 0)),
                     peer_sym=peers)
    barrier(world)  # every rank's model exists (its buffer zeroed) before any exchange
    kv = sm.KVCache(model, tree, b, x)
    if b == 1:
        if "prompt" in wl:
            lc_start = wl["prompt"]
        else:
            lc_start = max(128, min(args.lc_start, x - 5 * total_steps - 8))
        prompts = [synth.prompt_tokens(args.seed, rank if max(tp, pp) == 1 else 0, lc_start, cfg["vocab"])]
    else:  # ragged MT-Bench-length prompts (32 + h mod 129)
        prompts = [synth.prompt_tokens(args.seed, i, synth.prompt_length(args.seed, i), cfg["vocab"]) for i in range(b)]
        lc_start = int(np.mean([len(p) for p in prompts]))
    for i, p in enumerate(prompts):
        kv.prefill(i, torch.from_numpy(p).cuda())
    mode = sm.TYPICAL if wl["mode"] == "typical" else sm.GREEDY
    kv.prompts = prompts
    return cfg, tree, model, kv, mode, lc_start


# ------------------------------------------------------------------ our arm
def run_ours(args, world, rank, local) -> dict | None:
    import torch

    import paper_2506_01986_b200 as sm

    for kv_opt in filter(None, os.environ.get("SM_OPT", "").split(",")):  # experiment knobs (sm_set_option)
        k, v = kv_opt.split("=")
        sm.lib().sm_set_option(k.encode(), int(v))
    wl = WORKLOADS[args.config]
    tp = world if (wl.get("tp") and world > 1 and args.parallel == "tp") else 1
    pp = world if (wl.get("tp") and world > 1 and args.parallel == "pp") else 1
    cfg, tree, model, kv, mode, lc_start = build_workload(sm, wl, args, rank, world, tp, pp)
    grp = max(tp, pp)  # ranks that share one model (and emit one token stream)
    N, l, b = tree.N, tree.depth, kv.batch
    out = sm.AcceptOut(b, l)
    acfg = sm.accept_cfg(mode)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    for _ in range(args.warmup):
        kv.step(acfg, out)
    torch.cuda.synchronize()
    barrier(world)
    st = torch.cuda.current_stream()
    # the timed region: exactly K steps, bracketed by barrier + synchronize, device-timed with CUDA
    # events on the launching stream, max over ranks; repeated args.reps times, median reported
    reps = []
    for _ in range(max(1, args.reps)):
        L0 = kv.lengths().astype(np.int64)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(world)
        torch.cuda.synchronize()
        ev0.record(st)
        for _ in range(args.steps):
            kv.step(acfg, out)
        ev1.record(st)
        torch.cuda.synchronize()
        barrier(world)
        ms = reduce_max(ev0.elapsed_time(ev1), world)
        L1 = kv.lengths().astype(np.int64)
        # replicas: every rank's tokens count; tensor parallel: the group emits one stream
        tokens = reduce_sum(float((L1 - L0).sum()), world) if grp == 1 else float((L1 - L0).sum())
        reps.append((tokens / (ms / 1e3), ms, tokens, L0, L1))
    clk = clocks.stop()
    med = sorted(reps, key=lambda r: r[0])[len(reps) // 2]
    value, ms_max, tokens, L0, L1 = med
    tau = float((L1 - L0).sum()) / args.steps / b
    launches = kv.step_launches()

    # ---- kernel timing pass (event-instrumented replay of the same graph)
    kv.profile(True)
    g_ms, g_bytes, g_n, a_ms, a_n, lcs, s_ms = [], [], 0, [], 0, [], []
    for _ in range(args.prof_steps):
        lcs.append(float(kv.lengths().mean()))
        kv.step(acfg, out)
        n, gm, gb = kv.profile_read(0)
        na, am, _ = kv.profile_read(1)
        s_ms.append(kv.profile_read(3)[1])
        g_ms.append(gm)
        g_bytes.append(gb)
        g_n, a_n = n, na
        a_ms.append(am)
    kv.profile(False)
    gemm_ms = statistics.median(g_ms)
    step_prof_ms = statistics.median(s_ms) if s_ms else float("nan")
    gemm_bytes = g_bytes[0]
    attn_ms = statistics.median(a_ms)
    lc_prof = float(np.mean(lcs))

    # ---- end-to-end through the public API with host buffers (pinned), per step:
    # H2D of the turn budget, the step, D2H of the emitted tokens + counts into one of two
    # pinned slots; the host reads step k's tokens (event wait) while step k+1 runs -- the
    # device never waits for the host, and every step's result is read on the host.
    h_budget = torch.full((b,), 1 << 30, dtype=torch.int32).pin_memory()
    d_budget = torch.empty(b, dtype=torch.int32, device="cuda")
    h_emit = [torch.empty((b, l + 1), dtype=torch.int32).pin_memory() for _ in range(2)]
    h_n = [torch.empty((b,), dtype=torch.int32).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    ecfg = sm.accept_cfg(mode, max_new=d_budget)
    d_budget.copy_(h_budget)
    kv.step(ecfg, out)  # capture the e2e graph variant outside the timed region
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_tokens = 0
    e0.record(st)
    for k in range(args.e2e_steps + 1):
        if k < args.e2e_steps:
            d_budget.copy_(h_budget, non_blocking=True)
            kv.step(ecfg, out)
            h_emit[k % 2].copy_(out.emit_tok, non_blocking=True)
            h_n[k % 2].copy_(out.n_emit, non_blocking=True)
            done[k % 2].record(st)
        if k > 0:                          # the caller reads step k-1's tokens
            done[(k - 1) % 2].synchronize()
            e2e_tokens += int(h_n[(k - 1) % 2].sum())
    e1.record(st)
    torch.cuda.synchronize()
    e_ms = reduce_max(e0.elapsed_time(e1), world)
    e2e_val = (reduce_sum(e2e_tokens, world) if grp == 1 else e2e_tokens) / (e_ms / 1e3)

    # ---- vanilla greedy decoding on the same kernels and model: a 1-node tree (root
    # only: verify one row, accept the argmax) -- the speculative speed-up's denominator
    van = None
    if args.vanilla and grp == 1:
        vtree = sm.Tree([], topk=synth.TOPK)
        kv_v = sm.KVCache(model, vtree, b, wl["x_run"])
        for i, p in enumerate(kv.prompts):
            kv_v.prefill(i, torch.from_numpy(p).cuda())
        vout = sm.AcceptOut(b, 0)
        vcfg = sm.accept_cfg(sm.GREEDY)
        vsteps = min(args.steps, 50)
        for _ in range(3):
            kv_v.step(vcfg, vout)
        torch.cuda.synchronize()
        V0 = kv_v.lengths().astype(np.int64)
        v0e, v1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0e.record(st)
        for _ in range(vsteps):
            kv_v.step(vcfg, vout)
        v1e.record(st)
        torch.cuda.synchronize()
        vms = reduce_max(v0e.elapsed_time(v1e), world)
        vtok = reduce_sum(float((kv_v.lengths().astype(np.int64) - V0).sum()), world)
        van = {"value": round(vtok / (vms / 1e3), 3), "unit": "tokens/s", "ms_per_step": round(vms / vsteps, 4),
               "steps": vsteps, "what": "greedy, 1-node tree (no heads) on the same model and kernels"}
        del kv_v

    # ---- K1 tree-attention point of the C5 sweep (geometry A, N=64)
    k1 = run_k1_point(sm, args) if args.k1 and args.config == "c2" else None
    k1_grid = run_k1_grid(sm, args) if args.k1 and args.config == "c2" and world == 1 else None
    acc_lines = None
    if args.extra and args.config == "c2" and world == 1:
        acc_lines = run_c2_acceptance_lines(sm, cfg, model, tree, kv.prompts[0], wl["x_run"], wl)

    if rank != 0:
        return None
    pk = peaks()
    gemm_gbs = gemm_bytes / (gemm_ms / 1e3) / 1e9
    lc_mean = float((L0 + L1).mean() / 2)
    sb = step_bytes(cfg, N, lc_mean, b=b, n_medusa=wl["n_medusa"], tau=tau) / grp  # per GPU
    ms_step = ms_max / args.steps
    # the binding roofline of the whole step: max(bytes / HBM, flops / sustained bf16 tensor peak)
    sf = step_flops(cfg, tree.query()["node_depth"], lc_mean, b=b, n_medusa=wl["n_medusa"]) / grp
    t_hbm, t_tc = sb / pk["hbm"] / 1e6, sf / (pk["bf16_sus"] or pk["bf16"]) / 1e9  # ms
    step_roof = {"bound": "hbm" if t_hbm >= t_tc else "tensor", "alg_bytes": sb, "alg_flops": sf,
                 "roofline_ms": round(max(t_hbm, t_tc), 4), "hbm_ms": round(t_hbm, 4), "tensor_ms": round(t_tc, 4),
                 "frac": round(max(t_hbm, t_tc) / ms_step, 4),
                 "tensor_peak": "bf16 sustained (MEASURED_PEAKS.json)"}
    res = {
        "metric": METRIC, "value": round(value, 3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong" if grp > 1 else "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: counter-hash random-init weights (std 0.02), counter-hash prompt tokens",
        "config": {"workload": wl["desc"], "global_batch": b if grp > 1 else world * b, "seq_len": wl["x_run"],
                   "lc_start": lc_start, "lc_mean": lc_mean,
                   "parallelism": f"tp{tp} (peer-memory exchanges)" if tp > 1 else
                   (f"pp{pp} (layer split, P:252; residual hand-offs over peer memory)" if pp > 1 else
                    (f"replicas x{world}" if world > 1 else "single GPU")),
                   "l2": f"inputs larger than L2: {sb / 1e9:.1f} GB streamed every step (L2 126 MB)"},
        "tau": round(tau, 4), "steps_per_s": round(args.steps / (ms_max / 1e3), 3),
        "roofline": {"kernel": f"K2 tcgen05 GEMM (all {g_n} weight GEMM launches of one step)", "bound": "hbm",
                     "achieved": round(gemm_gbs, 1), "peak": pk["hbm"], "unit": "GB/s",
                     "frac": round(gemm_gbs / pk["hbm"], 4),
                     "traffic": gemm_traffic() if args.config == "c2" else None,
                     "launches_per_step": g_n, "ms_per_step": round(gemm_ms, 4),
                     "share_of_step": round(gemm_ms / ms_step, 4),
                     "share_of_profiled_step": round(gemm_ms / step_prof_ms, 4),
                     "alg_bytes_per_step": gemm_bytes,
                     "peak_source": pk["src"], "timing": "CUDA events around each launch inside the step graph"},
        "step_roofline": step_roof,
        "tree_attn_in_step": {"launches_per_step": a_n, "ms_per_step": round(attn_ms, 4), "lc": lc_prof,
                              "alg_bytes": attn_bytes(cfg, N, lc_prof, b=b),
                              "achieved_gbs": round(attn_bytes(cfg, N, lc_prof, b=b) / (attn_ms / 1e3) / 1e9, 1)},
        "e2e": {"value": round(e2e_val, 3), "unit": "tokens/s", "h2d_bytes_per_step": 4 * b,
                "d2h_bytes_per_step": b * (4 * (l + 1) + 4), "steps": args.e2e_steps,
                "host_loop": "per step: H2D budget, sm_step, D2H tokens + counts (pinned, two slots); the host "
                             "reads step k while step k+1 runs"},
        "gpu_launches": launches * args.steps,
        "clocks": clk,
        "repeats": {"n": len(reps), "values": [round(r[0], 3) for r in reps],
                    "median": round(value, 3), "min": round(min(r[0] for r in reps), 3),
                    "max": round(max(r[0] for r in reps), 3),
                    "what": f"the timed region (K = {args.steps} steps) run {len(reps)} times back to back; "
                            "value / ms_per_step are the median run"},
    }
    if van:
        van["speculative_speedup"] = round(value / van["value"], 3)
        res["vanilla"] = van
    if k1:
        res["k1_point"] = k1
    if k1_grid:
        res["k1_grid"] = k1_grid
    if acc_lines:
        res.update(acc_lines)
    return res


def run_chat(args, world, rank, local) -> dict | None:
    """C3 as a real multi-turn chat (P:22, P:405 multi-turn): for each of the 8
    turns, prefill the turn's prompt (CUDA-event timed on its own), then decode until 128 tokens
    were emitted (the per-turn budget d_max_new clamps the last step); the host reads each step's
    emitted count (the caller's loop).  value = generated tokens / decode time over all turns."""
    import torch

    import paper_2506_01986_b200 as sm
    wl = WORKLOADS[args.config]
    cfg = synth.model_cfg(wl["model"])
    tree = sm.Tree(synth.V64, topk=synth.TOPK)
    seq = rank  # replicas: each rank its own conversation
    P = [synth.prompt_length(args.seed, seq, t) for t in range(wl["turns"])]
    x = sum(p + wl["gen"] for p in P)
    W = sm.allocate_weights(cfg, wl["n_medusa"], seed=args.seed + rank)
    model = sm.Model(cfg, W, max_rows=256, max_batch=1, max_seq_len=x + tree.N)
    kv = sm.KVCache(model, tree, 1, x)
    out = sm.AcceptOut(1, tree.depth)
    budget = torch.zeros(1, dtype=torch.int32, device="cuda")
    acfg = sm.accept_cfg(sm.TYPICAL, max_new=budget, **synth.TYPICAL)
    st = torch.cuda.current_stream()
    h_n = torch.zeros(1, dtype=torch.int32).pin_memory()
    # warm-up conversation turn (graph capture, lazy loading) on a throwaway cache
    kvw = sm.KVCache(model, tree, 1, x)
    kvw.prefill(0, torch.from_numpy(synth.prompt_tokens(args.seed + 99, seq, 64, cfg["vocab"])).cuda())
    budget.fill_(1 << 20)
    for _ in range(max(3, args.warmup)):
        kvw.step(acfg, out)
    torch.cuda.synchronize()
    del kvw
    clocks = ClockSampler(local)
    turns, pre_ms, dec_ms, gen_tok, steps = [], 0.0, 0.0, 0, 0
    for t in range(wl["turns"]):
        prompt = torch.from_numpy(synth.prompt_tokens(args.seed, seq, P[t], cfg["vocab"], turn=t)).cuda()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        e0.record(st)
        kv.prefill(0, prompt)
        e1.record(st)
        budget.fill_(wl["gen"])
        n, k = 0, 0
        while n < wl["gen"]:
            kv.step(acfg, out)
            budget.sub_(out.n_emit)
            h_n.copy_(out.n_emit, non_blocking=True)
            st.synchronize()
            n += int(h_n[0])
            k += 1
        e2.record(st)
        torch.cuda.synchronize()
        pm, dm = e0.elapsed_time(e1), e1.elapsed_time(e2)
        turns.append({"prompt": P[t], "prefill_ms": round(pm, 3), "decode_ms": round(dm, 3), "steps": k,
                      "tau": round(n / k, 3)})
        pre_ms, dec_ms, gen_tok, steps = pre_ms + pm, dec_ms + dm, gen_tok + n, steps + k
    clk = clocks.stop()
    assert int(kv.lengths()[0]) == x
    dec_ms = reduce_max(dec_ms, world)
    pre_ms = reduce_max(pre_ms, world)
    tok_all = reduce_sum(gen_tok, world)
    # K2 share from one profiled replay at the end of the chat (the cache is full: a step there emits
    # nothing, which does not change the kernels' work)
    if rank != 0:
        return None
    pk = peaks()
    tau = gen_tok / steps
    lc_mean = x / 2
    sb = step_bytes(cfg, tree.N, lc_mean, tau=tau)
    sf = step_flops(cfg, tree.query()["node_depth"], lc_mean)
    t_hbm, t_tc = sb / pk["hbm"] / 1e6, sf / (pk["bf16_sus"] or pk["bf16"]) / 1e9
    ms_step = dec_ms / steps
    return {
        "metric": METRIC, "value": round(tok_all / (dec_ms / 1e3), 3), "unit": "tokens/s", "n_gpus": world,
        "steps": steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: counter-hash random-init weights (std 0.02), counter-hash prompts of MT-Bench length",
        "config": {"workload": wl["desc"], "global_batch": world, "seq_len": x, "turns": wl["turns"],
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": f"inputs larger than L2: {sb / 1e9:.1f} GB streamed every step (L2 126 MB)"},
        "tau": round(tau, 4),
        "prefill": {"tokens": sum(P), "ms": round(pre_ms, 3), "tokens_per_s": round(sum(P) / (pre_ms / 1e3), 1),
                    "what": "per-turn prefill (causal chunks through the verify path), timed separately"},
        "step_roofline": {"bound": "hbm" if t_hbm >= t_tc else "tensor", "roofline_ms": round(max(t_hbm, t_tc), 4),
                          "frac": round(max(t_hbm, t_tc) / ms_step, 4), "lc_mean": lc_mean},
        "turns": turns, "clocks": clk,
        "gpu_launches": kv.step_launches() * steps,
        "e2e": {"value": round(tok_all / (dec_ms / 1e3), 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 4, "what": "the chat loop itself: the host reads every step's emitted "
                                                 "count (pinned D2H) to end the turn"},
    }


def _time_steps(kv, cfgs, out, steps: int, st) -> tuple[float, float]:
    """(ms, tokens) of `steps` graph replays (cycling through the accept configs), CUDA events."""
    import torch
    L0 = kv.lengths().astype(np.int64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for k in range(steps):
        kv.step(cfgs[k % len(cfgs)], out)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), float((kv.lengths().astype(np.int64) - L0).sum())


def run_c2_acceptance_lines(sm, cfg, model, tree, prompt, x: int, wl: dict, steps: int = 20) -> dict:
    """C2 lines with tau > 1 (compaction inside the timed region), on the same layer weights:
    * medusa_init: heads R = 0, U = W_lm (reading Q18), greedy -- tau is whatever the random
      model accepts;
    * imposed: the Medusa-init model with acceptance imposed through the d_forced_path hook,
      depth s mod 5 along the first leaf's path (tau = 3 on average: compaction of up to 4 rows
      per layer and kv head every step) -- a cost measurement of the full step at tau = 3, not a
      model-quality number."""
    import torch
    d, l, N = cfg["d_model"], tree.depth, tree.N
    W = model.weights
    z = torch.zeros(d, d, dtype=torch.bfloat16, device="cuda")
    zb = torch.zeros(d, dtype=torch.bfloat16, device="cuda")
    W2 = dict(W)
    W2["medusa"] = [dict(R=z, b=zb, U=W["lm_head"]) for _ in range(wl["n_medusa"])]
    m2 = sm.Model(cfg, W2, max_rows=model.c.max_rows, max_batch=1, max_seq_len=x + N)
    kv = sm.KVCache(m2, tree, 1, x)
    kv.prefill(0, torch.from_numpy(prompt).cuda())
    out = sm.AcceptOut(1, l)
    st = torch.cuda.current_stream()
    g = [sm.accept_cfg(sm.GREEDY)]
    _time_steps(kv, g, out, 3, st)
    pk = peaks()
    res = {}
    lc0 = float(kv.lengths().mean())
    ms, tok = _time_steps(kv, g, out, steps, st)
    tau = tok / steps
    sb = step_bytes(cfg, N, lc0 + tok / 2, tau=tau)
    res["medusa_init"] = {"value": round(tok / (ms / 1e3), 3), "unit": "tokens/s", "tau": round(tau, 4),
                          "ms_per_step": round(ms / steps, 4), "steps": steps,
                          "step_roofline_frac": round(sb / pk["hbm"] / 1e6 / (ms / steps), 4),
                          "what": "C2 with Medusa-init heads (R = 0, U = W_lm), greedy"}
    path0 = [int(v) for v in tree.query()["leaf_paths"][0]]
    forced = []
    for dep in range(l + 1):
        row = path0[: dep + 1] + [-1] * (l - dep)
        forced.append(torch.tensor([row], dtype=torch.int32, device="cuda"))
    fcfgs = [sm.accept_cfg(sm.GREEDY, forced_path=f) for f in forced]
    _time_steps(kv, fcfgs, out, l + 1, st)  # capture the l + 1 graph variants
    lc0 = float(kv.lengths().mean())
    ms, tok = _time_steps(kv, fcfgs, out, steps, st)
    tau = tok / steps
    sb = step_bytes(cfg, N, lc0 + tok / 2, tau=tau)
    res["imposed_tau"] = {"value": round(tok / (ms / 1e3), 3), "unit": "tokens/s", "tau": round(tau, 4),
                          "ms_per_step": round(ms / steps, 4), "steps": steps,
                          "step_roofline_frac": round(sb / pk["hbm"] / 1e6 / (ms / steps), 4),
                          "what": f"Medusa-init C2 with acceptance imposed by the forced-path hook: depth "
                                  f"(step mod {l + 1}) along the first leaf's path -- the step's cost with "
                                  f"compaction in the timed region at tau = {tau:.1f}, not a model-quality number"}
    return res


ALPHA = (0.6, 0.4, 0.3, 0.2)   # stated tau model for tree selection (SPEC AcceptanceModel; unpinned)
RHO = 0.8


def c4_candidates():
    """Trees for 3 Medusa heads (C4): the V64 tree cut to depth 3 and R4-pruned to the
    tab:treefeatures sizes, the 16-node tree, and the 1-node tree (vanilla)."""
    from_v64 = [p for p in synth.V64 if len(p) <= 3]
    out = [("V64/3", from_v64)]

    def prune(ch, n):  # R4: drop the lexicographically largest leaf until n nodes remain
        cur = [tuple(p) for p in ch]
        while len(cur) + 1 > n:
            leaves = [p for p in cur if not any(len(q) == len(p) + 1 and q[:len(p)] == p for q in cur)]
            cur.remove(max(leaves))
        return [list(p) for p in cur]
    for n in (44, 31, 27):
        out.append((f"V64/3-R4-{n}", prune(from_v64, n)))
    out += [("tiny16", synth.TINY16), ("chain4", synth.CHAIN(3)), ("vanilla", [])]
    return out


def run_c4_line(sm, args) -> dict:
    """The bs = 10 part of the metric (BASELINE configs[3], C4 at TP1 on one B200): Llama-2-70B
    shape, 3 Medusa heads, 10 ragged prompts, greedy.  The tree is chosen by f1 tree-size selection
    (sm_select_tree): every candidate tree's step time is measured on this model and batch, and the
    candidate with the largest batch * E[tau] / step_ms under the stated tau model (ALPHA, RHO) is
    timed for the line; the 1-node candidate is vanilla bs = 10 (the paper's "2x over batched
    vanilla" comparison).  Random-init weights accept ~nothing (tau ~ 1): the line reports
    the measured tau, and the selection table the modelled one."""
    import copy

    import torch
    wl = dict(WORKLOADS["c4"])
    wl["max_rows"] = 640
    wl["max_tree_n"] = max(len(ch) + 1 for _, ch in c4_candidates())
    a2 = copy.copy(args)
    a2.steps, a2.warmup, a2.prof_steps, a2.e2e_steps = 10, 3, 0, 0
    cfg, tree0, model, kv0, mode, lc_start = build_workload(sm, wl, a2, 0)
    b, x = kv0.batch, wl["x_run"]
    st = torch.cuda.current_stream()
    acfg = [sm.accept_cfg(mode)]
    cands, kvs, step_ms, meas = [], [], [], []
    for name, ch in c4_candidates():
        t = sm.Tree(ch, topk=synth.TOPK)
        kv = sm.KVCache(model, t, b, x)
        for i, p in enumerate(kv0.prompts):
            kv.prefill(i, torch.from_numpy(p).cuda())
        out = sm.AcceptOut(b, t.depth)
        _time_steps(kv, acfg, out, 3, st)
        ms, tk = _time_steps(kv, acfg, out, 8, st)
        cands.append((name, t))
        kvs.append((kv, out))
        step_ms.append(ms / 8)
        meas.append((tk / 8 / b, tk / (ms / 1e3)))  # MedusaGenerate: acceptance length, tokens/s
    del kv0
    best, tps = sm.select_tree([t for _, t in cands], step_ms, ALPHA, RHO, batch=b)
    name, tree = cands[best]
    kv, out = kvs[best]
    runs = []
    for _ in range(3):
        lc0 = float(kv.lengths().mean())
        ms, tok = _time_steps(kv, acfg, out, 10, st)
        runs.append((tok / (ms / 1e3), ms, tok, lc0))
    val, ms, tok, lc0 = sorted(runs)[1]
    pk = peaks()
    N = tree.N
    tau = tok / 10 / b
    lcm = lc0 + tok / b / 2
    sb = step_bytes(cfg, N, lcm, b=b, n_medusa=wl["n_medusa"], tau=tau)
    sf = step_flops(cfg, tree.query()["node_depth"], lcm, b=b, n_medusa=wl["n_medusa"])
    t_hbm, t_tc = sb / pk["hbm"] / 1e6, sf / (pk["bf16_sus"] or pk["bf16"]) / 1e9
    van = [i for i, (n_, _) in enumerate(cands) if n_ == "vanilla"][0]
    vkv, vout = kvs[van]
    vms, vtok = _time_steps(vkv, acfg, vout, 10, st)
    res = {"value": round(val, 3), "unit": "tokens/s", "tau": round(tau, 4), "ms_per_step": round(ms / 10, 4),
           "steps": 10, "repeats": [round(r[0], 3) for r in runs], "tree": f"{name} (N = {N})",
           "step_roofline": {"bound": "hbm" if t_hbm >= t_tc else "tensor", "roofline_ms": round(max(t_hbm, t_tc), 4),
                             "frac": round(max(t_hbm, t_tc) / (ms / 10), 4)},
           "vanilla": {"value": round(vtok / (vms / 1e3), 3), "ms_per_step": round(vms / 10, 4)},
           "selection": {"tau_model": f"SPEC independent acceptance: alpha = {list(ALPHA)}, rho = {RHO} (stated, "
                                      f"unpinned)",
                         "candidates": [{"tree": n_, "N": t.N, "S": t.S, "heads": t.depth,
                                         "step_ms": round(step_ms[i], 4), "expected_tau": round(t.expected_tau(ALPHA, RHO), 4),
                                         "expected_tokens_per_s": round(tps[i], 1)} for i, (n_, t) in enumerate(cands)],
                         "chosen": name},
           "workload": wl["desc"] + " (TP1: one B200; tree chosen by sm_select_tree)"}
    res["speculative_speedup_measured"] = round(val / res["vanilla"]["value"], 3)
    # Algorithm 2: every candidate configuration's measured (acceptance length,
    # speedup over vanilla), best = Max(speedup) -- sm_alg2_select; with random-init heads tau ~ 1,
    # so the measured choice is the cheapest step, unlike the tau-model choice above
    v_tps = meas[van][1]
    idx = [i for i in range(len(cands)) if i != van]  # the tree configurations (vanilla is the reference)
    sp = [meas[i][1] / v_tps for i in idx]
    a2 = sm.alg2_select([meas[i][0] for i in idx], sp)
    res["alg2"] = {"configs": [{"tree": cands[i][0], "acceptance_length": round(meas[i][0], 4),
                                "speedup": round(sp[j], 4)} for j, i in enumerate(idx)],
                   "chosen": cands[idx[a2]][0],
                   "what": "Algorithm 2 over measured MedusaGenerate runs (8 sm_step calls per configuration on this "
                           "model and batch); speedup = tokens/s over the 1-node (vanilla) configuration's"}
    return res


def gemm_traffic():
    p = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get("dram_bytes_per_step")
    return None


def run_k1_point(sm, args) -> dict:
    """C5 geometry A (H = Hkv = 32, hd = 128), N = 64 (V64), b = 8, Lc = 4096:
    ~0.55 GB of K/V per launch; two buffer sets alternate (> 4x L2)."""
    import torch
    b, H, Hkv, hd, Lc = 8, 32, 32, 128, 4096
    tree = sm.Tree(synth.V64)
    N = tree.N
    cap = Lc + N
    sets = []
    for s in range(2):
        q = torch.empty(b, N, H, hd, dtype=torch.bfloat16, device="cuda")
        k = torch.empty(b, Hkv, cap, hd, dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        for i, t in enumerate((q, k, v)):
            sm.generate_bf16(t, 7 + s, 100 + i, mode=1)
        sets.append((q, k, v, torch.empty_like(q)))
    L = torch.full((b,), Lc, dtype=torch.int32, device="cuda")
    for i in range(4):
        q, k, v, o = sets[i % 2]
        sm.tree_attention(tree, q, k, v, L, H, Hkv, o)
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        q, k, v, o = sets[i % 2]
        sm.tree_attention(tree, q, k, v, L, H, Hkv, o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byt = b * Hkv * (Lc + N) * hd * 2 * 2 + 2 * b * N * H * hd * 2
    gbs = byt / (ms / 1e3) / 1e9
    pk = peaks()
    return {"geometry": "A: H=Hkv=32, hd=128", "N": N, "b": b, "Lc": Lc, "alg_bytes": byt, "ms": round(ms, 4),
            "achieved_gbs": round(gbs, 1), "peak": pk["hbm"], "frac": round(gbs / pk["hbm"], 4)}


def run_k1_grid(sm, args) -> dict:
    """C5 (BASELINE configs[4]) in brief, timed live: tree nodes {16, 64, 128} x KV length {1024, 4096,
    16384} x batch {1, 8, 32} in geometry A (one 7B layer: 32 q = 32 kv heads) and geometry B (one 70B TP8
    shard: 8 q heads on 1 kv head), head_dim 128, uniform lengths; bounded to <= 4 GB of K/V per point.
    Per point: 10 launches over two alternating buffer sets (> L2), CUDA events; frac = max(bytes / HBM
    peak, flops / bf16 peak) / time (the binding roofline).  The full 810-point grid is
    tools/k1_sweep.py --full (profiles/r02/k1_sweep_full.txt)."""
    import statistics

    import torch
    pk = peaks()
    trees = {16: sm.Tree(synth.SWEEP_TREES[16]), 64: sm.Tree(synth.V64), 128: sm.Tree(synth.SWEEP_TREES[128])}
    hd, pts = 128, []
    for geom, H, Hkv in (("A", 32, 32), ("B", 8, 1)):
        for b in (1, 8, 32):
            for N in (16, 64, 128):
                for Lc in (1024, 4096, 16384):
                    tree = trees[N]
                    cap = Lc + tree.N
                    if b * Hkv * cap * hd * 4 > 4e9:
                        continue
                    sets = []
                    for s_ in range(2):
                        q = torch.empty(b, tree.N, H, hd, dtype=torch.bfloat16, device="cuda")
                        k = torch.empty(b, Hkv, cap, hd, dtype=torch.bfloat16, device="cuda")
                        v = torch.empty_like(k)
                        for i, t in enumerate((q, k, v)):
                            sm.generate_bf16(t, 11 + s_, 200 + i, mode=1)
                        sets.append((q, k, v, torch.empty_like(q)))
                    L = torch.full((b,), Lc, dtype=torch.int32, device="cuda")
                    for i in range(2):
                        q, k, v, o = sets[i % 2]
                        sm.tree_attention(tree, q, k, v, L, H, Hkv, o)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for i in range(10):
                        q, k, v, o = sets[i % 2]
                        sm.tree_attention(tree, q, k, v, L, H, Hkv, o)
                    e1.record()
                    torch.cuda.synchronize()
                    us = e0.elapsed_time(e1) * 1e3 / 10
                    byt = b * Hkv * cap * hd * 4 + 2 * b * tree.N * H * hd * 2
                    depth = tree.query()["node_depth"]
                    flops = 4 * H * hd * b * (tree.N * Lc + int(sum(int(x) + 1 for x in depth)))
                    t_hbm, t_tc = byt / pk["hbm"] / 1e3, flops / pk["bf16"] / 1e6  # us
                    pts.append(dict(g=geom, b=b, N=tree.N, Lc=Lc, MB=round(byt / 1e6, 1), us=round(us, 1),
                                    bound="hbm" if t_hbm >= t_tc else "tensor", frac=round(max(t_hbm, t_tc) / us, 3)))
                    del sets
    torch.cuda.empty_cache()
    a_big = [p_["frac"] for p_ in pts if p_["g"] == "A" and p_["bound"] == "hbm" and p_["MB"] >= 64]
    b_big = [p_["frac"] for p_ in pts if p_["g"] == "B" and p_["b"] >= 8 and p_["Lc"] >= 4096]
    return {"what": run_k1_grid.__doc__.split("\n")[0].strip(),
            "points": len(pts),
            "A_hbm_bound_ge_64MB": {"n": len(a_big), "median_frac": round(statistics.median(a_big), 3),
                                    "n_ge_0.70": sum(f >= 0.7 for f in a_big)} if a_big else None,
            "B_b_ge_8_Lc_ge_4096": {"n": len(b_big), "median_frac": round(statistics.median(b_big), 3)} if b_big else None,
            "grid": [f"{p_['g']} b{p_['b']} N{p_['N']} Lc{p_['Lc']}: {p_['us']} us {p_['bound']} {p_['frac']}" for p_ in pts]}


# ------------------------------------------------------------------ oracle (CPU) arm
def host_info() -> dict:
    info = {"threads": host_threads(), "affinity": len(os.sched_getaffinity(0))}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu"] = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["mem_total_gb"] = round(int(line.split()[1]) / 1024 ** 2, 1)
                break
    except OSError:
        pass
    return info


def host_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        if info:
            return int(max(i.get("num_threads", 1) for i in info))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def oracle_c2_run(seed: int, n_layers: int, lc_start: int, warmup: int, steps: int) -> dict:
    """The oracle as it stands, in its timing variant (fp32 weights and
    arithmetic, the tree rows of a step batched through BLAS -- ``Model.forward_rows``, pinned to
    the row-at-a-time oracle), on the C2 workload: Vicuna-7B widths with ``n_layers`` layers, 4
    random-init Medusa heads, the V64 tree, x = 2048, greedy; the GPU arm's prompt (lc_start
    tokens, prefill timed separately) then ``warmup`` + ``steps`` real speculative steps, each
    timed on the host clock."""
    from oracle import model as OM
    from oracle import spec as OS
    cfg = synth.model_cfg("vicuna7b", n_layers=n_layers)
    t0 = time.perf_counter()
    W = OM.Weights(cfg, n_medusa=N_MEDUSA, seed=seed, dtype=np.float32)
    t1 = time.perf_counter()
    s = OS.Session(OM.Model(cfg, W, "fp32"), synth.V64, 1, X_BOUND, batched=True)
    s.prefill(0, synth.prompt_tokens(seed, 0, lc_start, cfg["vocab"]))
    t2 = time.perf_counter()
    times, toks = [], []
    for k in range(warmup + steps):
        a = time.perf_counter()
        r = s.step(0, "greedy")
        if k >= warmup:
            times.append(time.perf_counter() - a)
            toks.append(len(r["emitted"]))
    return {"gen_s": t1 - t0, "prefill_s": t2 - t1, "prefill_tokens": lc_start, "step_s": times, "tokens": toks}


def cpu_baseline(seed: int, lc_start: int) -> dict:
    """Bounded sample (~10-30 s of CPU work): the timing-variant oracle at C2 widths with 1 and 2
    of the 32 layers, prefill + 4 real steps each; the full-depth step time is extrapolated
    linearly in the layer count: t(32) = t(1) + 31 (t(2) - t(1))."""
    r1 = oracle_c2_run(seed, 1, lc_start, 1, 4)
    r2 = oracle_c2_run(seed, 2, lc_start, 1, 4)
    t1, t2 = statistics.median(r1["step_s"]), statistics.median(r2["step_s"])
    t_full = t1 + 31 * max(0.0, t2 - t1)
    tau = statistics.mean(r2["tokens"])
    hi = host_info()
    return {"value": round(tau / t_full, 5), "unit": "tokens/s", "cores": hi["threads"], "kind": "oracle",
            "sample": f"oracle timing variant (numpy fp32 BLAS, tree rows batched) at C2 widths with 1 and 2 of "
                      f"32 layers, {lc_start}-token prefill + 4 real greedy steps each: {t1:.3f} / {t2:.3f} s per "
                      f"step; full 32-layer step extrapolated linearly in the layer count = {t_full:.2f} s; "
                      f"tau {tau:.2f} (random heads)",
            "host": hi}


def run_reference(args, world, rank) -> dict | None:
    """--impl reference: the oracle (timing variant) on the full C2 workload -- all 32 layers,
    the same prompt, W warm-up + K timed real steps; ms_per_step is the host-clock time of those
    K steps (nothing extrapolated).  Under torchrun only rank 0 runs it."""
    if rank != 0:
        return None
    lc = args.lc_start
    r = oracle_c2_run(args.seed, 32, lc, args.warmup, args.steps)
    tot_s = sum(r["step_s"])
    tokens = sum(r["tokens"])
    val = tokens / tot_s
    hi = host_info()
    return {"impl": "reference", "metric": METRIC, "value": round(val, 5), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_s / args.steps * 1e3, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: counter-hash random-init weights, counter-hash prompt tokens",
            "config": {"workload": WORKLOADS["c2"]["desc"], "global_batch": 1, "seq_len": X_BOUND, "lc_start": lc,
                       "parallelism": "host CPU (numpy BLAS threads)"},
            "tau": round(tokens / args.steps, 4),
            "cpu_baseline": {"value": round(val, 5), "unit": "tokens/s", "cores": hi["threads"], "kind": "oracle",
                             "sample": f"full C2 workload: 32 layers, {lc}-token prompt (prefill "
                                       f"{r['prefill_s']:.1f} s, untimed), {args.warmup} warm-up + {args.steps} timed "
                                       f"real steps of the oracle's timing variant (numpy fp32 BLAS, tree rows "
                                       f"batched); weights generated in {r['gen_s']:.1f} s",
                             "host": hi},
            "e2e": {"value": round(val, 5), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--parallel", default="tp", choices=["tp", "pp"],
                    help="multi-GPU C4: tensor parallel (default) or the paper's layer-split pipeline (f4, P:252)")
    ap.add_argument("--lc-start", type=int, default=1024)
    ap.add_argument("--prof-steps", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3, help="repetitions of the K-step timed region (median)")
    ap.add_argument("--no-extra", dest="extra", action="store_false",
                    help="skip the C2 Medusa-init / imposed-tau lines and the C4 bs=10 line")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--no-vanilla", dest="vanilla", action="store_false", help="skip the vanilla (1-node) timing")
    ap.add_argument("--no-k1", dest="k1", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu", action="store_false")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        res = run_reference(args, world, rank)
        if res:
            print(json.dumps(res), flush=True)
        return
    world, rank, local = dist_setup()
    if "turns" in WORKLOADS[args.config]:
        res = run_chat(args, world, rank, local)
        if res is not None:
            print(json.dumps(res), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    res = run_ours(args, world, rank, local)
    if res is not None and args.extra and args.config == "c2" and world == 1:
        import gc

        import paper_2506_01986_b200 as sm
        import torch
        gc.collect()
        torch.cuda.empty_cache()  # the C2 model is gone: room for the 140 GB 70B-shaped weights
        res["bs10"] = run_c4_line(sm, args)
    if res is not None:
        if args.cpu and world == 1 and args.config == "c2":
            res["cpu_baseline"] = cpu_baseline(args.seed, res["config"]["lc_start"])
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
