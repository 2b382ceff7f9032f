"""B200-native Medusa tree-verification hot path (SpecMemo, arxiv 2506.01986).

Thin ctypes binding over ``libspecmemo.so`` (include/specmemo.h).  Argument
marshalling only: every step of the path runs in the library's sm_100a kernels.
PyTorch provides device memory and streams.  There is no CPU fallback: if the
library is missing or the device is not sm_100, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPECMEMO_LIB") or os.path.join(HERE, "libspecmemo.so")  # override: diagnostics builds

SM_OK, SM_ERR_INVALID_ARG, SM_ERR_INFEASIBLE_TREE, SM_ERR_KV_CAPACITY = 0, 1, 2, 3
SM_ERR_DEVICE_OOM, SM_ERR_CUDA, SM_ERR_NCCL, SM_ERR_UNSUPPORTED = 4, 5, 6, 7
GREEDY, TYPICAL = 0, 1


class SpecMemoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[sm_status {status}] {msg}")
        self.status = status


class KVCapacityError(SpecMemoError):
    pass


class InfeasibleTreeError(SpecMemoError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -m paper_2506_01986_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        L.sm_last_error.restype = ctypes.c_char_p
        L.sm_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != SM_OK:
        msg = lib().sm_last_error().decode()
        cls = {SM_ERR_KV_CAPACITY: KVCapacityError, SM_ERR_INFEASIBLE_TREE: InfeasibleTreeError}.get(status, SpecMemoError)
        raise cls(status, msg)


# ------------------------------------------------------------------ C structs
class ModelCfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn",
                                            "vocab", "n_medusa")] + \
               [("rms_eps", ctypes.c_float), ("rope_theta", ctypes.c_float)] + \
               [(n, ctypes.c_int) for n in ("max_rows", "max_batch", "max_seq_len", "dtype")]


DTYPES = {"bf16": 0, "fp32": 1}  # sm_model_cfg.dtype: bf16 path / fp32 parity mode


_PP = ctypes.POINTER(ctypes.c_void_p)


class Weights(ctypes.Structure):
    _fields_ = [("embed", ctypes.c_void_p), ("final_norm", ctypes.c_void_p), ("lm_head", ctypes.c_void_p)] + \
               [(n, _PP) for n in ("attn_norm", "wqkv", "wo", "mlp_norm", "wgate_up", "wdown",
                                   "medusa_R", "medusa_b", "medusa_U")]


MAX_TP = 8


class Dist(ctypes.Structure):
    _fields_ = [("tp_rank", ctypes.c_int), ("tp_size", ctypes.c_int), ("peer_sym", ctypes.c_void_p * MAX_TP),
                ("pp_rank", ctypes.c_int), ("pp_size", ctypes.c_int), ("emu_group", ctypes.c_void_p)]


def pp_layers(n_layers: int, pp_rank: int, pp_size: int) -> range:
    """Layers of pipeline rank pp_rank: equal-sized chunks (include/specmemo.h)."""
    if pp_size < 1 or n_layers % pp_size or not 0 <= pp_rank < pp_size:
        raise ValueError("pp_size must divide n_layers and 0 <= pp_rank < pp_size")
    per = n_layers // pp_size
    return range(pp_rank * per, (pp_rank + 1) * per)


class AcceptCfg(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("temperature", ctypes.c_float), ("eps", ctypes.c_float),
                ("alpha", ctypes.c_float), ("d_max_new", ctypes.c_void_p), ("d_forced_path", ctypes.c_void_p)]


class AcceptOutC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("acc_len", "best_leaf", "path", "emit_tok", "n_emit", "status")]


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


# ------------------------------------------------------------------ trees
class Tree:
    """Static Medusa tree from a path list (root implicit), canonical order
    (depth, rank path) -- Eq. 2 / P:67-72."""

    def __init__(self, choices, topk: int = 10, chain: int | None = None):
        self._h = ctypes.c_void_p()
        if chain is not None:
            _check(lib().sm_tree_create_chain(ctypes.c_int(chain), ctypes.byref(self._h)))
        else:
            flat = [int(r) for p in choices for r in p]
            offs = [0]
            for p in choices:
                offs.append(offs[-1] + len(p))
            fa = (ctypes.c_int32 * max(1, len(flat)))(*flat)
            oa = (ctypes.c_int32 * len(offs))(*offs)
            _check(lib().sm_tree_create(fa, oa, ctypes.c_int(len(choices)), ctypes.c_int(topk), ctypes.byref(self._h)))
        q = self.query()
        self.N, self.S, self.depth = q["N"], q["S"], q["depth"]
        self.topk = topk

    @classmethod
    def _from_handle(cls, h: ctypes.c_void_p, topk: int) -> "Tree":
        t = cls.__new__(cls)
        t._h = h
        q = t.query()
        t.N, t.S, t.depth = q["N"], q["S"], q["depth"]
        t.topk = topk
        return t

    # tree construction (f1; include/specmemo.h)
    @classmethod
    def full(cls, k: int, l: int) -> "Tree":
        h = ctypes.c_void_p()
        _check(lib().sm_tree_create_full(ctypes.c_int(k), ctypes.c_int(l), ctypes.byref(h)))
        return cls._from_handle(h, k)

    def pruned(self, target_nodes: int) -> "Tree":
        """R4 right-to-left in-place pruning to target_nodes."""
        h = ctypes.c_void_p()
        _check(lib().sm_tree_prune(self._h, ctypes.c_int(target_nodes), ctypes.byref(h)))
        return Tree._from_handle(h, self.topk)

    @classmethod
    def pruned_full(cls, k: int, l: int, r_min: float = 0.1, r_max: float = 0.95, mid: float = 2.5,
                    steep: float = 2.0) -> "Tree":
        h = ctypes.c_void_p()
        _check(lib().sm_tree_create_pruned_full(ctypes.c_int(k), ctypes.c_int(l), ctypes.c_float(r_min),
                                                ctypes.c_float(r_max), ctypes.c_float(mid), ctypes.c_float(steep),
                                                ctypes.byref(h)))
        return cls._from_handle(h, k)

    @classmethod
    def custom(cls, n_nodes: int, n_leaves: int, k: int, l: int) -> "Tree":
        h = ctypes.c_void_p()
        _check(lib().sm_tree_create_custom(ctypes.c_int(n_nodes), ctypes.c_int(n_leaves), ctypes.c_int(k),
                                           ctypes.c_int(l), ctypes.byref(h)))
        return cls._from_handle(h, k)

    def expected_tau(self, alpha, rho: float = 1.0) -> float:
        """E[tau] under SPEC's independent acceptance model (include/specmemo.h)."""
        a = (ctypes.c_float * len(alpha))(*[float(v) for v in alpha])
        t = ctypes.c_double()
        _check(lib().sm_tree_expected_tau(self._h, a, len(alpha), ctypes.c_float(rho), ctypes.byref(t)))
        return t.value

    def paths(self) -> list[list[int]]:
        """Rank paths of nodes 1..N-1 in canonical order (root implicit)."""
        q = self.query()
        out = []
        for n in range(1, q["N"]):
            p, x = [], n
            while x > 0:
                p.append(int(q["rank"][x]))
                x = int(q["parent"][x])
            out.append(p[::-1])
        return out

    def query(self) -> dict:
        N, S, dep = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().sm_tree_query(self._h, ctypes.byref(N), ctypes.byref(S), ctypes.byref(dep), None, None, None,
                                   None, None))
        n, s, l = N.value, S.value, dep.value
        parent = np.zeros(n, np.int32)
        nd = np.zeros(n, np.int32)
        rank = np.zeros(n, np.int32)
        anc = np.zeros((n, 4), np.uint64)
        lp = np.zeros((s, l + 1), np.int32)
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _check(lib().sm_tree_query(self._h, None, None, None, P(parent), P(nd), P(rank), P(anc), P(lp)))
        return dict(N=n, S=s, depth=l, parent=parent, node_depth=nd, rank=rank, anc=anc, leaf_paths=lp)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.sm_tree_destroy(self._h)


def select_tree(cands: list, step_ms, alpha, rho: float = 1.0, batch: int = 1) -> tuple[int, list[float]]:
    """sm_select_tree: index of the candidate Tree with the largest batch * E[tau] / step_ms, and
    every candidate's expected tokens/s."""
    n = len(cands)
    arr = (ctypes.c_void_p * n)(*[c._h.value for c in cands])
    ms = (ctypes.c_double * n)(*[float(v) for v in step_ms])
    a = (ctypes.c_float * len(alpha))(*[float(v) for v in alpha])
    best = ctypes.c_int()
    tps = (ctypes.c_double * n)()
    _check(lib().sm_select_tree(arr, n, ms, a, len(alpha), ctypes.c_float(rho), batch, ctypes.byref(best), tps))
    return best.value, list(tps)


def alg2_select(acc_len, speedup) -> int:
    """sm_alg2_select: Algorithm 2's choice -- the configuration with the largest
    measured speedup, ties to the first."""
    n = len(speedup)
    a = (ctypes.c_double * n)(*[float(v) for v in acc_len])
    sp = (ctypes.c_double * n)(*[float(v) for v in speedup])
    best = ctypes.c_int()
    _check(lib().sm_alg2_select(n, a, sp, ctypes.byref(best)))
    return best.value


# ------------------------------------------------------------------ tensor-parallel placement (host logic)
def tp_shard(cfg: dict, rank: int, t: int) -> dict:
    """Which rows / columns of each full weight rank `rank` of `t` holds
    (include/specmemo.h, sm_dist): half-open ranges in the full matrices."""
    d, H, Hkv, hd, F, V = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab"))
    if t not in (1, 2, 4, 8) or not 0 <= rank < t:
        raise ValueError("tp_size must be 1, 2, 4 or 8 and 0 <= rank < tp_size")
    if H % t or Hkv % t or F % (64 * t) or V % (4 * t):
        raise ValueError("tp_size must divide n_heads, n_kv_heads, d_ffn/64 and vocab/4")
    Hl, Hkvl, Fl, Vl = H // t, Hkv // t, F // t, V // t
    return dict(
        q_rows=(rank * Hl * hd, (rank + 1) * Hl * hd),                # of wq [H hd][d]
        k_rows=(rank * Hkvl * hd, (rank + 1) * Hkvl * hd),            # of wk [Hkv hd][d]
        v_rows=(rank * Hkvl * hd, (rank + 1) * Hkvl * hd),            # of wv
        o_cols=(rank * Hl * hd, (rank + 1) * Hl * hd),                # of wo [d][H hd]
        ffn=(rank * Fl, (rank + 1) * Fl),                             # gate/up rows, down columns
        vocab=(rank * Vl, (rank + 1) * Vl),                           # lm_head / medusa_U rows
        H=Hl, Hkv=Hkvl, F=Fl, V=Vl)


def generate_bf16_2d(t, full_cols: int, row0: int, col0: int, seed: int, stream_id: int, mode: int = 0,
                     stream=None) -> None:
    """t[i][j] = w[(row0 + i) * full_cols + col0 + j] of that stream (column shards)."""
    rows, cols = t.shape
    _check(lib().sm_generate_bf16_2d(ctypes.c_void_p(_ptr(t)), ctypes.c_int(rows), ctypes.c_int(cols),
                                     ctypes.c_int(full_cols), ctypes.c_int(row0), ctypes.c_int(col0),
                                     ctypes.c_uint64(seed), ctypes.c_uint64(stream_id), ctypes.c_int(mode),
                                     ctypes.c_void_p(_stream(stream))))


def tp_sym_bytes(cfg: dict, max_rows: int, max_batch: int, n_medusa: int) -> int:
    c = ModelCfg(cfg["n_layers"], cfg["d_model"], cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["d_ffn"],
                 cfg["vocab"], n_medusa, cfg.get("rms_eps", 1e-5), cfg.get("rope_theta", 1e4), max_rows, max_batch, 1)
    n = ctypes.c_size_t()
    _check(lib().sm_tp_sym_bytes(ctypes.byref(c), ctypes.byref(n)))
    return n.value


class EmuGroup:
    """Host-ordered emulation group for several ranks sharing one GPU in one process
    (sm_emu_group_create, include/specmemo.h): the ranks' exchanges run as segment launches
    joined by CUDA events instead of device-side flag waits.  Drive each rank from its own
    host thread (run_ranks); keep the group alive until the models are gone."""

    def __init__(self, n_ranks: int):
        self._h = ctypes.c_void_p()
        _check(lib().sm_emu_group_create(n_ranks, ctypes.byref(self._h)))
        self.n_ranks = n_ranks

    @property
    def handle(self) -> int:
        return self._h.value

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.sm_emu_group_destroy(self._h)
            self._h = ctypes.c_void_p()


def run_ranks(fns: list) -> list:
    """Run fns[r]() on one host thread per rank (the emulation contract: an exchange blocks its
    rank's thread until the peers have published) and return their results; re-raises the first
    exception after every thread has finished."""
    import threading
    res, err = [None] * len(fns), [None] * len(fns)

    def body(r):
        try:
            res[r] = fns[r]()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e
    th = [threading.Thread(target=body, args=(r,)) for r in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return res


def ipc_handle(t) -> bytes:
    h = (ctypes.c_ubyte * 64)()
    _check(lib().sm_ipc_get_handle(ctypes.c_void_p(_ptr(t)), h))
    return bytes(h)


def ipc_open(handle: bytes) -> int:
    h = (ctypes.c_ubyte * 64)(*handle)
    p = ctypes.c_void_p()
    _check(lib().sm_ipc_open(h, ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(lib().sm_ipc_close(ctypes.c_void_p(ptr)))


# ------------------------------------------------------------------ weights (device generator)
def generate_bf16(t, seed: int, stream_id: int, start: int = 0, mode: int = 0, stream=None) -> None:
    """Fill a bf16 CUDA tensor with the counter-hash law (synth.weight_bits /
    synth.normal_bits), on the device."""
    _check(lib().sm_generate_bf16(ctypes.c_void_p(_ptr(t)), ctypes.c_size_t(t.numel()), ctypes.c_uint64(seed),
                                  ctypes.c_uint64(stream_id), ctypes.c_uint64(start), ctypes.c_int(mode),
                                  ctypes.c_void_p(_stream(stream))))


def allocate_weights(cfg: dict, n_medusa: int, seed: int = 0, medusa_init: bool = False, device="cuda",
                     tp_rank: int = 0, tp_size: int = 1, pp_rank: int = 0, pp_size: int = 1) -> dict:
    """Random-init bf16 weights of a Llama + Medusa-1 model, generated on the GPU
    with the same streams as the oracle (synth stream registry).  tp_size > 1:
    the shard of rank tp_rank (tp_shard), generated in place from the full-matrix
    counter indices, so the shards of all ranks tile the tp_size = 1 weights.  pp_size > 1: the
    layers of pipeline rank pp_rank only (pp_layers), same streams as in the full model."""
    import torch

    import synth
    d, H, Hkv, hd, F, V, L = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab",
                                                "n_layers"))
    sh = tp_shard(cfg, tp_rank, tp_size)
    Hl, Hkvl, Fl, Vl = sh["H"], sh["Hkv"], sh["F"], sh["V"]
    bf = torch.bfloat16

    def rows(dst, stream_id, r0):  # rows [r0, r0 + len) of a [*][d] matrix
        generate_bf16(dst, seed, stream_id, start=r0 * dst.shape[1])

    W = {"embed": torch.empty(V, d, dtype=bf, device=device), "lm_head": torch.empty(Vl, d, dtype=bf, device=device),
         "final_norm": torch.ones(d, dtype=bf, device=device), "layers": [], "medusa": [], "tp": (tp_rank, tp_size),
         "pp": (pp_rank, pp_size)}
    generate_bf16(W["embed"], seed, synth.STREAM_EMBED)
    rows(W["lm_head"], synth.STREAM_LM_HEAD, sh["vocab"][0])
    if pp_size > 1 and tp_size > 1:
        raise ValueError("pipeline and tensor parallelism are not combined")
    for li in pp_layers(L, pp_rank, pp_size):
        wqkv = torch.empty((Hl + 2 * Hkvl) * hd, d, dtype=bf, device=device)
        rows(wqkv[: Hl * hd], synth.stream_layer(li, "wq"), sh["q_rows"][0])
        rows(wqkv[Hl * hd:(Hl + Hkvl) * hd], synth.stream_layer(li, "wk"), sh["k_rows"][0])
        rows(wqkv[(Hl + Hkvl) * hd:], synth.stream_layer(li, "wv"), sh["v_rows"][0])
        wo = torch.empty(d, Hl * hd, dtype=bf, device=device)
        generate_bf16_2d(wo, H * hd, 0, sh["o_cols"][0], seed, synth.stream_layer(li, "wo"))
        # gate/up fused with rows interleaved per 64: [g0..g63, u0..u63, g64..] so one
        # 128-row GEMM tile holds matching gate and up features (SiLU*mul epilogue)
        g = torch.empty(Fl, d, dtype=bf, device=device)
        u = torch.empty(Fl, d, dtype=bf, device=device)
        rows(g, synth.stream_layer(li, "wg"), sh["ffn"][0])
        rows(u, synth.stream_layer(li, "wu"), sh["ffn"][0])
        wgu = torch.stack([g.view(Fl // 64, 64, d), u.view(Fl // 64, 64, d)], dim=1).reshape(2 * Fl, d).contiguous()
        del g, u
        wd = torch.empty(d, Fl, dtype=bf, device=device)
        generate_bf16_2d(wd, F, 0, sh["ffn"][0], seed, synth.stream_layer(li, "wd"))
        W["layers"].append(dict(attn_norm=torch.ones(d, dtype=bf, device=device), wqkv=wqkv, wo=wo,
                                mlp_norm=torch.ones(d, dtype=bf, device=device), wgate_up=wgu, wdown=wd))
    for i in range(n_medusa):
        if medusa_init:
            R = torch.zeros(d, d, dtype=bf, device=device)
            U = W["lm_head"]
        else:
            R = torch.empty(d, d, dtype=bf, device=device)
            generate_bf16(R, seed, synth.stream_medusa(i, "R"))
            U = torch.empty(Vl, d, dtype=bf, device=device)
            rows(U, synth.stream_medusa(i, "U"), sh["vocab"][0])
        W["medusa"].append(dict(R=R, b=torch.zeros(d, dtype=bf, device=device), U=U))
    return W


def weights_bytes(cfg: dict, n_medusa: int) -> int:
    d, H, Hkv, hd, F, V, L = (cfg[k] for k in ("d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab",
                                                "n_layers"))
    layer = (H + 2 * Hkv) * hd * d + d * H * hd + 3 * F * d
    return 2 * (L * layer + 2 * V * d + n_medusa * (d * d + V * d))


# ------------------------------------------------------------------ model / kv
class Model:
    """sm_model over borrowed weights.  Tensor parallel: pass the rank's shard
    (allocate_weights(..., tp_rank, tp_size)) and peer_sym = every rank's
    symmetric buffer (tp_sym_bytes) as device pointers usable here; all ranks must
    be constructed before any rank issues work."""

    def __init__(self, cfg: dict, weights: dict, max_rows: int, max_batch: int, max_seq_len: int,
                 peer_sym: list | None = None, dtype: str = "bf16", emu_group: "EmuGroup | None" = None):
        c = ModelCfg(cfg["n_layers"], cfg["d_model"], cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"],
                     cfg["d_ffn"], cfg["vocab"], len(weights["medusa"]), cfg.get("rms_eps", 1e-5),
                     cfg.get("rope_theta", 1e4), max_rows, max_batch, max_seq_len, DTYPES[dtype])
        self.dtype = dtype
        L = len(weights["layers"])  # this rank's layers (all of them unless pipelined)
        arr = lambda key: (ctypes.c_void_p * max(1, L))(*[_ptr(l[key]) for l in weights["layers"]])  # noqa: E731
        marr = lambda key: (ctypes.c_void_p * max(1, len(weights["medusa"])))(  # noqa: E731
            *[_ptr(h[key]) for h in weights["medusa"]])
        self._arrays = [arr(k) for k in ("attn_norm", "wqkv", "wo", "mlp_norm", "wgate_up", "wdown")] + \
                       [marr(k) for k in ("R", "b", "U")]
        w = Weights(_ptr(weights["embed"]), _ptr(weights["final_norm"]), _ptr(weights["lm_head"]),
                    *[ctypes.cast(a, _PP) for a in self._arrays])
        self._h = ctypes.c_void_p()
        self.cfg, self.c = cfg, c
        self.weights = weights          # keep borrowed memory alive
        tp_rank, tp_size = weights.get("tp", (0, 1))
        pp_rank, pp_size = weights.get("pp", (0, 1))
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.pp_rank, self.pp_size = pp_rank, pp_size
        dist = None
        if tp_size > 1 or pp_size > 1:
            nr = max(tp_size, pp_size)
            if peer_sym is None or len(peer_sym) != nr:
                raise ValueError("a tensor-parallel or pipelined model needs peer_sym for every rank")
            dist = Dist(tp_rank, tp_size)
            dist.pp_rank, dist.pp_size = pp_rank, pp_size
            for q, p in enumerate(peer_sym):
                dist.peer_sym[q] = p
            if emu_group is not None:
                dist.emu_group = emu_group.handle
                self._emu = emu_group  # the group outlives this model
        _check(lib().sm_model_create(ctypes.byref(c), ctypes.byref(w), ctypes.byref(dist) if dist else None,
                                     ctypes.byref(self._h)))

    def tp_timed_out(self) -> bool:
        v = ctypes.c_int()
        _check(lib().sm_tp_status(self._h, ctypes.byref(v)))
        return bool(v.value)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.sm_model_destroy(self._h)


class PlanIn(ctypes.Structure):
    _fields_ = [("cfg", ModelCfg)] + [(n, ctypes.c_int) for n in ("batch", "n_queries", "max_tokens", "default_heads",
                                                                "prec_bytes", "accounting")] + \
               [("max_memory", ctypes.c_size_t), ("base_tree", ctypes.c_void_p)]


class PlanOut(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("status", "heads", "N", "S", "kind")] + [("x", ctypes.c_longlong)] + \
               [(n, ctypes.c_size_t) for n in ("max_memory", "base", "heads_bytes", "kv", "buffers", "total")]


PLAN_STATUS = {0: "default", 1: "pruned", 2: "fewer_heads", 3: "needs_quantization"}
PLAN_KIND = {0: "default", 1: "pruned", 2: "custom"}


def plan(cfg: dict, base_tree: "Tree", batch: int, n_queries: int, max_tokens: int, max_memory: int = 0,
         default_heads: int = 4, accounting: str = "b200", prec_bytes: int = 2) -> dict:
    """SpecMemo memory-budget planner (Algorithm 1 over Eqs. 1, 3-6; include/specmemo.h sm_plan).
    max_memory = 0: the current device's free memory is the budget."""
    c = ModelCfg(cfg["n_layers"], cfg["d_model"], cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["d_ffn"],
                 cfg["vocab"], 0, cfg.get("rms_eps", 1e-5), cfg.get("rope_theta", 1e4), 1, 1, 1, 0)
    pin = PlanIn(c, batch, n_queries, max_tokens, default_heads, prec_bytes, {"paper": 0, "b200": 1}[accounting],
                 max_memory, base_tree._h)
    out = PlanOut()
    _check(lib().sm_plan(ctypes.byref(pin), ctypes.byref(out)))
    return dict(status=PLAN_STATUS[out.status], heads=out.heads, N=out.N, S=out.S, kind=PLAN_KIND[out.kind], x=out.x,
                max_memory=out.max_memory, base=out.base, heads_bytes=out.heads_bytes, kv=out.kv,
                buffers=out.buffers, total=out.total)


def workspace_bytes(cfg: dict, max_rows: int, max_batch: int, max_seq_len: int, n_medusa: int,
                    dtype: str = "bf16") -> int:
    c = ModelCfg(cfg["n_layers"], cfg["d_model"], cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["d_ffn"],
                 cfg["vocab"], n_medusa, cfg.get("rms_eps", 1e-5), cfg.get("rope_theta", 1e4), max_rows, max_batch,
                 max_seq_len, DTYPES[dtype])
    n = ctypes.c_size_t()
    _check(lib().sm_workspace_bytes(ctypes.byref(c), ctypes.byref(n)))
    return n.value


def kv_bytes(cfg: dict, batch: int, max_seq_len: int, tree_nodes: int, tp_size: int = 1, dtype: str = "bf16") -> int:
    c = ModelCfg(cfg["n_layers"], cfg["d_model"], cfg["n_heads"], cfg["n_kv_heads"], cfg["head_dim"], cfg["d_ffn"],
                 cfg["vocab"], 0, 1e-5, 1e4, 1, 1, 1, DTYPES[dtype])
    out = ctypes.c_size_t()
    _check(lib().sm_kv_bytes(ctypes.byref(c), tp_size, batch, max_seq_len, tree_nodes, ctypes.byref(out)))
    return out.value


class AcceptOut:
    """Device int32 outputs of one step (sm_accept_out)."""

    def __init__(self, batch: int, depth: int, device="cuda"):
        import torch
        z = lambda *s: torch.zeros(*s, dtype=torch.int32, device=device)  # noqa: E731
        self.acc_len, self.best_leaf, self.n_emit, self.status = z(batch), z(batch), z(batch), z(batch)
        self.path, self.emit_tok = z(batch, depth + 1), z(batch, depth + 1)
        self.c = AcceptOutC(*[_ptr(t) for t in (self.acc_len, self.best_leaf, self.path, self.emit_tok, self.n_emit,
                                                 self.status)])


def accept_cfg(mode: int = GREEDY, temperature: float = 0.7, eps: float = 0.09, alpha: float = 0.3,
               max_new=None, forced_path=None) -> AcceptCfg:
    return AcceptCfg(mode, temperature, eps, alpha, _ptr(max_new), _ptr(forced_path))


class KVCache:
    """Bounded KV cache (Eq. 1 with d + N tree-scratch slots) bound to one tree."""

    def __init__(self, model: Model, tree: Tree, batch: int, max_seq_len: int):
        import torch
        self.model, self.tree, self.batch, self.x = model, tree, batch, max_seq_len
        cfg = dict(model.cfg, n_layers=model.cfg["n_layers"] // model.pp_size)  # this rank's layers
        self.nbytes = kv_bytes(cfg, batch, max_seq_len, tree.N, model.tp_size, model.dtype)
        self.mem = torch.empty(self.nbytes // 2, dtype=torch.bfloat16, device="cuda")
        self._h = ctypes.c_void_p()
        _check(lib().sm_kv_bind(model._h, tree._h, batch, max_seq_len, ctypes.c_void_p(_ptr(self.mem)),
                                ctypes.c_size_t(self.nbytes), ctypes.byref(self._h)))

    def layout(self):
        """[L][2][b][Hkv/tp][x+N][hd] view of the cache memory (this rank's kv heads;
        bf16, or fp32 in the parity mode)."""
        import torch
        c = self.model.cfg
        mem = self.mem.view(torch.float32) if self.model.dtype == "fp32" else self.mem
        return mem.view(c["n_layers"] // self.model.pp_size, 2, self.batch, c["n_kv_heads"] // self.model.tp_size,
                        self.x + self.tree.N, c["head_dim"])

    def set_pad_mode(self, on: bool = True) -> None:
        """Pad batching (f4): uniform cache advance, pads masked (include/specmemo.h)."""
        _check(lib().sm_kv_set_pad_mode(self._h, ctypes.c_int(1 if on else 0)))

    def positions(self) -> np.ndarray:
        """Tokens committed per sequence (= lengths() in the ragged mode)."""
        out = np.zeros(self.batch, np.int32)
        _check(lib().sm_kv_positions(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def status(self) -> int:
        """sm_kv_status: latched device-detected status (3 = a sequence reached the bound x), cleared."""
        v = ctypes.c_int()
        _check(lib().sm_kv_status(self._h, ctypes.byref(v)))
        return v.value

    def lengths(self) -> np.ndarray:
        out = np.zeros(self.batch, np.int32)
        _check(lib().sm_kv_lengths(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def state(self):
        """(root[b], topk[b][n_medusa][K]) device tensors (views, not copies)."""
        import torch
        r, t = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().sm_state_device(self._h, ctypes.byref(r), ctypes.byref(t)))
        nmed = max(1, self.model.c.n_medusa)
        return r.value, t.value, nmed

    def prefill(self, seq: int, tokens, stream=None) -> None:
        _check(lib().sm_prefill(self.model._h, self._h, seq, ctypes.c_void_p(_ptr(tokens)), tokens.numel(),
                                ctypes.c_void_p(_stream(stream))))

    def propose(self, tree_tok, pos=None, stream=None) -> None:
        _check(lib().sm_propose(self.model._h, self._h, ctypes.c_void_p(_ptr(tree_tok)), ctypes.c_void_p(_ptr(pos)),
                                ctypes.c_void_p(_stream(stream))))

    def verify(self, tree_tok, logits=None, stream=None) -> None:
        _check(lib().sm_verify(self.model._h, self._h, ctypes.c_void_p(_ptr(tree_tok)), ctypes.c_void_p(_ptr(logits)),
                               ctypes.c_void_p(_stream(stream))))

    def accept(self, cfg: AcceptCfg, out: AcceptOut, stream=None) -> None:
        _check(lib().sm_accept(self.model._h, self._h, ctypes.byref(cfg), ctypes.byref(out.c),
                               ctypes.c_void_p(_stream(stream))))

    def step(self, cfg: AcceptCfg, out: AcceptOut, stream=None) -> None:
        _check(lib().sm_step(self.model._h, self._h, ctypes.byref(cfg), ctypes.byref(out.c),
                             ctypes.c_void_p(_stream(stream))))

    def profile(self, enable: bool) -> None:
        """Next step() replays an event-instrumented graph (K2 / K1 timing)."""
        _check(lib().sm_step_profile(self._h, ctypes.c_int(1 if enable else 0)))

    def profile_read(self, kind: int):
        """(launch count, summed ms, algorithmic bytes) of the last profiled replay;
        kind 0 = K2 GEMM, 1 = K1 tree attention."""
        n, ms, by = ctypes.c_int(), ctypes.c_float(), ctypes.c_double()
        _check(lib().sm_profile_read(self._h, ctypes.c_int(kind), ctypes.byref(n), ctypes.byref(ms),
                                     ctypes.byref(by)))
        return n.value, ms.value, by.value

    def step_launches(self) -> int:
        n = ctypes.c_int()
        _check(lib().sm_step_launches(self._h, ctypes.byref(n)))
        return n.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.sm_kv_destroy(self._h)


# ------------------------------------------------------------------ stage kernels
def tree_attention(tree: Tree, q, k, v, lengths, n_heads: int, n_kv_heads: int, out, stream=None) -> None:
    """K1 on caller buffers: q/out [b][N][H][hd], k/v [b][Hkv][cap][hd] bf16, lengths int32 [b]."""
    b, cap, hd = k.shape[0], k.shape[2], k.shape[3]
    _check(lib().sm_tree_attention(tree._h, ctypes.c_void_p(_ptr(q)), ctypes.c_void_p(_ptr(k)),
                                   ctypes.c_void_p(_ptr(v)), ctypes.c_void_p(_ptr(lengths)), b, n_heads, n_kv_heads,
                                   hd, cap, ctypes.c_void_p(_ptr(out)), ctypes.c_void_p(_stream(stream))))


def causal_attention(q, k, v, lengths, n_heads: int, n_kv_heads: int, out, stream=None) -> None:
    """K1 prefill mode: q/out [b][n][H][hd] (token i at slot Lc + i attends [0, Lc + i])."""
    b, n = q.shape[0], q.shape[1]
    cap, hd = k.shape[2], k.shape[3]
    _check(lib().sm_causal_attention(n, ctypes.c_void_p(_ptr(q)), ctypes.c_void_p(_ptr(k)), ctypes.c_void_p(_ptr(v)),
                                     ctypes.c_void_p(_ptr(lengths)), b, n_heads, n_kv_heads, hd, cap,
                                     ctypes.c_void_p(_ptr(out)), ctypes.c_void_p(_stream(stream))))


def gemm_bf16(x, w, out, stream=None) -> None:
    """K2: out[M][N] fp32 = x[M][K] @ w[N][K]^T (tcgen05); out None = GEMM only (timing)."""
    M, K = x.shape
    N = w.shape[0]
    _check(lib().sm_gemm_bf16(ctypes.c_void_p(_ptr(x)), ctypes.c_void_p(_ptr(w)), ctypes.c_void_p(_ptr(out)), M, N, K,
                              ctypes.c_void_p(_stream(stream))))


def topk_f32(logits, k: int, out, stream=None) -> None:
    rows, V = logits.shape
    _check(lib().sm_topk_f32(ctypes.c_void_p(_ptr(logits)), rows, V, k, ctypes.c_void_p(_ptr(out)),
                             ctypes.c_void_p(_stream(stream))))


def version() -> str:
    return lib().sm_version().decode()


def set_option(name: str, value: int) -> None:
    """sm_set_option: process-wide launch knobs ("pdl", "gemm_ctas", "attn_tc", ...)."""
    _check(lib().sm_set_option(name.encode(), int(value)))


def reset_options() -> None:
    """sm_reset_options: every knob back to the library default."""
    _check(lib().sm_reset_options())
