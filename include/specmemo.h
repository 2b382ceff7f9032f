/*
 * specmemo.h -- C ABI of the B200-native Medusa tree-verification hot path
 * (SpecMemo, arxiv 2506.01986).  Implemented by libspecmemo.so (sm_100a).
 *
 * Citations: P:<n> = /root/reference/PAPER.md line n, S:<n> = SPEC.md line n.
 * Readings of the paper (Q1..Q26, R0..R11) are listed in DESIGN.md §3.
 *
 * Conventions
 *  - Every call returns sm_status; nothing throws across the ABI.  On error,
 *    sm_last_error() returns a thread-local message.  Argument errors are
 *    detected on the host before anything is enqueued.
 *  - Pointers named d_* are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *    h_* are HOST pointers.  Weights and the KV-cache memory are allocated by
 *    the caller and BORROWED: they must outlive the handles.  Handles and the
 *    library's internal workspace are owned by the library (freed by *_destroy).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All device work is stream-ordered; sm_step is CUDA-graph replayed and
 *    never synchronises with the host.
 *  - bf16 tensors are row-major, PyTorch nn.Linear layout [out][in].
 */
#ifndef SPECMEMO_H
#define SPECMEMO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SM_OK = 0,
  SM_ERR_INVALID_ARG = 1,      /* bad pointer / shape / config; nothing enqueued (SPEC exit 1) */
  SM_ERR_INFEASIBLE_TREE = 2,  /* orphan / duplicate path, rank >= topk, depth > heads (SPEC exit 2)   */
  SM_ERR_KV_CAPACITY = 3,      /* prefill / verify would exceed the bound x (OOM reason "Cache") */
  SM_ERR_DEVICE_OOM = 4,       /* workspace allocation failed (reason Model|Cache|Buffer)        */
  SM_ERR_CUDA = 5,
  SM_ERR_NCCL = 6,              /* reserved: the exchanges are the library's own peer-memory kernels (no
                                  * NCCL; a wait that times out is reported by sm_tp_status instead)   */
  SM_ERR_UNSUPPORTED = 7
} sm_status;

typedef struct sm_tree sm_tree;
typedef struct sm_model sm_model;
typedef struct sm_kv sm_kv;

/* ------------------------------------------------------------------ trees
 * A static Medusa tree in path-list form ("choices", root implicit), e.g.
 * [[0],[0,0],[1],...] (P:55 static pre-built trees; S:227 path-list format).
 * Eq. 2: node n attends to its ancestors and itself ("attention mask
 * assumes full acceptance").  Canonical node order: root = 0, then sort
 * by (depth, lexicographic rank path) (reading Q4).
 *   ranks_flat    concatenated rank paths (host)
 *   path_offsets  n_paths+1 offsets into ranks_flat (host)
 *   topk          arity K ("arity-k equals top-k sampling from heads")
 * Errors: SM_ERR_INFEASIBLE_TREE (orphan, duplicate, empty path, rank >= topk),
 *         SM_ERR_INVALID_ARG (n_paths > 255, i.e. N > 256).
 * n_paths = 0 gives the 1-node tree (vanilla decoding).                      */
sm_status sm_tree_create(const int32_t *h_ranks_flat, const int32_t *h_path_offsets, int n_paths, int topk,
                         sm_tree **out);
/* Chain tree of n nodes (node i = depth i): used for prefill chunks.        */
sm_status sm_tree_create_chain(int n, sm_tree **out);
/* Tree construction ("Optimizing attention mask").  Host
 * only (no device work); results are ordinary trees in canonical order.  Readings in
 * DESIGN.md (Q30, R4).  Errors: SM_ERR_INVALID_ARG (more than 256 nodes, bad k / l),
 * SM_ERR_INFEASIBLE_TREE (target / features no tree of this kind can meet).
 *   full        Eq. 2 full tree: sum_{i<=l} k^i nodes.
 *   prune       R4 in-place pruning of an existing mask to target_nodes (Medusa's
 *               right-to-left pruning: repeatedly drop the lexicographically largest leaf).
 *   pruned_full full tree pruned by the scaled logistic per-level rate
 *               r(i) = r_min + (r_max - r_min) / (1 + exp(-steep (i - mid))) (fig:prunefunc,
 *               parameters unreadable in the paper: SPEC defaults 0.1 / 0.95 / 2.5 / 2);
 *               level 1 keeps all k nodes, level i its first ceil((1 - r(i)) k^i).
 *   custom      a tree with exactly n_nodes nodes and n_leaves leaves, arity <= k, depth
 *               <= l ("directly builds tree mask structures with exact features"). */
sm_status sm_tree_create_full(int k, int l, sm_tree **out);
sm_status sm_tree_prune(const sm_tree *t, int target_nodes, sm_tree **out);
sm_status sm_tree_create_pruned_full(int k, int l, float r_min, float r_max, float mid, float steep, sm_tree **out);
sm_status sm_tree_create_custom(int n_nodes, int n_leaves, int k, int l, sm_tree **out);
/* Tree-size selection (the paper's choice of heads x mask by measured per-token
 * latency, fig:maskmodel P:326-401, "Using 3 heads with mask of size 44 gives the best latency",
 * P:399).  Host only.
 *   sm_tree_expected_tau  E[tau] of tree t under the independent acceptance model of SPEC's simulator
 *       (S:336-337): the node at level j with sibling rank r is accepted with probability
 *       alpha[j-1] * rho^r; the longest all-accepted root path is taken; tau = its depth + 1.
 *       h_alpha[n_alpha >= depth] in [0, 1]; 0 < rho <= 1.  Errors: SM_ERR_INVALID_ARG.
 *   sm_select_tree  among n candidate trees with MEASURED step times h_step_ms[n] (the caller
 *       times sm_step on its model, batch and cache length), the index maximising the expected
 *       decode throughput batch * E[tau] / step_ms (ties: fewer nodes, then lower index);
 *       h_tokens_per_s[n] (nullable) receives every candidate's expected tokens/s.           */
sm_status sm_tree_expected_tau(const sm_tree *t, const float *h_alpha, int n_alpha, float rho, double *tau);
sm_status sm_select_tree(const sm_tree *const *cands, int n, const double *h_step_ms, const float *h_alpha,
                         int n_alpha, float rho, int batch, int *best, double *h_tokens_per_s);
/* Algorithm 2 ("SpecMemo for Medusa"): for every pruned tree configuration the
 * caller runs MedusaGenerate over its queries and records (acceptance_length, speedup); the
 * result is the configuration with the largest measured speedup ("best_config <- Max(results.
 * speedup)"), ties to the first in list order (reading Q32).  acceptance_length is recorded by
 * the algorithm but does not enter the choice.  h_acc_len[n] (nullable), h_speedup[n] finite;
 * *best = index.  Errors: SM_ERR_INVALID_ARG (n < 1, null, non-finite speedup).             */
sm_status sm_alg2_select(int n, const double *h_acc_len, const double *h_speedup, int *best);
/* Query the canonical tables (host outputs, any pointer may be NULL):
 *   N, S (leaves), depth (max depth l), parent[N], node_depth[N], rank[N],
 *   anc_bits[N][4] (bit j of word j/64 = node j is n or an ancestor of n),
 *   leaf_paths[S][depth+1] node ids root..leaf in DFS order, -1 padded.      */
sm_status sm_tree_query(const sm_tree *t, int *N, int *S, int *depth, int32_t *h_parent, int32_t *h_node_depth,
                        int32_t *h_rank, uint64_t *h_anc_bits, int32_t *h_leaf_paths);
void sm_tree_destroy(sm_tree *t);

/* ------------------------------------------------------------------ model */
typedef struct {
  int n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ffn, vocab, n_medusa;
  float rms_eps, rope_theta;
  int max_rows;      /* max token rows per forward (b*N; prefill chunks use <= 256), <= 1024
                        (<= 341 with SM_DTYPE_FP32)                               */
  int max_batch;     /* max sequences b                                          */
  int max_seq_len;   /* max positions (RoPE table length) = x + N                */
  int dtype;         /* SM_DTYPE_BF16 (0, default): bf16 activations and K/V, fp32
                        accumulation (rounding contract R0..R10).
                        SM_DTYPE_FP32 (1): fp32 parity mode (north star: logits and
                        KV within 1e-4 of the oracle's fp32 mode) -- activations,
                        K/V and softmax in fp32; the weights stay the same bf16
                        tensors (R0); each GEMM multiplies the three exact bf16
                        planes of its fp32 input on the tensor cores.  tp_size 1 only. */
} sm_model_cfg;
#define SM_DTYPE_BF16 0
#define SM_DTYPE_FP32 1

/* Device pointers to bf16 weights ([out][in]); arrays are host arrays of
 * device pointers, one entry per layer / Medusa head.  Medusa-1 head i:
 * u_i = U_i (h + SiLU(R_i h + b_i)) (Eq. 4 size pin; reading Q6).       */
typedef struct {
  const void *embed;       /* [V][d]                          */
  const void *final_norm;  /* [d]                             */
  const void *lm_head;     /* [V][d]                          */
  const void *const *attn_norm, *const *wqkv, *const *wo;           /* [d], [(H+2Hkv)hd][d], [d][H hd] */
  const void *const *mlp_norm, *const *wgate_up, *const *wdown;     /* [d], [2F][d], [d][F]            */
  /* wgate_up rows are interleaved in blocks of 64: rows [128t, 128t+64) = gate
   * rows [64t, 64t+64), rows [128t+64, 128t+128) = up rows [64t, 64t+64); one
   * 128-row GEMM tile then holds matching gate/up features for the fused
   * SiLU(gate)*up epilogue.  F must be a multiple of 64.                      */
  const void *const *medusa_R, *const *medusa_b, *const *medusa_U;  /* [d][d], [d], [V][d]             */
} sm_weights;

/* ------------------------------------------------------------------ tensor parallelism (a7, e)
 * North star: TP over NVLink for C4 (SURVEY §8 rows a7 / e).  Rank r of t owns
 * q heads [r*H/t, (r+1)*H/t), kv heads [r*Hkv/t, ...), FFN features
 * [r*F/t, ...) and vocabulary rows [r*V/t, ...) (Megatron-style placement; the
 * paper itself splits layers instead).  sm_weights then holds SHARDS:
 *   wqkv     [(H/t + 2 Hkv/t) hd][d]  rows of the rank's q heads, then k, then v heads
 *   wo       [d][H/t hd]              the rank's columns of the full [d][H hd]
 *   wgate_up [2F/t][d]                the rank's features, 64-row gate/up interleave as above
 *   wdown    [d][F/t]                 the rank's columns of the full [d][F]
 *   lm_head, medusa_U [V/t][d]        the rank's vocabulary rows
 *   embed, norms, medusa_R, medusa_b  full (replicated)
 * Exchanges (all inside the library's kernels, no NCCL): the residual all-reduce
 * after o_proj and down_proj is fused into the residual+RMSNorm consumer (each rank
 * reduces its own split-K partials, publishes the fp32 row slice in its symmetric
 * buffer, and sums all ranks' slices in rank order, so every rank holds bitwise
 * the same residual); the LM head's (argmax, max, m, s, t, candidate logit) and
 * the heads' top-K candidates are merged across ranks by (value desc, index asc).
 * Synchronisation: per-CTA epoch flags written with st.release.sys into every
 * peer's buffer and polled with ld.acquire.sys; a wait that exceeds ~10 s sets the
 * flag read by sm_tp_status and continues (results then invalid).
 * peer_sym[q] = rank q's symmetric buffer (sm_tp_sym_bytes bytes, caller-owned;
 * sm_model_create zero-fills the rank's own, so every rank must have returned from
 * sm_model_create before any rank issues work) as a device pointer usable on this rank's
 * device: cudaIpcOpenMemHandle across processes (sm_ipc_*), or the plain pointer
 * when several ranks share one device in one process (tests).  All ranks must
 * issue the same sequence of prefill / propose / verify / accept / step calls. */
#define SM_MAX_TP 8
typedef struct {
  int tp_rank, tp_size;          /* tp_size in {1, 2, 4, 8}; divides H, Hkv, F/64 and V/4   */
  void *peer_sym[SM_MAX_TP];     /* [tp_size] (or [pp_size]) device pointers, [rank] = own  */
  int pp_rank, pp_size;          /* layer-split pipeline (f4; pp_size 0 or 1 = off), below  */
  void *emu_group;               /* NULL on real multi-GPU placements; see sm_emu_group_create */
} sm_dist;
/* Host-ordered emulation: several ranks sharing ONE GPU in one process (tests on a 1-GPU box).
 * There a kernel must never spin on a flag raised by another rank's launch -- nothing guarantees
 * that the two run at the same time -- so with emu_group set every exchange runs as segment
 * launches (publish; [reduce-scatter;] merge) with no device-side wait, and the ranks' host
 * threads order the segments with CUDA events: a rank records "published" on its stream and its
 * peers' streams wait for that record before their next segment.  The arithmetic, the rank-order
 * sums and therefore the results are bitwise those of the fused flag protocol.  Contract: every
 * rank's calls are issued from its own host thread (an exchange blocks the thread until its
 * peers have published, ~60 s at most, then SM_ERR_CUDA), all ranks share one group, and
 * sm_step runs eagerly (no step graph) on such a model.  One group per set of ranks; destroy it
 * after the models. */
sm_status sm_emu_group_create(int n_ranks, void **group);
void sm_emu_group_destroy(void *group);
/* Layer-split pipeline (f4 comparison mode, the paper's own distribution: "partitioning its
 * layers into equal-sized chunks across all available GPUs, with each GPU also hosting the
 * corresponding slices of the KV cache alongside the layers").  pp_size in 2..8 with
 * tp_size = 1, bf16, n_layers % pp_size == 0: rank r owns layers [r L/pp, (r+1) L/pp) --
 * sm_weights' per-layer arrays then hold those L/pp layers only and the KV cache (sm_kv_bytes
 * with n_layers = L/pp) holds their slices -- plus a full copy of the embedding, final norm, LM
 * head and Medusa heads.  Every forward (prefill chunk or verify) runs stage by stage: rank 0
 * embeds the rows, each rank runs its layers and hands the fp32 residual rows [M][d] to the next
 * rank (published in its symmetric buffer, pulled by the receiver after per-CTA epoch flags, the
 * protocol above); the last rank's final residual goes to every rank, which then runs the final
 * norm, the LM head, acceptance, compaction of its own layers' K/V and the heads replicated
 * (bitwise the same on every rank).  Results equal pp_size = 1 bit for bit: the same kernels run
 * on the same operands.  peer_sym / zero-fill / call-sequence rules as for tensor parallelism. */
/* Bytes of one rank's symmetric exchange buffer for cfg (max_rows, max_batch). */
sm_status sm_tp_sym_bytes(const sm_model_cfg *cfg, size_t *bytes);
/* *timed_out = 1 if any exchange wait of this model gave up (synchronises).    */
sm_status sm_tp_status(const sm_model *m, int *timed_out);
/* CUDA IPC plumbing for multi-process TP: 64-byte handle of a cudaMalloc'd
 * device buffer, and its mapping in this process (close with sm_ipc_close).   */
sm_status sm_ipc_get_handle(const void *d_ptr, unsigned char handle[64]);
sm_status sm_ipc_open(const unsigned char handle[64], void **d_ptr);
sm_status sm_ipc_close(void *d_ptr);

sm_status sm_model_create(const sm_model_cfg *cfg, const sm_weights *w, const sm_dist *dist, sm_model **out);
void sm_model_destroy(sm_model *m);

/* Fill a bf16 buffer with the counter-hash weights of SURVEY §8.d.1:
 * w[i] = bf16(f32((h>>40) - 2^23) * 2^-23 * f32(0.02*sqrt(3))),
 * h = splitmix64(seed ^ stream<<40 ^ (start+i)).  mode 1 = N(0,1)-ish (sum of
 * four 16-bit uniforms, for the K1 sweep), mode 0 = the weight law above.     */
sm_status sm_generate_bf16(void *d_dst, size_t numel, uint64_t seed, uint64_t stream_id, uint64_t start, int mode,
                           void *stream);
/* Block [rows][cols] of the full [*][full_cols] matrix of that stream, starting at
 * (row0, col0): dst[i][j] = w[(row0 + i) * full_cols + col0 + j] (TP column shards). */
sm_status sm_generate_bf16_2d(void *d_dst, int rows, int cols, int full_cols, int row0, int col0, uint64_t seed,
                              uint64_t stream_id, int mode, void *stream);

/* ------------------------------------------------------------------ memory-budget planner (f2)
 * SpecMemo's OptimizerEngine (Algorithm 1) over the memory model of §3.1:
 *   Eq. 1 KV = 2 h b k d x p, x = n m (d restored, Q14)      Eq. 4 heads = 0.6 GB * l
 *   Eq. 3 buffers = (b N w + b S l w + b S l l w) p          Eq. 5 base = B p
 *   Eq. 6 total = base + heads + KV + buffers
 * accounting = SM_ACCT_B200 binds it to this library instead: KV = sm_kv_bytes (x + N
 * scratch slots), heads = l (d^2 + d + V d) p, buffers = only the fp32 node logits b N V 4
 * (the S-indexed gathers of Eq. 3 terms 2-3 do not exist on this path).
 * Algorithm (readings Q31): default config (default_heads, base tree) if it fits;
 * else the largest fitting candidate of ExploreTree for the current head count -- the base
 * tree cut to depth = heads and R4-pruned to 64/44/31/27/16/5 nodes, plus the custom
 * (64, 56) and (44, 37) trees of tab:treefeatures at 4 heads; else the largest head count
 * in [2, heads-1] whose default config fits, and explore again; else NEEDS_QUANTIZATION
 * (QuantizeBaseModel, is not part of this build).  Host only unless max_memory = 0
 * (then cudaMemGetInfo's free bytes of the current device are the budget).            */
typedef struct sm_plan_in {
  sm_model_cfg cfg;          /* shapes; cfg.n_medusa is ignored                          */
  int batch, n_queries, max_tokens;  /* b, n, m                                           */
  int default_heads;         /* Alg. 1 default_heads (4)                                  */
  int prec_bytes;            /* p: 2 (bf16)                                               */
  int accounting;            /* SM_ACCT_PAPER (0) or SM_ACCT_B200 (1)                     */
  size_t max_memory;         /* bytes; 0 = free device memory                             */
  const struct sm_tree *base_tree;   /* default tree (the (64, 42) Medusa tree)           */
} sm_plan_in;
typedef struct sm_plan_out {
  int status;                /* SM_PLAN_DEFAULT 0, _PRUNED 1, _FEWER_HEADS 2, _NEEDS_QUANTIZATION 3 */
  int heads, N, S;
  int kind;                  /* 0 default tree, 1 R4-pruned base tree, 2 custom (N, S) tree */
  long long x;               /* KV bound in committed tokens per sequence = n m           */
  size_t max_memory, base, heads_bytes, kv, buffers, total;  /* of the returned config   */
} sm_plan_out;
#define SM_ACCT_PAPER 0
#define SM_ACCT_B200 1
sm_status sm_plan(const sm_plan_in *in, sm_plan_out *out);
/* Bytes sm_model_create allocates as workspace for cfg (activations, fp32 logits,
 * stream-K partial slots, tables), excluding weights and KV.                          */
sm_status sm_workspace_bytes(const sm_model_cfg *cfg, size_t *bytes);

/* ------------------------------------------------------------------ bounded KV cache
 * Eq. 1 with d restored (reading Q14): bytes =
 *   2 * layers * batch * kv_heads/tp * head_dim * (max_seq_len + tree_nodes) * w,
 * w = 2 (bf16) or 4 (cfg->dtype == SM_DTYPE_FP32).
 * The last N slots of each sequence are the tree scratch ("scratch space").
 * Layout: [layer][K|V][b][Hkv][x+N][hd] of bf16 (fp32 in the parity mode).      */
sm_status sm_kv_bytes(const sm_model_cfg *cfg, int tp_size, int batch, int max_seq_len, int tree_nodes,
                      size_t *bytes);
/* Bind caller memory (>= sm_kv_bytes) as the cache of `batch` sequences for
 * tree t; zero-fills it and sets every length to 0.                           */
sm_status sm_kv_bind(sm_model *m, const sm_tree *t, int batch, int max_seq_len, void *d_mem, size_t bytes,
                     sm_kv **out);
/* Device pointer to the int32 committed lengths Lc[b] (for stage tests).    */
sm_status sm_kv_lengths_device(const sm_kv *kv, int32_t **d_len);
/* Copy Lc[b] to the host (synchronises the kv's stream).                    */
sm_status sm_kv_lengths(const sm_kv *kv, int32_t *h_len);
void sm_kv_destroy(sm_kv *kv);

/* Pad batching (the paper's batched decoding), a comparison mode
 * to the default ragged lengths: every step all sequences' caches advance by the batch's
 * longest acceptance (tau_max); a sequence that accepted fewer tokens leaves pad slots, which
 * attention masks (-inf); RoPE positions count only real tokens ("positional embeddings
 * continue from the latest sequence length").  Per-sequence results equal the ragged
 * mode's up to summation order; the cost is KV slots (and attention over them).  Call before
 * the first step (after prefill is fine: the next step aligns the lengths with pads); single
 * GPU only.  sm_kv_lengths then reports cache slots, sm_kv_positions the token counts.      */
sm_status sm_kv_set_pad_mode(sm_kv *kv, int on);
sm_status sm_kv_positions(const sm_kv *kv, int32_t *h_pos);

/* Prefill one turn of n tokens of sequence `seq` (causal forward at positions
 * [Lc, Lc+n)), then set the pending root (argmax) and the heads' top-k
 * at the last token.  A pending root of a previous turn is dropped (Q15).
 * The turn runs through the verify path in chunks: bf16 on one GPU, causal chunks of up
 * to max_rows tokens (K1 masks cache slot Lc + j for token i by j <= i, no ancestor
 * table); fp32 mode and tensor parallel, chain trees of <= 256 tokens.  Larger max_rows
 * means larger GEMMs (closer to the tensor-core roofline) at the cost of workspace.
 * SM_ERR_KV_CAPACITY if the host-tracked Lc + n > x.  d_tokens: device int32. */
sm_status sm_prefill(sm_model *m, sm_kv *kv, int seq, const int32_t *d_tokens, int n, void *stream);

typedef enum { SM_ACCEPT_GREEDY = 0, SM_ACCEPT_TYPICAL = 1 } sm_accept_mode;
typedef struct {
  sm_accept_mode mode;
  float temperature, eps, alpha;   /* typical: P[tok] > min(eps, alpha*exp(-H)) at temperature T (Q10) */
  const int32_t *d_max_new;        /* [b] remaining per-turn budget, NULL = unbounded (Q15)           */
  const int32_t *d_forced_path;    /* [b][l+1] test hook, NULL = off: accept this node path instead;
                                      a row starting with -1 leaves that sequence unforced          */
} sm_accept_cfg;

/* Device outputs of one step (caller-allocated int32 buffers):
 *   acc_len[b] = a (max accepted depth), best_leaf[b] (DFS leaf index),
 *   path[b][l+1] accepted node ids (-1 padded), emit_tok[b][l+1] emitted tokens,
 *   n_emit[b] = tau = a_eff + 1 (0 if inactive), status[b] (0 ok, 3 capacity). */
typedef struct {
  int32_t *acc_len, *best_leaf, *path, *emit_tok, *n_emit, *status;
} sm_accept_out;

/* a1 propose: tree tokens tok[n] = topk[depth(n)-1][rank(n)], tok[0] = root
 * (P:67); positions Lc + depth.  d_tree_tok [b][N], d_pos [b][N]. */
sm_status sm_propose(sm_model *m, sm_kv *kv, int32_t *d_tree_tok, int32_t *d_pos, void *stream);
/* a2+a3 verify: one forward of all b*N nodes with the tree mask (Eq. 2), K/V
 * written to slots [Lc, Lc+N).  d_logits nullable: fp32 [b][N][V] copy.      */
sm_status sm_verify(sm_model *m, sm_kv *kv, const int32_t *d_tree_tok, float *d_logits, void *stream);
/* a4+a5 accept (greedy/typical tree DP) + in-place compaction of the
 * accepted nodes' K/V + next-state heads/top-k at the accepted node.   */
sm_status sm_accept(sm_model *m, sm_kv *kv, const sm_accept_cfg *cfg, const sm_accept_out *out, void *stream);
/* Full step a1..a5 for the whole batch (P:252-257 batched decoding, ragged
 * lengths).  Captured into a CUDA graph on first use per (mode, hooks) and
 * replayed; graph-capturable itself.                                          */
sm_status sm_step(sm_model *m, sm_kv *kv, const sm_accept_cfg *cfg, const sm_accept_out *out, void *stream);
/* Device-detected conditions (SURVEY §8(b) "surfaced by the next call's return code"): when the
 * accept kernel writes status[b] = 3 (sequence b reached the bound x, nothing emitted for it;
 * OOM reason "Cache", bound P:62-65) it also latches a mapped host word of the kv.  The
 * next sm_verify / sm_accept / sm_step whose host call runs after that step completed returns
 * SM_ERR_KV_CAPACITY without enqueuing anything and clears the latch (no synchronisation: a call
 * enqueued while the detecting step still runs reports it on a later call).  With tp_size > 1
 * the latch is reported only by sm_kv_status (ranks must issue identical calls).
 * sm_kv_status synchronises the device and returns (and clears) the latched status (0 = none). */
sm_status sm_kv_status(sm_kv *kv, int *h_status);
/* Number of kernels one sm_step launches (for the bench's gpu_launches).     */
sm_status sm_step_launches(const sm_kv *kv, int *n);
/* Kernel timing for the bench's roofline: with enable = 1 the next sm_step
 * captures (and then replays) a graph variant that brackets every K2 GEMM
 * launch (kind 0), every K1 tree-attention launch + combine (kind 1) and the
 * whole step (kind 3) with CUDA events on the launch stream (the events
 * serialise the launches they bracket).  sm_profile_read synchronises and returns,
 * for the most recent replay, the number of bracketed launches, their summed
 * duration in ms, and (kind 0) the algorithmic bytes of those launches = their weight
 * matrices (activations and fp32 partial slots excluded).      */
sm_status sm_step_profile(sm_kv *kv, int enable);
sm_status sm_profile_read(const sm_kv *kv, int kind, int *count, float *total_ms, double *alg_bytes);
/* Device pointers to the pending state: root[b], topk[b][n_medusa][K] (int32). */
sm_status sm_state_device(const sm_kv *kv, int32_t **d_root, int32_t **d_topk);

/* ------------------------------------------------------------------ stage kernels (parity tests)
 * K1 tree attention on caller buffers.  q [b][N][H][hd] bf16; k/v caches
 * [b][Hkv][cap][hd] bf16 with the N tree rows at [Lc, Lc+N); d_len[b] int32 Lc;
 * out [b][N][H][hd] bf16.  Node n attends keys [0, Lc) and the tree slots of
 * its ancestors and itself, scale 1/sqrt(hd), softmax in fp32.               */
sm_status sm_tree_attention(const sm_tree *t, const void *d_q, const void *d_k, const void *d_v,
                            const int32_t *d_len, int batch, int n_heads, int n_kv_heads, int head_dim, int cap,
                            void *d_out, void *stream);
/* K1 in prefill mode (f3): the n tokens of a chunk sit at slots [Lc, Lc+n) and token i
 * attends keys [0, Lc) and slots Lc..Lc+i (causal) -- the mask of a chain tree of n
 * nodes, computed without an ancestor table, so n may exceed the 256-node tree limit.
 * Buffers as sm_tree_attention with N = n (1 <= n <= 1024).                       */
sm_status sm_causal_attention(int n, const void *d_q, const void *d_k, const void *d_v, const int32_t *d_len,
                              int batch, int n_heads, int n_kv_heads, int head_dim, int cap, void *d_out,
                              void *stream);
/* K2 tcgen05 GEMM: out[M][N] fp32 = x[M][K] bf16 * w[N][K]^T bf16.  M <= 1024.
 * d_out NULL: only the GEMM runs (its partials stay in library scratch; timing).
 * The stream-K partial sums live in library scratch owned per stream (calls on different streams
 * never share it).  Growing it synchronises the device, so under stream capture the first call of
 * that size on that stream must have run uncaptured (else SM_ERR_UNSUPPORTED).               */
sm_status sm_gemm_bf16(const void *d_x, const void *d_w, float *d_out, int M, int N, int K, void *stream);
/* K3 top-k rows of fp32 logits: idx[r][k] by (value desc, index asc).        */
sm_status sm_topk_f32(const float *d_logits, int rows, int V, int k, int32_t *d_idx, void *stream);

/* Runtime options for experiments (take effect for launches enqueued or graphs
 * captured afterwards): "pdl" (0/1, programmatic dependent launch of the step's
 * kernels), "gemm_ctas" (persistent K2 grid size, 0 = one CTA per SM), "gemm_rep" (1, default:
 * when M spans several token tiles, groups of that many CTAs walk the same weight k-blocks
 * together so each weight stage leaves HBM once; 0: plain stream-K).
 * Unknown names return SM_ERR_INVALID_ARG.                                     */
sm_status sm_set_option(const char *name, int value);
/* Restore every sm_set_option knob to the library default.  Both calls invalidate the per-step
 * graphs captured under the previous knobs (the next sm_step re-captures).                  */
sm_status sm_reset_options(void);

const char *sm_last_error(void);
const char *sm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPECMEMO_H */
