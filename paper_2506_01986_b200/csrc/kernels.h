// kernels.h -- host-visible launch interfaces of the sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sm {

typedef __nv_bfloat16 bf16;
constexpr int kNumSMs = 148;
constexpr int kMaxGemmBatch = 5;
constexpr int kMaxTreeNodes = 256;
constexpr int kAncWords = kMaxTreeNodes / 64;

// ---------------------------------------------------------------- K2 GEMM
struct GemmArgs {
  CUtensorMap tmW[kMaxGemmBatch];  // weight [N][K] bf16, box 64(k) x 128(rows), SWIZZLE_128B
  CUtensorMap tmX[kMaxGemmBatch];  // activation [rows][K] bf16, box 64(k) x 16(rows), SWIZZLE_128B
  float *out[kMaxGemmBatch];       // fp32 partials [splits][ldm][ldo]
  int N, K, M, batch, bn;
  int kb_total, kb_per_split, splits;
  int ldo;                         // leading dim of out (>= N)
  int x_row0;                      // first activation row (TMA row offset)
  long long split_stride;          // elements between split slices
};
void gemm_plan(GemmArgs &a, int N, int K, int M, int batch);
cudaError_t gemm_launch(const GemmArgs &a, cudaStream_t st);
int gemm_pick_bn(int M);

// ---------------------------------------------------------------- K1 tree attention
struct AttnArgs {
  CUtensorMap tmK, tmV;       // 2D views [rows][hd] of the K and V caches, box 64 rows x min(hd,64)
  const bf16 *q;              // [rows M][H][hd]
  bf16 *out;                  // [M][H][hd]
  float *part_o;              // [nsplit][M][H][hd]   (nsplit > 1)
  float *part_ml;             // [nsplit][M][H][2]
  const int32_t *len;         // Lc by absolute sequence index
  const uint64_t *anc;        // [Nq][kAncWords]
  long long k_row0, v_row0;   // tmap row of (seq 0, head 0, slot 0) for K and V of this layer
  long long seq_rows;         // rows per sequence block = Hkv * cap
  int cap;                    // slots per (seq, head)
  int Nq, H, Hkv, G, nseq, seq_base, chunk, nsplit;
  float scale_log2;           // log2(e) / sqrt(hd)
};
cudaError_t attention_launch(const AttnArgs &a, int head_dim, cudaStream_t st);
int attention_row_blocks(int Nq, int G);

// ---------------------------------------------------------------- elementwise / epilogues
struct RowCtx {                // forward rows m = (seq - seq_base) * Nq + n
  int M, Nq, seq_base;
  const int32_t *len;          // Lc[seq]
  const int32_t *depth;        // [Nq]
};
// out[m][n] = sum_s part[s][m][n]
cudaError_t sum_splits_launch(const float *part, int splits, long long split_stride, int ldp, float *out, int M, int N,
                              cudaStream_t st);
cudaError_t embed_launch(const int32_t *tok, const bf16 *E, float *x, int M, int d, cudaStream_t st);
// x[m] += sum_s part[s][m] (if part), then h = bf16(rmsnorm(x) * g)
cudaError_t resid_norm_launch(const float *part, int splits, long long split_stride, int ldp, float *x,
                              const bf16 *g, bf16 *h, int M, int d, float eps, cudaStream_t st);
cudaError_t qkv_epilogue_launch(const float *part, int splits, long long split_stride, int ldp, RowCtx rc, int H,
                                int Hkv, int hd, const float2 *rope, bf16 *q, bf16 *kcache, bf16 *vcache, int cap,
                                cudaStream_t st);
cudaError_t silu_mul_launch(const float *part, int splits, long long split_stride, int ldp, int F, bf16 *act, int M,
                            cudaStream_t st);
// logits rows: z = sum of partials; argmax (lowest index on ties) and the
// single-pass typical stats (m, s, t) of y = z / T; optional fp32 copy.
cudaError_t logits_finalize_launch(const float *part, int splits, long long split_stride, int ldp, int V,
                                   const int32_t *row_index, int rows, float inv_temp, float *z_out, int ldz,
                                   int32_t *argmax, float *stats, cudaStream_t st);
cudaError_t topk_launch(const float *part, int splits, long long split_stride, int ldp, int V, int rows, int k,
                        int32_t *idx, int ld_idx, cudaStream_t st);
// rows = groups * rows_per_group; row (grp, rr) reads part + grp*group_stride + rr*ldp
// and writes idx[rr * ld_idx + grp * k + kk]
cudaError_t topk_grouped_launch(const float *part, int splits, long long split_stride, int ldp, int V, int groups,
                                int rows_per_group, long long group_stride, int k, int32_t *idx, int ld_idx,
                                cudaStream_t st);

// ---------------------------------------------------------------- decode control (K3/K4/K5)
struct TreeDev {
  int N, S, l;
  const int32_t *parent, *depth, *rank, *dfs_pos, *first_leaf;
  const uint64_t *anc;
};
cudaError_t propose_launch(TreeDev t, const int32_t *root, const int32_t *topk, int K, int nmed, int b,
                           int32_t *tree_tok, int32_t *pos, const int32_t *len, cudaStream_t st);
struct AcceptArgs {
  TreeDev t;
  int b, K, V, x_bound;
  int mode;                    // 0 greedy, 1 typical
  float inv_temp, eps, alpha;
  const int32_t *tok;          // [b][N]
  const int32_t *argmax;       // [b*N]
  const float *stats;          // [b*N][3] (m, s, t) of y = z/T
  const float *z;              // [b*N][V] logits (typical gather)
  const int32_t *len;          // Lc[b]
  const int32_t *max_new;      // nullable
  const int32_t *forced_path;  // nullable [b][l+1]
  int32_t *acc_len, *best_leaf, *path, *emit_tok, *n_emit, *status;
  int32_t *acc_row;            // [b] row index of the last emitted node
  int32_t *root_next;          // [b]
};
cudaError_t accept_launch(const AcceptArgs &a, cudaStream_t st);
cudaError_t compact_launch(bf16 *kv_base, int L, int b, int Hkv, int cap, int hd, const int32_t *len,
                           const int32_t *path, int path_ld, const int32_t *n_emit, cudaStream_t st);
cudaError_t commit_launch(int b, int32_t *len, const int32_t *n_emit, int32_t *root, const int32_t *root_next,
                          const int32_t *acc_row, const bf16 *hf, int d, bf16 *head_in, int32_t *emitted_total,
                          cudaStream_t st);
cudaError_t advance_len_launch(int32_t *len, int seq, int n, cudaStream_t st);
cudaError_t set_root_launch(int32_t *root, int seq, const int32_t *argmax_row, const bf16 *hf_row, int d,
                            bf16 *head_in_row, cudaStream_t st);
cudaError_t heads_epilogue_grouped_launch(const float *part, int splits, long long split_stride, int ldp,
                                          long long head_stride, int nmed, int b, int d, const bf16 *head_in,
                                          const bf16 *const *beta, bf16 *r_out, long long r_stride, cudaStream_t st);
cudaError_t generate_bf16_launch(void *dst, size_t numel, uint64_t seed, uint64_t stream_id, uint64_t start, int mode,
                                 cudaStream_t st);

}  // namespace sm
