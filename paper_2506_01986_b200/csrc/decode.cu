// decode.cu -- device-resident control of one speculative step (no host syncs):
//   propose  (a1, K3)  tree tokens from the heads' top-k at the accepted node
//   accept   (a4, K4)  greedy / typical tree DP, longest accepted path
//   compact  (a5, K5)  in-place gather/scatter of the accepted nodes' K/V
//   commit            Lc += tau, pending root, head input row
// plus the counter-hash weight generator.
#include "common.cuh"
#include "kernels.h"

namespace sm {

// ------------------------------------------------------------------ propose
// tok[n] = root for n = 0, else topk[b][depth(n)-1][rank(n)]
__global__ void propose_kernel(TreeDev t, const int32_t *root, const int32_t *topk, int K, int nmed, int32_t *tree_tok,
                               int32_t *pos, const int32_t *len) {
  pdl_trigger();
  pdl_wait();
  const int bb = blockIdx.x, n = threadIdx.x;
  if (n >= t.N) return;
  int tok;
  if (n == 0) {
    tok = root[bb];
  } else {
    tok = topk[((size_t)bb * nmed + (t.depth[n] - 1)) * K + t.rank[n]];
  }
  tree_tok[(size_t)bb * t.N + n] = tok;
  if (pos) pos[(size_t)bb * t.N + n] = len[bb] + t.depth[n];  // P:255 (len = the position base passed in)
}
cudaError_t propose_launch(TreeDev t, const int32_t *root, const int32_t *topk, int K, int nmed, int b,
                           int32_t *tree_tok, int32_t *pos, const int32_t *len, cudaStream_t st) {
  return launch_pdl(propose_kernel, dim3(b), dim3(256), 0, st, t, root, topk, K, nmed, tree_tok, pos, len);
}

// ------------------------------------------------------------------ accept (tree DP)
// acc(0) = 1; acc(c) = acc(parent) & C(parent, c).
//   greedy : C = tok[c] == argmax z[parent]                        (reading Q9)
//   typical: C = P_p[tok_c] > min(eps, alpha * exp(-H_p)), P at temperature T,
//            H = log s - t/s from the single-pass (m, s, t) stats   (Q10)
// a = deepest accepted depth; among those, max log-likelihood then lowest DFS
// position (Q11); emission clamped by the turn budget and the KV bound x.
__global__ void __launch_bounds__(256) accept_kernel(const __grid_constant__ AcceptArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ int s_cond[kMaxTreeNodes];
  __shared__ float s_lp[kMaxTreeNodes];
  __shared__ int s_chosen;
  const int bb = blockIdx.x, n = threadIdx.x;
  const int N = a.t.N;
  const size_t rowbase = (size_t)bb * N;
  if (n < N) {
    int cond = 1;
    float lp = 0.f;
    if (n > 0) {
      const int p = a.t.parent[n];
      const int tokc = a.tok[rowbase + n];
      if (a.mode == 0) {
        cond = tokc == a.argmax[rowbase + p];
      } else {
        const float *st = a.stats + 3 * (rowbase + p);
        const float m = st[0], s = st[1], tt = st[2];
        const float zc = a.cand ? a.cand[rowbase + n] : a.z[(rowbase + p) * (size_t)a.V + tokc];
        const float y = zc * a.inv_temp;
        const float logs = logf(s);
        const float logP = (y - m) - logs;
        const float H = logs - tt / s;
        const float thr = fminf(a.eps, a.alpha * expf(-H));
        cond = expf(logP) > thr;
        lp = logP;
      }
    }
    s_cond[n] = cond;
    s_lp[n] = lp;
  }
  __syncthreads();
  if (n == 0) {
    // walk every node's ancestor chain (depth <= l), pick (depth, ll, -dfs) max
    int best = 0, bdep = 0, bdfs = a.t.dfs_pos[0];
    float bll = 0.f;
    const int32_t *fp = a.forced_path ? a.forced_path + (size_t)bb * (a.t.l + 1) : nullptr;
    if (fp && fp[0] >= 0) {  // test hook: this sequence accepts the given path (row -1.. = not forced)
      for (int j = 0; j <= a.t.l; ++j)
        if (fp[j] >= 0) best = fp[j];
    } else {
      for (int c = 1; c < N; ++c) {
        int ok = 1, x = c;
        float ll = 0.f;
        while (x > 0) {
          ok &= s_cond[x];
          ll += s_lp[x];
          x = a.t.parent[x];
        }
        if (!ok) continue;
        const int dep = a.t.depth[c], dfs = a.t.dfs_pos[c];
        if (dep > bdep || (dep == bdep && (ll > bll || (ll == bll && dfs < bdfs)))) {
          best = c;
          bdep = dep;
          bll = ll;
          bdfs = dfs;
        }
      }
    }
    s_chosen = best;
  }
  __syncthreads();
  if (n != 0) return;
  const int chosen = s_chosen;
  const int adepth = a.t.depth[chosen];
  const int L1 = a.t.l + 1;
  int path[8];
  {
    int x = chosen;
    for (int j = adepth; j >= 0; --j) {
      path[j] = x;
      x = a.t.parent[x];
    }
  }
  const int Lc = a.len[bb];
  const int budget = a.max_new ? a.max_new[bb] : 0x7fffffff;
  int a_eff, status = 0;
  if (budget <= 0) {
    a_eff = -1;
  } else if (Lc >= a.x_bound) {
    a_eff = -1;
    status = 3;  // SM_ERR_KV_CAPACITY
  } else {
    a_eff = min(adepth, min(budget - 1, a.x_bound - Lc - 1));
  }
  a.acc_len[bb] = adepth;
  a.best_leaf[bb] = a.t.first_leaf[chosen];
  for (int j = 0; j < L1; ++j) {
    a.path[(size_t)bb * L1 + j] = j <= adepth ? path[j] : -1;
    a.emit_tok[(size_t)bb * L1 + j] = j <= a_eff ? a.tok[rowbase + path[j]] : -1;
  }
  a.n_emit[bb] = a_eff + 1;
  a.status[bb] = status;
  if (status && a.sticky) *(volatile int32_t *)a.sticky = status;  // surfaced by the next host call
  if (a_eff >= 0) {
    const int row = (int)rowbase + path[a_eff];
    a.acc_row[bb] = row;
    a.root_next[bb] = a.argmax[row];
  }
}
cudaError_t accept_launch(const AcceptArgs &a, cudaStream_t st) {
  return launch_pdl(accept_kernel, dim3(a.b), dim3(256), 0, st, a);
}

// ------------------------------------------------------------------ compaction
// For j = 1..a_eff: K/V[Lc + j] <- K/V[Lc + path[j]] (all layers, kv heads).
// Reads of every source row complete (barrier) before any write: a parallel
// copy would otherwise race where path[j'] = j for j' < j.
// grid = (L * 2, b, Hkv); 16-byte chunks.
__global__ void compact_kernel(bf16 *kv_base, int b, int Hkv, int cap, int hd, const int32_t *len,
                               const int32_t *path, int path_ld, const int32_t *n_emit) {
  pdl_trigger();
  pdl_wait();
  const int lk = blockIdx.x, bb = blockIdx.y, h = blockIdx.z;
  const int a_eff = n_emit[bb] - 1;
  if (a_eff <= 0) return;
  const int Lc = len[bb];
  const int chunks = hd / 8;  // uint4 per row
  bf16 *base = kv_base + (((size_t)lk * b + bb) * Hkv + h) * (size_t)cap * hd;
  const int total = a_eff * chunks;
  uint4 v[2];
  int cnt = 0;
  for (int i = threadIdx.x; i < total && cnt < 2; i += blockDim.x, ++cnt) {
    const int j = 1 + i / chunks, c = i % chunks;
    const int src = path[(size_t)bb * path_ld + j];
    v[cnt] = reinterpret_cast<const uint4 *>(base + (size_t)(Lc + src) * hd)[c];
  }
  __syncthreads();
  cnt = 0;
  for (int i = threadIdx.x; i < total && cnt < 2; i += blockDim.x, ++cnt) {
    const int j = 1 + i / chunks, c = i % chunks;
    const int src = path[(size_t)bb * path_ld + j];
    if (src != j) reinterpret_cast<uint4 *>(base + (size_t)(Lc + j) * hd)[c] = v[cnt];
  }
}
cudaError_t compact_launch(bf16 *kv_base, int L, int b, int Hkv, int cap, int hd, const int32_t *len,
                           const int32_t *path, int path_ld, const int32_t *n_emit, cudaStream_t st) {
  // each thread holds up to 2 chunks: threads >= ceil(l * hd/8 / 2)
  const int threads = 128;  // covers a_eff <= 16 rows at hd = 128 (256 chunks)
  dim3 grid(L * 2, b, Hkv);
  return launch_pdl(compact_kernel, grid, dim3(threads), 0, st, kv_base, b, Hkv, cap, hd, len, path, path_ld, n_emit);
}

// ------------------------------------------------------------------ commit
// LATE: trigger dependents only after the Lc write is fenced (common.cuh).  Inside the step's
// CUDA graph nothing after the commit reads Lc before its wait and the next replay is a full
// dependency, so the captured commit triggers at entry (the heads GEMM then streams its first
// weight stages while accept / compact / commit run); eager launches (sm_accept) use LATE.
template <bool LATE>
__global__ void commit_kernel(int32_t *len, const int32_t *n_emit, int32_t *root, const int32_t *root_next,
                              const int32_t *acc_row, const bf16 *hf, int d, bf16 *head_in, int32_t *emitted_total) {
  if (!LATE) pdl_trigger();
  pdl_wait();
  const int bb = blockIdx.x;
  const int ne = n_emit[bb];
  if (ne > 0) {
    const bf16 *src = hf + (size_t)acc_row[bb] * d;
    bf16 *dst = head_in + (size_t)bb * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0) {
      if (len) len[bb] += ne;
      root[bb] = root_next[bb];
      if (emitted_total) emitted_total[bb] += ne;
    }
  }
  if (LATE) pdl_trigger_after_writes();  // Lc changed: see common.cuh
}
cudaError_t commit_launch(int b, int32_t *len, const int32_t *n_emit, int32_t *root, const int32_t *root_next,
                          const int32_t *acc_row, const bf16 *hf, int d, bf16 *head_in, int32_t *emitted_total,
                          bool early, cudaStream_t st) {
  // early (entry) trigger only inside the library's own per-step graph (sm_step's capture): a
  // caller that captures several steps into its own graph gets the late trigger, so the next
  // step's tree attention (it reads Lc before its griddepcontrol.wait) cannot race this write.
  if (early)
    return launch_pdl(commit_kernel<false>, dim3(b), dim3(256), 0, st, len, n_emit, root, root_next, acc_row, hf, d,
                      head_in, emitted_total);
  return launch_pdl(commit_kernel<true>, dim3(b), dim3(256), 0, st, len, n_emit, root, root_next, acc_row, hf, d,
                    head_in, emitted_total);
}

__global__ void advance_len_kernel(int32_t *len, int seq, int n, int32_t *pos_len) {
  pdl_wait();
  len[seq] += n;
  if (pos_len) pos_len[seq] += n;
  pdl_trigger_after_writes();
}
cudaError_t advance_len_launch(int32_t *len, int seq, int n, int32_t *pos_len, cudaStream_t st) {
  return launch_pdl(advance_len_kernel, dim3(1), dim3(1), 0, st, len, seq, n, pos_len);
}

// ------------------------------------------------------------------ device-to-device copy as a kernel
// (sm_verify's tree-token and logits copies).  cudaMemcpyAsync D2D goes to a copy engine whose
// queue other streams share: in the single-GPU multi-rank emulations (TP / pipeline ranks on
// several streams) a rank's copy queued behind a peer's copy that waits on a spinning exchange
// kernel stalled the rank until the exchange timed out.  A kernel runs beside the spinner.
__global__ void d2d_copy_kernel(uint4 *dst, const uint4 *src, size_t n16, uint8_t *dst_b, const uint8_t *src_b,
                                size_t tail0, size_t nbytes) {
  pdl_wait();
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = src[i];
  if (blockIdx.x == 0)
    for (size_t i = tail0 + threadIdx.x; i < nbytes; i += blockDim.x) dst_b[i] = src_b[i];
  pdl_trigger_after_writes();
}
cudaError_t d2d_copy_launch(void *dst, const void *src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  const bool al = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  const size_t n16 = al ? bytes / 16 : 0;
  const int grid = (int)std::min<size_t>(4 * kNumSMs, std::max<size_t>(1, (n16 + 255) / 256));
  return launch_pdl(d2d_copy_kernel, dim3(grid), dim3(256), 0, st, static_cast<uint4 *>(dst),
                    static_cast<const uint4 *>(src), n16, static_cast<uint8_t *>(dst), static_cast<const uint8_t *>(src),
                    n16 * 16, bytes);
}

// ------------------------------------------------------------------ pad batching (f4)
SM_DEV void pad_mark(uint32_t *row, int s0, int s1) {  // slots [s0, s1) -> pad (one thread)
  for (int s = s0; s < s1; ++s) row[s >> 5] |= 1u << (s & 31);
}
__global__ void pad_align_kernel(int b, int32_t *len, uint32_t *pad, int pad_words) {
  pdl_wait();
  __shared__ int mx;
  if (threadIdx.x == 0) {
    int m = 0;
    for (int i = 0; i < b; ++i) m = max(m, len[i]);
    mx = m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    pad_mark(pad + (size_t)i * pad_words, len[i], mx);
    len[i] = mx;
  }
  pdl_trigger_after_writes();
}
cudaError_t pad_align_launch(int b, int32_t *len, uint32_t *pad, int pad_words, cudaStream_t st) {
  return launch_pdl(pad_align_kernel, dim3(1), dim3(32), 0, st, b, len, pad, pad_words);
}
__global__ void pad_commit_kernel(int b, int32_t *len, int32_t *pos_len, const int32_t *n_emit, uint32_t *pad,
                                  int pad_words) {
  pdl_wait();
  __shared__ int A;
  if (threadIdx.x == 0) {
    int m = 0;
    for (int i = 0; i < b; ++i) m = max(m, n_emit[i]);
    A = m;  // the batch's longest acceptance: every sequence's cache advances by it
  }
  __syncthreads();
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    const int ne = max(0, n_emit[i]);
    pad_mark(pad + (size_t)i * pad_words, len[i] + ne, len[i] + A);
    len[i] += A;
    pos_len[i] += ne;
  }
  pdl_trigger_after_writes();
}
cudaError_t pad_commit_launch(int b, int32_t *len, int32_t *pos_len, const int32_t *n_emit, uint32_t *pad,
                              int pad_words, cudaStream_t st) {
  return launch_pdl(pad_commit_kernel, dim3(1), dim3(32), 0, st, b, len, pos_len, n_emit, pad, pad_words);
}

__global__ void set_root_kernel(int32_t *root, int seq, const int32_t *argmax_row, const bf16 *hf_row, int d,
                                bf16 *head_in_row) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) root[seq] = argmax_row[0];
  for (int i = threadIdx.x; i < d; i += blockDim.x) head_in_row[i] = hf_row[i];
}
cudaError_t set_root_launch(int32_t *root, int seq, const int32_t *argmax_row, const bf16 *hf_row, int d,
                            bf16 *head_in_row, cudaStream_t st) {
  return launch_pdl(set_root_kernel, dim3(1), dim3(256), 0, st, root, seq, argmax_row, hf_row, d, head_in_row);
}

// ------------------------------------------------------------------ weight generator
SM_DEV uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// dst[i] = w[start + i] (cols == 0) or, for a [rows][cols] block of a [*][full_cols]
// matrix at (row0, col0), w[(row0 + i / cols) * full_cols + col0 + i % cols]
__global__ void generate_kernel(uint16_t *dst, size_t numel, uint64_t seed, uint64_t stream_id, uint64_t start,
                                int mode, int cols, int full_cols, int col0) {
  const uint64_t base = seed ^ (stream_id << 40);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < numel; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t src = cols ? start + (i / cols) * (uint64_t)full_cols + col0 + i % cols : start + i;
    const uint64_t h = splitmix64(base ^ src);
    float w;
    if (mode == 0) {
      const int k = (int)(h >> 40) - (1 << 23);
      w = __fmul_rn(__fmul_rn((float)k, 1.1920928955078125e-07f /* 2^-23 */), 0.034641016151377546f);
    } else {
      float acc = 0.f;
#pragma unroll
      for (int sh = 0; sh < 64; sh += 16) {
        const int k = (int)((h >> sh) & 0xFFFFull) - (1 << 15);
        acc = __fadd_rn(acc, __fmul_rn((float)k, 3.0517578125e-05f /* 2^-15 */));
      }
      w = __fmul_rn(acc, 0.8660254037844386f);
    }
    const __nv_bfloat16 b = __float2bfloat16_rn(w);
    dst[i] = *reinterpret_cast<const uint16_t *>(&b);
  }
}
cudaError_t generate_bf16_launch(void *dst, size_t numel, uint64_t seed, uint64_t stream_id, uint64_t start, int mode,
                                 cudaStream_t st) {
  if (numel == 0) return cudaSuccess;
  size_t blocks = (numel + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  generate_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<uint16_t *>(dst), numel, seed, stream_id, start, mode,
                                                     0, 0, 0);
  return cudaGetLastError();
}
cudaError_t generate_bf16_2d_launch(void *dst, int rows, int cols, int full_cols, int row0, int col0, uint64_t seed,
                                    uint64_t stream_id, int mode, cudaStream_t st) {
  const size_t numel = (size_t)rows * cols;
  if (numel == 0) return cudaSuccess;
  size_t blocks = (numel + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  generate_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<uint16_t *>(dst), numel, seed, stream_id,
                                                     (uint64_t)row0 * full_cols, mode, cols, full_cols, col0);
  return cudaGetLastError();
}

void decode_preload() {  // force-load (see gemm_preload)
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, propose_kernel);
  cudaFuncGetAttributes(&fa, accept_kernel);
  cudaFuncGetAttributes(&fa, compact_kernel);
  cudaFuncGetAttributes(&fa, commit_kernel<false>);
  cudaFuncGetAttributes(&fa, commit_kernel<true>);
  cudaFuncGetAttributes(&fa, advance_len_kernel);
  cudaFuncGetAttributes(&fa, pad_align_kernel);
  cudaFuncGetAttributes(&fa, d2d_copy_kernel);
  cudaFuncGetAttributes(&fa, pad_commit_kernel);
  cudaFuncGetAttributes(&fa, set_root_kernel);
  cudaFuncGetAttributes(&fa, generate_kernel);
}

}  // namespace sm
