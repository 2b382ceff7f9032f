// attention_f32.cu -- K1 in the fp32 parity mode (north star: logits and KV within
// 1e-4 of the oracle in fp32 mode).  Same operation as the bf16 kernels (Eq. 2,
// node n attends the committed keys [0, Lc) plus the tree slots of its
// ancestors and itself, scale 1/sqrt(hd), softmax), computed in plain fp32 on the
// CUDA cores: the parity mode is a correctness instrument, not a timed path.
//
// One CTA per (token row, q head).  Scores of every key are staged in shared
// memory, then softmax and P.V; the output is written as three bf16 planes
// (hi, mid, lo) whose sum is the fp32 value, ready for the o_proj GEMM.
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace sm {

constexpr int kF32Threads = 128;

__global__ void __launch_bounds__(kF32Threads) tree_attn_f32_kernel(const float *q, const float *k, const float *v,
                                                                    const int32_t *len, const uint64_t *anc, int Nq,
                                                                    int H, int Hkv, int hd, int cap, int seq_base,
                                                                    const uint32_t *pad, int pad_words, float scale,
                                                                    bf16 *out) {
  extern __shared__ float f32_smem[];
  __shared__ float red[kF32Threads / 32];
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
  const int n = m % Nq, seq = seq_base + m / Nq;
  const int Lc = len[seq];
  const int kvh = h / (H / Hkv);
  const float *kb = k + ((size_t)seq * Hkv + kvh) * cap * hd;
  const float *vb = v + ((size_t)seq * Hkv + kvh) * cap * hd;
  float *sq = f32_smem, *ss = f32_smem + hd;
  for (int i = tid; i < hd; i += kF32Threads) sq[i] = q[((size_t)m * H + h) * hd + i];
  __syncthreads();
  const uint64_t *an = anc + (size_t)n * kAncWords;
  const int nk = Lc + Nq;
  const uint32_t *pw = pad ? pad + (size_t)seq * pad_words : nullptr;  // pad batching (f4)
  auto visible = [&](int j) {
    if (j < Lc) return !(pw && ((pw[j >> 5] >> (j & 31)) & 1u));
    return ((an[(j - Lc) >> 6] >> ((j - Lc) & 63)) & 1ull) != 0;
  };
  float mx = -FLT_MAX;
  for (int j = tid; j < nk; j += kF32Threads) {
    float s = -FLT_MAX;
    if (visible(j)) {
      const float *kr = kb + (size_t)j * hd;
      float dot = 0.f;
      for (int i = 0; i < hd; ++i) dot = fmaf(sq[i], kr[i], dot);
      s = dot * scale;
    }
    ss[j] = s;
    mx = fmaxf(mx, s);
  }
  mx = warp_max(mx);
  if ((tid & 31) == 0) red[tid >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < kF32Threads / 32; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int j = tid; j < nk; j += kF32Threads) {
    const float p = visible(j) ? expf(ss[j] - mx) : 0.f;
    ss[j] = p;
    sum += p;
  }
  sum = warp_sum(sum);
  if ((tid & 31) == 0) red[tid >> 5] = sum;
  __syncthreads();
  sum = 0.f;
  for (int w = 0; w < kF32Threads / 32; ++w) sum += red[w];
  const float inv = 1.0f / sum;
  for (int i = tid; i < hd; i += kF32Threads) {
    float o = 0.f;
    for (int j = 0; j < nk; ++j) {
      const float p = ss[j];
      if (p != 0.f) o = fmaf(p, vb[(size_t)j * hd + i], o);
    }
    bf16 a, b, c;
    split3_bf16(o * inv, a, b, c);
    const size_t col = (size_t)h * hd + i, w = (size_t)H * hd;
    out[((size_t)m * 3 + 0) * w + col] = a;
    out[((size_t)m * 3 + 1) * w + col] = b;
    out[((size_t)m * 3 + 2) * w + col] = c;
  }
}

cudaError_t attention_f32_launch(const float *q, const float *k, const float *v, const int32_t *len,
                                 const uint64_t *anc, int Nq, int H, int Hkv, int hd, int cap, int nseq, int seq_base,
                                 const uint32_t *pad, int pad_words, bf16 *out, cudaStream_t st) {
  const size_t smem = (size_t)(hd + cap) * sizeof(float);
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(tree_attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  const float scale = (float)(1.0 / std::sqrt((double)hd));
  return launch_pdl(tree_attn_f32_kernel, dim3(nseq * Nq, H), dim3(kF32Threads), smem, st, q, k, v, len, anc, Nq, H,
                    Hkv, hd, cap, seq_base, pad, pad_words, scale, out);
}

void attention_f32_preload() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, tree_attn_f32_kernel);
}

}  // namespace sm
