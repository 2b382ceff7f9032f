// epilogue.cu -- the consumers of the GEMM partials, each fusing the fixed-order
// split-K reduction with the next elementwise step of the verify forward
// (rounding contract R1..R10):
//   embed         x = E[tok]                                  (R1)
//   resid_norm    x += sum_s o/down partials; h = bf16(rms(x)*g)   (R5/R7 + R2/R8)
//   qkv_epilogue  q,k,v = sum_s; RoPE(fp32, fp64-built table); q -> bf16,
//                 k,v -> bf16 into cache slots Lc + n at position Lc + depth(n)   (R3)
//   silu_mul      a = bf16(SiLU(g) * u)                       (R6)
//   logits        z = sum_s (fp32), argmax (lowest index on ties) and the
//                 single-pass typical statistics (m, s, t) of y = z/T   (R9)
//   heads         r_i = bf16(h + SiLU(R_i h + b_i))          (R10)
//   topk          top-K of head logits by (value desc, index asc)  (K3)
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace sm {

template <int NT>
SM_DEV float block_sum(float v, float *red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = 0.f;
  if (threadIdx.x < 32) {
    r = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.f;
    r = warp_sum(r);
    if (threadIdx.x == 0) red[0] = r;
  }
  __syncthreads();
  r = red[0];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ split sum (stage API)
__global__ void sum_splits_kernel(const float *part, int splits, long long sstride, int ldp, float *out, int N) {
  const int m = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float acc = 0.f;
  for (int s = 0; s < splits; ++s) acc += part[s * sstride + (size_t)m * ldp + n];
  out[(size_t)m * N + n] = acc;
}
cudaError_t sum_splits_launch(const float *part, int splits, long long split_stride, int ldp, float *out, int M, int N,
                              cudaStream_t st) {
  dim3 grid((N + 255) / 256, M);
  sum_splits_kernel<<<grid, 256, 0, st>>>(part, splits, split_stride, ldp, out, N);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ embed
__global__ void embed_kernel(const int32_t *tok, const bf16 *E, float *x, int d) {
  const int m = blockIdx.x;
  const bf16 *row = E + (size_t)tok[m] * d;
  float *xr = x + (size_t)m * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) xr[i] = bf2f(row[i]);
}
cudaError_t embed_launch(const int32_t *tok, const bf16 *E, float *x, int M, int d, cudaStream_t st) {
  embed_kernel<<<M, 256, 0, st>>>(tok, E, x, d);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ residual + RMSNorm
__global__ void __launch_bounds__(256) resid_norm_kernel(const float *part, int splits, long long sstride, int ldp,
                                                         float *x, const bf16 *g, bf16 *h, int d, float eps) {
  __shared__ float red[32];
  const int m = blockIdx.x;
  float *xr = x + (size_t)m * d;
  float ss = 0.f;
  for (int i = threadIdx.x * 4; i < d; i += 256 * 4) {
    float4 v = *reinterpret_cast<float4 *>(xr + i);
    if (part) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < splits; ++s) {  // fixed split order -> deterministic
        const float4 p = *reinterpret_cast<const float4 *>(part + s * sstride + (size_t)m * ldp + i);
        acc.x += p.x;
        acc.y += p.y;
        acc.z += p.z;
        acc.w += p.w;
      }
      v.x += acc.x;  // R5/R7: fp32 residual += fp32 projection
      v.y += acc.y;
      v.z += acc.z;
      v.w += acc.w;
      *reinterpret_cast<float4 *>(xr + i) = v;
    }
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = block_sum<256>(ss, red);
  const float rs = 1.0f / sqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x * 4; i < d; i += 256 * 4) {
    const float4 v = *reinterpret_cast<const float4 *>(xr + i);
    const __nv_bfloat162 g01 = *reinterpret_cast<const __nv_bfloat162 *>(g + i);
    const __nv_bfloat162 g23 = *reinterpret_cast<const __nv_bfloat162 *>(g + i + 2);
    uint2 o;
    o.x = pack_bf16(v.x * rs * __low2float(g01), v.y * rs * __high2float(g01));
    o.y = pack_bf16(v.z * rs * __low2float(g23), v.w * rs * __high2float(g23));
    *reinterpret_cast<uint2 *>(h + (size_t)m * d + i) = o;
  }
}
cudaError_t resid_norm_launch(const float *part, int splits, long long split_stride, int ldp, float *x,
                              const bf16 *g, bf16 *h, int M, int d, float eps, cudaStream_t st) {
  resid_norm_kernel<<<M, 256, 0, st>>>(part, splits, split_stride, ldp, x, g, h, d, eps);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ QKV epilogue (RoPE + cache write)
__global__ void __launch_bounds__(256) qkv_epilogue_kernel(const float *part, int splits, long long sstride, int ldp,
                                                           RowCtx rc, int H, int Hkv, int hd, const float2 *rope,
                                                           bf16 *q, bf16 *kc, bf16 *vc, int cap) {
  const int m = blockIdx.x;
  const int sl = m / rc.Nq, n = m % rc.Nq;
  const int seq = rc.seq_base + sl;
  const int Lc = rc.len[seq];
  const int pos = Lc + rc.depth[n];
  const int slot = Lc + n;
  const int half = hd / 2;
  const int npairs = (H + 2 * Hkv) * half;
  const float *pr = part + (size_t)m * ldp;
  for (int i = threadIdx.x; i < npairs; i += blockDim.x) {
    const int hh = i / half, c = i % half;
    const int col = hh * hd + c;
    float v0 = 0.f, v1 = 0.f;
    for (int s = 0; s < splits; ++s) {
      v0 += pr[s * sstride + col];
      v1 += pr[s * sstride + col + half];
    }
    if (hh < H + Hkv) {  // q and k heads: rotate-half RoPE at pos
      const float2 cs = rope[(size_t)pos * half + c];
      const float r0 = v0 * cs.x - v1 * cs.y;
      const float r1 = v1 * cs.x + v0 * cs.y;
      v0 = r0;
      v1 = r1;
    }
    bf16 *dst;
    if (hh < H) {
      dst = q + ((size_t)m * H + hh) * hd;
    } else if (hh < H + Hkv) {
      dst = kc + (((size_t)seq * Hkv + (hh - H)) * cap + slot) * hd;
    } else {
      dst = vc + (((size_t)seq * Hkv + (hh - H - Hkv)) * cap + slot) * hd;
    }
    dst[c] = f2bf(v0);
    dst[c + half] = f2bf(v1);
  }
}
cudaError_t qkv_epilogue_launch(const float *part, int splits, long long split_stride, int ldp, RowCtx rc, int H,
                                int Hkv, int hd, const float2 *rope, bf16 *q, bf16 *kcache, bf16 *vcache, int cap,
                                cudaStream_t st) {
  qkv_epilogue_kernel<<<rc.M, 256, 0, st>>>(part, splits, split_stride, ldp, rc, H, Hkv, hd, rope, q, kcache, vcache,
                                            cap);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ SiLU(g) * u
__global__ void __launch_bounds__(256) silu_mul_kernel(const float *part, int splits, long long sstride, int ldp, int F,
                                                       bf16 *act) {
  const int m = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= F) return;
  const float *pr = part + (size_t)m * ldp;
  float gg = 0.f, uu = 0.f;
  for (int s = 0; s < splits; ++s) {
    gg += pr[s * sstride + j];
    uu += pr[s * sstride + F + j];
  }
  const float si = gg / (1.0f + expf(-gg));
  act[(size_t)m * F + j] = f2bf(si * uu);
}
cudaError_t silu_mul_launch(const float *part, int splits, long long split_stride, int ldp, int F, bf16 *act, int M,
                            cudaStream_t st) {
  dim3 grid((F + 255) / 256, M);
  silu_mul_kernel<<<grid, 256, 0, st>>>(part, splits, split_stride, ldp, F, act);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ logits: argmax + typical stats
struct MST {
  float m, s, t;
};
SM_DEV MST mst_merge(MST a, MST b) {
  if (a.m == -INFINITY) return b;
  if (b.m == -INFINITY) return a;
  const float M = fmaxf(a.m, b.m);
  const float ea = expf(a.m - M), eb = expf(b.m - M);
  MST r;
  r.m = M;
  r.s = a.s * ea + b.s * eb;
  r.t = ea * (a.t + (a.m - M) * a.s) + eb * (b.t + (b.m - M) * b.s);
  return r;
}
SM_DEV void argmax_merge(float &v, int &i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__global__ void __launch_bounds__(512) logits_finalize_kernel(const float *part, int splits, long long sstride,
                                                              int ldp, int V, const int32_t *row_index,
                                                              float inv_temp, float *z_out, int ldz, int32_t *argmax,
                                                              float *stats) {
  __shared__ float sv[32];
  __shared__ int si[32];
  __shared__ MST smst[32];
  const int r = blockIdx.x;
  const int m = row_index ? row_index[r] : r;
  const float *pr = part + (size_t)m * ldp;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  MST acc{-INFINITY, 0.f, 0.f};
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    float z = 0.f;
    for (int s = 0; s < splits; ++s) z += pr[s * sstride + j];
    if (z_out) z_out[(size_t)r * ldz + j] = z;
    argmax_merge(bv, bi, z, j);
    const float y = z * inv_temp;
    if (y > acc.m) {
      const float e = (acc.m == -INFINITY) ? 0.f : expf(acc.m - y);
      acc.t = (acc.m == -INFINITY) ? 0.f : e * (acc.t + (acc.m - y) * acc.s);
      acc.s = acc.s * e + 1.f;
      acc.m = y;
    } else {
      const float e = expf(y - acc.m);
      acc.s += e;
      acc.t += e * (y - acc.m);
    }
  }
  // warp reduce
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    argmax_merge(bv, bi, v2, i2);
    MST b{__shfl_xor_sync(0xffffffffu, acc.m, o), __shfl_xor_sync(0xffffffffu, acc.s, o),
          __shfl_xor_sync(0xffffffffu, acc.t, o)};
    acc = mst_merge(acc, b);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[w] = bv;
    si[w] = bi;
    smst[w] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      argmax_merge(bv, bi, sv[k], si[k]);
      acc = mst_merge(acc, smst[k]);
    }
    argmax[r] = bi;
    if (stats) {
      stats[3 * r + 0] = acc.m;
      stats[3 * r + 1] = acc.s;
      stats[3 * r + 2] = acc.t;
    }
  }
}
cudaError_t logits_finalize_launch(const float *part, int splits, long long split_stride, int ldp, int V,
                                   const int32_t *row_index, int rows, float inv_temp, float *z_out, int ldz,
                                   int32_t *argmax, float *stats, cudaStream_t st) {
  logits_finalize_kernel<<<rows, 512, 0, st>>>(part, splits, split_stride, ldp, V, row_index, inv_temp, z_out, ldz,
                                               argmax, stats);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ top-k (K3)
// One block per row: the split-summed row is staged in shared memory, then K
// rounds of a block argmax by (value desc, index asc); taken entries become NaN.
__global__ void __launch_bounds__(1024) topk_kernel(const float *part, int splits, long long sstride, int ldp, int V,
                                                    int k, int32_t *idx, int ld_idx, int rows_per_group,
                                                    long long group_stride) {
  extern __shared__ float srow[];
  __shared__ float wv[32];
  __shared__ int wi[32];
  const int r = blockIdx.x;
  const int grp = r / rows_per_group, rr = r % rows_per_group;
  const float *pr = part + grp * group_stride + (size_t)rr * ldp;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    float z = 0.f;
    for (int s = 0; s < splits; ++s) z += pr[s * sstride + j];
    srow[j] = z;
  }
  __syncthreads();
  for (int kk = 0; kk < k; ++kk) {
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int j = threadIdx.x; j < V; j += blockDim.x) {
      const float z = srow[j];
      if (z == z) argmax_merge(bv, bi, z, j);  // skip NaN (taken)
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(bv, bi, v2, i2);
    }
    if ((threadIdx.x & 31) == 0) {
      wv[threadIdx.x >> 5] = bv;
      wi[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) argmax_merge(bv, bi, wv[w], wi[w]);
      // output layout: row r = grp * rows_per_group + rr -> idx[(rr * groups + grp) * k]
      idx[(size_t)rr * ld_idx + grp * k + kk] = bi;
      if (bi >= 0 && bi < V) srow[bi] = __int_as_float(0x7fc00000);
    }
    __syncthreads();
  }
}
cudaError_t topk_launch(const float *part, int splits, long long split_stride, int ldp, int V, int rows, int k,
                        int32_t *idx, int ld_idx, cudaStream_t st) {
  // generic single-group form (rows independent, idx[r * ld_idx + kk])
  const size_t smem = (size_t)V * sizeof(float);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  topk_kernel<<<rows, 1024, smem, st>>>(part, splits, split_stride, ldp, V, k, idx, ld_idx, rows, 0);
  return cudaGetLastError();
}
// grouped form used by the Medusa heads: rows = groups * rows_per_group
cudaError_t topk_grouped_launch(const float *part, int splits, long long split_stride, int ldp, int V, int groups,
                                int rows_per_group, long long group_stride, int k, int32_t *idx, int ld_idx,
                                cudaStream_t st) {
  const size_t smem = (size_t)V * sizeof(float);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  topk_kernel<<<groups * rows_per_group, 1024, smem, st>>>(part, splits, split_stride, ldp, V, k, idx, ld_idx,
                                                           rows_per_group, group_stride);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Medusa head ResBlock epilogue
struct BetaPtrs {
  const bf16 *p[kMaxGemmBatch];
};
__global__ void heads_epilogue_kernel(const float *part, int splits, long long sstride, int ldp, long long head_stride,
                                      int b, int d, const bf16 *head_in, BetaPtrs beta, bf16 *r_out,
                                      long long r_stride) {
  const int i = blockIdx.z, bb = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const float *pr = part + i * head_stride + (size_t)bb * ldp;
  float t = 0.f;
  for (int s = 0; s < splits; ++s) t += pr[s * sstride + j];
  t += bf2f(beta.p[i][j]);
  const float hv = bf2f(head_in[(size_t)bb * d + j]);
  r_out[i * r_stride + (size_t)bb * d + j] = f2bf(hv + t / (1.0f + expf(-t)));
}
cudaError_t heads_epilogue_grouped_launch(const float *part, int splits, long long split_stride, int ldp,
                                          long long head_stride, int nmed, int b, int d, const bf16 *head_in,
                                          const bf16 *const *beta, bf16 *r_out, long long r_stride, cudaStream_t st) {
  BetaPtrs bp{};
  for (int i = 0; i < nmed && i < kMaxGemmBatch; ++i) bp.p[i] = beta[i];
  dim3 grid((d + 255) / 256, b, nmed);
  heads_epilogue_kernel<<<grid, 256, 0, st>>>(part, splits, split_stride, ldp, head_stride, b, d, head_in, bp, r_out,
                                             r_stride);
  return cudaGetLastError();
}

}  // namespace sm
