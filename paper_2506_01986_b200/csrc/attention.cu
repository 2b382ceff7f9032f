// attention.cu -- K1: tree-masked attention of N candidate nodes (x G query heads
// per kv head) against the committed prefix [0, Lc) and the tree slots
// [Lc, Lc+N) of the bounded KV cache.
//
// Eq. 2: node n attends to its ancestors and itself ("attention mask
// assumes full acceptance"), plus the whole cached prefix.  Scale
// 1/sqrt(hd), fp32 softmax.
//
// Design (memory-bound for N*G < ~250 flop/B):
//  * one CTA = (split of the key range, 64 query rows, (seq, kv head)); GQA rows
//    r = n*G + g share every K/V tile;
//  * K/V tiles of 64 keys are staged by TMA (cp.async.bulk.tensor, SWIZZLE_128B)
//    into a 3-4 deep mbarrier ring -- whole 16 KB tiles per request, coalesced;
//  * Q K^T and P V on tensor cores (mma.sync m16n8k16 bf16, ldmatrix from the
//    swizzled tiles), fp32 online softmax with quad warp-shuffle max/sum;
//  * the ancestor bitmask (N x 4 u64) masks only tiles that reach past Lc;
//  * split-KV for parallelism at b*Hkv < 148: the nsplit CTAs of one (row block,
//    seq, kv head) form a thread-block cluster; each stages its (m, l, O) rows in
//    shared memory and the cluster combines them through DSMEM (no combine
//    kernel, no global partials).  Key ranges come from the device-side Lc, so
//    the launch is CUDA-graph safe;
//  * programmatic dependent launch: the committed prefix [0, Lc) does not change
//    during the forward, so its first K/V tiles are requested before
//    griddepcontrol.wait; Q and the tree tiles only after it.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace sm {

template <int HD>
struct AttnCfg {
  static constexpr int kTile = 64 * HD * 2;  // bytes of one 64-key K (or V) tile
  static constexpr int kStages = HD >= 128 ? 3 : 4;
  static constexpr int kSmem = kStages * 2 * kTile + 1024 + 64 * kAncWords * 8 + 128;
};

// byte offset of 16-byte chunk c of key row `row` inside a [64][HD] tile.
template <int HD>
SM_DEV uint32_t tile_off(int row, int c) {
  if constexpr (HD >= 64) {
    return (uint32_t)((c >> 3) * 8192 + row * 128 + (((c & 7) ^ (row & 7)) << 4));  // TMA SWIZZLE_128B
  } else {
    return (uint32_t)(row * (HD * 2) + (c << 4));
  }
}

template <int HD>
__global__ void __launch_bounds__(128) tree_attn_kernel(const __grid_constant__ AttnArgs a) {
  using C = AttnCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *s_anc = reinterpret_cast<uint64_t *>(smem + C::kStages * 2 * C::kTile);  // [64 rows][kAncWords]
  uint64_t *full = s_anc + 64 * kAncWords;

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, rblk = blockIdx.y;  // split = rank inside the (nsplit, 1, 1) cluster
  const int sl = blockIdx.z / a.Hkv, h = blockIdx.z % a.Hkv;
  const int seq = a.seq_base + sl;
  const int Lc = a.len[seq];  // only the step's last kernels change Lc: safe before the wait
  const int R = a.Nq * a.G;
  // causal prefill chunk: keys past the block's last node are invisible to every row of it
  const int T = Lc + (a.causal ? min(a.Nq, (min(R, (rblk + 1) * 64) - 1) / a.G + 1) : a.Nq);
  const int chunk = ((T + a.nsplit - 1) / a.nsplit + 63) / 64 * 64;
  const int key0 = min(T, split * chunk);
  const int key1 = min(T, key0 + chunk);
  const int ntiles = (key1 - key0 + 63) / 64;

  // tree mask rows of this CTA (node of each query row); constant tables
  if (!a.causal) {
    for (int i = threadIdx.x; i < 64 * kAncWords; i += blockDim.x) {
      const int r = rblk * 64 + i / kAncWords;
      s_anc[i] = (r < R) ? a.anc[(r / a.G) * kAncWords + (i % kAncWords)] : 0ull;
    }
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&a.tmK);
    tma_prefetch_desc(&a.tmV);
    for (int s = 0; s < C::kStages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  const long long kbase_row = a.k_row0 + (long long)seq * a.seq_rows + (long long)h * a.cap;
  const long long vbase_row = a.v_row0 + (long long)seq * a.seq_rows + (long long)h * a.cap;
  auto issue = [&](int i) {
    const int s = i % C::kStages;
    uint8_t *kb = smem + s * 2 * C::kTile;
    uint8_t *vb = kb + C::kTile;
    const int p = key0 + i * 64;
    mbar_arrive_expect_tx(&full[s], 2 * C::kTile);
    if constexpr (HD >= 64) {
#pragma unroll
      for (int hf = 0; hf < HD / 64; ++hf) {
        tma_load_2d(kb + hf * 8192, &a.tmK, &full[s], hf * 64, (int)(kbase_row + p));
        tma_load_2d(vb + hf * 8192, &a.tmV, &full[s], hf * 64, (int)(vbase_row + p));
      }
    } else {
      tma_load_2d(kb, &a.tmK, &full[s], 0, (int)(kbase_row + p));
      tma_load_2d(vb, &a.tmV, &full[s], 0, (int)(vbase_row + p));
    }
  };
  const int first = min(C::kStages, ntiles);
  int pre = 0;  // prefix tiles (entirely below Lc) requested before the dependency wait
  if (threadIdx.x == 0)
    while (pre < first && key0 + (pre + 1) * 64 <= Lc) issue(pre++);
  pdl_wait();  // q and the tree K/V rows come from the preceding kernel
  if (threadIdx.x == 0)
    for (int i = pre; i < first; ++i) issue(i);

  // ---- per-thread rows: ra = r0 + g, rb = r0 + g + 8 (mma C-fragment layout)
  const int r0 = rblk * 64 + warp * 16;
  const bool warp_active = r0 < R;
  const int g = lane >> 2, t = lane & 3;
  const int ra = r0 + g, rb = r0 + g + 8;
  const int la = warp * 16 + g, lb = la + 8;  // local rows for s_anc

  uint32_t qf[HD / 16][4];
  {
    auto qptr = [&](int r) -> const bf16 * {
      const int n = r / a.G, gg = r % a.G;
      const long long m = (long long)sl * a.Nq + n;
      return a.q + (m * a.H + (long long)h * a.G + gg) * HD;
    };
    const bf16 *qa = ra < R ? qptr(ra) : nullptr;
    const bf16 *qb = rb < R ? qptr(rb) : nullptr;
#pragma unroll
    for (int kc = 0; kc < HD / 16; ++kc) {
      const int c = kc * 16 + 2 * t;
      qf[kc][0] = qa ? *reinterpret_cast<const uint32_t *>(qa + c) : 0u;
      qf[kc][1] = qb ? *reinterpret_cast<const uint32_t *>(qb + c) : 0u;
      qf[kc][2] = qa ? *reinterpret_cast<const uint32_t *>(qa + c + 8) : 0u;
      qf[kc][3] = qb ? *reinterpret_cast<const uint32_t *>(qb + c + 8) : 0u;
    }
  }

  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  const float sl2 = a.scale_log2;

  for (int i = 0; i < ntiles; ++i) {
    const int s = i % C::kStages;
    mbar_wait(&full[s], (i / C::kStages) & 1);
    if (warp_active) {
      const uint32_t kb = smem_u32(smem + s * 2 * C::kTile);
      const uint32_t vb = kb + C::kTile;
      const int p0 = key0 + i * 64;
      float sc[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < HD / 16; ++kc) {
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          uint32_t b0, b1, b2, b3;
          const int key = jp * 16 + ((lane >> 4) << 3) + (lane & 7);
          const int ch = kc * 2 + ((lane >> 3) & 1);
          ldmatrix_x4(kb + tile_off<HD>(key, ch), b0, b1, b2, b3);
          mma_bf16_16816(sc[2 * jp], qf[kc], b0, b1);
          mma_bf16_16816(sc[2 * jp + 1], qf[kc], b2, b3);
        }
      }
      if (a.pad && p0 < Lc) {  // pad batching (f4): masked cache slots of this sequence's prefix
        const uint32_t *pw = a.pad + (size_t)seq * a.pad_words + (p0 >> 5);
        const uint64_t pm = (uint64_t)pw[0] | ((uint64_t)pw[1] << 32);
        if (pm) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              if ((pm >> (8 * j + 2 * t + e)) & 1ull) {
                sc[j][e] = -INFINITY;
                sc[j][2 + e] = -INFINITY;
              }
            }
          }
        }
      }
      // mask: keys >= Lc need the ancestor bit, keys >= T / tail are invisible
      if (p0 + 64 > Lc) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int p = p0 + 8 * j + 2 * t + e;
            if (p >= Lc) {
              const int jj = p - Lc;
              const bool va = jj < a.Nq && (a.causal ? jj <= ra / a.G
                                                      : ((s_anc[la * kAncWords + (jj >> 6)] >> (jj & 63)) & 1ull));
              const bool vbb = jj < a.Nq && (a.causal ? jj <= rb / a.G
                                                       : ((s_anc[lb * kAncWords + (jj >> 6)] >> (jj & 63)) & 1ull));
              if (!va) sc[j][e] = -INFINITY;
              if (!vbb) sc[j][2 + e] = -INFINITY;
            }
          }
        }
      }
      // online softmax (rows a: c0,c1; rows b: c2,c3), reductions over the quad
      float mxa = -INFINITY, mxb = -INFINITY;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        mxa = fmaxf(mxa, fmaxf(sc[j][0], sc[j][1]));
        mxb = fmaxf(mxb, fmaxf(sc[j][2], sc[j][3]));
      }
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 1));
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 2));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 1));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 2));
      const float mna = fmaxf(m_a, mxa), mnb = fmaxf(m_b, mxb);
      const float basea = (mna == -INFINITY) ? 0.f : mna * sl2;
      const float baseb = (mnb == -INFINITY) ? 0.f : mnb * sl2;
      const float alpha_a = exp2f(m_a * sl2 - basea);
      const float alpha_b = exp2f(m_b * sl2 - baseb);
      m_a = mna;
      m_b = mnb;
      float suma = 0.f, sumb = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sc[j][0] = exp2f(sc[j][0] * sl2 - basea);
        sc[j][1] = exp2f(sc[j][1] * sl2 - basea);
        sc[j][2] = exp2f(sc[j][2] * sl2 - baseb);
        sc[j][3] = exp2f(sc[j][3] * sl2 - baseb);
        suma += sc[j][0] + sc[j][1];
        sumb += sc[j][2] + sc[j][3];
      }
      l_a = l_a * alpha_a + suma;
      l_b = l_b * alpha_b + sumb;
#pragma unroll
      for (int j = 0; j < HD / 8; ++j) {
        o[j][0] *= alpha_a;
        o[j][1] *= alpha_a;
        o[j][2] *= alpha_b;
        o[j][3] *= alpha_b;
      }
      // O += P V   (P from registers as the A operand, V via ldmatrix.trans)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t pa[4];
        pa[0] = pack_bf16(sc[2 * kk][0], sc[2 * kk][1]);
        pa[1] = pack_bf16(sc[2 * kk][2], sc[2 * kk][3]);
        pa[2] = pack_bf16(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
        pa[3] = pack_bf16(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
        for (int jq = 0; jq < HD / 16; ++jq) {
          uint32_t b0, b1, b2, b3;
          const int key = kk * 16 + (((lane >> 3) & 1) << 3) + (lane & 7);
          const int ch = jq * 2 + (lane >> 4);
          ldmatrix_x4_trans(vb + tile_off<HD>(key, ch), b0, b1, b2, b3);
          mma_bf16_16816(o[2 * jq], pa, b0, b1);
          mma_bf16_16816(o[2 * jq + 1], pa, b2, b3);
        }
      }
    }
    __syncthreads();  // every warp is done with stage s
    if (threadIdx.x == 0 && i + C::kStages < ntiles) issue(i + C::kStages);
  }

  l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);

  auto out_row = [&](int r) -> bf16 * {  // global output row of query row r
    const int n = r / a.G, gg = r % a.G;
    const long long m = (long long)sl * a.Nq + n;
    return a.out + (m * a.H + (long long)h * a.G + gg) * HD;
  };
  if (a.nsplit == 1) {
    if (!warp_active) return;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int r = half ? rb : ra;
      if (r >= R) continue;
      const float inv = 1.f / (half ? l_b : l_a);
      bf16 *dst = out_row(r);
#pragma unroll
      for (int j = 0; j < HD / 8; ++j) {
        const float v0 = o[j][2 * half] * inv, v1 = o[j][2 * half + 1] * inv;
        *reinterpret_cast<uint32_t *>(dst + 8 * j + 2 * t) = pack_bf16(v0, v1);
      }
    }
    return;
  }
  // ---- cluster combine: stage (m, l, O) of the 64 local rows in shared memory
  // (the K/V ring is idle: every issued tile has been consumed)
  float *so = reinterpret_cast<float *>(smem);  // [64][HD]
  float *sml = so + 64 * HD;                    // [64][2]
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int lr = half ? lb : la;
    const bool live = warp_active && (half ? rb : ra) < R;
#pragma unroll
    for (int j = 0; j < HD / 8; ++j)
      *reinterpret_cast<float2 *>(so + lr * HD + 8 * j + 2 * t) =
          live ? make_float2(o[j][2 * half], o[j][2 * half + 1]) : make_float2(0.f, 0.f);
    if (t == 0) {
      sml[2 * lr] = live ? (half ? m_b : m_a) : -INFINITY;
      sml[2 * lr + 1] = live ? (half ? l_b : l_a) : 0.f;
    }
  }
  cluster_sync_all();
  // rank `split` combines local rows [split * 64/nsplit, (split+1) * 64/nsplit)
  const int rows_per = 64 / a.nsplit;
  const uint32_t so_u = smem_u32(so), sml_u = smem_u32(sml);
  for (int e = threadIdx.x; e < rows_per * HD; e += blockDim.x) {
    const int lr = split * rows_per + e / HD, dcol = e % HD;
    const int r = rblk * 64 + lr;
    if (r >= R) continue;
    // every rank's (m, l, o) is loaded before any is used: one DSMEM round trip
    float mq[8], lq[8], oq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const bool ok = q < a.nsplit;
      mq[q] = ok ? ld_dsmem_f32(mapa_u32(sml_u + 8 * lr, q)) : -INFINITY;
      lq[q] = ok ? ld_dsmem_f32(mapa_u32(sml_u + 8 * lr + 4, q)) : 0.f;
      oq[q] = ok ? ld_dsmem_f32(mapa_u32(so_u + 4 * (lr * HD + dcol), q)) : 0.f;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < 8; ++q) mx = fmaxf(mx, mq[q]);
    const float base = mx * sl2;
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // fixed rank order -> deterministic
      const float w = mq[q] == -INFINITY ? 0.f : exp2f(mq[q] * sl2 - base);
      L += w * lq[q];
      acc += w * oq[q];
    }
    out_row(r)[dcol] = f2bf(acc / L);
  }
  cluster_sync_all();  // keep every CTA's shared memory alive until all remote reads are done
}

static int g_attn_tc = 1;  // head_dim 128 on tcgen05 (sm_set_option "attn_tc")
static int g_attn_splits = 0;  // experiments: force the key-split count (sm_set_option "attn_splits", 0 = auto)
// tree mode, head_dim 128: the stream-K ("lean") tcgen05 kernel (1, default) or the cluster-split one (0)
static int g_attn_lean = 0;
static int g_lean_div = 16;  // lean K1: minimum tiles per CTA = max(2, live rows per unit / g_lean_div)
void attention_set_lean(int on) { g_attn_lean = on; }
void attention_set_lean_div(int d) { g_lean_div = d < 1 ? 1 : d; }
int attention_lean_min_tiles(int Nq, int G) { return std::max(2, std::min(128, Nq * G) / g_lean_div); }
void attention_set_tc(int on) { g_attn_tc = on; }
void attention_set_splits(int n) { g_attn_splits = n; }
static bool use_tc(int head_dim) { return g_attn_tc && head_dim == 128; }
int attention_row_blocks(int Nq, int G, int head_dim) {
  const int rows = use_tc(head_dim) ? 128 : 64;
  return (Nq * G + rows - 1) / rows;
}

template <int HD>
static cudaError_t launch_hd(const AttnArgs &a, cudaStream_t st) {
  using C = AttnCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tree_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.nsplit, (a.Nq * a.G + 63) / 64, a.nseq * a.Hkv);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = gemm_pdl() ? 1 : 0;
  attrs[1].id = cudaLaunchAttributeClusterDimension;
  attrs[1].val.clusterDim.x = a.nsplit;
  attrs[1].val.clusterDim.y = 1;
  attrs[1].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = a.nsplit > 1 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, tree_attn_kernel<HD>, a);
}

// nsplit = cluster size in {1, 2, 4, 8}: enough CTAs to cover ~2 waves of SMs
int attention_tc_nsplit(int units, int cap);
cudaError_t attention_tc_launch(const AttnArgs &a, cudaStream_t st);

int attention_nsplit(int units, int head_dim, int cap) {
  if (g_attn_splits >= 1 && g_attn_splits <= 8) return g_attn_splits;
  if (use_tc(head_dim)) return attention_tc_nsplit(units, cap);
  int ns = 1;
  while (ns < 8 && units * ns < 2 * kNumSMs) ns *= 2;
  return ns;
}

cudaError_t attention_launch(const AttnArgs &a, int head_dim, cudaStream_t st) {
  switch (head_dim) {
    case 16: return launch_hd<16>(a, st);
    case 32: return launch_hd<32>(a, st);
    case 64: return launch_hd<64>(a, st);
    case 128:
      if (use_tc(128) && g_attn_lean && !a.causal && a.lean_part && a.nseq <= kLeanMaxSeq)
        return attention_lean_launch(a, st);
      return use_tc(128) ? attention_tc_launch(a, st) : launch_hd<128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

void attention_preload() {  // force-load (see gemm_preload)
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, tree_attn_kernel<16>);
  cudaFuncGetAttributes(&fa, tree_attn_kernel<32>);
  cudaFuncGetAttributes(&fa, tree_attn_kernel<64>);
  cudaFuncGetAttributes(&fa, tree_attn_kernel<128>);
}

}  // namespace sm
