// gemm.cu -- K2: small-M bf16 GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA),
// persistent and stream-K balanced; fp32 partials reduced by the consumer.
//
//   y[m][n] = sum_k x[m][k] * w[n][k]      (x: token rows, w: nn.Linear weight)
//
// Swap-AB: the weight tile (128 output features x 64 k, K-major, SWIZZLE_128B)
// is the UMMA A operand (M = 128 TMEM lanes); the token rows (BN <= 256, padded
// to 16) are the UMMA N dimension, so b*N = 1..256 rows never waste the 128-row
// MMA.  The path is HBM-bound: every weight byte is read once.
//
// Work split: U = tiles x k-blocks units are divided evenly over P CTAs (one per
// SM), so no SM idles in a partial wave.  A CTA walks its contiguous unit range;
// each maximal run inside one tile is a "segment" whose fp32 accumulator goes to
// the partial slot (tile, contributor) -- no atomics, no fences, no serial
// fixup tail.  The consumer kernels (epilogue.cu) sum a tile's contributors in
// CTA order (deterministic) and fuse the next elementwise step.
//
// Warp roles (192 threads): warp 0 = TMA producer (1 lane), warp 1 = tcgen05.mma
// issuer (1 lane) + TMEM allocator, warps 2..5 = epilogue (tcgen05.ld; warp w
// reads TMEM lanes 32*(w%4)..+31).  Two TMEM accumulators let the MMA of the
// next segment overlap the write-out of the previous one.
//
// Programmatic dependent launch: weights do not depend on the previous kernel,
// so the producer streams the first STAGES weight tiles before
// griddepcontrol.wait; activations are loaded after it.
#include "common.cuh"
#include "kernels.h"

namespace sm {

template <int BN, int SMEMKB>
struct GemmCfg {
  static constexpr int kA = 128 * 64 * 2;  // weight tile bytes
  static constexpr int kB = BN * 64 * 2;   // activation tile bytes
  static constexpr int kStage = kA + kB;
  static constexpr int kStages = (SMEMKB * 1024) / kStage;  // 216 KB: 1 CTA/SM; 104 KB: 2 may co-reside
  static constexpr int kChunk = BN < 32 ? BN : 32;  // token columns per tcgen05.ld
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr int kSmem = kStages * kStage + 1024 + 256;
};

SM_DEV void tmem_ld32(uint32_t taddr, float *v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
      "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
template <int C>
SM_DEV void tmem_ldc(uint32_t taddr, float *v) {
  if constexpr (C == 32) {
    tmem_ld32(taddr, v);
  } else {
    float t[16];
    tmem_ld16(taddr, t);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = t[i];
  }
}

SM_DEV void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }  // the 4 epilogue warps

// Fused tile epilogue (see kernels.h, kEpi*), run by the last contributor of tile t
// with the 128 epilogue threads: thread et owns the feature pair (p, p + 64) of the
// tile -- a RoPE pair (hd = 128), a gate/up pair, or two residual columns -- for the
// token columns ml = half, half + 2, ... of the tile.  Partial slots are read from L2.
template <int BN>
SM_DEV void fused_fixup(const GemmArgs &a, int t, int nc, int et) {
  const SplitPlan &pl = a.plan;
  const EpiArgs &e = a.e;
  int bi, tt, mt;
  sk_decode(t, pl, bi, tt, mt);
  const int p = et & 63, half = et >> 6, w = et >> 5;
  const int rows = min(BN, a.M - tt * BN);
  const float *base = a.ws + (size_t)t * pl.maxc * BN * 128 + p;
  const size_t kstride = (size_t)BN * 128;
  constexpr int CB = BN >= 8 ? 4 : 1;  // token columns per batch: CB x 8 contributors x 2 loads in flight
  constexpr int KM = 8;
  for (int ml0 = half * CB; ml0 < rows; ml0 += 2 * CB) {
    float v0[CB][KM], v1[CB][KM];
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const float *col = base + (size_t)(ml0 + c) * 128;
#pragma unroll
      for (int k = 0; k < KM; ++k) {
        const bool ok = k < nc && ml0 + c < rows;
        v0[c][k] = ok ? __ldcg(col + k * kstride) : 0.f;
        v1[c][k] = ok ? __ldcg(col + k * kstride + 64) : 0.f;
      }
    }
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const int ml = ml0 + c;
      float y0 = 0.f, y1 = 0.f;
#pragma unroll
      for (int k = 0; k < KM; ++k) {  // contributor order: identical to the consumer kernels' sums
        if (k < nc) {
          y0 += v0[c][k];
          y1 += v1[c][k];
        }
      }
      for (int k = KM; k < nc; ++k) {
        const float *col = base + (size_t)ml * 128;
        y0 += __ldcg(col + k * kstride);
        y1 += __ldcg(col + k * kstride + 64);
      }
      const bool live = ml < rows;  // all lanes of a warp share ml (warp_sum below)
      const int m = tt * BN + (live ? ml : 0);
      if (a.epi == kEpiQKV) {
        if (!live) continue;
        const float r = e.rs_in[m];
        float x0 = y0 * r, x1 = y1 * r;
        const int hh = mt, sl = m / e.rc.Nq, node = m % e.rc.Nq;
        const int seq = e.rc.seq_base + sl;
        const int Lc = e.rc.len[seq];
        if (hh < e.H + e.Hkv) {  // rotate-half RoPE at pos = Lc + depth
          const float2 cs = e.rope[(size_t)((e.rc.pos ? e.rc.pos[seq] : Lc) + e.rc.depth[node]) * 64 + p];
          const float o0 = x0 * cs.x - x1 * cs.y;
          const float o1 = x1 * cs.x + x0 * cs.y;
          x0 = o0;
          x1 = o1;
        }
        bf16 *dst;
        if (hh < e.H)
          dst = e.q + ((size_t)m * e.H + hh) * 128;
        else if (hh < e.H + e.Hkv)
          dst = e.kc + (((size_t)seq * e.Hkv + (hh - e.H)) * e.cap + Lc + node) * 128;
        else
          dst = e.vc + (((size_t)seq * e.Hkv + (hh - e.H - e.Hkv)) * e.cap + Lc + node) * 128;
        dst[p] = __float2bfloat16_rn(x0);
        dst[p + 64] = __float2bfloat16_rn(x1);
      } else if (a.epi == kEpiSiLU) {
        if (!live) continue;
        const float r = e.rs_in[m];
        const float gg = y0 * r, uu = y1 * r;
        e.act[(size_t)m * e.F + mt * 64 + p] = __float2bfloat16_rn(gg / (1.0f + expf(-gg)) * uu);
      } else {  // kEpiResid
        const int n0 = mt * 128 + p, n1 = n0 + 64;
        float sq = 0.f;
        if (live) {
          float *xr = e.x + (size_t)m * e.d;
          const float x0 = xr[n0] + y0, x1 = xr[n1] + y1;
          xr[n0] = x0;
          xr[n1] = x1;
          e.h[(size_t)m * e.d + n0] = __float2bfloat16_rn(x0 * __bfloat162float(e.g[n0]));
          e.h[(size_t)m * e.d + n1] = __float2bfloat16_rn(x1 * __bfloat162float(e.g[n1]));
          sq = x0 * x0 + x1 * x1;
        }
        sq = warp_sum(sq);  // lanes of a warp share (half, ml)
        if (live && (et & 31) == 0) e.ss[(size_t)m * (e.d / 64) + mt * 2 + (w & 1)] = sq;
      }
    }
  }
}

// kEpiResid: the last tile of the launch turns the sum-of-squares partials into the
// deferred-norm scale rs[m] = 1/sqrt(sum/d + eps), fixed summation order (warp w: rows w, w+4, ...).
SM_DEV void resid_rs(const GemmArgs &a, int et) {
  const EpiArgs &e = a.e;
  const int nss = e.d / 64, lane = et & 31;
  for (int m = et >> 5; m < a.M; m += 4) {
    float s = 0.f;
    for (int j = lane; j < nss; j += 32) s += __ldcg(e.ss + (size_t)m * nss + j);
    s = warp_sum(s);
    if (lane == 0) e.rs_out[m] = 1.0f / sqrtf(s / (float)e.d + e.eps);
  }
}

// FUSED: compiled with the tile-epilogue fixup (GemmArgs.epi != 0).  The plain variant
// carries none of that code: its register count (96) leaves room on an SM for the
// consumer kernel's CTAs to become resident (and wait) while the GEMM still runs.
// GROUPS: compiled for token-tile CTA groups (SplitPlan::rep > 1, BN = 256 only); the decode
// variants keep rep = 1 as a compile-time constant (their index math folds away).
template <int BN, int SMEMKB, bool FUSED, bool GROUPS = false>
__global__ void __launch_bounds__(192, 1) gemm_streamk_kernel(const __grid_constant__ GemmArgs a) {
  using C = GemmCfg<BN, SMEMKB>;
  constexpr int CH = C::kChunk;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::kStages * C::kA;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::kStages * C::kStage);
  uint64_t *empty = full + C::kStages;
  uint64_t *tfull = empty + C::kStages;  // [2]
  uint64_t *tempty = tfull + 2;          // [2]
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);
  int *s_flag = reinterpret_cast<int *>(tslot + 1);  // fused epilogue: "this CTA fixes up the tile"

  SM_GT_BEGIN();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const SplitPlan &pl = a.plan;
  const int c = blockIdx.x;
  const int rep = GROUPS ? pl.rep : 1;
  const int g = c / rep, ttr = c % rep;  // CTA group and token-tile lane (SplitPlan::rep)
  const long long u0 = sk_unit0(g, pl), u1 = sk_unit0(g + 1, pl);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.tmW[0]);
    tma_prefetch_desc(&a.tmX[0]);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();  // let the consumer launch now and wait on our completion
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      // weights stream through once; with several token tiles they are re-read right away
      const uint64_t pol_w = pl.token_tiles > 1 ? policy_evict_last() : policy_evict_first();
      const bool wonly = a.dbg_mode == 1;
      const uint32_t stage_bytes = wonly ? (uint32_t)C::kA : (uint32_t)C::kStage;
      auto issue_x = [&](int s, int bi, int tt, int kc) {  // activation rows [tt*BN, tt*BN + BN)
        if (wonly) return;
        if constexpr (BN >= 64) {  // tmX64 is encoded with a BN-row box: one request per stage
          tma_load_2d(sB + s * C::kB, &a.tmX64[bi], &full[s], kc, a.x_row0 + tt * BN);
        } else {
#pragma unroll
          for (int r = 0; r < BN / 16; ++r)
            tma_load_2d(sB + s * C::kB + r * 2048, &a.tmX[bi], &full[s], kc, a.x_row0 + tt * BN + r * 16);
        }
      };
      int pre = (u1 - u0) < (long long)C::kStages ? (int)(u1 - u0) : C::kStages;
      if (a.pre_stages >= 0 && a.pre_stages < pre) pre = a.pre_stages;
      for (int i = 0; i < pre; ++i) {  // weights first: independent of the previous kernel
        const long long u = u0 + i;
        int bi, tt, mt;
        sk_decode((int)(u / pl.kb_total) * rep + ttr, pl, bi, tt, mt);
        mbar_arrive_expect_tx(&full[i], stage_bytes);
        tma_load_2d_hint(sA + i * C::kA, &a.tmW[bi], &full[i], sk_kb(u, pl) * 64, mt * 128, pol_w);
      }
      // optionally pull the following weight tiles into L2 across the kernel boundary
      for (int i = pre; i < pre + a.l2_prefetch && u0 + i < u1; ++i) {
        const long long u = u0 + i;
        int bi, tt, mt;
        sk_decode((int)(u / pl.kb_total) * rep + ttr, pl, bi, tt, mt);
        tma_prefetch_l2_2d(&a.tmW[bi], sk_kb(u, pl) * 64, mt * 128);
      }
      pdl_wait();  // activations only after the producer kernel completed
      SM_GT_WAITED();
      for (int i = 0; i < pre; ++i) {
        const long long u = u0 + i;
        int bi, tt, mt;
        sk_decode((int)(u / pl.kb_total) * rep + ttr, pl, bi, tt, mt);
        issue_x(i, bi, tt, sk_kb(u, pl) * 64);
      }
      for (long long u = u0 + pre; u < u1; ++u) {
        const int i = (int)(u - u0);
        const int s = i % C::kStages;
        if (i >= C::kStages) mbar_wait(&empty[s], ((i / C::kStages) - 1) & 1);
        int bi, tt, mt;
        sk_decode((int)(u / pl.kb_total) * rep + ttr, pl, bi, tt, mt);
        const int kc = sk_kb(u, pl) * 64;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        tma_load_2d_hint(sA + s * C::kA, &a.tmW[bi], &full[s], kc, mt * 128, pol_w);
        issue_x(s, bi, tt, kc);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
      int seg = 0;
      bool seg_start = true;
      for (long long u = u0; u < u1; ++u) {
        const int i = (int)(u - u0);
        const int s = i % C::kStages;
        const int buf = seg & 1;
        if (seg_start && seg >= 2) mbar_wait(&tempty[buf], ((seg >> 1) - 1) & 1);
        mbar_wait(&full[s], (i / C::kStages) & 1);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * C::kA));
        const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * C::kB));
        const uint32_t td = tmem + buf * BN;
        if (a.dbg_mode == 1) {  // weights-only streaming experiment: no MMA
          mbar_arrive(&empty[s]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_bf16(td, ad + 2 * k, bd + 2 * k, idesc, (!seg_start || k > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        seg_start = false;
        if ((u + 1) % pl.kb_total == 0 || u + 1 == u1) {
          if (a.dbg_mode == 1)
            mbar_arrive(&tfull[buf]);
          else
            umma_commit(&tfull[buf]);
          ++seg;
          seg_start = true;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31
    const int wq = warp & 3;
    const int lrow = wq * 32 + lane;  // feature row inside the tile (= TMEM lane)
    int seg = 0;
    long long u = u0;
    while (u < u1) {
      const int t = (int)(u / pl.kb_total) * rep + ttr;
      const long long seg_end = min(u1, (long long)(t / rep + 1) * pl.kb_total);
      const int buf = seg & 1;
      mbar_wait(&tfull[buf], (seg >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(wq * 32) << 16) + buf * BN;
      float *dst = sk_partial(a.ws, pl, t, g - sk_cta_of((long long)(t / rep) * pl.kb_total, pl));
      for (int c0 = 0; c0 < BN; c0 += CH) {
        float v[CH];
        tmem_ldc<CH>(tbase + c0, v);
#pragma unroll
        for (int j = 0; j < CH; ++j) dst[(size_t)(c0 + j) * 128 + lrow] = v[j];  // coalesced 512 B rows
      }
      tc_fence_before();
      mbar_arrive(&tempty[buf]);
      if (FUSED && a.epi != kEpiPartial) {  // last contributor of tile t applies the fused epilogue
        const int et = threadIdx.x - 64;
        const int nc = sk_ncontrib(t, pl);
        __threadfence();
        epi_bar();
        if (et == 0) *s_flag = atomicAdd(&a.e.tile_cnt[t], 1) == nc - 1;
        epi_bar();
        if (*s_flag) {
          __threadfence();
          if (a.dbg_mode != 2) fused_fixup<BN>(a, t, nc, et);  // experiments: 2 = protocol only
          if (a.epi == kEpiResid) {
            __threadfence();
            epi_bar();
            if (et == 0) {
              a.e.tile_cnt[t] = 0;
              *s_flag = atomicAdd(a.e.done_cnt, 1) == pl.tiles - 1;
            }
            epi_bar();
            if (*s_flag) {
              __threadfence();
              resid_rs(a, et);
              if (et == 0) *a.e.done_cnt = 0;
            }
          } else if (et == 0) {
            a.e.tile_cnt[t] = 0;
          }
        }
        epi_bar();  // s_flag is reused by the next segment
      }
      u = seg_end;
      ++seg;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
  if (threadIdx.x == 0) SM_GT_END(1000 + a.N / 128);
}

// ------------------------------------------------------------------ 2-SM variant (cta_group::2)
// The CTA pair of a cluster computes a 256-row weight tile x BN token rows per unit: CTA r
// loads weight rows [256 t + 128 r, +128) and token rows [BN/2 r, +BN/2) of the stage, the
// leader (rank 0) issues tcgen05.mma.cta_group::2 (M = 256, N = BN) reading both CTAs'
// shared memory, and each CTA's TMEM receives its own 128 weight rows x BN tokens.  Per SM
// the activation bytes per stage halve (BN/2 rows instead of BN), which is what limits the
// single-SM kernel for BN >= 96: every stage re-reads the activation tile from L2.
template <int BN, int SMEMKB>
struct PairCfg {
  static constexpr int kA = 128 * 64 * 2;
  static constexpr int kB = (BN / 2) * 64 * 2;
  static constexpr int kStage = kA + kB;
  static constexpr int kStages = (SMEMKB * 1024) / kStage;
  // TMEM accumulator buffers: two (the MMA of the next segment overlaps the epilogue) unless
  // two CTAs share the SM and 2 x BN columns would not fit twice into its 512 columns
  static constexpr int kNBuf = (2 * BN <= 256 || SMEMKB > 104) ? 2 : 1;
  static constexpr int kTmemCols = kNBuf * BN <= 128 ? 128 : kNBuf * BN <= 256 ? 256 : 512;
  static constexpr int kSmem = kStages * kStage + 1024 + 256;
};

template <int BN, int SMEMKB, bool GROUPS = false>
__global__ void __launch_bounds__(192, 1) gemm_pair_kernel(const __grid_constant__ GemmArgs a) {
  using C = PairCfg<BN, SMEMKB>;
  static_assert(BN % 32 == 0 && BN >= 64, "pair tiles: BN >= 64, BN/2 a multiple of 16");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::kStages * C::kA;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::kStages * C::kStage);
  uint64_t *empty = full + C::kStages;
  uint64_t *tfull = empty + C::kStages;  // [2]
  uint64_t *tempty = tfull + 2;          // [2] (leader's: 128 arrivals from each CTA)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);

  SM_GT_BEGIN();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const SplitPlan &pl = a.plan;
  const int rank = (int)cluster_ctarank();
  const int c = blockIdx.x >> 1;  // cluster = work unit owner
  const int rep = GROUPS ? pl.rep : 1;
  const int g = c / rep, ttr = c % rep;  // cluster group and token-tile lane (SplitPlan::rep)
  const long long u0 = sk_unit0(g, pl), u1 = sk_unit0(g + 1, pl);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.tmW[0]);
    tma_prefetch_desc(&a.tmX64[0]);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2<C::kTmemCols>(tslot);
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA arrive / TMA
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs; completion counted on the leader's barriers)
      const uint64_t pol_w = pl.token_tiles > 1 ? policy_evict_last() : policy_evict_first();
      const uint32_t full_cl0 = mapa_u32(smem_u32(&full[0]), 0);
      auto load_w = [&](int s, long long u) {
        int bi, tt, mt;
        sk_decode((int)(u / pl.kb_total) * rep + ttr, pl, bi, tt, mt);
        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * C::kStage);  // both CTAs' W and X bytes
        tma_load_2d_cg2_hint(sA + s * C::kA, &a.tmW[0], full_cl0 + 8 * s, sk_kb(u, pl) * 64, (mt * 2 + rank) * 128,
                             pol_w);
      };
      auto load_x = [&](int s, long long u) {
        int bi, tt, mt;
        sk_decode((int)(u / pl.kb_total) * rep + ttr, pl, bi, tt, mt);
        tma_load_2d_cg2(sB + s * C::kB, &a.tmX64[0], full_cl0 + 8 * s, sk_kb(u, pl) * 64,
                        a.x_row0 + tt * BN + rank * (BN / 2));
      };
      int pre = (u1 - u0) < (long long)C::kStages ? (int)(u1 - u0) : C::kStages;
      if (a.pre_stages >= 0 && a.pre_stages < pre) pre = a.pre_stages;
      for (int i = 0; i < pre; ++i) load_w(i, u0 + i);  // weights: independent of the previous kernel
      pdl_wait();
      SM_GT_WAITED();
      for (int i = 0; i < pre; ++i) load_x(i, u0 + i);
      for (long long u = u0 + pre; u < u1; ++u) {
        const int i = (int)(u - u0);
        const int s = i % C::kStages;
        if (i >= C::kStages) mbar_wait(&empty[s], ((i / C::kStages) - 1) & 1);
        load_w(s, u);
        load_x(s, u);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader only): M = 256 across the pair
      constexpr uint32_t idesc = umma_idesc_bf16(256, BN);
      int seg = 0;
      bool seg_start = true;
      for (long long u = u0; u < u1; ++u) {
        const int i = (int)(u - u0);
        const int s = i % C::kStages;
        const int buf = seg % C::kNBuf;
        if (seg_start && seg >= C::kNBuf) mbar_wait(&tempty[buf], ((seg / C::kNBuf) - 1) & 1);
        mbar_wait(&full[s], (i / C::kStages) & 1);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * C::kA));
        const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * C::kB));
        const uint32_t td = tmem + buf * BN;
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_bf16_cg2(td, ad + 2 * k, bd + 2 * k, idesc, (!seg_start || k > 0) ? 1u : 0u);
        umma_commit_cg2(&empty[s], 0x3);
        seg_start = false;
        if ((u + 1) % pl.kb_total == 0 || u + 1 == u1) {
          umma_commit_cg2(&tfull[buf], 0x3);
          ++seg;
          seg_start = true;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 of both CTAs: this CTA's 128 weight rows
    const int wq = warp & 3;
    const int lrow = wq * 32 + lane;
    const uint32_t tempty_cl0 = mapa_u32(smem_u32(&tempty[0]), 0);
    int seg = 0;
    long long u = u0;
    while (u < u1) {
      const int t = (int)(u / pl.kb_total) * rep + ttr;
      const long long seg_end = min(u1, (long long)(t / rep + 1) * pl.kb_total);
      const int buf = seg % C::kNBuf;
      mbar_wait(&tfull[buf], (seg / C::kNBuf) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(wq * 32) << 16) + buf * BN;
      float *dst = sk_partial(a.ws, pl, t, g - sk_cta_of((long long)(t / rep) * pl.kb_total, pl), rank);
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(tbase + c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[(size_t)(c0 + j) * 128 + lrow] = v[j];
      }
      tc_fence_before();
      mbar_arrive_cluster(tempty_cl0 + 8 * buf);
      u = seg_end;
      ++seg;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no cross-CTA arrivals or MMAs remain
  tc_fence_after();
  if (warp == 1) tmem_dealloc_cg2<C::kTmemCols>(tmem);
  if (threadIdx.x == 0) SM_GT_END(2000 + a.N / 128);
}

static bool g_pdl = true;
static int g_ctas = 0;
static int g_rep = 1;  // sm_set_option("gemm_rep"): token-tile CTA groups (SplitPlan::rep); 0 = plain stream-K
static int g_l2pf = 0;
static int g_dbg_mode = 0;
static int g_force_bn = 0;
// 2-SM MMA (cta_group::2): 0 off; 1 (default) for token tiles of 96..160 rows and for 256-row
// tiles when there are several (measured faster there, slower at M = 64 and for one 192- or
// 256-row tile); 2 for every tile of >= 64 rows (experiments)
static int g_pair = 1;
// weight stages issued before griddepcontrol.wait: -2 (default) = 2 for single-SM GEMMs of one token tile
// (decode: measured -0.5 % C2 step vs the whole ring, tools/bench A/B), the whole ring otherwise;
// -1 = the whole ring; n >= 0 = n stages (sm_set_option "gemm_pre")
static int g_pre_stages = -2;
static int g_occ = 2;  // GEMM CTAs per SM for BN <= 64 (1..4); grid = 148 * occ
void gemm_set_bn(int bn) { g_force_bn = bn; }
void gemm_set_pair(int mode) { g_pair = mode < 0 ? 0 : (mode > 2 ? 2 : mode); }
void gemm_set_pre_stages(int n) { g_pre_stages = n; }
static int g_occ_smalln = 0;  // experiments: occupancy for GEMMs with N <= 8192 (0 = g_occ)
void gemm_set_small(int v) { g_occ = v < 1 ? 1 : (v > 4 ? 4 : v); }
void gemm_set_occ_smalln(int v) { g_occ_smalln = v < 0 ? 0 : (v > 4 ? 4 : v); }
int gemm_occ_for(int bn, int N = 1 << 30) {
  if (bn > 64) return 1;
  return (g_occ_smalln > 0 && N <= 8192) ? g_occ_smalln : g_occ;
}
void gemm_set_debug_mode(int m) { g_dbg_mode = m; }
void gemm_set_pdl(bool on) { g_pdl = on; }
bool gemm_pdl() { return g_pdl; }
void gemm_set_ctas(int n) { g_ctas = n; }
void gemm_set_rep(int on) { g_rep = on ? 1 : 0; }
void gemm_set_l2_prefetch(int kblocks) { g_l2pf = kblocks < 0 ? 0 : kblocks; }

template <int BN, int SMEMKB>
static cudaError_t launch_bn(const GemmArgs &a, cudaStream_t st) {
  if constexpr (BN == 256) {
    if (a.plan.rep > 1) {  // token-tile groups (plain partial epilogue only)
      static bool gattr = false;
      if (!gattr) {
        cudaError_t e = cudaFuncSetAttribute(gemm_streamk_kernel<BN, SMEMKB, false, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN, SMEMKB>::kSmem);
        if (e != cudaSuccess) return e;
        gattr = true;
      }
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(a.plan.P * a.plan.rep);
      cfg.blockDim = dim3(192);
      cfg.dynamicSmemBytes = GemmCfg<BN, SMEMKB>::kSmem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, gemm_streamk_kernel<BN, SMEMKB, false, true>, a);
    }
  }
  if (a.plan.rep > 1) return cudaErrorInvalidValue;
  using C = GemmCfg<BN, SMEMKB>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_streamk_kernel<BN, SMEMKB, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_streamk_kernel<BN, SMEMKB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.plan.P);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.epi != kEpiPartial) return cudaLaunchKernelEx(&cfg, gemm_streamk_kernel<BN, SMEMKB, true>, a);
  return cudaLaunchKernelEx(&cfg, gemm_streamk_kernel<BN, SMEMKB, false>, a);
}

// Token-tile width: the smallest supported UMMA N (multiple of 16) covering M, so one
// token tile holds every row up to 256 (each weight tile then crosses shared memory
// once) and padding MMA work stays small (C4: b*N = 10 x 16 = 160 rows -> BN 160).
template <int BN, int SMEMKB, bool GROUPS>
static cudaError_t launch_pair_v(const GemmArgs &a, cudaStream_t st) {
  using C = PairCfg<BN, SMEMKB>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_pair_kernel<BN, SMEMKB, GROUPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * a.plan.P * (GROUPS ? a.plan.rep : 1));
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, gemm_pair_kernel<BN, SMEMKB, GROUPS>, a);
}
template <int BN, int SMEMKB>
static cudaError_t launch_pair(const GemmArgs &a, cudaStream_t st) {
  if constexpr (BN == 256) {
    if (a.plan.rep > 1) return launch_pair_v<BN, SMEMKB, true>(a, st);
  }
  if (a.plan.rep > 1) return cudaErrorInvalidValue;
  return launch_pair_v<BN, SMEMKB, false>(a, st);
}

int gemm_pick_bn(int M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 96) return 96;
  if (M <= 128) return 128;
  if (M <= 160) return 160;
  if (M <= 192) return 192;
  return 256;
}

void gemm_plan(GemmArgs &a, int N, int K, int M, int batch) {
  a.N = N;
  a.K = K;
  a.M = M;
  a.batch = batch;
  SplitPlan &p = a.plan;
  p.bn = g_force_bn > 0 ? g_force_bn : gemm_pick_bn(M);
  const int ttiles = (M + p.bn - 1) / p.bn;
  // measured (tools/gemm_pair.py, tools/gemm_m128.py): the pair wins for 96..160-row tiles and for several
  // 256-row tiles, loses for 64-row tiles, a single 192- or 256-row tile
  const bool pair_ok = (g_pair == 1 && ((p.bn >= 96 && p.bn <= 160) || (p.bn == 256 && ttiles > 1))) ||
                       (g_pair == 2 && p.bn >= 64);
  p.pair = (!a.no_pair && batch == 1 && pair_ok) ? 2 : 1;
  p.m_tiles = (N + 128 * p.pair - 1) / (128 * p.pair);
  p.token_tiles = (M + p.bn - 1) / p.bn;
  p.tiles = p.m_tiles * p.token_tiles * batch;
  p.kb_total = (K + 63) / 64;
  p.occ = gemm_occ_for(p.bn, N);
  int want = g_ctas > 0 ? g_ctas : kNumSMs * p.occ;
  if (p.pair == 2) want = g_ctas > 0 ? g_ctas / 2 : kNumSMs;  // clusters of 2 CTAs, 2 CTAs per SM
  // several token tiles (tensor-bound M): groups of token_tiles CTAs walk the same weight
  // k-blocks together (SplitPlan::rep) -- measured: plain stream-K re-read the weights from HBM
  // ~3.7x at M = 1024 (the token tiles of a weight tile ran far apart in time)
  p.rep = (g_rep && p.bn == 256 && p.token_tiles > 1 && !a.no_pair && want / p.token_tiles >= 1) ? p.token_tiles
                                                                                                  : 1;  // not fused
  const long long U = (long long)(p.tiles / p.rep) * p.kb_total;
  want /= p.rep;
  p.P = (int)(U < want ? U : want);
  p.U = U;
  // contributors per tile <= ceil(KB / floor(U/P)) + 1
  const long long per = U / p.P;
  p.maxc = (int)((p.kb_total + per - 1) / per) + 1;
}

size_t gemm_ws_floats(const GemmArgs &a) {
  return (size_t)a.plan.tiles * sk_pair(a.plan) * a.plan.maxc * a.plan.bn * 128;
}

cudaError_t gemm_launch(const GemmArgs &a0, cudaStream_t st) {
  GemmArgs a = a0;
  a.l2_prefetch = g_pdl ? g_l2pf : 0;
  a.pre_stages = g_pre_stages != -2 ? g_pre_stages : (a.plan.pair == 1 && a.plan.token_tiles == 1 ? 2 : -1);
  a.dbg_mode = g_dbg_mode;
  if (a.plan.pair == 2) {
    switch (a.plan.bn) {
      case 64: return launch_pair<64, 104>(a, st);
      case 96: return launch_pair<96, 104>(a, st);
      case 128: return launch_pair<128, 104>(a, st);
      // BN >= 160: two CTAs per SM with one TMEM accumulator buffer each (PairCfg::kNBuf)
      case 160: return launch_pair<160, 104>(a, st);
      case 192: return launch_pair<192, 104>(a, st);
      case 256: return launch_pair<256, 104>(a, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (a.plan.bn) {
    case 16: return a.plan.occ == 4 ? launch_bn<16, 50>(a, st) : a.plan.occ == 3 ? launch_bn<16, 68>(a, st)
                    : a.plan.occ == 2 ? launch_bn<16, 104>(a, st) : launch_bn<16, 216>(a, st);
    case 32: return a.plan.occ == 4 ? launch_bn<32, 50>(a, st) : a.plan.occ == 3 ? launch_bn<32, 68>(a, st)
                    : a.plan.occ == 2 ? launch_bn<32, 104>(a, st) : launch_bn<32, 216>(a, st);
    case 64: return a.plan.occ == 4 ? launch_bn<64, 50>(a, st) : a.plan.occ == 3 ? launch_bn<64, 68>(a, st)
                    : a.plan.occ == 2 ? launch_bn<64, 104>(a, st) : launch_bn<64, 216>(a, st);
    case 80: return launch_bn<80, 104>(a, st);  // experiments (gemm_bn): 2 CTAs per SM at 2 x 80 TMEM columns
    case 96: return launch_bn<96, 216>(a, st);
    case 128: return launch_bn<128, 216>(a, st);
    case 160: return launch_bn<160, 216>(a, st);
    case 192: return launch_bn<192, 216>(a, st);
    default: return launch_bn<256, 216>(a, st);
  }
}

// Force-load every instantiation (lazy module loading would otherwise load a kernel at
// its first launch, which can wait for running kernels -- fatal when those spin on a
// tensor-parallel peer whose work is enqueued later).
template <int BN, int SK>
static void preload_one() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, gemm_streamk_kernel<BN, SK, false>);
  cudaFuncGetAttributes(&fa, gemm_streamk_kernel<BN, SK, true>);
}
void gemm_preload() {
  preload_one<16, 50>(), preload_one<16, 68>(), preload_one<16, 104>(), preload_one<16, 216>();
  preload_one<32, 50>(), preload_one<32, 68>(), preload_one<32, 104>(), preload_one<32, 216>();
  preload_one<64, 50>(), preload_one<64, 68>(), preload_one<64, 104>(), preload_one<64, 216>();
  preload_one<80, 104>(), preload_one<96, 216>(), preload_one<128, 216>(), preload_one<160, 216>();
  preload_one<192, 216>();
  preload_one<256, 216>();
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, gemm_pair_kernel<64, 104>);
  cudaFuncGetAttributes(&fa, gemm_pair_kernel<96, 104>);
  cudaFuncGetAttributes(&fa, gemm_pair_kernel<128, 104>);
  cudaFuncGetAttributes(&fa, gemm_pair_kernel<160, 104>);
  cudaFuncGetAttributes(&fa, gemm_pair_kernel<192, 104>);
  cudaFuncGetAttributes(&fa, gemm_pair_kernel<256, 104>);
  cudaFuncGetAttributes(&fa, gemm_pair_kernel<256, 104, true>);
  cudaFuncGetAttributes(&fa, gemm_streamk_kernel<256, 216, false, true>);
}

SM_GT_READER(sm_gtrace_read_gemm)
}  // namespace sm
