// kernels.h -- host-visible launch interfaces of the sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace sm {

typedef __nv_bfloat16 bf16;
constexpr int kNumSMs = 148;
constexpr int kMaxGemmBatch = 5;
constexpr int kMaxTreeNodes = 256;
constexpr int kAncWords = kMaxTreeNodes / 64;

struct RowCtx {                // forward rows m = (seq - seq_base) * Nq + n
  int M, Nq, seq_base;
  const int32_t *len;          // Lc[seq]: cache slot of node 0
  const int32_t *depth;        // [Nq]
  const int32_t *pos;          // nullable: RoPE position of node 0 (pad batching: tokens, not slots)
};

// ---------------------------------------------------------------- K2 GEMM split plan
// Stream-K partition: U = tiles * kb_total units split evenly over P CTAs, CTA c
// owns [U*c/P, U*(c+1)/P).  Tile t = (bi * m_tiles + mt) * token_tiles + tt
// covers 128 output features x bn token rows.  Every (tile, contributing CTA)
// writes an fp32 partial [bn][128] at slot t * maxc + (c - first CTA of t).
// pair = 2 (2-SM MMA, tcgen05 cta_group::2): a unit's weight tile is 256 rows, held as two
// 128-row halves by the two CTAs of a cluster; P counts clusters, m_tiles counts 256-row
// tiles, and the partial slot of 128-row half r of tile t is (t * pair + r) * maxc + k.
struct SplitPlan {
  long long U;
  int P, bn, m_tiles, token_tiles, tiles, kb_total, maxc;
  int pair;
  int occ;  // GEMM CTAs per SM of the launch (smem variant)
  // rep > 1 (several token tiles, tensor-bound M): U and P count weight-tile units and CTA
  // groups; group g is rep CTAs (clusters) that run the same k-range of the same weight tile,
  // one per token tile, so the weight stage is fetched from HBM once and hit in L2 by the
  // others.  CTA c = g * rep + token tile.  rep = 1: the plain stream-K partition.
  int rep;
};
__host__ __device__ inline long long sk_unit0(int c, const SplitPlan &p) { return p.U * c / p.P; }
__host__ __device__ inline int sk_cta_of(long long u, const SplitPlan &p) {
  return (int)(((u + 1) * p.P + p.U - 1) / p.U) - 1;
}
__host__ __device__ inline int sk_tile(long long u, const SplitPlan &p) { return (int)(u / p.kb_total); }
// real tile of unit u for the CTA at token-tile lane ttr of its group (rep = token_tiles: the
// tile index (bi * m_tiles + mt) * token_tiles + tt with tt = ttr)
__host__ __device__ inline int sk_tile_r(long long u, const SplitPlan &p, int ttr) {
  return (int)(u / p.kb_total) * p.rep + ttr;
}
// first and last CTA group contributing to real tile t
__host__ __device__ inline int sk_first_grp(int t, const SplitPlan &p) {
  return sk_cta_of((long long)(p.rep == 1 ? t : t / p.rep) * p.kb_total, p);
}
__host__ __device__ inline int sk_ncontrib(int t, const SplitPlan &p) {
  const int tw = p.rep == 1 ? t : t / p.rep;  // (no division on the decode path)
  return sk_cta_of((long long)(tw + 1) * p.kb_total - 1, p) - sk_cta_of((long long)tw * p.kb_total, p) + 1;
}
__host__ __device__ inline int sk_kb(long long u, const SplitPlan &p) { return (int)(u % p.kb_total); }
// token tiles of one weight tile are adjacent units, so a re-read of the same
// 128 x K weight rows for the next token tile is a near-term L2 hit
__host__ __device__ inline void sk_decode(int t, const SplitPlan &p, int &bi, int &tt, int &mt) {
  tt = t % p.token_tiles;
  const int r = t / p.token_tiles;
  mt = r % p.m_tiles;
  bi = r / p.m_tiles;
}
__host__ __device__ inline int sk_tile_of(const SplitPlan &p, int bi, int tt, int mt) {
  return (bi * p.m_tiles + mt) * p.token_tiles + tt;
}
__host__ __device__ inline int sk_pair(const SplitPlan &p) { return p.pair > 1 ? 2 : 1; }
__host__ __device__ inline float *sk_partial(float *ws, const SplitPlan &p, int t, int k, int r = 0) {
  return ws + (((size_t)t * sk_pair(p) + r) * p.maxc + k) * p.bn * 128;
}
// (unit tile t, first partial slot) of output column n (any 128-row half) for token row m
// tw: the tile's index in the unit space (t itself; the weight tile when rep > 1) -- no division
__host__ __device__ inline void sk_locate(const SplitPlan &p, int bi, int m, int n, int &t, size_t &slot0, int &tw) {
  const int pr = sk_pair(p);
  const int tt = m / p.bn, mt = n >> 7;
  t = sk_tile_of(p, bi, tt, mt / pr);
  tw = p.rep > 1 ? bi * p.m_tiles + mt / pr : t;
  slot0 = ((size_t)t * pr + (mt % pr)) * p.maxc;
}
__host__ __device__ inline int sk_ncontrib_w(int tw, const SplitPlan &p) {
  return sk_cta_of((long long)(tw + 1) * p.kb_total - 1, p) - sk_cta_of((long long)tw * p.kb_total, p) + 1;
}
// Where a GEMM's partials live, for the consumer kernels.  planes = 3 in the fp32
// parity mode: every logical activation row m was fed to the GEMM as three bf16
// rows 3m, 3m+1, 3m+2 (hi, mid, lo with hi + mid + lo == the fp32 value exactly),
// so the logical output row is the sum of those three GEMM rows; M counts logical rows.
struct PartialView {
  SplitPlan plan;
  const float *ws;
  int N, M;
  int planes;  // 0 or 1: bf16 activations; 3: fp32 split into three bf16 planes
};
// Deterministic sum (contributor order) of y[bi][m][n .. n+3] (n % 4 == 0).
// Loads of up to 8 contributors are issued before any add (one memory round
// trip instead of one per contributor).
__device__ inline float4 sk_sum4(const PartialView &v, int bi, int m, int n) {
  const SplitPlan &p = v.plan;
  const int tt = m / p.bn;
  int t;
  size_t slot0;
  int tw;
  sk_locate(p, bi, m, n, t, slot0, tw);
  const int nc = sk_ncontrib_w(tw, p);
  const float4 *base =
      reinterpret_cast<const float4 *>(v.ws + slot0 * p.bn * 128 + (size_t)(m - tt * p.bn) * 128 + (n & 127));
  const size_t stride = (size_t)p.bn * 128 / 4;  // float4 between contributors
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k0 = 0; k0 < nc; k0 += 8) {
    float4 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (k0 + k < nc) ? __ldcg(base + (k0 + k) * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k0 + k < nc) {
        acc.x += x[k].x;
        acc.y += x[k].y;
        acc.z += x[k].z;
        acc.w += x[k].w;
      }
    }
  }
  return acc;
}
// Split form of sk_sum4 for consumers that need several sums: sk_ref locates the
// contributors, sk_load issues up to NMAX loads at once, sk_reduce adds them (and any
// beyond NMAX) in contributor order -- the same order as sk_sum4, so identical results.
struct SkRef {
  const float4 *base;
  size_t stride;  // float4 between contributors
  int nc;
};
__device__ inline SkRef sk_ref(const PartialView &v, int bi, int m, int n) {
  const SplitPlan &p = v.plan;
  const int tt = m / p.bn;
  int t;
  size_t slot0;
  int tw;
  sk_locate(p, bi, m, n, t, slot0, tw);
  SkRef r;
  r.nc = sk_ncontrib_w(tw, p);
  r.base = reinterpret_cast<const float4 *>(v.ws + slot0 * p.bn * 128 + (size_t)(m - tt * p.bn) * 128 + (n & 127));
  r.stride = (size_t)p.bn * 128 / 4;
  return r;
}
template <int NMAX>
__device__ inline void sk_load(const SkRef &r, float4 (&x)[NMAX]) {
#pragma unroll
  for (int k = 0; k < NMAX; ++k) x[k] = (k < r.nc) ? __ldcg(r.base + k * r.stride) : make_float4(0.f, 0.f, 0.f, 0.f);
}
template <int NMAX>
__device__ inline float4 sk_reduce(const SkRef &r, const float4 (&x)[NMAX]) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < NMAX; ++k) {
    if (k < r.nc) {
      acc.x += x[k].x;
      acc.y += x[k].y;
      acc.z += x[k].z;
      acc.w += x[k].w;
    }
  }
  for (int k = NMAX; k < r.nc; ++k) {
    const float4 y = __ldcg(r.base + k * r.stride);
    acc.x += y.x;
    acc.y += y.y;
    acc.z += y.z;
    acc.w += y.w;
  }
  return acc;
}
__device__ inline float sk_sum1(const PartialView &v, int bi, int m, int n) {
  const SplitPlan &p = v.plan;
  const int tt = m / p.bn;
  int t;
  size_t slot0;
  int tw;
  sk_locate(p, bi, m, n, t, slot0, tw);
  const int nc = sk_ncontrib_w(tw, p);
  const float *base = v.ws + slot0 * p.bn * 128 + (size_t)(m - tt * p.bn) * 128 + (n & 127);
  const size_t stride = (size_t)p.bn * 128;
  float acc = 0.f;
  for (int k0 = 0; k0 < nc; k0 += 8) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = (k0 + k < nc) ? __ldcg(base + (k0 + k) * stride) : 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k0 + k < nc) acc += x[k];
  }
  return acc;
}

// Logical-row sums for consumers that accept either activation format (the fp32
// mode adds the three planes in order hi, mid, lo after each plane's contributor sum).
__device__ inline float4 sk_get4(const PartialView &v, int bi, int m, int n) {
  if (v.planes <= 1) return sk_sum4(v, bi, m, n);
  float4 acc = sk_sum4(v, bi, 3 * m, n);
#pragma unroll
  for (int p = 1; p < 3; ++p) {
    const float4 y = sk_sum4(v, bi, 3 * m + p, n);
    acc.x += y.x;
    acc.y += y.y;
    acc.z += y.z;
    acc.w += y.w;
  }
  return acc;
}
__device__ inline float sk_get1(const PartialView &v, int bi, int m, int n) {
  if (v.planes <= 1) return sk_sum1(v, bi, m, n);
  return sk_sum1(v, bi, 3 * m, n) + sk_sum1(v, bi, 3 * m + 1, n) + sk_sum1(v, bi, 3 * m + 2, n);
}
// fp32 -> three bf16 planes whose sum is exactly x (each residual is exact in fp32).
__device__ inline void split3_bf16(float x, __nv_bfloat16 &hi, __nv_bfloat16 &mid, __nv_bfloat16 &lo) {
  hi = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r1);
  lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
}
// Store 4 consecutive values of logical row m at column c of a [rows * planes][width]
// bf16 activation buffer (planes = 1: plain bf16 row; 3: interleaved hi/mid/lo rows).
__device__ inline void store_act4(__nv_bfloat16 *buf, int planes, int m, int width, int c, float a, float b, float cc,
                                  float d) {
  if (planes <= 1) {
    __nv_bfloat162 lo2 = __floats2bfloat162_rn(a, b), hi2 = __floats2bfloat162_rn(cc, d);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t *>(&lo2);
    o.y = *reinterpret_cast<uint32_t *>(&hi2);
    *reinterpret_cast<uint2 *>(buf + (size_t)m * width + c) = o;
    return;
  }
  const float v[4] = {a, b, cc, d};
  __nv_bfloat16 p[3][4];
#pragma unroll
  for (int e = 0; e < 4; ++e) split3_bf16(v[e], p[0][e], p[1][e], p[2][e]);
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    __nv_bfloat16 *dst = buf + ((size_t)m * 3 + q) * width + c;
#pragma unroll
    for (int e = 0; e < 4; ++e) dst[e] = p[q][e];
  }
}
// Value of logical row m, column c of such a buffer (exact fp32 in the split form).
__device__ inline float load_act1(const __nv_bfloat16 *buf, int planes, int m, int width, int c) {
  if (planes <= 1) return __bfloat162float(buf[(size_t)m * width + c]);
  const __nv_bfloat16 *r = buf + (size_t)m * 3 * width + c;
  return __bfloat162float(r[0]) + __bfloat162float(r[width]) + __bfloat162float(r[2 * width]);
}

// Fused tile epilogues of K2 (GemmArgs.epi != 0, bf16 path with tp = 1): every
// contributor writes its partial slot, the LAST contributor of a 128-feature tile
// (arrival counter) sums the slots in contributor order -- the same deterministic
// order as the consumer kernels -- and applies the next step of the forward itself:
//   kEpiQKV   y *= rs[m]; RoPE at Lc + depth (hd = 128: tile = head); q, K/V -> cache (R3)
//   kEpiSiLU  act = bf16(SiLU(rs g) * rs u) from the 64/64 gate/up rows of the tile (R6)
//   kEpiResid x += y (R5/R7); h = bf16(x * g) for the next GEMM (deferred R2); per-row
//             sum-of-squares partials; the last tile of the GEMM turns them into rs[m]
enum { kEpiPartial = 0, kEpiQKV = 1, kEpiSiLU = 2, kEpiResid = 3 };
struct EpiArgs {
  const float *rs_in;        // kEpiQKV / kEpiSiLU: deferred-norm scale of the input rows
  const float2 *rope;        // kEpiQKV
  RowCtx rc;
  int H, Hkv, cap;
  bf16 *q, *kc, *vc;         // q [M][H][128]; this layer's K / V cache base ([b][Hkv][cap][128])
  bf16 *act;                 // kEpiSiLU: [M][F]
  int F;
  float *x;                  // kEpiResid: fp32 residual [M][d]
  const bf16 *g;             //            next norm's gain [d]
  bf16 *h;                   //            next GEMM input [M][d] = bf16(x * g)
  float *ss;                 //            [M][d / 64] sum-of-squares partials
  float *rs_out;             //            [M]
  int d;
  float eps;
  int *tile_cnt;             // arrival counters (zero between launches; the fixup resets its own)
  int *done_cnt;             // tiles fixed up in this launch (kEpiResid), reset by the last
};

// Deferred RMSNorm scale of a GEMM's input rows (rounding contract R2): either precomputed
// (rs[m]: TP / fused paths) or from the per-slice sums of squares the split residual+norm
// kernel wrote (ss[m][cs], summed in slice order -- the cluster kernel's order).
struct RsArgs {
  const float *rs;
  const float *ss;
  int cs, d;
  float eps;
};
__device__ inline float rs_of(const RsArgs &a, int m) {
  if (a.rs) return a.rs[m];
  if (!a.ss) return 1.0f;
  float s = 0.f;
  for (int q = 0; q < a.cs; ++q) s += a.ss[(size_t)m * a.cs + q];
  return 1.0f / sqrtf(s / (float)a.d + a.eps);
}

struct GemmArgs {
  CUtensorMap tmW[kMaxGemmBatch];  // weight [N][K] bf16, box 64(k) x 128(rows), SWIZZLE_128B
  CUtensorMap tmX[kMaxGemmBatch];  // activation [rows][K] bf16, box 64(k) x 16(rows), SWIZZLE_128B
  CUtensorMap tmX64[kMaxGemmBatch];  // same activation, box 64(k) x BN rows (BN >= 64): one TMA per stage
  const void *x_base[kMaxGemmBatch];  // host bookkeeping: activation base / rows (re-encode tmX64 per BN)
  int x_rows[kMaxGemmBatch];
  int x_box;                          // box rows tmX64 is currently encoded with
  int N, K, M, batch;
  int x_row0;                      // first activation row (TMA row offset)
  int l2_prefetch;                 // weight k-blocks per CTA prefetched into L2 before the PDL wait
  int dbg_mode;                    // experiments: 1 = stream weights only (no X, no MMA)
  int pre_stages;                  // weight stages issued before griddepcontrol.wait (-1 = the ring)
  int no_pair;                     // 1: plan without the 2-SM (cta_group::2) variant
  SplitPlan plan;
  float *ws;                       // partial slots, gemm_ws_floats() floats
  int epi;                         // kEpi*: fused tile epilogue (batch 1 only)
  EpiArgs e;
};
void gemm_plan(GemmArgs &a, int N, int K, int M, int batch);
cudaError_t gemm_launch(const GemmArgs &a, cudaStream_t st);
int gemm_pick_bn(int M);
size_t gemm_ws_floats(const GemmArgs &a);
void gemm_set_pdl(bool on);
bool gemm_pdl();
void gemm_set_ctas(int n);
void gemm_set_rep(int on);
void gemm_set_l2_prefetch(int kblocks);
void gemm_set_debug_mode(int m);
void gemm_set_small(int v);
void gemm_set_bn(int bn);
void gemm_set_pair(int mode);
void gemm_set_occ_smalln(int v);  // experiments: occupancy of GEMMs with N <= 8192  // 2-SM MMA for token tiles >= 96 rows (1), >= 64 (2), off (0)
void gemm_set_pre_stages(int n);  // experiments: force the token-tile width (16..256 supported set; 0 = auto)

// ---------------------------------------------------------------- K1 tree attention
struct AttnArgs {
  CUtensorMap tmK, tmV;       // 2D views [rows][hd] of the K and V caches, box 64 rows x min(hd,64)
  const bf16 *q;              // [rows M][H][hd]
  bf16 *out;                  // [M][H][hd]
  const int32_t *len;         // Lc by absolute sequence index
  const uint64_t *anc;        // [Nq][kAncWords]
  long long k_row0, v_row0;   // tmap row of (seq 0, head 0, slot 0) for K and V of this layer
  long long seq_rows;         // rows per sequence block = Hkv * cap
  int cap;                    // slots per (seq, head)
  int Nq, H, Hkv, G, nseq, seq_base;
  int nsplit;                 // key splits = cluster size (1, 2, 4, 8), combined through DSMEM
  float scale_log2;           // log2(e) / sqrt(hd)
  // L2 prefetch of the next GEMM's weights (the o_proj, which cannot start its own prefetch
  // while the attention CTAs fill the SMs' shared memory); nullable
  const void *l2_pf;
  unsigned long long l2_pf_bytes;
  const uint32_t *pad;        // nullable: pad-batching bitmap [seq][pad_words] of masked cache slots (f4)
  int pad_words;
  int causal;                 // prefill chunk (f3): anc unused, tree slot j visible to node n iff j <= n
  // stream-K ("lean") tree kernel (attention_tc.cu): partial slots, barrier counters (zeroed once,
  // reset by the kernel), minimum tiles per CTA
  float *lean_part;
  int *lean_sync;
  int lean_min_tiles;
  // raw K / V bases of tmK / tmV (tmap row r = base + r hd elements) for L2 prefetch ahead of the
  // TMA ring (K1 row-copy kernel): l2_ahead bit 0 = this CTA's own key range past the ring, bit 1 =
  // the first ring's worth of the CTA one wave later (set by attention_tc_launch from the option)
  const bf16 *k_base, *v_base;
  int l2_ahead;
  int q_early;  // row-copy kernel: Q loads issued before the CTA barrier (set by attention_tc_launch)
};
cudaError_t attention_launch(const AttnArgs &a, int head_dim, cudaStream_t st);
int attention_row_blocks(int Nq, int G, int head_dim);
// fp32 parity mode: plain fp32 tree attention (SIMT), q [M][H][hd] fp32, caches fp32
// [b][Hkv][cap][hd] at (k, v) for this layer, output as three bf16 planes per row.
cudaError_t attention_f32_launch(const float *q, const float *k, const float *v, const int32_t *len,
                                 const uint64_t *anc, int Nq, int H, int Hkv, int hd, int cap, int nseq, int seq_base,
                                 const uint32_t *pad, int pad_words, bf16 *out, cudaStream_t st);
int attention_nsplit(int units, int head_dim, int cap);  // units = row blocks * sequences * kv heads; cap = keys
constexpr int kLeanMaxSeq = 64;                 // sequences per lean K1 launch
cudaError_t attention_lean_launch(const AttnArgs &a, cudaStream_t st);
size_t attention_lean_part_floats(int nunits);
void attention_set_lean(int on);
void attention_set_ks(int on);
void attention_set_l2ahead(int mode);
void attention_set_ksp(int on);
void attention_set_split_model(int m);
void attention_set_w2(int on);
void attention_set_qearly(int on);
void consumer_set_rpc(int n);
void consumer_set_nm(int n);
void resid_set_nm(int n);
void attention_set_lean_div(int d);
int attention_lean_min_tiles(int Nq, int G);
void attention_set_splits(int n);               // experiments: force key splits (0 = auto)
void attention_set_tc(int on);                  // head_dim 128: tcgen05 kernel (1, default) or mma.sync (0)
void attention_set_l2pf(int on);                // experiments: L2 prefetch of AttnArgs.l2_pf (0, default)

// ---------------------------------------------------------------- GEMM consumers (epilogue.cu)
// Every consumer waits on the producer GEMM with griddepcontrol.wait and lets
// its own dependent launch early (programmatic dependent launch).
cudaError_t embed_launch(const int32_t *tok, const bf16 *E, float *x, int M, int d, cudaStream_t st);
// x[m] += y[m] (if pv), then h = bf16(rmsnorm(x) * g)    (R5/R7 + R2/R8)
// hp = planes of h (1: bf16; 3: fp32 parity mode, split rows).  rs_out != nullptr:
// deferred RMSNorm (R2): h = x * g, rs_out[m] = 1/sqrt(mean(x^2) + eps); else h = rms(x) * g.
cudaError_t resid_norm_launch(const PartialView *pv, float *x, const bf16 *g, bf16 *h, int M, int d, float eps,
                              int hp, float *rs_out, cudaStream_t st);
// q/k/v = y; RoPE(q, k) at pos Lc + depth; q -> q[m][H][hd], k/v -> cache slot Lc + node   (R3)
// pv.planes == 3 (fp32 parity mode): q and the caches are fp32, else bf16.
cudaError_t qkv_consumer_launch(const PartialView &pv, RowCtx rc, int H, int Hkv, int hd, const float2 *rope, void *q,
                                void *kcache, void *vcache, int cap, RsArgs rs, cudaStream_t st);
// act[m][f] = bf16(SiLU(gate) * up), gate/up interleaved per 64 rows    (R6)
cudaError_t silu_consumer_launch(const PartialView &pv, int F, bf16 *act, RsArgs rs, cudaStream_t st);
// Residual + deferred RMSNorm without the cluster exchange: one CTA per (row, 1024-column
// slice) adds the partials into x, writes h = bf16(x * g) and the slice's sum of squares
// ss[m][slice]; the next GEMM's consumer forms rs from them (rs_of).
cudaError_t resid_norm_split_launch(const PartialView *pv, float *x, const bf16 *g, bf16 *h, int M, int d, int hp,
                                    float *ss, cudaStream_t st);
int resid_norm_slices(int d);
// LM rows: z = y (fp32, optional copy), argmax (lowest index on ties) and the
// single-pass typical statistics (m, s, t) of z * inv_temp    (R9)
cudaError_t logits_consumer_launch(const PartialView &pv, float inv_temp, float *z_out, int32_t *argmax, float *stats,
                                   int idx_offset, float *amax,
                                   cudaStream_t st);
// plain fp32 rows (z or head logits) -> argmax/stats
cudaError_t logits_finalize_launch(const float *z, int V, int rows, float inv_temp, int32_t *argmax, float *stats,
                                   int idx_offset, float *amax,
                                   cudaStream_t st);
// Medusa ResBlock: r[i][b][:] = bf16(h[b] + SiLU(y_i[b] + beta_i))    (R10)
cudaError_t heads_r_consumer_launch(const PartialView &pv, int nmed, int nb, int d, const bf16 *head_in,
                                    const bf16 *const *beta, bf16 *r_out, long long r_stride, cudaStream_t st);
// top-k of the U-head logits y_i[b][:]: idx[b][i][k], (value desc, index asc)    (K3)
cudaError_t topk_consumer_launch(const PartialView &pv, int nmed, int nb, int V, int k, int32_t *idx, int idx_offset,
                                 float *vals, cudaStream_t st);
void consumer_set_threads(int n);  // experiments: qkv / SiLU consumer block size  // experiments: cap the consumer grids (persistent), 0 = uncapped
// stage API: top-k of plain fp32 rows
cudaError_t topk_launch(const float *logits, int rows, int V, int k, int32_t *idx, cudaStream_t st);
// stage API: out[m][n] = y[m][n]
cudaError_t plain_consumer_launch(const PartialView &pv, float *out, cudaStream_t st);

// ---------------------------------------------------------------- decode control (K3/K4/K5)
struct TreeDev {
  int N, S, l;
  const int32_t *parent, *depth, *rank, *dfs_pos, *first_leaf;
  const uint64_t *anc;
};
cudaError_t propose_launch(TreeDev t, const int32_t *root, const int32_t *topk, int K, int nmed, int b,
                           int32_t *tree_tok, int32_t *pos, const int32_t *len, cudaStream_t st);
// ---- pad batching (f4): all sequences advance their cache by the batch's longest
// acceptance; the shorter ones' extra slots are pads, masked in attention; positions count tokens.
// pad_align: len[b] = max len (slots [len_b, max) marked pad); pad_commit: len[b] += max n_emit,
// pos_len[b] += n_emit[b], slots [len + n_emit_b, len + A) marked pad.
cudaError_t d2d_copy_launch(void *dst, const void *src, size_t bytes, cudaStream_t st);  // copy as a kernel
cudaError_t pad_align_launch(int b, int32_t *len, uint32_t *pad, int pad_words, cudaStream_t st);
cudaError_t pad_commit_launch(int b, int32_t *len, int32_t *pos_len, const int32_t *n_emit, uint32_t *pad,
                              int pad_words, cudaStream_t st);
struct AcceptArgs {
  TreeDev t;
  int b, K, V, x_bound;
  int mode;                    // 0 greedy, 1 typical
  float inv_temp, eps, alpha;
  const int32_t *tok;          // [b][N]
  const int32_t *argmax;       // [b*N]
  const float *stats;          // [b*N][3] (m, s, t) of y = z/T
  const float *z;              // [b*N][V] logits (typical gather)
  const float *cand;           // nullable: [b*N] z[parent(n)][tok[n]] (tensor parallel: merged)
  const int32_t *len;          // Lc[b]
  const int32_t *max_new;      // nullable
  const int32_t *forced_path;  // nullable [b][l+1]
  int32_t *acc_len, *best_leaf, *path, *emit_tok, *n_emit, *status;
  int32_t *acc_row;            // [b] row index of the last emitted node
  int32_t *root_next;          // [b]
  int32_t *sticky;             // nullable: mapped host word, set to a nonzero status (sm_kv surfacing)
};
cudaError_t accept_launch(const AcceptArgs &a, cudaStream_t st);
cudaError_t compact_launch(bf16 *kv_base, int L, int b, int Hkv, int cap, int hd, const int32_t *len,
                           const int32_t *path, int path_ld, const int32_t *n_emit, cudaStream_t st);
cudaError_t commit_launch(int b, int32_t *len, const int32_t *n_emit, int32_t *root, const int32_t *root_next,
                          const int32_t *acc_row, const bf16 *hf, int d, bf16 *head_in, int32_t *emitted_total,
                          bool early, cudaStream_t st);  // len == nullptr: lengths advanced elsewhere (pad batching)
cudaError_t advance_len_launch(int32_t *len, int seq, int n, int32_t *pos_len, cudaStream_t st);
cudaError_t set_root_launch(int32_t *root, int seq, const int32_t *argmax_row, const bf16 *hf_row, int d,
                            bf16 *head_in_row, cudaStream_t st);
cudaError_t generate_bf16_launch(void *dst, size_t numel, uint64_t seed, uint64_t stream_id, uint64_t start, int mode,
                                 cudaStream_t st);
cudaError_t generate_bf16_2d_launch(void *dst, int rows, int cols, int full_cols, int row0, int col0, uint64_t seed,
                                    uint64_t stream_id, int mode, cudaStream_t st);

// ---------------------------------------------------------------- tensor parallelism (a7)
constexpr int kMaxTP = 8;
constexpr int kTpFlagSlots = 8192;  // flags per source rank = max CTAs of one exchange point
// Symmetric buffer of one rank: [flags: kMaxTP src x kTpFlagSlots int64][data slot 0][data slot 1]
struct TpArgs {
  int rank, t;
  float *data[kMaxTP];            // each rank's data slot of this exchange (point parity), mapped here
  long long *flags[kMaxTP];       // each rank's flags region, mapped here
  const long long *seq;           // this rank's epoch base (device)
  int point;                      // exchange index within the current top-level call
  int *err;                       // set to 1 when a wait times out
  // Host-ordered emulation (several ranks on one GPU; guide: kernels that wait on one another must
  // not run as separate launches there).  phase 0 = the fused kernel with flag waits; phase p >= 1 =
  // only segment p of it, no flag wait: the launch function orders the segments of all ranks with
  // CUDA events (emu_publish / emu_wait) between launches instead.
  int phase;
  void *emu;                      // host only: EmuGroup of the ranks (nullptr = real multi-GPU)
  long long gen;                  // host only: this exchange's generation (monotone per rank)
};
// Host-ordered exchange emulation: rank `rank` of the group records "segment `sub` of exchange gen
// done" on st (emu_publish); emu_wait makes st wait for rank q's record of the same (gen, sub).
// emu_wait blocks the calling host thread until rank q has published (each rank is driven by its
// own host thread), ~60 s at most (then cudaErrorTimeout).
struct EmuGroup;
EmuGroup *emu_group_create(int t);
void emu_group_destroy(EmuGroup *g);
cudaError_t emu_publish(const TpArgs &tp, int sub, cudaStream_t st);
cudaError_t emu_wait(const TpArgs &tp, int q, int sub, cudaStream_t st);
cudaError_t emu_exchange(const TpArgs &tp, int sub, cudaStream_t st);  // publish, then wait for every peer
// Residual all-reduce fused into residual + RMSNorm (pv = this rank's o_proj / down partials).
void tp_set_rsag(int mode);  // -1 auto (t >= 4), 0 one-shot, 1 reduce-scatter + all-gather
cudaError_t resid_norm_tp_launch(const PartialView &pv, float *x, const bf16 *g, bf16 *h, int M, int d, float eps,
                                 const TpArgs &tp, float *rs_out, cudaStream_t st);
// Merge the vocab-parallel LM head statistics of rows [0, rows): in = this rank's
// (amax, argmax, m, s, t) per row; cand (nullable) = z[parent(n)][tok[n]] when the rank
// owns tok[n] (tree rows, typical acceptance); out: merged argmax / stats / cand.
cudaError_t tp_merge_logits_launch(int rows, const float *amax, int32_t *argmax, float *stats, const float *z_local,
                                   int Vl, int v0, const int32_t *parent, int N, const int32_t *tok, float *cand,
                                   const TpArgs &tp, cudaStream_t st);
// Merge per-rank top-K (value, global index) lists of `entries` (b x head) into idx.
cudaError_t tp_merge_topk_launch(int entries, int K, const float *vals, const int32_t *idx_local, int32_t *idx_out,
                                 int nmed, int nb, const TpArgs &tp, cudaStream_t st);
cudaError_t tp_advance_launch(long long *seq, int n, cudaStream_t st);
// Layer-split pipeline (f4): hand the fp32 residual rows x[n4 float4] from rank src to the ranks
// in dst_mask (bit q = rank q).  The sender publishes them in its data slot and raises per-CTA
// epoch flags in each receiver; a receiver's CTA waits for its flag and pulls its chunk into x.
cudaError_t pp_xfer_launch(float *x, int n4, int src, unsigned dst_mask, const TpArgs &tp, cudaStream_t st);

// Force-load every kernel of the library (lazy module loading).
void gemm_preload();
void attention_preload();
void attention_tc_preload();
void attention_f32_preload();
void decode_preload();
void epilogue_preload();
void tp_preload();

// ---------------------------------------------------------------- PDL launch helpers
// Launch with programmatic stream serialization when enabled (gemm_pdl()).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = gemm_pdl() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// Same, with a (cx, 1, 1) thread-block cluster.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                      int cx, Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = gemm_pdl() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cx;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace sm
