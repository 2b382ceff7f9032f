// attention_tc.cu -- K1 on 5th-gen tensor cores (head_dim 128): tree-masked
// attention of up to 128 query rows (N nodes x G query heads of one kv head)
// per CTA against the committed prefix [0, Lc) and the tree slots [Lc, Lc+N).
//
// Eq. 2: node n attends to its ancestors and itself ("attention mask
// assumes full acceptance") plus the whole cached prefix; scale 1/sqrt(hd).
//
//  * S = Q K^T and O += P V are tcgen05.mma (kind::f16, M = 128 query rows) with
//    fp32 accumulators in TMEM: S double-buffered (2 x 64 columns) so the MMA of
//    tile i+1 overlaps the softmax of tile i; O (128 columns) stays in TMEM for
//    the whole key range.  K (K-major) and V (MN-major) tiles of 64 keys are
//    TMA-loaded (SWIZZLE_128B) into a 4-deep mbarrier ring and used in place;
//    P is double-buffered so the softmax of tile i+1 does not wait for PV(i).
//  * softmax: one thread per query row reads its S row with tcgen05.ld, applies
//    the ancestor mask on tiles past Lc, and keeps a running max that is only
//    raised when a tile exceeds it by more than 2^8 (then that warp rescales its
//    O rows in TMEM with tcgen05.ld/st) -- the result is exact because l and O
//    use the same stale max.  P (bf16) goes to shared memory in the UMMA A
//    layout.
//  * split-KV: the nsplit CTAs of a (row block, seq, kv head) form a cluster; each
//    stages its (m, l, O) rows in its idle K/V ring and the CTA owning a row pulls
//    the nsplit partials over DSMEM and combines them in a fixed rank order.
//  * programmatic dependent launch: prefix K/V tiles are requested before
//    griddepcontrol.wait; Q and the tree tiles after it.
// Warp roles (192 threads): warps 0-3 softmax / epilogue (TMEM lanes = rows),
// warp 4 TMA producer, warp 5 MMA issuer + TMEM allocator.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace sm {

namespace tc {
constexpr int HD = 128;
constexpr int ROWS = 128;                     // query rows per CTA (UMMA M)
constexpr int KEYS = 64;                      // keys per tile
constexpr int TILE = KEYS * HD * 2;           // 16 KB: one K (or V) tile
// P never touches shared memory: the softmax writes it (bf16 pairs) over its S buffer in TMEM and
// the PV MMA reads its A operand from there (tcgen05.mma ... [a_tmem]), so the ring gets the 32 KB
// the two P buffers took: 6 stages = 192 KB of K/V in flight per SM (4 stages held ~4.6 TB/s)
constexpr int STAGES = 6;
constexpr int QB = ROWS * HD * 2;             // 32 KB
constexpr int OFF_Q = 0;
constexpr int OFF_KV = OFF_Q + QB;
constexpr int OFF_BAR = OFF_KV + STAGES * 2 * TILE;
constexpr int SMEM = OFF_BAR + 256 + 1024;    // + barriers + alignment slack
static_assert(SMEM <= 232448, "K1 shared memory");
constexpr float RESCALE_LOG2 = 8.0f;          // lazy-rescale threshold (log2 units)
}  // namespace tc

// K-major SWIZZLE_128B operand: byte offset of 16-byte chunk c of row r in a
// [rows][64 bf16] block (8-row atoms of 1024 B)
SM_DEV uint32_t sw128_off(int r, int c) { return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((c ^ r) & 7) << 4)); }

// UMMA descriptor, MN-major SWIZZLE_128B: 64-element MN atoms LBO apart, 8-row
// K groups SBO = 1024 B apart
SM_DEV uint64_t umma_desc_mn_sw128(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// kind::f16 instruction descriptor with operand majors (0 = K, 1 = MN)
__host__ __device__ constexpr uint32_t idesc_bf16_major(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

SM_DEV float ex2(float x) {  // 2^x, flush-to-zero (MUFU.EX2; -inf -> 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
SM_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

SM_DEV void tmem_ld32_f(uint32_t taddr, float *v) {
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
SM_DEV void tmem_ld64_f(uint32_t taddr, float *v) {  // 64 consecutive columns, one wait
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}
SM_DEV void tmem_ld16_f(uint32_t taddr, float *v) {  // 16 consecutive columns
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
SM_DEV void tmem_st32_f(uint32_t taddr, const float *v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

SM_DEV void tmem_st32_u(uint32_t taddr, const uint32_t *v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// sm_set_option("attn_l2pf"): prefetch the o_proj weights into L2 during attention.  Measured:
// the o_proj GEMM gains ~0.8 us per layer, attention loses ~2.3 us (its K/V reads compete) -> off.
__device__ int g_attn_l2pf = 0;
// CAUSAL: prefill chunk (AttnArgs::causal), compiled separately so the tree kernel keeps its code
template <bool CAUSAL>
__global__ void __launch_bounds__(192, 1) tree_attn_tc_kernel(const __grid_constant__ AttnArgs a) {
  using namespace tc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem + OFF_Q;
  uint8_t *sKV = smem + OFF_KV;
  uint64_t *kv_full = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *kv_empty = kv_full + STAGES;
  uint64_t *s_full = kv_empty + STAGES;  // [2]
  uint64_t *s_free = s_full + 2;         // [2] (unused: S(i+2) is issued after PV(i), in order)
  uint64_t *p_full = s_free + 2;         // [2] P(i) written over S buffer i & 1
  uint64_t *o_done = p_full + 2;         // [2] PV(i) commits to o_done[i & 1]
  uint64_t *q_full = o_done + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(q_full + 1);

  pdl_trigger();
  SM_GT_BEGIN();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) SM_STAMP(0);
  const int split = blockIdx.x, rblk = blockIdx.y;  // split = rank in the (nsplit, 1, 1) cluster
  const int sl = blockIdx.z / a.Hkv, h = blockIdx.z % a.Hkv;
  const int seq = a.seq_base + sl;
  const int Lc = a.len[seq];  // changed only by the step's last kernels: safe before the wait
  const int R = a.Nq * a.G;
  // causal prefill chunk (f3): keys past the block's last node are invisible to every row of it
  const int T = Lc + (CAUSAL ? min(a.Nq, (min(R, (rblk + 1) * ROWS) - 1) / a.G + 1) : a.Nq);
  const int chunk = ((T + a.nsplit - 1) / a.nsplit + KEYS - 1) / KEYS * KEYS;
  const int key0 = min(T, split * chunk);
  const int key1 = min(T, key0 + chunk);
  const int ntiles = (key1 - key0 + KEYS - 1) / KEYS;
  const float sl2 = a.scale_log2;

  const long long kbase_row = a.k_row0 + (long long)seq * a.seq_rows + (long long)h * a.cap;
  const long long vbase_row = a.v_row0 + (long long)seq * a.seq_rows + (long long)h * a.cap;
  auto issue = [&](int i) {  // TMA: K and V of key tile i -> ring stage i % STAGES
    const int s = i % STAGES;
    uint8_t *kb = sKV + s * 2 * TILE;
    uint8_t *vb = kb + TILE;
    const int p = key0 + i * KEYS;
    mbar_arrive_expect_tx(&kv_full[s], 2 * TILE);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      tma_load_2d(kb + hf * 8192, &a.tmK, &kv_full[s], hf * 64, (int)(kbase_row + p));
      tma_load_2d(vb + hf * 8192, &a.tmV, &kv_full[s], hf * 64, (int)(vbase_row + p));
    }
  };
  const int first = min(STAGES, ntiles);
  int pre = 0;
  if (threadIdx.x == 128) {  // producer thread: barriers, then the prefix tiles (independent of this step)
    tma_prefetch_desc(&a.tmK);
    tma_prefetch_desc(&a.tmV);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 128);
      mbar_init(&p_full[b], 128);
      mbar_init(&o_done[b], 1);
    }
    mbar_init(q_full, 128);
    fence_barrier_init();
    while (pre < first && key0 + (pre + 1) * KEYS <= Lc) issue(pre++);
    SM_STAMP(11);
    if (a.l2_pf && g_attn_l2pf) {  // experiments: this CTA's slice of the next GEMM's weights -> L2
      const unsigned ctas = gridDim.x * gridDim.y * gridDim.z;
      const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
      const unsigned long long per = ((a.l2_pf_bytes + ctas - 1) / ctas + 4095) & ~4095ull;
      const unsigned long long b0 = per * cta, b1 = min(a.l2_pf_bytes, b0 + per);
      for (unsigned long long off = b0; off < b1; off += 65536)
        prefetch_l2_bulk(static_cast<const char *>(a.l2_pf) + off, (uint32_t)min(65536ull, b1 - off));
    }
  }
  // softmax threads: the ancestor words of their row's node (static tree tables: safe before the wait)
  uint64_t anc0 = 0, anc1 = 0, anc2 = 0, anc3 = 0;
  if (warp < 4 && !CAUSAL) {
    const int r = rblk * ROWS + threadIdx.x;
    if (r < R) {
      const uint64_t *w = a.anc + (r / a.G) * kAncWords;
      anc0 = w[0];
      anc1 = w[1];
      anc2 = w[2];
      anc3 = w[3];
    }
  }
  static_assert(kAncWords == 4, "ancestor words are kept in 4 registers");
  if (warp == 5) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) SM_STAMP(1);
  const uint32_t tmem = *tslot;  // S0: cols [0,64), S1: [64,128), O: [128,256)

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      pdl_wait();
      SM_STAMP(12);
      for (int i = pre; i < first; ++i) issue(i);
      for (int i = STAGES; i < ntiles; ++i) {
        mbar_wait(&kv_empty[i % STAGES], ((i / STAGES) - 1) & 1);
        if (i == 9) SM_STAMP(22);
        issue(i);
      }
      SM_STAMP(13);
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && ntiles > 0) {
      constexpr uint32_t idesc_s = idesc_bf16_major(ROWS, KEYS, 0, 0);  // Q (K-major) x K^T (K-major)
      constexpr uint32_t idesc_o = idesc_bf16_major(ROWS, HD, 0, 1);    // P (K-major) x V (MN-major)
      const uint32_t q_u = smem_u32(sQ), kv_u = smem_u32(sKV);
      mbar_wait(q_full, 0);
      SM_STAMP(14);
      auto issue_s = [&](int i) {
        const int sb = i & 1, st = i % STAGES;
        // S buffer sb last held S(i-2) / P(i-2): its PV was issued before this MMA (tensor pipe order)
        mbar_wait(&kv_full[st], (i / STAGES) & 1);
        if (i == 9) SM_STAMP(20);
        tc_fence_after();
        const uint32_t kb = kv_u + st * 2 * TILE;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {  // hd in 16-element steps; halves of 64 are separate 8/16 KB blocks
          const uint64_t ad = umma_desc_sw128(q_u + (k >> 2) * 16384 + (k & 3) * 32);
          const uint64_t bd = umma_desc_sw128(kb + (k >> 2) * 8192 + (k & 3) * 32);
          umma_bf16(tmem + sb * KEYS, ad, bd, idesc_s, k > 0);
        }
        umma_commit(&s_full[sb]);
      };
      issue_s(0);
      for (int i = 0; i < ntiles; ++i) {
        if (i + 1 < ntiles) issue_s(i + 1);
        mbar_wait(&p_full[i & 1], (i >> 1) & 1);
        if (i == 8) SM_STAMP(19);
        tc_fence_after();
        const uint32_t vb = kv_u + (i % STAGES) * 2 * TILE + TILE;
#pragma unroll
        for (int k = 0; k < KEYS / 16; ++k) {  // keys in 16-row steps: 8 TMEM columns of bf16 pairs
          const uint64_t bd = umma_desc_mn_sw128(vb + k * 2048, 8192);
          umma_bf16_ts(tmem + 2 * KEYS, tmem + (i & 1) * KEYS + k * 8, bd, idesc_o, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&kv_empty[i % STAGES]);
        umma_commit(&o_done[i & 1]);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps 0..3 (row = TMEM lane)
    const int r = warp * 32 + lane;
    const int rr = rblk * ROWS + r;
    const bool live = rr < R;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    pdl_wait();  // q comes from the preceding kernel
    SM_GT_WAITED();
    if (threadIdx.x == 0) SM_STAMP(2);
    {  // stage this row of Q into the K-major SW128 layout (two 64-column halves)
      const uint4 *src = nullptr;
      if (live) {
        const int n = rr / a.G, gg = rr % a.G;
        src = reinterpret_cast<const uint4 *>(a.q + (((long long)sl * a.Nq + n) * a.H + (long long)h * a.G + gg) * HD);
      }
      uint4 v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = live ? __ldg(src + c) : make_uint4(0, 0, 0, 0);  // all loads in flight
      const uint32_t q_u = smem_u32(sQ);
#pragma unroll
      for (int c = 0; c < 16; ++c) st_shared_v4(q_u + (c >> 3) * 16384 + sw128_off(r, c), v[c].x, v[c].y, v[c].z, v[c].w);
      fence_proxy_async();
      mbar_arrive(q_full);
    }
    if (threadIdx.x == 0) SM_STAMP(3);
    const int Nq = a.Nq;
    float m_run = -INFINITY, l = 0.f;  // running max in log2 units (lazy), running sum
    const bool warp_live = rblk * ROWS + warp * 32 < R;  // warps of padding rows only keep the handshakes
    for (int i = 0; i < ntiles; ++i) {
      const int sb = i & 1;
      mbar_wait(&s_full[sb], (i >> 1) & 1);
      tc_fence_after();
      if (threadIdx.x == 0) {
        if (i == 0) SM_STAMP(4);
        if (i == ntiles - 1) SM_STAMP(5);
        if (i == 8) SM_STAMP(15);
        if (i == 9) SM_STAMP(21);
      }
      if (!warp_live) {
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
        continue;
      }
      float y[64];
      tmem_ld64_f(lane_base + sb * KEYS, y);
      if (threadIdx.x == 0 && i == 8) SM_STAMP(16);
      const int p0 = key0 + i * KEYS;
      if (a.pad && p0 < Lc) {  // pad batching (f4): masked cache slots of this sequence's prefix
        const uint32_t *pw = a.pad + (size_t)seq * a.pad_words + (p0 >> 5);
        const uint64_t pm = (uint64_t)pw[0] | ((uint64_t)pw[1] << 32);
        if (pm) {
#pragma unroll
          for (int j = 0; j < 64; ++j) y[j] = ((pm >> j) & 1ull) ? -INFINITY : y[j];
        }
      }
      if (CAUSAL && p0 + KEYS > Lc) {  // prefill chunk: key p visible iff p <= Lc + node
        const int lim = Lc + rr / a.G + 1 - p0;  // visible keys of this tile
        const uint64_t vis = lim >= 64 ? ~0ull : (lim <= 0 ? 0ull : (~0ull >> (64 - lim)));
#pragma unroll
        for (int j = 0; j < 64; ++j) y[j] = ((vis >> j) & 1ull) ? y[j] : -INFINITY;
      } else if (p0 + KEYS > Lc) {  // tile reaches past the prefix: visibility bitmask of its 64 keys (Eq. 2)
        const int off = p0 - Lc;  // tree slot of key 0 (may be negative)
        auto word = [&](int q) { return q == 0 ? anc0 : q == 1 ? anc1 : q == 2 ? anc2 : q == 3 ? anc3 : 0ull; };
        uint64_t vis;
        if (off < 0) {
          vis = (~0ull >> (64 + off)) | (anc0 << (-off));  // prefix keys, then tree slots 0..
        } else {
          const int q = off >> 6, sh = off & 63;
          const uint64_t lo = word(q), hi = word(q + 1);
          vis = sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
        }
        if (Nq - off < 64) vis &= (Nq - off <= 0) ? 0ull : (~0ull >> (64 - (Nq - off)));
#pragma unroll
        for (int j = 0; j < 64; ++j) y[j] = ((vis >> j) & 1ull) ? y[j] : -INFINITY;
      }
      float mx0 = y[0], mx1 = y[1], mx2 = y[2], mx3 = y[3];  // four independent chains
#pragma unroll
      for (int j = 4; j < 64; j += 4) {
        mx0 = fmaxf(mx0, y[j]);
        mx1 = fmaxf(mx1, y[j + 1]);
        mx2 = fmaxf(mx2, y[j + 2]);
        mx3 = fmaxf(mx3, y[j + 3]);
      }
      const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
      // lazy max: raised only when a tile exceeds it by more than 2^8 (exact: l and O share the stale max)
      float m_new = m_run, alpha = 1.f;
      bool resc = false;
      if (m_run == -INFINITY) {
        m_new = mx;
      } else if (mx > m_run + RESCALE_LOG2) {
        m_new = mx;
        alpha = exp2f(m_run - m_new);
        resc = true;
      }
      const float nb = (m_new == -INFINITY) ? 0.f : -m_new;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float e0 = ex2(fmaf(y[2 * j], sl2, nb)), e1 = ex2(fmaf(y[2 * j + 1], sl2, nb));
        const float e2 = ex2(fmaf(y[2 * j + 2], sl2, nb)), e3 = ex2(fmaf(y[2 * j + 3], sl2, nb));
        s0 += e0;
        s1 += e1;
        s2 += e2;
        s3 += e3;
        pk[j] = pack_bf16(e0, e1);
        pk[j + 1] = pack_bf16(e2, e3);
      }
      l = l * alpha + ((s0 + s1) + (s2 + s3));
      m_run = m_new;
      if (__any_sync(0xffffffffu, resc) && i > 0) {
        mbar_wait(&o_done[sb ^ 1], ((i - 1) >> 1) & 1);  // PV(i-1) done: O is stable
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < HD; c0 += 32) {
          float o[32];
          tmem_ld32_f(lane_base + 2 * KEYS + c0, o);
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] *= alpha;
          tmem_st32_f(lane_base + 2 * KEYS + c0, o);
        }
      }
      if (threadIdx.x == 0 && i == 8) SM_STAMP(17);
      tmem_st32_u(lane_base + sb * KEYS, pk);  // P(i) over S(i): columns [sb * 64, sb * 64 + 32)
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
      if (threadIdx.x == 0 && i == 8) SM_STAMP(18);
    }
    // final O row
    if (ntiles > 0) {
      mbar_wait(&o_done[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1);
      tc_fence_after();
    }
    if (threadIdx.x == 0) SM_STAMP(6);
    const float fin_m = live ? m_run : -INFINITY, fin_l = live ? l : 0.f;
    if (a.nsplit == 1 && warp_live && ntiles > 0) {  // warp-uniform: tcgen05.ld is .sync.aligned
      const float inv = live ? 1.f / l : 0.f;
      bf16 *dst = a.out + (((long long)sl * a.Nq + rr / a.G) * a.H + (long long)h * a.G + rr % a.G) * HD;
#pragma unroll
      for (int c0 = 0; c0 < HD; c0 += 32) {
        float o[32];
        tmem_ld32_f(lane_base + 2 * KEYS + c0, o);
        if (live) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 w;
            w.x = pack_bf16(o[8 * c] * inv, o[8 * c + 1] * inv);
            w.y = pack_bf16(o[8 * c + 2] * inv, o[8 * c + 3] * inv);
            w.z = pack_bf16(o[8 * c + 4] * inv, o[8 * c + 5] * inv);
            w.w = pack_bf16(o[8 * c + 6] * inv, o[8 * c + 7] * inv);
            reinterpret_cast<uint4 *>(dst + c0)[c] = w;
          }
        }
      }
    } else if (a.nsplit > 1) {
      // stage (m, l, O) of this split in the idle K/V ring (own MMAs and loads are complete);
      // 16-byte chunk c of row r at chunk c ^ (r & 7): conflict-free
      float *so = reinterpret_cast<float *>(sKV);  // [128][HD]
      float *sml = so + ROWS * HD;                 // [128][2]
      sml[2 * r] = fin_m;
      sml[2 * r + 1] = fin_l;
      if (warp_live) {  // (padding warps stage nothing: their rows are never read)
#pragma unroll
        for (int c0 = 0; c0 < HD; c0 += 32) {
          float o[32];
          if (ntiles > 0) {
            tmem_ld32_f(lane_base + 2 * KEYS + c0, o);
          } else {  // empty split: weight 0, but the slot must hold finite values
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = 0.f;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4 *>(so + r * HD + 4 * ((c0 / 4 + c) ^ (r & 7))) =
                make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
        }
      }
    }
  }

  if (a.nsplit > 1) {
    // split-KV combine over DSMEM (pull): rank q owns rows [q*rows_per, (q+1)*rows_per) of the
    // block and reads only live rows (DSMEM moves ~20 B/clk per SM, so padding rows are skipped)
    cluster_sync_all();
    if (threadIdx.x == 0) SM_STAMP(8);
    const float *so = reinterpret_cast<const float *>(sKV);
    const float *sml = so + ROWS * HD;
    float *swt = reinterpret_cast<float *>(sKV + ROWS * HD * 4 + ROWS * 2 * 4);  // [rows_per][8] weights w_q / L
    const uint32_t so_u = smem_u32(so), sml_u = smem_u32(sml);
    // the block's LIVE rows are dealt evenly to the ranks (N*G = 64 of 128 rows: 16 per rank
    // at 4 splits instead of 32 on two ranks and none on the others)
    const int live_tot = max(0, min(ROWS, R - rblk * ROWS));
    const int rows_per = (live_tot + a.nsplit - 1) / a.nsplit;
    const int lr0 = split * rows_per;
    const int live_rows = max(0, min(rows_per, live_tot - lr0));
    for (int lr = threadIdx.x; lr < live_rows; lr += blockDim.x) {
      float mq[8], lq[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 v = q < a.nsplit ? ld_dsmem_f32x2(mapa_u32(sml_u + 8 * (lr0 + lr), q)) : make_float2(-INFINITY, 0.f);
        mq[q] = v.x;
        lq[q] = v.y;
      }
      float M = -INFINITY;
#pragma unroll
      for (int q = 0; q < 8; ++q) M = fmaxf(M, mq[q]);
      float wq[8], L = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // fixed rank order -> deterministic
        wq[q] = mq[q] == -INFINITY ? 0.f : exp2f(mq[q] - M);
        L += wq[q] * lq[q];
      }
      const float inv = 1.f / L;
#pragma unroll
      for (int q = 0; q < 8; ++q) swt[lr * 8 + q] = wq[q] * inv;
    }
    __syncthreads();
    const int items = live_rows * (HD / 4);
    for (int e0 = threadIdx.x; e0 < items; e0 += 2 * blockDim.x) {  // two items per pass: 2 x nsplit loads in flight
      float4 v[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = min(e0 + u * (int)blockDim.x, items - 1);
        const int lr = e / (HD / 4), c4 = e % (HD / 4);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < a.nsplit) v[u][q] = ld_dsmem_f32x4(mapa_u32(so_u + 4 * ((lr0 + lr) * HD + 4 * (c4 ^ ((lr0 + lr) & 7))), q));
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = e0 + u * (int)blockDim.x;
        if (e >= items) continue;
        const int lr = e / (HD / 4), c4 = e % (HD / 4);
        const int row = rblk * ROWS + lr0 + lr;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < a.nsplit) {  // fixed rank order -> deterministic
            const float w = swt[lr * 8 + q];
            acc.x += w * v[u][q].x;
            acc.y += w * v[u][q].y;
            acc.z += w * v[u][q].z;
            acc.w += w * v[u][q].w;
          }
        }
        const int n = row / a.G, gg = row % a.G;
        uint2 pk2;
        pk2.x = pack_bf16(acc.x, acc.y);
        pk2.y = pack_bf16(acc.z, acc.w);
        *reinterpret_cast<uint2 *>(a.out + (((long long)sl * a.Nq + n) * a.H + (long long)h * a.G + gg) * HD + 4 * c4) =
            pk2;
      }
    }
    if (threadIdx.x == 0) SM_STAMP(9);
    cluster_sync_all();  // peers may still be reading this CTA's shared memory
    if (threadIdx.x == 0) SM_STAMP(10);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc<256>(tmem);
  if (threadIdx.x == 0) SM_GT_END(5);
}

// ============================================================================ K1, key-split row packing (KS)
// For N G <= 64 live query rows (the C2 in-step shape: 64 nodes x 1 head per kv head; N 16-32 with
// G <= 2) half or more of the tree kernel's 128 MMA rows are padding, and the softmax of the live
// rows runs on two (or one) of the four SM sub-partitions (TMEM lane quadrant = sub-partition).
// Here the live rows are replicated F = 128 / RP times (RP = 64 or 32 rows per copy) and the key
// tile is 128 keys: copy f of row r (MMA row f RP + r) owns keys [f 128/F, (f+1) 128/F) of every
// tile -- its P is zero at the other keys -- so all four sub-partitions share the softmax of a
// 128-key tile and each thread handles 128/F keys of it.  Tensor work per key is unchanged (S:
// M 128 x N 128 x K 128, PV: M 128 x N 128 x K 128 per 128 keys = the tree kernel's per-64-key
// work twice).  Each copy keeps its own (m, l, O); the F partials of a row are merged in the CTA
// (fixed copy order) and the result enters the split-KV cluster combine as in tree_attn_tc_kernel.
namespace ks {
// KEYS = 128: 3 stages of 64 KB.  (KEYS = 64, 6 stages of 32 KB, for the short split ranges of the C2
// in-step shape measured 13 % slower than the 128-row kernel there: profiles/r02/k1_experiments.txt)
constexpr int HD = 128, ROWS = 128;
template <int KEYS> struct Cfg {
  static constexpr int HALF = KEYS * 64 * 2;        // one hd-half (64 columns) of a K or V tile
  static constexpr int TILE = 2 * HALF;             // a K (or V) tile
  static constexpr int STAGES = KEYS == 128 ? 3 : 6;
};
constexpr int QB = ROWS * HD * 2;          // 32 KB
constexpr int OFF_Q = 0;
constexpr int OFF_KV = OFF_Q + QB;
constexpr int OFF_BAR = OFF_KV + 192 * 1024;
constexpr int OFF_SMAX = OFF_BAR + 256;    // W2: [2 key halves][128 rows] fp32 row-max / row-sum exchange
constexpr int SMEM = OFF_SMAX + 1024 + 1024;
static_assert(SMEM <= 232448, "K1 (KS) shared memory");
// end-of-kernel staging in the idle ring: merged rows for the cluster combine at offset 0 (the tree
// kernel's layout: so [128][HD] fp32 + sml [128][2] + swt), the copies' partials above 80 KB
constexpr int OFF_PART = 80 * 1024;        // [ROWS][HD] fp32 (copy f of row r at f RP + r) + [ROWS] (m, l)
}  // namespace ks

#ifdef SM_TRACE
// diagnostics build: per-CTA %globaltimer stamps of the row-copy kernel, by linear CTA index:
// [smid, entry, Q staged (MMA sees q_full), first K/V tile landed, last PV retired, exit, partials
// staged, copies merged]
constexpr int kKsTr = 8192;
static __device__ long long g_ks_tr[kKsTr][8];
#define KS_TR(slot, v) do { if (ks_lin < kKsTr) g_ks_tr[ks_lin][slot] = (v); } while (0)
extern "C" int sm_trace_read_ks(long long *dst, int n) {
  return (int)cudaMemcpyFromSymbol(dst, g_ks_tr, sizeof(long long) * 8 * (size_t)min(n, kKsTr));
}
#else
#define KS_TR(slot, v) do { } while (0)
#endif

// K and V rows [p0, p1) of (seq, kv head h) -> L2 (bulk prefetch, 64 KB pieces): a hint that lets a
// CTA's whole key range stream at HBM rate while the ring holds only STAGES tiles
SM_DEV void ks_prefetch_l2(const AttnArgs &a, int seq, int h, int p0, int p1) {
  if (p1 <= p0) return;
  const long long r0 = (long long)seq * a.seq_rows + (long long)h * a.cap + p0;
  const char *kb = reinterpret_cast<const char *>(a.k_base + (a.k_row0 + r0) * ks::HD);
  const char *vb = reinterpret_cast<const char *>(a.v_base + (a.v_row0 + r0) * ks::HD);
  const long long bytes = (long long)(p1 - p0) * ks::HD * 2;
  for (long long off = 0; off < bytes; off += 65536) {
    const uint32_t n = (uint32_t)min(65536ll, bytes - off);
    prefetch_l2_bulk(kb + off, n);
    prefetch_l2_bulk(vb + off, n);
  }
}

// W2 (F = 1 only): eight softmax warps, two per TMEM lane quadrant -- warp w and w + 4 share the rows of
// quadrant w & 3 and take the two 64-key halves of every tile (the row max is exchanged through shared
// memory; the lower half's warp does the O rescales and the epilogue): the per-thread softmax work of the
// F = 2 kernel for 128 live rows.
template <int F, int KEYS, bool W2 = false>
__global__ void __launch_bounds__(W2 ? 320 : 192, 1) tree_attn_ks_kernel(const __grid_constant__ AttnArgs a) {
  constexpr int HD = ks::HD, ROWS = ks::ROWS, STAGES = ks::Cfg<KEYS>::STAGES;
  constexpr int NSW = W2 ? 8 : 4;   // softmax warps; producer = warp NSW, MMA issuer = warp NSW + 1
  constexpr int NST = NSW * 32;     // softmax threads
  static_assert(!W2 || (F == 1 && KEYS == 128), "W2: 128 live rows, 128-key tiles");
  constexpr int HALF = ks::Cfg<KEYS>::HALF, TILE = ks::Cfg<KEYS>::TILE;
  constexpr int TCOLS = KEYS == 128 ? 512 : 256;  // S0, S1 (KEYS columns each), O (128)
  constexpr int RP = ROWS / F;      // rows per copy
  constexpr int KT = W2 ? KEYS / 2 : KEYS / F;  // keys per thread per tile
  static_assert(F == 1 || F == 2 || F == 4, "copies");
  static_assert(KEYS == 64 || KEYS == 128, "key tile");
  static_assert(KT >= 16, "keys per thread");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem + ks::OFF_Q;
  uint8_t *sKV = smem + ks::OFF_KV;
  uint64_t *kv_full = reinterpret_cast<uint64_t *>(smem + ks::OFF_BAR);
  uint64_t *kv_empty = kv_full + STAGES;
  uint64_t *s_full = kv_empty + STAGES;  // [2]
  uint64_t *p_full = s_full + 2;         // [2]
  uint64_t *o_done = p_full + 2;         // [2]
  uint64_t *q_full = o_done + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(q_full + 1);

  pdl_trigger();
#ifdef SM_TRACE
  const long long ks_lin = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    KS_TR(0, smid);
    KS_TR(1, gtime());
  }
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x;
  const int row0 = F == 1 ? blockIdx.y * ROWS : 0;  // query rows of this block (several blocks only with F = 1)
  const int sl = blockIdx.z / a.Hkv, h = blockIdx.z % a.Hkv;
  const int seq = a.seq_base + sl;
  const int Lc = a.len[seq];  // changed only by the step's last kernels: safe before the wait
  const int R = a.Nq * a.G;
  const int T = Lc + a.Nq;
  const int chunk = ((T + a.nsplit - 1) / a.nsplit + KEYS - 1) / KEYS * KEYS;
  const int key0 = min(T, split * chunk);
  const int key1 = min(T, key0 + chunk);
  const int ntiles = (key1 - key0 + KEYS - 1) / KEYS;
  const float sl2 = a.scale_log2;

  const long long kbase_row = a.k_row0 + (long long)seq * a.seq_rows + (long long)h * a.cap;
  const long long vbase_row = a.v_row0 + (long long)seq * a.seq_rows + (long long)h * a.cap;
  auto issue = [&](int i) {  // K and V of keys [p, p + KEYS) -> stage i % STAGES, [hd half][KEYS keys][64]
    const int s = i % STAGES;
    uint8_t *kb = sKV + s * 2 * TILE;
    uint8_t *vb = kb + TILE;
    const int p = key0 + i * KEYS;
    mbar_arrive_expect_tx(&kv_full[s], 2 * TILE);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
      for (int kh = 0; kh < KEYS / 64; ++kh) {  // 64-key boxes per hd half, consecutive rows
        tma_load_2d(kb + hf * HALF + kh * 8192, &a.tmK, &kv_full[s], hf * 64, (int)(kbase_row + p + kh * 64));
        tma_load_2d(vb + hf * HALF + kh * 8192, &a.tmV, &kv_full[s], hf * 64, (int)(vbase_row + p + kh * 64));
      }
    }
  };
  const int first = min(STAGES, ntiles);
  int pre = 0;
  if (threadIdx.x == NST) {
    tma_prefetch_desc(&a.tmK);
    tma_prefetch_desc(&a.tmV);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], NST);
      mbar_init(&o_done[b], 1);
    }
    mbar_init(q_full, 128);
    fence_barrier_init();
    while (pre < first && key0 + (pre + 1) * KEYS <= Lc) issue(pre++);
    if (a.l2_ahead & 1)  // the rest of this CTA's cached prefix -> L2 now (the ring then refills from L2)
      ks_prefetch_l2(a, seq, h, key0 + first * KEYS, min(key1, Lc));
  }
  // softmax threads: copy f of query row r; the ancestor words of its node
  const int rr_lane = (warp < NSW) ? (warp & 3) * 32 + lane : 0;
  const int cf = W2 ? (warp < NSW ? warp >> 2 : 0) : rr_lane / RP;  // copy (W2: key half), query row
  const int qr = row0 + rr_lane % RP;
  uint64_t anc0 = 0, anc1 = 0, anc2 = 0, anc3 = 0;
  if (warp < NSW && qr < R) {
    const uint64_t *w = a.anc + (qr / a.G) * kAncWords;
    anc0 = w[0];
    anc1 = w[1];
    anc2 = w[2];
    anc3 = w[3];
  }
  static_assert(kAncWords == 4, "ancestor words are kept in 4 registers");
  // Q row qr in registers before the CTA barrier (option attn_qearly): its load latency overlaps the barrier
  // and the TMEM allocation; staged into shared memory after the barrier (which publishes q_full's init)
  uint4 qv[16];
  const bool qearly = a.q_early && warp < NSW && (!W2 || cf == 0);
  if (qearly) {
    pdl_wait();
    const uint4 *src = nullptr;
    if (qr < R) {
      const int n = qr / a.G, gg = qr % a.G;
      src = reinterpret_cast<const uint4 *>(a.q + (((long long)sl * a.Nq + n) * a.H + (long long)h * a.G + gg) * HD);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) qv[c] = qr < R ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
  }
  if (warp == NSW + 1) tmem_alloc<TCOLS>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;  // S0: cols [0, KEYS), S1: [KEYS, 2 KEYS), O: [2 KEYS, 2 KEYS + 128)

  if (warp == NSW) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      pdl_wait();
      for (int i = pre; i < first; ++i) issue(i);
      for (int i = STAGES; i < ntiles; ++i) {
        mbar_wait(&kv_empty[i % STAGES], ((i / STAGES) - 1) & 1);
        issue(i);
      }
    }
    __syncwarp();
    if (a.l2_ahead & 2) {  // Q rows and the first ring's worth of K/V of the CTA one wave later -> L2
      const long long lin = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
      const long long nx = lin + kNumSMs;  // 1 CTA per SM: roughly the CTA that takes this SM next
      const long long per_z = (long long)gridDim.x * gridDim.y;
      if (nx < per_z * gridDim.z) {
        const int nz = (int)(nx / per_z), nsplit_i = (int)(nx % gridDim.x), nrb = (int)((nx / gridDim.x) % gridDim.y);
        const int nsl = nz / a.Hkv, nh = nz % a.Hkv, nseq = a.seq_base + nsl;
        if (lane == 0) {
          const int nLc = a.len[nseq], nT = nLc + a.Nq;
          const int nchunk = ((nT + a.nsplit - 1) / a.nsplit + KEYS - 1) / KEYS * KEYS;
          const int nk0 = min(nT, nsplit_i * nchunk), nk1 = min(nT, nk0 + nchunk);
          ks_prefetch_l2(a, nseq, nh, nk0, min(min(nk1, nLc), nk0 + STAGES * KEYS));
        }
        // its query rows: nodes of row block nrb, G heads (contiguous) each
        const int r0 = F == 1 ? nrb * ROWS : 0, r1 = min(R, r0 + (F == 1 ? ROWS : RP));
        for (int n = r0 / a.G + lane; n * a.G < r1; n += 32)
          prefetch_l2_bulk(a.q + (((long long)nsl * a.Nq + n) * a.H + (long long)nh * a.G) * HD, a.G * HD * 2);
      }
    }
  } else if (warp == NSW + 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && ntiles > 0) {
      constexpr uint32_t idesc_s = idesc_bf16_major(ROWS, KEYS, 0, 0);  // Q (K-major) x K^T (K-major)
      constexpr uint32_t idesc_o = idesc_bf16_major(ROWS, HD, 0, 1);    // P (TMEM) x V (MN-major)
      const uint32_t q_u = smem_u32(sQ), kv_u = smem_u32(sKV);
      mbar_wait(q_full, 0);
      KS_TR(2, gtime());
      auto issue_s = [&](int i) {
        const int sb = i & 1, st = i % STAGES;
        mbar_wait(&kv_full[st], (i / STAGES) & 1);
        if (i == 0) KS_TR(3, gtime());
        tc_fence_after();
        const uint32_t kb = kv_u + st * 2 * TILE;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint64_t ad = umma_desc_sw128(q_u + (k >> 2) * 16384 + (k & 3) * 32);
          const uint64_t bd = umma_desc_sw128(kb + (k >> 2) * HALF + (k & 3) * 32);
          umma_bf16(tmem + sb * KEYS, ad, bd, idesc_s, k > 0);
        }
        umma_commit(&s_full[sb]);
      };
      issue_s(0);
      for (int i = 0; i < ntiles; ++i) {
        if (i + 1 < ntiles) issue_s(i + 1);
        mbar_wait(&p_full[i & 1], (i >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = kv_u + (i % STAGES) * 2 * TILE + TILE;
#pragma unroll
        for (int k = 0; k < KEYS / 16; ++k) {  // 16 keys per step: 8 TMEM columns of packed P
          const uint64_t bd = umma_desc_mn_sw128(vb + k * 2048, HALF);
          umma_bf16_ts(tmem + 2 * KEYS, tmem + (i & 1) * KEYS + k * 8, bd, idesc_o, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&kv_empty[i % STAGES]);
        umma_commit(&o_done[i & 1]);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps 0..3 (MMA row = TMEM lane)
    const int r = (warp & 3) * 32 + lane;  // MMA row = TMEM lane (F > 1: cf RP + (qr - row0))
    const bool live = qr < R;
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    float *smax = reinterpret_cast<float *>(smem + ks::OFF_SMAX);  // W2: [2 key halves][128 rows]
    if (!qearly) pdl_wait();
    if (!W2 || cf == 0) {  // stage Q row qr (every copy) into the K-major SW128 layout
      uint4 v[16];
      if (qearly) {
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = qv[c];
      } else {
        const uint4 *src = nullptr;
        if (live) {
          const int n = qr / a.G, gg = qr % a.G;
          src = reinterpret_cast<const uint4 *>(a.q + (((long long)sl * a.Nq + n) * a.H + (long long)h * a.G + gg) * HD);
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = live ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
      }
      const uint32_t q_u = smem_u32(sQ);
#pragma unroll
      for (int c = 0; c < 16; ++c) st_shared_v4(q_u + (c >> 3) * 16384 + sw128_off(r, c), v[c].x, v[c].y, v[c].z, v[c].w);
      fence_proxy_async();
      mbar_arrive(q_full);
    }
    const int Nq = a.Nq;
    float m_run = -INFINITY, l = 0.f;
    // warps of padding rows only keep the handshakes (W2: they run the tile loop, whose named barriers
    // count every softmax warp; their rows are never written)
    const bool warp_live = W2 || row0 + ((warp & 3) * 32) % RP < R;
    for (int i = 0; i < ntiles; ++i) {
      const int sb = i & 1;
      mbar_wait(&s_full[sb], (i >> 1) & 1);
      tc_fence_after();
      if (!warp_live) {
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
        continue;
      }
      float y[KT];
      if constexpr (KT == 128) {
        tmem_ld64_f(lane_base + sb * KEYS, y);
        tmem_ld64_f(lane_base + sb * KEYS + 64, y + 64);
      } else if constexpr (KT == 64) {
        tmem_ld64_f(lane_base + sb * KEYS + cf * KT, y);
      } else if constexpr (KT == 32) {
        tmem_ld32_f(lane_base + sb * KEYS + cf * KT, y);
      } else {
        tmem_ld16_f(lane_base + sb * KEYS + cf * KT, y);
      }
      const int pt = key0 + i * KEYS + cf * KT;  // this thread's first key
      constexpr int NH = KT >= 64 ? KT / 64 : 1;  // 64-key windows of this thread's keys
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        constexpr int W = KT >= 64 ? 64 : KT;
        float *yw = y + hh * 64;
        const int p0 = pt + hh * 64;
        if (a.pad && p0 < Lc) {  // pad batching (f4): masked cache slots of the prefix
          const uint32_t *pw = a.pad + (size_t)seq * a.pad_words + (p0 >> 5);
          const uint64_t pm = (uint64_t)pw[0] | (W == 64 ? ((uint64_t)pw[1] << 32) : 0ull);
          if (pm) {
#pragma unroll
            for (int j = 0; j < W; ++j) yw[j] = ((pm >> j) & 1ull) ? -INFINITY : yw[j];
          }
        }
        if (p0 + W > Lc) {  // keys past the prefix: visibility bitmask (Eq. 2)
          const int off = p0 - Lc;
          auto word = [&](int q) { return q == 0 ? anc0 : q == 1 ? anc1 : q == 2 ? anc2 : q == 3 ? anc3 : 0ull; };
          uint64_t vis;
          if (off < 0) {
            vis = (off <= -64 ? ~0ull : (~0ull >> (64 + off))) | (off <= -64 ? 0ull : (anc0 << (-off)));
          } else {
            const int q = off >> 6, sh = off & 63;
            const uint64_t lo = word(q), hi = word(q + 1);
            vis = sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
          }
          if (Nq - off < 64) vis &= (Nq - off <= 0) ? 0ull : (~0ull >> (64 - (Nq - off)));
#pragma unroll
          for (int j = 0; j < W; ++j) yw[j] = ((vis >> j) & 1ull) ? yw[j] : -INFINITY;
        }
      }
      float mx0 = y[0], mx1 = y[1], mx2 = y[2], mx3 = y[3];
#pragma unroll
      for (int j = 4; j < KT; j += 4) {
        mx0 = fmaxf(mx0, y[j]);
        mx1 = fmaxf(mx1, y[j + 1]);
        mx2 = fmaxf(mx2, y[j + 2]);
        mx3 = fmaxf(mx3, y[j + 3]);
      }
      float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
      if constexpr (W2) {  // both halves' maxima (every S read of the tile is complete before P is written)
        smax[cf * 128 + r] = mx;
        asm volatile("bar.sync 2, 256;" ::: "memory");
        mx = fmaxf(mx, smax[(cf ^ 1) * 128 + r]);
      }
      float m_new = m_run, alpha = 1.f;
      bool resc = false;
      if (m_run == -INFINITY) {
        m_new = mx;
      } else if (mx > m_run + tc::RESCALE_LOG2) {
        m_new = mx;
        alpha = exp2f(m_run - m_new);
        resc = true;
      }
      const float nb = (m_new == -INFINITY) ? 0.f : -m_new;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      uint32_t pe[KT / 2];  // this copy's keys, packed in pairs
#pragma unroll
      for (int j = 0; j < KT / 2; j += 2) {
        const float e0 = ex2(fmaf(y[2 * j], sl2, nb)), e1 = ex2(fmaf(y[2 * j + 1], sl2, nb));
        const float e2 = ex2(fmaf(y[2 * j + 2], sl2, nb)), e3 = ex2(fmaf(y[2 * j + 3], sl2, nb));
        s0 += e0;
        s1 += e1;
        s2 += e2;
        s3 += e3;
        pe[j] = pack_bf16(e0, e1);
        pe[j + 1] = pack_bf16(e2, e3);
      }
      uint32_t pk[KEYS / 2];  // the row's packed P columns: this copy's keys, zeros elsewhere
#pragma unroll
      for (int j = 0; j < KEYS / 2; ++j) pk[j] = (j / (KT / 2) == cf) ? pe[j % (KT / 2)] : 0u;
      l = l * alpha + ((s0 + s1) + (s2 + s3));
      m_run = m_new;
      if (__any_sync(0xffffffffu, resc) && i > 0 && (!W2 || cf == 0)) {
        mbar_wait(&o_done[sb ^ 1], ((i - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < HD; c0 += 32) {
          float o[32];
          tmem_ld32_f(lane_base + 2 * KEYS + c0, o);
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] *= alpha;
          tmem_st32_f(lane_base + 2 * KEYS + c0, o);
        }
      }
      if constexpr (W2) {
        tmem_st32_u(lane_base + sb * KEYS + cf * 32, pe);  // this half's 32 packed columns
        asm volatile("bar.sync 3, 256;" ::: "memory");     // both halves have read smax before its reuse
      } else {
        tmem_st32_u(lane_base + sb * KEYS, pk);  // P(i) over S(i): packed columns [sb KEYS, sb KEYS + KEYS / 2)
        if constexpr (KEYS == 128) tmem_st32_u(lane_base + sb * KEYS + 32, pk + 32);
      }
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
    }
    if (ntiles > 0) {
      mbar_wait(&o_done[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1);
      tc_fence_after();
    }
    if (threadIdx.x == 0) KS_TR(4, gtime());
    // ---- stage this copy's (m, l, O) at MMA row r (ring idle: every MMA and load is complete)
    float *spart = reinterpret_cast<float *>(sKV + ks::OFF_PART);  // [ROWS][HD]
    float *spml = spart + ROWS * HD;                                // [ROWS][2]
    if constexpr (W2) {  // the row's sum is the two halves' sums (same running max)
      if (cf == 1) smax[r] = l;
      asm volatile("bar.sync 2, 256;" ::: "memory");
      if (cf == 0) l += smax[r];
    }
    if (!W2 || cf == 0) {
      spml[2 * r] = live ? m_run : -INFINITY;
      spml[2 * r + 1] = live ? l : 0.f;
    }
    if (warp_live && (!W2 || cf == 0)) {
#pragma unroll
      for (int c0 = 0; c0 < HD; c0 += 32) {
        float o[32];
        if (ntiles > 0) {
          tmem_ld32_f(lane_base + 2 * KEYS + c0, o);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<float4 *>(spart + r * HD + 4 * ((c0 / 4 + c) ^ (r & 7))) =
              make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
      }
    }
    if (threadIdx.x == 0) KS_TR(6, gtime());
    asm volatile("bar.sync 1, %0;" ::"n"(NST) : "memory");  // the softmax warps
    // ---- merge the F copies of query row qr (copy order), threads of copy 0 only
    if (cf == 0 && live) {
      float mq[F], lq[F];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        mq[f] = spml[2 * (f * RP + qr - row0)];
        lq[f] = spml[2 * (f * RP + qr - row0) + 1];
      }
      float M = mq[0];
#pragma unroll
      for (int f = 1; f < F; ++f) M = fmaxf(M, mq[f]);
      float wq[F], L = 0.f;
#pragma unroll
      for (int f = 0; f < F; ++f) {
        wq[f] = mq[f] == -INFINITY ? 0.f : exp2f(mq[f] - M);
        L += wq[f] * lq[f];
      }
      float *so = reinterpret_cast<float *>(sKV);  // [128][HD]: the tree kernel's staging layout
      float *sml = so + ROWS * HD;
      bf16 *dst = a.out + (((long long)sl * a.Nq + qr / a.G) * a.H + (long long)h * a.G + qr % a.G) * HD;
      const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll 4
      for (int c4 = 0; c4 < HD / 4; ++c4) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const int rf = f * RP + qr - row0;
          const float4 v = *reinterpret_cast<const float4 *>(spart + rf * HD + 4 * (c4 ^ (rf & 7)));
          acc.x += wq[f] * v.x;
          acc.y += wq[f] * v.y;
          acc.z += wq[f] * v.z;
          acc.w += wq[f] * v.w;
        }
        if (a.nsplit == 1) {
          uint2 pk2;
          pk2.x = pack_bf16(acc.x * inv, acc.y * inv);
          pk2.y = pack_bf16(acc.z * inv, acc.w * inv);
          *reinterpret_cast<uint2 *>(dst + 4 * c4) = pk2;
        } else {
          *reinterpret_cast<float4 *>(so + (qr - row0) * HD + 4 * (c4 ^ ((qr - row0) & 7))) = acc;
        }
      }
      if (a.nsplit > 1) {
        sml[2 * (qr - row0)] = M;
        sml[2 * (qr - row0) + 1] = L;
      }
    }
  }

  if (threadIdx.x == 0) KS_TR(7, gtime());
  if (a.nsplit > 1) {
    // split-KV combine over DSMEM (pull), as tree_attn_tc_kernel: rank q owns live rows
    // [q rows_per, (q+1) rows_per) and reads only live rows
    cluster_sync_all();
    const float *so = reinterpret_cast<const float *>(sKV);
    const float *sml = so + ROWS * HD;
    float *swt = reinterpret_cast<float *>(sKV + ROWS * HD * 4 + ROWS * 2 * 4);
    const uint32_t so_u = smem_u32(so), sml_u = smem_u32(sml);
    const int live_tot = max(0, min(RP, R - row0));
    const int rows_per = (live_tot + a.nsplit - 1) / a.nsplit;
    const int lr0 = split * rows_per;
    const int live_rows = max(0, min(rows_per, live_tot - lr0));
    for (int lr = threadIdx.x; lr < live_rows; lr += blockDim.x) {
      float mq[8], lq[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 v = q < a.nsplit ? ld_dsmem_f32x2(mapa_u32(sml_u + 8 * (lr0 + lr), q)) : make_float2(-INFINITY, 0.f);
        mq[q] = v.x;
        lq[q] = v.y;
      }
      float M = -INFINITY;
#pragma unroll
      for (int q = 0; q < 8; ++q) M = fmaxf(M, mq[q]);
      float wq[8], L = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        wq[q] = mq[q] == -INFINITY ? 0.f : exp2f(mq[q] - M);
        L += wq[q] * lq[q];
      }
      const float inv = 1.f / L;
#pragma unroll
      for (int q = 0; q < 8; ++q) swt[lr * 8 + q] = wq[q] * inv;
    }
    __syncthreads();
    const int items = live_rows * (HD / 4);
    for (int e0 = threadIdx.x; e0 < items; e0 += 2 * blockDim.x) {
      float4 v[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = min(e0 + u * (int)blockDim.x, items - 1);
        const int lr = e / (HD / 4), c4 = e % (HD / 4);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < a.nsplit) v[u][q] = ld_dsmem_f32x4(mapa_u32(so_u + 4 * ((lr0 + lr) * HD + 4 * (c4 ^ ((lr0 + lr) & 7))), q));
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = e0 + u * (int)blockDim.x;
        if (e >= items) continue;
        const int lr = e / (HD / 4), c4 = e % (HD / 4);
        const int row = row0 + lr0 + lr;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < a.nsplit) {
            const float w = swt[lr * 8 + q];
            acc.x += w * v[u][q].x;
            acc.y += w * v[u][q].y;
            acc.z += w * v[u][q].z;
            acc.w += w * v[u][q].w;
          }
        }
        const int n = row / a.G, gg = row % a.G;
        uint2 pk2;
        pk2.x = pack_bf16(acc.x, acc.y);
        pk2.y = pack_bf16(acc.z, acc.w);
        *reinterpret_cast<uint2 *>(a.out + (((long long)sl * a.Nq + n) * a.H + (long long)h * a.G + gg) * HD + 4 * c4) =
            pk2;
      }
    }
    cluster_sync_all();  // peers may still be reading this CTA's shared memory
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) KS_TR(5, gtime());
  if (warp == NSW + 1) tmem_dealloc<TCOLS>(tmem);
}

// ============================================================================ K1, persistent row-copy kernel (KSP)
// The row-copy kernel above runs one (sequence, kv head, row block) unit per CTA.  With one key split
// and more units than SMs (C5 b >= 8 at geometry A: 256-1024 units) every SM runs several CTAs back to
// back, and each pays its entry (barriers, TMEM, Q and first tiles: 2.5-4 us under load) and its exit
// (staging and merging the copies: ~2.8 us) while its ring is empty (profiles/r02/k1_experiments.txt:
// the SMs streamed for 0.56 of the span at b 32 / Lc 1024).  Here min(units, 148) CTAs walk units
// c, c + P, c + 2P, ...: the producer streams the key tiles of consecutive units through the same
// 3-stage ring without a break, so the next unit's first tiles land while this unit's epilogue runs.
// The epilogue stages the copies' O in the (then idle) Q buffer, one 64-column half at a time, and
// frees the O accumulator as soon as it is read; the next unit's Q is staged after it.  Arithmetic,
// copy order and merge order are the row-copy kernel's: the output is bitwise the same.
namespace ksp {
constexpr int HD = 128, ROWS = 128, KEYS = 128, STAGES = 3;
constexpr int HALF = KEYS * 64 * 2, TILE = 2 * HALF;
constexpr int OFF_Q = 0;                               // Q [128][128] bf16; epilogue: O half [128][64] fp32
constexpr int OFF_KV = 32 * 1024;
constexpr int OFF_BAR = OFF_KV + STAGES * 2 * TILE;    // 229376
constexpr int OFF_ML = OFF_BAR + 256;                  // (m, l) of every MMA row [128][2] fp32
constexpr int SMEM = OFF_ML + 1024 + 1024;
static_assert(SMEM <= 232448, "K1 (KSP) shared memory");
}  // namespace ksp

template <int F, bool W2 = false>  // W2: as tree_attn_ks_kernel (F = 1, eight softmax warps)
__global__ void __launch_bounds__(W2 ? 320 : 192, 1) tree_attn_ksp_kernel(const __grid_constant__ AttnArgs a,
                                                                         int units, int nrb, int dyn) {
  constexpr int HD = ksp::HD, ROWS = ksp::ROWS, KEYS = ksp::KEYS, STAGES = ksp::STAGES;
  constexpr int HALF = ksp::HALF, TILE = ksp::TILE;
  constexpr int TCOLS = 512;        // S0, S1 (128 columns each), O (128)
  // Units after the first come from a launch-wide counter (a CTA that finishes early takes the next
  // unit: ragged lengths balance like separate CTAs would), handed to the MMA and softmax warps in
  // order through a kUq-slot queue: the producer is at most STAGES units ahead (every unit has a tile)
  constexpr int kUq = 8;
  constexpr int RP = ROWS / F;      // rows per copy
  constexpr int KT = W2 ? KEYS / 2 : KEYS / F;  // keys per thread per tile
  constexpr int NSW = W2 ? 8 : 4;   // softmax warps; producer = warp NSW, MMA issuer = warp NSW + 1
  constexpr int NST = NSW * 32;
  static_assert(!W2 || F == 1, "W2: 128 live rows");
  static_assert(F == 1 || F == 2 || F == 4, "copies");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem + ksp::OFF_Q;
  uint8_t *sKV = smem + ksp::OFF_KV;
  uint64_t *kv_full = reinterpret_cast<uint64_t *>(smem + ksp::OFF_BAR);
  uint64_t *kv_empty = kv_full + STAGES;
  uint64_t *s_full = kv_empty + STAGES;  // [2]
  uint64_t *p_full = s_full + 2;         // [2]
  uint64_t *o_done = p_full + 2;         // [2]
  uint64_t *q_full = o_done + 2;         // one phase per unit
  uint64_t *o_free = q_full + 1;         // one phase per unit: its O has been read out of TMEM
  uint64_t *u_full = o_free + 1;         // [kUq] unit queue slots (producer -> MMA / softmax)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(u_full + kUq);
  int *uq = reinterpret_cast<int *>(tslot + 1);  // [kUq] unit ids, -1 = no more work
  float *sml = reinterpret_cast<float *>(smem + ksp::OFF_ML);

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = a.Nq * a.G;
  const int P = gridDim.x;
  const float sl2 = a.scale_log2;
  struct Unit {
    int seq, sl, h, row0, Lc, ntiles;
    long long kb, vb;  // tmap rows of slot 0 of this (seq, kv head)
  };
  auto unit_of = [&](int u) {
    Unit x;
    const int rb = u % nrb, z = u / nrb;
    x.sl = z / a.Hkv;
    x.h = z % a.Hkv;
    x.seq = a.seq_base + x.sl;
    x.row0 = F == 1 ? rb * ROWS : 0;
    x.Lc = a.len[x.seq];  // changed only by the step's last kernels: safe before the wait
    x.ntiles = (x.Lc + a.Nq + KEYS - 1) / KEYS;
    x.kb = a.k_row0 + (long long)x.seq * a.seq_rows + (long long)x.h * a.cap;
    x.vb = a.v_row0 + (long long)x.seq * a.seq_rows + (long long)x.h * a.cap;
    return x;
  };
  auto issue = [&](const Unit &x, int i, long long g) {  // K and V of keys [i KEYS, +KEYS) -> stage g % STAGES
    const int s = (int)(g % STAGES);
    uint8_t *kb = sKV + s * 2 * TILE;
    uint8_t *vb = kb + TILE;
    const int p = i * KEYS;
    mbar_arrive_expect_tx(&kv_full[s], 2 * TILE);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
      for (int kh = 0; kh < KEYS / 64; ++kh) {
        tma_load_2d(kb + hf * HALF + kh * 8192, &a.tmK, &kv_full[s], hf * 64, (int)(x.kb + p + kh * 64));
        tma_load_2d(vb + hf * HALF + kh * 8192, &a.tmV, &kv_full[s], hf * 64, (int)(x.vb + p + kh * 64));
      }
    }
  };
  int pre = 0;  // prefix tiles of the first unit issued before the wait
  if (threadIdx.x == NST) {
    tma_prefetch_desc(&a.tmK);
    tma_prefetch_desc(&a.tmV);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], NST);
      mbar_init(&o_done[b], 1);
    }
    mbar_init(q_full, 128);
    mbar_init(o_free, 128);
    for (int j = 0; j < kUq; ++j) mbar_init(&u_full[j], 1);
    fence_barrier_init();
    const Unit x = unit_of(blockIdx.x);
    const int first = min(STAGES, x.ntiles);
    while (pre < first && (pre + 1) * KEYS <= x.Lc) {
      issue(x, pre, pre);
      ++pre;
    }
  }
  const int rr_lane = (warp < NSW) ? (warp & 3) * 32 + lane : 0;
  const int cf = W2 ? (warp < NSW ? warp >> 2 : 0) : rr_lane / RP;  // copy of this softmax thread (W2: key half)
  if (warp == NSW + 1) tmem_alloc<TCOLS>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;  // S0: [0, 128), S1: [128, 256), O: [256, 384)

  if (warp == NSW) {
    // ------------------------------------------------------------ TMA producer: every unit's tiles, one ring
    if (lane == 0) {
      pdl_wait();
      long long g = 0;
      int *work = a.lean_sync + 2, *done = a.lean_sync + 3;  // zero between launches
      for (int u = blockIdx.x, k = 0;; ++k) {
        if (k > 0) {
          u = dyn ? P + atomicAdd(work, 1) : blockIdx.x + k * P;  // dyn 0: static round robin (experiments)
          if (u >= units) u = -1;
          uq[(k - 1) % kUq] = u;
          mbar_arrive(&u_full[(k - 1) % kUq]);
          if (u < 0) {
            if (dyn && atomicAdd(done, 1) == P - 1) {  // the last CTA out resets the counters
              *work = 0;
              *done = 0;
            }
            break;
          }
        }
        const Unit x = unit_of(u);
        if (k > 0) {  // this unit's Q rows -> L2 while the previous unit finishes (its softmax warps load them next)
          const int r0 = x.row0, r1 = min(R, x.row0 + (F == 1 ? ROWS : RP));
          for (int n = r0 / a.G; n * a.G < r1; ++n)
            prefetch_l2_bulk(a.q + (((long long)x.sl * a.Nq + n) * a.H + (long long)x.h * a.G) * HD, a.G * HD * 2);
        }
        for (int i = 0; i < x.ntiles; ++i, ++g) {
          if (k == 0 && i < pre) continue;
          if (g >= STAGES) mbar_wait(&kv_empty[g % STAGES], (int)(((g / STAGES) - 1) & 1));
          issue(x, i, g);
        }
      }
    }
  } else if (warp == NSW + 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_major(ROWS, KEYS, 0, 0);  // Q (K-major) x K^T (K-major)
      constexpr uint32_t idesc_o = idesc_bf16_major(ROWS, HD, 0, 1);    // P (TMEM) x V (MN-major)
      const uint32_t q_u = smem_u32(sQ), kv_u = smem_u32(sKV);
      long long g0 = 0;
      for (int u = blockIdx.x, k = 0;; ++k) {
        if (k > 0) {
          mbar_wait(&u_full[(k - 1) % kUq], ((k - 1) / kUq) & 1);
          u = *(volatile int *)&uq[(k - 1) % kUq];
          if (u < 0) break;
        }
        const int ntiles = unit_of(u).ntiles;
        mbar_wait(q_full, k & 1);
        auto issue_s = [&](long long g) {
          const int sb = (int)(g & 1), st = (int)(g % STAGES);
          mbar_wait(&kv_full[st], (int)((g / STAGES) & 1));
          tc_fence_after();
          const uint32_t kb = kv_u + st * 2 * TILE;
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(q_u + (kk >> 2) * 16384 + (kk & 3) * 32);
            const uint64_t bd = umma_desc_sw128(kb + (kk >> 2) * HALF + (kk & 3) * 32);
            umma_bf16(tmem + sb * KEYS, ad, bd, idesc_s, kk > 0);
          }
          umma_commit(&s_full[sb]);
        };
        issue_s(g0);
        for (int i = 0; i < ntiles; ++i) {
          const long long g = g0 + i;
          if (i + 1 < ntiles) issue_s(g + 1);
          mbar_wait(&p_full[g & 1], (int)((g >> 1) & 1));
          if (i == 0 && k > 0) mbar_wait(o_free, (k - 1) & 1);  // the previous unit's O has been read
          tc_fence_after();
          const uint32_t vb = kv_u + (int)(g % STAGES) * 2 * TILE + TILE;
#pragma unroll
          for (int kk = 0; kk < KEYS / 16; ++kk) {
            const uint64_t bd = umma_desc_mn_sw128(vb + kk * 2048, HALF);
            umma_bf16_ts(tmem + 2 * KEYS, tmem + (int)(g & 1) * KEYS + kk * 8, bd, idesc_o, (i > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&kv_empty[g % STAGES]);
          umma_commit(&o_done[g & 1]);
        }
        g0 += ntiles;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps 0..3 (MMA row = TMEM lane)
    const int r = (warp & 3) * 32 + lane;  // MMA row = cf RP + (query row - row0) (W2: the quadrant's row)
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const int Nq = a.Nq;
    pdl_wait();
    long long g0 = 0;
    uint64_t anc0 = 0, anc1 = 0, anc2 = 0, anc3 = 0;
    int anc_row0 = -1;
    for (int u = blockIdx.x, k = 0;; ++k) {
      if (k > 0) {
        mbar_wait(&u_full[(k - 1) % kUq], ((k - 1) / kUq) & 1);
        u = *(volatile int *)&uq[(k - 1) % kUq];
        if (u < 0) break;
      }
      const Unit x = unit_of(u);
      const int qr = x.row0 + r % RP;  // this thread's query row
      const bool live = qr < R;
      const bool warp_live = W2 || x.row0 + ((warp & 3) * 32) % RP < R;  // W2: every warp keeps the barriers
      if (x.row0 != anc_row0) {  // ancestor words of the row's node (static tree tables)
        anc_row0 = x.row0;
        anc0 = anc1 = anc2 = anc3 = 0;
        if (live) {
          const uint64_t *w = a.anc + (qr / a.G) * kAncWords;
          anc0 = w[0];
          anc1 = w[1];
          anc2 = w[2];
          anc3 = w[3];
        }
      }
      if (!W2 || cf == 0) {  // stage Q row qr (every copy) into the K-major SW128 layout (buffer free: epilogue)
        const uint4 *src = nullptr;
        if (live) {
          const int n = qr / a.G, gg = qr % a.G;
          src = reinterpret_cast<const uint4 *>(a.q + (((long long)x.sl * Nq + n) * a.H + (long long)x.h * a.G + gg) * HD);
        }
        uint4 v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = live ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
        const uint32_t q_u = smem_u32(sQ);
#pragma unroll
        for (int c = 0; c < 16; ++c) st_shared_v4(q_u + (c >> 3) * 16384 + sw128_off(r, c), v[c].x, v[c].y, v[c].z, v[c].w);
        fence_proxy_async();
        mbar_arrive(q_full);
      }
      const int Lc = x.Lc;
      float m_run = -INFINITY, l = 0.f;
      for (int i = 0; i < x.ntiles; ++i) {
        const long long g = g0 + i;
        const int sb = (int)(g & 1);
        mbar_wait(&s_full[sb], (int)((g >> 1) & 1));
        tc_fence_after();
        if (!warp_live) {
          tc_fence_before();
          mbar_arrive(&p_full[sb]);
          continue;
        }
        float y[KT];
        if constexpr (KT == 128) {
          tmem_ld64_f(lane_base + sb * KEYS, y);
          tmem_ld64_f(lane_base + sb * KEYS + 64, y + 64);
        } else if constexpr (KT == 64) {
          tmem_ld64_f(lane_base + sb * KEYS + cf * KT, y);
        } else {
          tmem_ld32_f(lane_base + sb * KEYS + cf * KT, y);
        }
        const int pt = i * KEYS + cf * KT;  // this thread's first key
        constexpr int NH = KT >= 64 ? KT / 64 : 1;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
          constexpr int W = KT >= 64 ? 64 : KT;
          float *yw = y + hh * 64;
          const int p0 = pt + hh * 64;
          if (a.pad && p0 < Lc) {  // pad batching (f4): masked cache slots of the prefix
            const uint32_t *pw = a.pad + (size_t)x.seq * a.pad_words + (p0 >> 5);
            const uint64_t pm = (uint64_t)pw[0] | (W == 64 ? ((uint64_t)pw[1] << 32) : 0ull);
            if (pm) {
#pragma unroll
              for (int j = 0; j < W; ++j) yw[j] = ((pm >> j) & 1ull) ? -INFINITY : yw[j];
            }
          }
          if (p0 + W > Lc) {  // keys past the prefix: visibility bitmask (Eq. 2)
            const int off = p0 - Lc;
            auto word = [&](int q) { return q == 0 ? anc0 : q == 1 ? anc1 : q == 2 ? anc2 : q == 3 ? anc3 : 0ull; };
            uint64_t vis;
            if (off < 0) {
              vis = (off <= -64 ? ~0ull : (~0ull >> (64 + off))) | (off <= -64 ? 0ull : (anc0 << (-off)));
            } else {
              const int q = off >> 6, sh = off & 63;
              const uint64_t lo = word(q), hi = word(q + 1);
              vis = sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
            }
            if (Nq - off < 64) vis &= (Nq - off <= 0) ? 0ull : (~0ull >> (64 - (Nq - off)));
#pragma unroll
            for (int j = 0; j < W; ++j) yw[j] = ((vis >> j) & 1ull) ? yw[j] : -INFINITY;
          }
        }
        float mx0 = y[0], mx1 = y[1], mx2 = y[2], mx3 = y[3];
#pragma unroll
        for (int j = 4; j < KT; j += 4) {
          mx0 = fmaxf(mx0, y[j]);
          mx1 = fmaxf(mx1, y[j + 1]);
          mx2 = fmaxf(mx2, y[j + 2]);
          mx3 = fmaxf(mx3, y[j + 3]);
        }
        float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
        if constexpr (W2) {  // both halves' maxima (sml doubles as the exchange buffer outside the epilogue)
          sml[cf * 128 + r] = mx;
          asm volatile("bar.sync 2, 256;" ::: "memory");
          mx = fmaxf(mx, sml[(cf ^ 1) * 128 + r]);
        }
        float m_new = m_run, alpha = 1.f;
        bool resc = false;
        if (m_run == -INFINITY) {
          m_new = mx;
        } else if (mx > m_run + tc::RESCALE_LOG2) {
          m_new = mx;
          alpha = exp2f(m_run - m_new);
          resc = true;
        }
        const float nb = (m_new == -INFINITY) ? 0.f : -m_new;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        uint32_t pe[KT / 2];
#pragma unroll
        for (int j = 0; j < KT / 2; j += 2) {
          const float e0 = ex2(fmaf(y[2 * j], sl2, nb)), e1 = ex2(fmaf(y[2 * j + 1], sl2, nb));
          const float e2 = ex2(fmaf(y[2 * j + 2], sl2, nb)), e3 = ex2(fmaf(y[2 * j + 3], sl2, nb));
          s0 += e0;
          s1 += e1;
          s2 += e2;
          s3 += e3;
          pe[j] = pack_bf16(e0, e1);
          pe[j + 1] = pack_bf16(e2, e3);
        }
        uint32_t pk[KEYS / 2];
#pragma unroll
        for (int j = 0; j < KEYS / 2; ++j) pk[j] = (j / (KT / 2) == cf) ? pe[j % (KT / 2)] : 0u;
        l = l * alpha + ((s0 + s1) + (s2 + s3));
        m_run = m_new;
        if (__any_sync(0xffffffffu, resc) && i > 0 && (!W2 || cf == 0)) {
          mbar_wait(&o_done[(g - 1) & 1], (int)(((g - 1) >> 1) & 1));
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < HD; c0 += 32) {
            float o[32];
            tmem_ld32_f(lane_base + 2 * KEYS + c0, o);
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] *= alpha;
            tmem_st32_f(lane_base + 2 * KEYS + c0, o);
          }
        }
        if constexpr (W2) {
          tmem_st32_u(lane_base + sb * KEYS + cf * 32, pe);  // this half's 32 packed columns
          asm volatile("bar.sync 3, 256;" ::: "memory");     // both halves have read the exchange slots
        } else {
          tmem_st32_u(lane_base + sb * KEYS, pk);
          tmem_st32_u(lane_base + sb * KEYS + 32, pk + 32);
        }
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
      }
      {  // last PV of this unit
        const long long gl = g0 + x.ntiles - 1;
        mbar_wait(&o_done[gl & 1], (int)((gl >> 1) & 1));
        tc_fence_after();
      }
      // ---- epilogue: (m, l) of every MMA row; O staged in the Q buffer one 64-column half at a time
      // ([128][64] fp32 = 32 KB, 16-byte chunks XOR-swizzled by row), merged by the copy-0 threads
      if constexpr (W2) {  // the row's sum is the two halves' sums (same running max)
        if (cf == 1) sml[128 + r] = l;
        asm volatile("bar.sync 2, 256;" ::: "memory");
        if (cf == 0) l += sml[128 + r];
        asm volatile("bar.sync 2, 256;" ::: "memory");
      }
      if (!W2 || cf == 0) {
        sml[2 * r] = live ? m_run : -INFINITY;
        sml[2 * r + 1] = live ? l : 0.f;
      }
      float *spart = reinterpret_cast<float *>(sQ);
      bf16 *dst = a.out + (((long long)x.sl * Nq + qr / a.G) * a.H + (long long)x.h * a.G + qr % a.G) * HD;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        if (warp_live && (!W2 || cf == 0)) {
#pragma unroll
          for (int c0 = 0; c0 < 64; c0 += 32) {
            float o[32];
            tmem_ld32_f(lane_base + 2 * KEYS + half * 64 + c0, o);
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<float4 *>(spart + r * 64 + 4 * ((c0 / 4 + c) ^ (r & 7))) =
                  make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
          }
        }
        if (half == 1 && (!W2 || cf == 0)) {  // every O column has been read: the next unit's first PV may overwrite it
          tc_fence_before();
          mbar_arrive(o_free);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NST) : "memory");  // the softmax warps
        if (cf == 0 && live) {  // merge the F copies of row qr (copy order), as tree_attn_ks_kernel
          float mq[F], lq[F];
#pragma unroll
          for (int f = 0; f < F; ++f) {
            mq[f] = sml[2 * (f * RP + qr - x.row0)];
            lq[f] = sml[2 * (f * RP + qr - x.row0) + 1];
          }
          float M = mq[0];
#pragma unroll
          for (int f = 1; f < F; ++f) M = fmaxf(M, mq[f]);
          float wq[F], L = 0.f;
#pragma unroll
          for (int f = 0; f < F; ++f) {
            wq[f] = mq[f] == -INFINITY ? 0.f : exp2f(mq[f] - M);
            L += wq[f] * lq[f];
          }
          const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll 4
          for (int c4 = 0; c4 < 16; ++c4) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int f = 0; f < F; ++f) {
              const int rf = f * RP + qr - x.row0;
              const float4 v = *reinterpret_cast<const float4 *>(spart + rf * 64 + 4 * (c4 ^ (rf & 7)));
              acc.x += wq[f] * v.x;
              acc.y += wq[f] * v.y;
              acc.z += wq[f] * v.z;
              acc.w += wq[f] * v.w;
            }
            uint2 pk2;
            pk2.x = pack_bf16(acc.x * inv, acc.y * inv);
            pk2.y = pack_bf16(acc.z * inv, acc.w * inv);
            *reinterpret_cast<uint2 *>(dst + half * 64 + 4 * c4) = pk2;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NST) : "memory");  // staging buffer (then Q) reused
      }
      g0 += x.ntiles;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == NSW + 1) tmem_dealloc<TCOLS>(tmem);
}

// ============================================================================ K1, stream-K ("lean") variant
// The tree-mode kernel above gives every (row block, sequence, kv head) unit nsplit CTAs of a
// cluster (nsplit <= 8, combined over DSMEM): with 1 CTA per SM (192 KB of shared memory) the grid
// is units x nsplit CTAs, so b Hkv = 8 units (C2 b = 8) run 256 CTAs = 1.73 waves on 148 SMs and
// b Hkv = 32 (C2 in-step) runs 64 CTAs.  Here the key tiles of ALL units are one flat sequence
// (unit-major, Ttot tiles in total, known only on the device: Lc lives there) and CTA c of
// Peff <= 148 persistent CTAs takes tiles [c Ttot / Peff, (c+1) Ttot / Peff): every SM streams the
// same number of tiles.  A CTA's range crosses unit boundaries ("segments"); a unit fully inside
// one CTA is written directly, otherwise each covering CTA (a "piece") stores its (m, l, O) rows
// unnormalised to a global slot, and after a grid barrier (all Peff CTAs are co-resident: one per
// SM) the CTAs combine those units in piece order (deterministic), rows spread over all warps.
// Per CTA: two Q buffers (the next segment's Q is staged while this one runs), S double-buffered
// in TMEM, two O accumulators (the next segment's PV starts while this one's O is drained).
namespace lean {
// P in TMEM (over its S buffer, as in the cluster kernel): 2 Q buffers + 5 K/V stages
constexpr int HD = 128, ROWS = 128, KEYS = 64, TILE = KEYS * HD * 2, STAGES = 5;
constexpr int QB = ROWS * HD * 2;   // 32 KB
constexpr int OFF_Q = 0;            // 2 Q buffers
constexpr int OFF_KV = 2 * QB;
constexpr int OFF_BAR = OFF_KV + STAGES * 2 * TILE;  // 229376
constexpr int OFF_SPRE = OFF_BAR + 256;
constexpr int SMEM = OFF_SPRE + (kLeanMaxSeq + 1) * 4 + 16 + 1024;
static_assert(SMEM <= 232448, "lean K1 shared memory");
constexpr int WARPS = 6;
}  // namespace lean

struct LeanSeg {
  int s, u, h, rb, t0, t1, Ts;  // sequence, unit, kv head, row block, tiles [t0, t1) of Ts
  long long pre;                // first global tile of the unit
};

__global__ void __launch_bounds__(192, 1) tree_attn_lean_kernel(const __grid_constant__ AttnArgs a) {
  using namespace lean;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem + OFF_Q;
  uint8_t *sKV = smem + OFF_KV;
  uint64_t *kv_full = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
  uint64_t *kv_empty = kv_full + STAGES;
  uint64_t *s_full = kv_empty + STAGES;  // [2]
  uint64_t *s_free = s_full + 2;         // [2]
  uint64_t *p_full = s_free + 2;         // [2]
  uint64_t *o_done = p_full + 2;         // [2] PV(i) commits to o_done[i & 1]
  uint64_t *q_full = o_done + 2;         // [2] Q buffers
  uint64_t *q_free = q_full + 2;         // [2]
  uint64_t *o_free = q_free + 2;         // [2] O accumulators
  int *spre = reinterpret_cast<int *>(smem + OFF_SPRE);  // per-sequence first global tile, [nseq + 1]
  uint32_t *tslot = reinterpret_cast<uint32_t *>(spre + kLeanMaxSeq + 1);

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = a.Nq * a.G;
  const int RB = (R + ROWS - 1) / ROWS;
  const int UPS = a.Hkv * RB;  // units per sequence
  // ---- the flat tile sequence (Lc is read before griddepcontrol.wait: only the step's last kernels
  // change it, see common.cuh)
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < a.nseq; ++s) {
      spre[s] = acc;
      acc += ((a.len[a.seq_base + s] + a.Nq + KEYS - 1) / KEYS) * UPS;
    }
    spre[a.nseq] = acc;
  }
  __syncthreads();
  const long long Ttot = spre[a.nseq];
  const int Peff = (int)min((long long)gridDim.x, max(1LL, Ttot / max(1, a.lean_min_tiles)));
  const int c = blockIdx.x;
  if (c >= Peff) return;
  const long long g_lo = (long long)c * Ttot / Peff, g_hi = (long long)(c + 1) * Ttot / Peff;
  auto owner = [&](long long g) { return (int)(((g + 1) * Peff - 1) / Ttot); };
  auto seg_at = [&](long long g, LeanSeg &sg) {
    int s = 0;
    while (s + 1 < a.nseq && spre[s + 1] <= g) ++s;
    sg.s = s;
    sg.Ts = (spre[s + 1] - spre[s]) / UPS;
    const long long within = g - spre[s];
    const int ui = (int)(within / sg.Ts);
    sg.u = s * UPS + ui;
    sg.h = ui / RB;
    sg.rb = ui % RB;
    sg.t0 = (int)(within % sg.Ts);
    sg.t1 = (int)min((long long)sg.Ts, sg.t0 + (g_hi - g));
    sg.pre = spre[s] + (long long)ui * sg.Ts;
  };
  const float sl2 = a.scale_log2;
  auto kv_rows = [&](const LeanSeg &sg, long long &kr, long long &vr) {
    const int seq = a.seq_base + sg.s;
    kr = a.k_row0 + (long long)seq * a.seq_rows + (long long)sg.h * a.cap;
    vr = a.v_row0 + (long long)seq * a.seq_rows + (long long)sg.h * a.cap;
  };
  auto issue = [&](int i, long long kr, long long vr, int p) {  // K and V of keys [p, p+64) -> ring stage
    const int st = i % STAGES;
    uint8_t *kb = sKV + st * 2 * TILE;
    uint8_t *vb = kb + TILE;
    mbar_arrive_expect_tx(&kv_full[st], 2 * TILE);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      tma_load_2d(kb + hf * 8192, &a.tmK, &kv_full[st], hf * 64, (int)(kr + p));
      tma_load_2d(vb + hf * 8192, &a.tmV, &kv_full[st], hf * 64, (int)(vr + p));
    }
  };

  if (threadIdx.x == 128) {
    tma_prefetch_desc(&a.tmK);
    tma_prefetch_desc(&a.tmV);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 128);
      mbar_init(&p_full[b], 128);
      mbar_init(&o_done[b], 1);
      mbar_init(&q_full[b], 128);
      mbar_init(&q_free[b], 1);
      mbar_init(&o_free[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;  // S0 [0,64), S1 [64,128), O0 [128,256), O1 [256,384)

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      bool waited = false;
      int i = 0;
      for (long long g = g_lo; g < g_hi;) {
        LeanSeg sg;
        seg_at(g, sg);
        long long kr, vr;
        kv_rows(sg, kr, vr);
        const int Lc = a.len[a.seq_base + sg.s];
        for (int t = sg.t0; t < sg.t1; ++t, ++i) {
          const int p = t * KEYS;
          // tiles entirely inside the committed prefix do not depend on this step: the first ring
          // fill of them is issued before griddepcontrol.wait
          if (!waited && (i >= STAGES || p + KEYS > Lc)) {
            pdl_wait();
            waited = true;
          }
          if (i >= STAGES) mbar_wait(&kv_empty[i % STAGES], ((i / STAGES) - 1) & 1);
          issue(i, kr, vr, p);
        }
        g += sg.t1 - sg.t0;
      }
      if (!waited) pdl_wait();
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_major(ROWS, KEYS, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16_major(ROWS, HD, 0, 1);
      const uint32_t q_u0 = smem_u32(sQ), kv_u = smem_u32(sKV);
      int i = 0, k = 0;
      for (long long g = g_lo; g < g_hi; ++k) {
        LeanSeg sg;
        seg_at(g, sg);
        const int nt = sg.t1 - sg.t0;
        const uint32_t q_u = q_u0 + (k & 1) * QB;
        const uint32_t o_col = 2 * KEYS + (k & 1) * HD;
        mbar_wait(&q_full[k & 1], (k >> 1) & 1);
        auto issue_s = [&](int ii) {
          const int sb = ii & 1, st = ii % STAGES;  // S buffer: PV(ii - 2) was issued before (pipe order)
          mbar_wait(&kv_full[st], (ii / STAGES) & 1);
          tc_fence_after();
          const uint32_t kb = kv_u + st * 2 * TILE;
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(q_u + (kk >> 2) * 16384 + (kk & 3) * 32);
            const uint64_t bd = umma_desc_sw128(kb + (kk >> 2) * 8192 + (kk & 3) * 32);
            umma_bf16(tmem + sb * KEYS, ad, bd, idesc_s, kk > 0);
          }
          umma_commit(&s_full[sb]);
        };
        issue_s(i);
        if (nt == 1) umma_commit(&q_free[k & 1]);
        if (k >= 2) mbar_wait(&o_free[k & 1], ((k >> 1) - 1) & 1);  // segment k-2 drained this O
        for (int j = 0; j < nt; ++j, ++i) {
          if (j + 1 < nt) {
            issue_s(i + 1);
            if (j + 2 == nt) umma_commit(&q_free[k & 1]);  // the segment's last S reads Q
          }
          mbar_wait(&p_full[i & 1], (i >> 1) & 1);
          tc_fence_after();
          const uint32_t vb = kv_u + (i % STAGES) * 2 * TILE + TILE;
#pragma unroll
          for (int kk = 0; kk < KEYS / 16; ++kk) {
            const uint64_t bd = umma_desc_mn_sw128(vb + kk * 2048, 8192);
            umma_bf16_ts(tmem + o_col, tmem + (i & 1) * KEYS + kk * 8, bd, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&kv_empty[i % STAGES]);
          umma_commit(&o_done[i & 1]);
        }
        g += nt;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps 0..3 (row = TMEM lane)
    const int r = warp * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    pdl_wait();  // q comes from the preceding kernel; partial slots are rewritten below
    auto load_q = [&](const LeanSeg &sg, int buf) {  // this row of the unit's Q -> K-major SW128 layout
      const int rr = sg.rb * ROWS + r;
      const bool live = rr < R;
      const uint4 *src = nullptr;
      if (live) {
        const int n = rr / a.G, gg = rr % a.G;
        src = reinterpret_cast<const uint4 *>(a.q + (((long long)sg.s * a.Nq + n) * a.H + (long long)sg.h * a.G + gg) *
                                                        HD);
      }
      uint4 v[16];
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) v[cc] = live ? __ldg(src + cc) : make_uint4(0, 0, 0, 0);
      const uint32_t q_u = smem_u32(sQ) + buf * QB;
#pragma unroll
      for (int cc = 0; cc < 16; ++cc)
        st_shared_v4(q_u + (cc >> 3) * 16384 + sw128_off(r, cc), v[cc].x, v[cc].y, v[cc].z, v[cc].w);
      fence_proxy_async();
      mbar_arrive(&q_full[buf]);
    };
    const int Nq = a.Nq;
    int i = 0, k = 0;
    LeanSeg sg;
    if (g_lo < g_hi) {
      seg_at(g_lo, sg);
      load_q(sg, 0);
    }
    for (long long g = g_lo; g < g_hi; ++k) {
      const int nt = sg.t1 - sg.t0;
      const long long gn = g + nt;
      LeanSeg nx;
      if (gn < g_hi) {  // stage the next segment's Q now (its buffer's last S MMAs are done: k - 1)
        seg_at(gn, nx);
        if (k + 1 >= 2) mbar_wait(&q_free[(k + 1) & 1], (((k + 1) >> 1) - 1) & 1);
        load_q(nx, (k + 1) & 1);
      }
      const int ob = k & 1;
      const uint32_t o_col = 2 * KEYS + ob * HD;
      const int rr = sg.rb * ROWS + r;
      const bool live = rr < R;
      const bool warp_live = sg.rb * ROWS + warp * 32 < R;
      const int seq = a.seq_base + sg.s;
      const int Lc = a.len[seq];
      uint64_t anc0 = 0, anc1 = 0, anc2 = 0, anc3 = 0;
      if (live) {
        const uint64_t *w = a.anc + (rr / a.G) * kAncWords;
        anc0 = w[0];
        anc1 = w[1];
        anc2 = w[2];
        anc3 = w[3];
      }
      float m_run = -INFINITY, l = 0.f;
      for (int j = 0; j < nt; ++j, ++i) {
        const int sb = i & 1;
        mbar_wait(&s_full[sb], (i >> 1) & 1);
        tc_fence_after();
        if (!warp_live) {
          tc_fence_before();
          mbar_arrive(&p_full[sb]);
          continue;
        }
        float y[64];
        tmem_ld64_f(lane_base + sb * KEYS, y);
        const int p0 = (sg.t0 + j) * KEYS;
        if (a.pad && p0 < Lc) {  // pad batching (f4): masked cache slots of this sequence's prefix
          const uint32_t *pw = a.pad + (size_t)seq * a.pad_words + (p0 >> 5);
          const uint64_t pm = (uint64_t)pw[0] | ((uint64_t)pw[1] << 32);
          if (pm) {
#pragma unroll
            for (int jj = 0; jj < 64; ++jj) y[jj] = ((pm >> jj) & 1ull) ? -INFINITY : y[jj];
          }
        }
        if (p0 + KEYS > Lc) {  // tile reaches past the prefix: visibility of its 64 keys (Eq. 2)
          const int off = p0 - Lc;
          auto word = [&](int q) { return q == 0 ? anc0 : q == 1 ? anc1 : q == 2 ? anc2 : q == 3 ? anc3 : 0ull; };
          uint64_t vis;
          if (off < 0) {
            vis = (~0ull >> (64 + off)) | (anc0 << (-off));
          } else {
            const int q = off >> 6, sh = off & 63;
            const uint64_t lo = word(q), hi = word(q + 1);
            vis = sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
          }
          if (Nq - off < 64) vis &= (Nq - off <= 0) ? 0ull : (~0ull >> (64 - (Nq - off)));
#pragma unroll
          for (int jj = 0; jj < 64; ++jj) y[jj] = ((vis >> jj) & 1ull) ? y[jj] : -INFINITY;
        }
        float mx0 = y[0], mx1 = y[1];
#pragma unroll
        for (int jj = 2; jj < 64; jj += 2) {
          mx0 = fmaxf(mx0, y[jj]);
          mx1 = fmaxf(mx1, y[jj + 1]);
        }
        const float mx = fmaxf(mx0, mx1) * sl2;
        float m_new = m_run, alpha = 1.f;
        bool resc = false;
        if (m_run == -INFINITY) {
          m_new = mx;
        } else if (mx > m_run + tc::RESCALE_LOG2) {
          m_new = mx;
          alpha = exp2f(m_run - m_new);
          resc = true;
        }
        const float nb = (m_new == -INFINITY) ? 0.f : -m_new;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        uint32_t pk[32];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) {
          const float e0 = ex2(fmaf(y[2 * jj], sl2, nb)), e1 = ex2(fmaf(y[2 * jj + 1], sl2, nb));
          const float e2 = ex2(fmaf(y[2 * jj + 2], sl2, nb)), e3 = ex2(fmaf(y[2 * jj + 3], sl2, nb));
          s0 += e0;
          s1 += e1;
          s2 += e2;
          s3 += e3;
          pk[jj] = pack_bf16(e0, e1);
          pk[jj + 1] = pack_bf16(e2, e3);
        }
        l = l * alpha + ((s0 + s1) + (s2 + s3));
        m_run = m_new;
        if (__any_sync(0xffffffffu, resc) && j > 0) {
          mbar_wait(&o_done[sb ^ 1], ((i - 1) >> 1) & 1);  // PV(i-1) done: O is stable
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < HD; c0 += 32) {
            float o[32];
            tmem_ld32_f(lane_base + o_col + c0, o);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) o[jj] *= alpha;
            tmem_st32_f(lane_base + o_col + c0, o);
          }
        }
        tmem_st32_u(lane_base + sb * KEYS, pk);  // P(i) over S(i)
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
      }
      // ---- segment end: O of this unit's piece
      const int il = i - 1;
      mbar_wait(&o_done[il & 1], (il >> 1) & 1);
      tc_fence_after();
      const int own0 = owner(sg.pre);
      const int npieces = owner(sg.pre + sg.Ts - 1) - own0 + 1;
      if (warp_live) {
        if (npieces == 1) {  // the whole unit in this CTA: final output
          const float inv = live ? 1.f / l : 0.f;
          bf16 *dst = a.out + (((long long)sg.s * a.Nq + rr / a.G) * a.H + (long long)sg.h * a.G + rr % a.G) * HD;
#pragma unroll
          for (int c0 = 0; c0 < HD; c0 += 32) {
            float o[32];
            tmem_ld32_f(lane_base + o_col + c0, o);
            if (live) {
#pragma unroll
              for (int cc = 0; cc < 4; ++cc) {
                uint4 w;
                w.x = pack_bf16(o[8 * cc] * inv, o[8 * cc + 1] * inv);
                w.y = pack_bf16(o[8 * cc + 2] * inv, o[8 * cc + 3] * inv);
                w.z = pack_bf16(o[8 * cc + 4] * inv, o[8 * cc + 5] * inv);
                w.w = pack_bf16(o[8 * cc + 6] * inv, o[8 * cc + 7] * inv);
                reinterpret_cast<uint4 *>(dst + c0)[cc] = w;
              }
            }
          }
        } else {  // a piece: unnormalised (m, l, O) column-major in its slot (coalesced over rows)
          const long long slot = (long long)sg.u + own0 + (c - own0);
          float *po = a.lean_part + slot * (long long)(ROWS * (HD + 2));
#pragma unroll
          for (int c0 = 0; c0 < HD; c0 += 32) {
            float o[32];
            tmem_ld32_f(lane_base + o_col + c0, o);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) __stcg(po + (size_t)(c0 + jj) * ROWS + r, o[jj]);
          }
          __stcg(po + (size_t)HD * ROWS + r, live ? m_run : -INFINITY);
          __stcg(po + (size_t)(HD + 1) * ROWS + r, live ? l : 0.f);
        }
      }
      tc_fence_before();
      mbar_arrive(&o_free[ob]);
      g = gn;
      sg = nx;
    }
  }

  // ---- grid barrier (all Peff CTAs are resident: one per SM, Peff <= SMs), then the combine
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&a.lean_sync[0], 1);
    while (ld_acquire_gpu(&a.lean_sync[0]) < Peff) __nanosleep(64);
  }
  __syncthreads();
  {
    // Units with more than one piece are exactly those a CTA boundary falls inside; unit u is
    // enumerated once, by the first boundary inside it (CTA b starts inside u and CTA b - 1 starts
    // at or before u's first tile).  Work item = (boundary b, 32-row group, 32-column chunk), one
    // warp each, lane = row; decoded directly (no per-item scan).  Loads are batched (8 pieces'
    // (m, l), then 2 pieces x 32 columns): ~np / 2 + 2 dependent L2 round trips per item.
    const int gw = c * WARPS + warp, nw = Peff * WARPS;
    constexpr long long PS = (long long)ROWS * (HD + 2);  // floats per piece slot
    const int n_items = (Peff - 1) * 16;
    for (int it2 = gw; it2 < n_items; it2 += nw) {
      const int b = it2 / 16 + 1, rg = (it2 / 4) % 4, c0 = (it2 % 4) * 32;
      const long long gb = (long long)b * Ttot / Peff;  // first tile of CTA b
      LeanSeg su;
      {
        int s = 0;
        while (s + 1 < a.nseq && spre[s + 1] <= gb) ++s;
        su.s = s;
        su.Ts = (spre[s + 1] - spre[s]) / UPS;
        const int ui = (int)((gb - spre[s]) / su.Ts);
        su.u = s * UPS + ui;
        su.h = ui / RB;
        su.rb = ui % RB;
        su.pre = spre[s] + (long long)ui * su.Ts;
      }
      if (gb == su.pre || owner(su.pre) != b - 1) continue;  // not split here, or not its first boundary
      const int u = su.u, s = su.s, h = su.h, rb = su.rb;
      const int own0 = b - 1;
      const int np = owner(su.pre + su.Ts - 1) - own0 + 1;
      const int live_rows = min(ROWS, R - rb * ROWS);
      const int w0 = rg * 32;
      if (w0 >= live_rows) continue;
      {
        {
          const int r = w0 + lane;
          const bool live = r < live_rows;
          const float *base = a.lean_part + ((long long)u + own0) * PS;
          float M = -INFINITY, L = 0.f;
          for (int q0 = 0; q0 < np; q0 += 8) {
            float mq[8], lq[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const bool ok = q0 + e < np;
              mq[e] = ok ? __ldcg(base + (q0 + e) * PS + HD * ROWS + r) : -INFINITY;
              lq[e] = ok ? __ldcg(base + (q0 + e) * PS + (HD + 1) * ROWS + r) : 0.f;
            }
            float Mb = -INFINITY;
#pragma unroll
            for (int e = 0; e < 8; ++e) Mb = fmaxf(Mb, mq[e]);
            const float Mn = fmaxf(M, Mb);
            float Lb = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) Lb += mq[e] == -INFINITY ? 0.f : exp2f(mq[e] - Mn) * lq[e];
            L = (M == -INFINITY ? 0.f : L * exp2f(M - Mn)) + Lb;
            M = Mn;
          }
          const float invL = live ? 1.f / L : 0.f;
          float acc[32];
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) acc[jj] = 0.f;
          for (int q = 0; q < np; q += 2) {  // piece order: deterministic
            float v0[32], v1[32], w[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const bool ok = q + e < np;
              const float mq = ok ? __ldcg(base + (q + e) * PS + HD * ROWS + r) : -INFINITY;
              w[e] = mq == -INFINITY ? 0.f : exp2f(mq - M) * invL;
            }
            const float *b0 = base + q * PS + (size_t)c0 * ROWS + r;
            const float *b1 = q + 1 < np ? b0 + PS : b0;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              v0[jj] = __ldcg(b0 + (size_t)jj * ROWS);
              v1[jj] = __ldcg(b1 + (size_t)jj * ROWS);
            }
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) acc[jj] += w[0] * v0[jj] + w[1] * v1[jj];
          }
          if (live) {
            const int rr = rb * ROWS + r;
            bf16 *dst = a.out + (((long long)s * a.Nq + rr / a.G) * a.H + (long long)h * a.G + rr % a.G) * HD + c0;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              uint4 wv;
              wv.x = pack_bf16(acc[8 * cc], acc[8 * cc + 1]);
              wv.y = pack_bf16(acc[8 * cc + 2], acc[8 * cc + 3]);
              wv.z = pack_bf16(acc[8 * cc + 4], acc[8 * cc + 5]);
              wv.w = pack_bf16(acc[8 * cc + 6], acc[8 * cc + 7]);
              reinterpret_cast<uint4 *>(dst)[cc] = wv;
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the last CTA out resets the barrier for the next launch (every CTA has passed the wait)
    if (atomicAdd(&a.lean_sync[1], 1) == Peff - 1) {
      a.lean_sync[0] = 0;
      a.lean_sync[1] = 0;
      __threadfence();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc<512>(tmem);
}

cudaError_t attention_lean_launch(const AttnArgs &a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tree_attn_lean_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lean::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (a.nseq > kLeanMaxSeq || !a.lean_part || !a.lean_sync) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kNumSMs);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = lean::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = gemm_pdl() ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, tree_attn_lean_kernel, a);
}

// Partial slots the lean kernel may use for nunits units: nunits + 148 of [128 rows][hd + 2] fp32.
size_t attention_lean_part_floats(int nunits) { return (size_t)(nunits + kNumSMs) * lean::ROWS * (lean::HD + 2); }

SM_GT_READER(sm_gtrace_read_attn)
#ifdef SM_TRACE
extern "C" int sm_trace_read(long long *dst, int n) {  // diagnostics build only
  return (int)cudaMemcpyFromSymbol(dst, g_trace, sizeof(long long) * (size_t)n);
}
#endif

// Most clusters of ns CTAs of the one-CTA-per-SM K1 kernels that can be co-resident, queried once per ns:
// clusters must fit inside a GPC, so e.g. only 15 clusters of 8 run at a time (120 of 148 SMs) and
// 16 units x 8 splits took two waves (profiles/r02/k1_experiments.txt, geometry B b 16 / Lc 32K).
static int active_clusters(int ns) {
  static int cache[9] = {0};
  if (ns <= 1) return kNumSMs;
  if (cache[ns] == 0) {
    int n = 0;
    if (cudaFuncSetAttribute(tree_attn_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM) ==
        cudaSuccess) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(ns, 1, 256);
      cfg.blockDim = dim3(192);
      cfg.dynamicSmemBytes = tc::SMEM;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = ns;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, (void *)tree_attn_tc_kernel<false>, &cfg) != cudaSuccess) n = 0;
    }
    cudaGetLastError();
    cache[ns] = n > 0 ? n : kNumSMs / ns;
  }
  return cache[ns];
}

// Key splits (= cluster size, 1..8) for `units` (sequence, kv head, row block) units of up to cap keys:
// minimise waves x (keys per CTA + a fixed per-CTA cost of ~256 keys), waves = units over the clusters of
// that size that fit at once.
static int g_attn_ksp = 1;  // sm_set_option("attn_ksp"), see attention_tc_launch
static int g_split_model = 1;  // sm_set_option("attn_split_model"): 1 occupancy-aware (default), 0 round-1 rule
void attention_set_split_model(int m) { g_split_model = m; }
int attention_tc_nsplit(int units, int cap) {
  if (g_split_model == 0) {  // round 1: powers of two up to ~one wave of 148 CTAs
    int ns = 1;
    while (ns < 8 && units * ns * 2 <= kNumSMs) ns *= 2;
    return ns;
  }
  constexpr double kOverheadKeys = 256;
  int best = 1;
  double best_cost = -1;
  for (int ns = 1; ns <= 8; ++ns) {
    const int act = active_clusters(ns);
    double cost = std::ceil((double)units / act) * ((cap + ns - 1) / ns + kOverheadKeys);
    if (ns == 1 && units > kNumSMs && g_attn_ksp)  // persistent KSP: units stream back to back, no waves
      cost = (double)units / kNumSMs * (cap + kOverheadKeys / 2);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = ns;
    }
  }
  return best;
}

// sm_set_option("attn_l2ahead"), AttnArgs::l2_ahead.  Default 2: the next wave's first ring and Q rows go
// to L2 once a CTA has issued its last tile (profiles/r02/k1_experiments.txt: 3-5 % on multi-wave launches,
// neutral elsewhere); bit 0 (the CTA's own range at entry) measured 5-40 % slower (it floods the
// memory system ahead of the ring's own loads) and stays off
static int g_attn_l2ahead = 2;
// sm_set_option("attn_w2"): row-copy kernels with 128 live rows on 8 softmax warps (1, default: 5-10 % on those
// launches, profiles/r02/k1_experiments.txt) or 4 (0)
static int g_attn_w2 = 1;
// sm_set_option("attn_qearly"): row-copy kernel loads Q before its CTA barrier (1, default: 0-3 %, never slower,
// profiles/r02/k1_experiments.txt) or after it (0)
static int g_attn_qearly = 1;
void attention_set_qearly(int on) { g_attn_qearly = on; }
void attention_set_w2(int on) { g_attn_w2 = on; }
void attention_set_l2ahead(int mode) { g_attn_l2ahead = mode & 3; }
// sm_set_option("attn_ksp"): persistent row-copy kernel when a one-split launch has more units than SMs (1,
// default: 3-14 % faster on every multi-wave C5 point, profiles/r02/k1_experiments.txt) or never (0)
void attention_set_ksp(int on) { g_attn_ksp = on; }
static int g_attn_ks = 2;  // sm_set_option("attn_ks"): 128-key-tile kernel on long key ranges, all N G (2, default), N G <= 64 (1), off (0)
void attention_set_ks(int on) { g_attn_ks = on; }

cudaError_t attention_tc_launch(const AttnArgs &a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tree_attn_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         tc::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tree_attn_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.nsplit, (a.Nq * a.G + tc::ROWS - 1) / tc::ROWS, a.nseq * a.Hkv);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = tc::SMEM;
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
  const int R = a.Nq * a.G;
  // 128-key-tile kernel (row copies F = 128 / RP for <= 64 live rows) unless the key range is cut into
  // short splits (cache capacity / nsplit < 1024: the C2 in-step shape, ~530 keys per split), where
  // the 128-row kernel measured faster (profiles/r02/k1_experiments.txt)
  const bool long_range = a.nsplit == 1 || a.cap >= 1024 * a.nsplit;
  if (g_attn_ks && !a.causal && (g_attn_ks > 1 || R <= 64) && long_range) {
    static bool ks_attr = false;
    if (!ks_attr) {
      const auto A = cudaFuncAttributeMaxDynamicSharedMemorySize;
      cudaError_t e = cudaSuccess;
      for (auto fn : {tree_attn_ks_kernel<4, 128>, tree_attn_ks_kernel<2, 128>, tree_attn_ks_kernel<1, 128>,
                      tree_attn_ks_kernel<1, 128, true>})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, A, ks::SMEM);
      if (e != cudaSuccess) return e;
      ks_attr = true;
    }
    const int nrb = R <= 64 ? 1 : (R + 127) / 128;
    const int units = a.nseq * a.Hkv * nrb;
    if (g_attn_ksp && a.nsplit == 1 && units > kNumSMs && a.lean_sync) {  // several units per SM: persistent (KSP)
      static bool ksp_attr = false;
      if (!ksp_attr) {
        const auto A = cudaFuncAttributeMaxDynamicSharedMemorySize;
        cudaError_t e = cudaSuccess;
        for (auto fn : {tree_attn_ksp_kernel<4>, tree_attn_ksp_kernel<2>, tree_attn_ksp_kernel<1>,
                        tree_attn_ksp_kernel<1, true>})
          if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, A, ksp::SMEM);
        if (e != cudaSuccess) return e;
        ksp_attr = true;
      }
      cfg.gridDim = dim3(kNumSMs);
      cfg.dynamicSmemBytes = ksp::SMEM;
      cfg.numAttrs = 1;
      const int dyn = g_attn_ksp == 3 ? 0 : 1;
      if (R <= 32) return cudaLaunchKernelEx(&cfg, tree_attn_ksp_kernel<4>, a, units, nrb, dyn);
      if (R <= 64) return cudaLaunchKernelEx(&cfg, tree_attn_ksp_kernel<2>, a, units, nrb, dyn);
      if (g_attn_w2) {
        cfg.blockDim = dim3(320);
        return cudaLaunchKernelEx(&cfg, tree_attn_ksp_kernel<1, true>, a, units, nrb, dyn);
      }
      return cudaLaunchKernelEx(&cfg, tree_attn_ksp_kernel<1>, a, units, nrb, dyn);
    }
    cfg.dynamicSmemBytes = ks::SMEM;
    AttnArgs b = a;
    b.l2_ahead = (a.k_base && a.v_base) ? g_attn_l2ahead : 0;
    b.q_early = g_attn_qearly;
    if (R <= 32) return cudaLaunchKernelEx(&cfg, tree_attn_ks_kernel<4, 128>, b);
    if (R <= 64) return cudaLaunchKernelEx(&cfg, tree_attn_ks_kernel<2, 128>, b);
    if (g_attn_w2) {  // two softmax warps per row (W2)
      cfg.blockDim = dim3(320);
      return cudaLaunchKernelEx(&cfg, tree_attn_ks_kernel<1, 128, true>, b);
    }
    return cudaLaunchKernelEx(&cfg, tree_attn_ks_kernel<1, 128>, b);  // ceil(R / 128) row blocks (grid y)
  }
  if (a.causal) return cudaLaunchKernelEx(&cfg, tree_attn_tc_kernel<true>, a);
  return cudaLaunchKernelEx(&cfg, tree_attn_tc_kernel<false>, a);
}

void attention_set_l2pf(int on) { cudaMemcpyToSymbol(g_attn_l2pf, &on, sizeof(int)); }

void attention_tc_preload() {  // force-load (see gemm_preload)
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, tree_attn_lean_kernel);
  cudaFuncGetAttributes(&fa, tree_attn_tc_kernel<false>);
  cudaFuncGetAttributes(&fa, tree_attn_tc_kernel<true>);
  cudaFuncGetAttributes(&fa, tree_attn_ks_kernel<4, 128>);
  cudaFuncGetAttributes(&fa, tree_attn_ks_kernel<2, 128>);
  cudaFuncGetAttributes(&fa, tree_attn_ks_kernel<1, 128>);
}

}  // namespace sm
