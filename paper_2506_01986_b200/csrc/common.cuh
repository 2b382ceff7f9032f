// common.cuh -- shared device helpers for the sm_100a kernels: bf16 conversion,
// mbarrier / TMA (cp.async.bulk.tensor) / tcgen05 PTX wrappers, warp reductions.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

#define SM_DEV __device__ __forceinline__

namespace sm {



SM_DEV float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
SM_DEV __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }
SM_DEV float bfbits2f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

SM_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Programmatic dependent launch: wait for the preceding kernel (all reads of its
// outputs and all writes must come after), and let the next kernel launch.
SM_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SM_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Kernels that change step-static state (Lc, positions, pad bitmaps) trigger their dependents
// only after those writes are fenced: kernels downstream read Lc before their own
// griddepcontrol.wait, and every trigger-at-entry kernel in between would otherwise let them
// start while the writer still runs.  Every thread of the block must reach this call.
SM_DEV void pdl_trigger_after_writes() {
  __threadfence();
  __syncthreads();
  pdl_trigger();
}

SM_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SM_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------------------------ clusters / DSMEM
SM_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
SM_DEV void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
SM_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
SM_DEV uint32_t mapa_u32(uint32_t smem_addr, int rank) {  // this CTA's smem address -> rank's copy
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
SM_DEV float ld_dsmem_f32(uint32_t cluster_addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cluster_addr) : "memory");
  return v;
}
SM_DEV void st_dsmem_f32(uint32_t cluster_addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(cluster_addr), "f"(v) : "memory");
}
SM_DEV float2 ld_dsmem_f32x2(uint32_t cluster_addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(cluster_addr) : "memory");
  return v;
}
SM_DEV void st_dsmem_f32x4(uint32_t cluster_addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(cluster_addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
SM_DEV void st_dsmem_f32x2(uint32_t cluster_addr, float a, float b) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(cluster_addr), "f"(a), "f"(b) : "memory");
}
SM_DEV float4 ld_dsmem_f32x4(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}

// ------------------------------------------------------------------ logits statistics
// Single-pass typical statistics of y over a row: m = max y, s = sum e^(y-m),
// t = sum e^(y-m) (y-m), so H = log s - t/s (reading Q10); merges are exact
// re-basings, applied in a fixed order.
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
SM_DEV void mst_add(MST &acc, float y) {
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
SM_DEV void argmax_merge(float &v, int &i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

// ------------------------------------------------------------------ cross-GPU flags (tensor parallel)
SM_DEV void st_release_sys(long long *p, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SM_DEV int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SM_DEV long long ld_acquire_sys(const long long *p) {
  long long v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
SM_DEV unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait until *f >= ep; after ~10 s give up, raise *err and continue (no hung GPU).
SM_DEV void tp_wait_flag(const long long *f, long long ep, int *err) {
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_sys(f) < ep) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > 10000000000ull) {
      atomicExch(err, 1);
      break;
    }
  }
}

// Diagnostics build only (-DSM_TRACE, build(trace=True)): per-CTA clock64 stamps.
#ifdef SM_TRACE
constexpr int kTraceCtas = 1024, kTraceSlots = 24;
static __device__ long long g_trace[kTraceCtas][kTraceSlots];  // per translation unit
#define SM_STAMP(slot)                                                                           \
  do {                                                                                           \
    const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);             \
    if (cta_ < kTraceCtas) g_trace[cta_][slot] = clock64();                                      \
  } while (0)
// Cross-kernel timeline (diagnostics build): one record per CTA {kernel id, globaltimer at
// entry, after griddepcontrol.wait, at exit}; per translation unit, read by sm_gtrace_read_*.
constexpr int kGtRecs = 1 << 17;
static __device__ long long g_gt[kGtRecs][4];
static __device__ unsigned int g_gt_n;
SM_DEV long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SM_GT_BEGIN() long long gt0_ = gtime(), gt1_ = 0
#define SM_GT_WAITED() gt1_ = gtime()
#define SM_GT_END(kid)                                  \
  do {                                                  \
    const unsigned i_ = atomicAdd(&g_gt_n, 1u);         \
    if (i_ < (unsigned)kGtRecs) {                       \
      g_gt[i_][0] = (kid);                              \
      g_gt[i_][1] = gt0_;                               \
      g_gt[i_][2] = gt1_;                               \
      g_gt[i_][3] = gtime();                            \
    }                                                   \
  } while (0)
#define SM_GT_READER(name)                                                                   \
  extern "C" int name(long long *dst, int max_recs) {                                        \
    unsigned n = 0;                                                                          \
    cudaMemcpyFromSymbol(&n, g_gt_n, sizeof(n));                                             \
    n = n < (unsigned)max_recs ? n : (unsigned)max_recs;                                     \
    n = n < (unsigned)kGtRecs ? n : (unsigned)kGtRecs;                                       \
    cudaMemcpyFromSymbol(dst, g_gt, sizeof(long long) * 4 * (size_t)n);                      \
    const unsigned z = 0;                                                                    \
    cudaMemcpyToSymbol(g_gt_n, &z, sizeof(z));                                               \
    return (int)n;                                                                           \
  }
#else
#define SM_STAMP(slot) \
  do {                 \
  } while (0)
#define SM_GT_BEGIN() \
  do {                \
  } while (0)
#define SM_GT_WAITED() \
  do {                 \
  } while (0)
#define SM_GT_END(kid) \
  do {                 \
  } while (0)
#define SM_GT_READER(name)
#endif

// ------------------------------------------------------------------ mbarrier
SM_DEV void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
SM_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SM_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
SM_DEV void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
SM_DEV void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
SM_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------ TMA
SM_DEV void tma_prefetch_desc(const CUtensorMap *m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)m) : "memory");
}
// 2D tiled load: box at (c0 = inner/column coordinate, c1 = row coordinate).
SM_DEV void tma_load_2d(void *smem_dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
SM_DEV void tma_load_2d_hint(void *smem_dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
// TMA prefetch of a 2D box into L2 only (no shared memory, no completion)
SM_DEV void tma_prefetch_l2_2d(const CUtensorMap *m, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"((uint64_t)m), "r"(c0), "r"(c1)
               : "memory");
}
// bulk prefetch of [ptr, ptr + bytes) into L2 (bytes a multiple of 16)
SM_DEV void prefetch_l2_bulk(const void *ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((uint64_t)ptr), "r"(bytes) : "memory");
}
SM_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SM_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------------ tcgen05
// UMMA shared-memory descriptor, K-major operand, SWIZZLE_128B canonical layout:
// 8-row x 128-byte swizzle atoms stacked along M/N with SBO = 1024 B.
SM_DEV uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);        // start address [0,14)
  d |= (uint64_t)1 << 16;                            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                  // SBO [32,46)
  d |= (uint64_t)1 << 46;                            // version = 1 (sm_100)
  d |= (uint64_t)2 << 61;                            // layout: SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
SM_DEV void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// A operand from tensor memory (K-major, 16-bit: lane = row, column c = elements 2c, 2c+1 packed)
SM_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
SM_DEV void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
SM_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SM_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// ---- 2-SM (CTA pair) variants: tcgen05 cta_group::2 (cluster of 2 CTAs on one TPC)
SM_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// D[256 x N] (lanes of both CTAs) += A[256 x K] (128 rows from each CTA's smem at the same
// address) * B[N x K] (N/2 rows from each CTA's smem).  Issued by the leader CTA only.
SM_DEV void umma_bf16_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// completion of the leader's MMAs arrives on the mbarrier at this offset in every CTA of mask
SM_DEV void umma_commit_cg2(uint64_t *bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                   "r"(smem_u32(bar)),
               "h"(mask)
               : "memory");
}
// TMA into this CTA's smem, completion counted on the mbarrier at cluster address mbar_cl
// (the leader's barrier: both CTAs' bytes complete one transaction count)
SM_DEV void tma_load_2d_cg2(void *smem_dst, const CUtensorMap *m, uint32_t mbar_cl, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem_dst)),
      "l"((uint64_t)m), "r"(mbar_cl), "r"(c0), "r"(c1)
      : "memory");
}
SM_DEV void tma_load_2d_cg2_hint(void *smem_dst, const CUtensorMap *m, uint32_t mbar_cl, int c0, int c1,
                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"((uint64_t)m), "r"(mbar_cl), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
SM_DEV void mbar_arrive_cluster(uint32_t mbar_cl) {  // arrive on a (possibly peer) CTA's mbarrier
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mbar_cl) : "memory");
}
template <int NCOLS>
SM_DEV void tmem_alloc_cg2(uint32_t *smem_dst) {  // one warp of EACH CTA of the pair
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <int NCOLS>
SM_DEV void tmem_dealloc_cg2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}

template <int NCOLS>
SM_DEV void tmem_alloc(uint32_t *smem_dst) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int NCOLS>
SM_DEV void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}
// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread.
SM_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
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

// ------------------------------------------------------------------ legacy mma.sync (attention)
SM_DEV void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
SM_DEV void ldmatrix_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SM_DEV void ldmatrix_x4_trans(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SM_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

}  // namespace sm
