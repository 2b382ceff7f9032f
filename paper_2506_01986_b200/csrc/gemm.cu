// gemm.cu -- K2: small-M bf16 GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
//   out[split][m][n] = sum_{k in split} x[m][k] * w[n][k]        (fp32 partials)
//
// Swap-AB: the weight tile (128 output features x 64 k, K-major, SWIZZLE_128B)
// is the UMMA A operand (M = 128 lanes of TMEM), the token rows (BN <= 256,
// padded to 16) are the UMMA N dimension.  This keeps M = b*N = 1..256 token
// rows from wasting the 128-row MMA.  Warp roles: warp 0 lane 0
// issues TMA into a STAGES-deep mbarrier ring, warp 1 lane 0 issues tcgen05.mma
// and tcgen05.commit (frees the smem slot), then all 4 warps drain the fp32
// accumulator with tcgen05.ld and write coalesced fp32 partials.  Split-K over
// CTAs fills the 148 SMs; the fixed-order reduction of the partials is fused
// into the consumer kernels (epilogue.cu), so results are deterministic.
#include "common.cuh"
#include "kernels.h"

namespace sm {

template <int BN>
struct GemmCfg {
  static constexpr int kA = 128 * 64 * 2;          // weight tile bytes
  static constexpr int kB = BN * 64 * 2;           // activation tile bytes
  static constexpr int kStage = kA + kB;
  static constexpr int kStages = BN <= 16 ? 6 : BN <= 32 ? 5 : BN <= 64 ? 4 : BN <= 128 ? 6 : 4;
  static constexpr int kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int kSmem = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__global__ void __launch_bounds__(128, 1) gemm_bf16_tc_kernel(const __grid_constant__ GemmArgs args) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::kStages * C::kA;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::kStages * C::kStage);
  uint64_t *empty = full + C::kStages;
  uint64_t *done = empty + C::kStages;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, split = blockIdx.y;
  const int bi = blockIdx.z % args.batch, tt = blockIdx.z / args.batch;
  const int kb0 = split * args.kb_per_split;
  const int nkb = min(args.kb_total - kb0, args.kb_per_split);
  const CUtensorMap *tmW = &args.tmW[bi];
  const CUtensorMap *tmX = &args.tmX[bi];

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(tmW);
    tma_prefetch_desc(tmX);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const uint64_t pol_w = policy_evict_first();   // weights stream through once
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      if (i >= C::kStages) mbar_wait(&empty[s], ((i / C::kStages) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], C::kStage);
      const int kc = (kb0 + i) * 64;
      tma_load_2d_hint(sA + s * C::kA, tmW, &full[s], kc, mt * 128, pol_w);
#pragma unroll
      for (int r = 0; r < BN / 16; ++r) tma_load_2d(sB + s * C::kB + r * 2048, tmX, &full[s], kc, args.x_row0 + tt * BN + r * 16);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread)
    constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      mbar_wait(&full[s], (i / C::kStages) & 1);
      tc_fence_after();
      const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * C::kA));
      const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * C::kB));
#pragma unroll
      for (int k = 0; k < 4; ++k)  // UMMA_K = 16 bf16 = 32 B -> +2 in the 16-byte address field
        umma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();

  // ---------------- epilogue: TMEM -> registers -> fp32 partials (all 4 warps)
  mbar_wait(done, 0);
  tc_fence_after();
  const int n = mt * 128 + warp * 32 + lane;  // output feature = TMEM lane
  float *out = args.out[bi] + (size_t)split * args.split_stride;
  const int m_base = tt * BN;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    if (n < args.N) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = m_base + c0 + j;
        if (m < args.M) out[(size_t)m * args.ldo + n] = v[j];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

template <int BN>
static cudaError_t launch_bn(const GemmArgs &a, int m_tiles, int token_tiles, cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(m_tiles, a.splits, a.batch * token_tiles);
  gemm_bf16_tc_kernel<BN><<<grid, 128, C::kSmem, st>>>(a);
  return cudaGetLastError();
}

int gemm_pick_bn(int M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 128) return 128;
  return 256;
}

// Choose split-K so that tiles * splits covers >= 2 waves of 148 SMs (memory-bound
// regime: every SM must be streaming weights), keeping >= 2 k-blocks per split.
void gemm_plan(GemmArgs &a, int N, int K, int M, int batch) {
  a.N = N;
  a.K = K;
  a.M = M;
  a.batch = batch;
  a.bn = gemm_pick_bn(M);
  const int m_tiles = (N + 127) / 128;
  const int token_tiles = (M + a.bn - 1) / a.bn;
  const int tiles = m_tiles * token_tiles * batch;
  a.kb_total = (K + 63) / 64;
  int splits = (2 * kNumSMs + tiles - 1) / tiles;
  splits = max(1, min(splits, a.kb_total / 2 > 0 ? a.kb_total / 2 : 1));
  a.kb_per_split = (a.kb_total + splits - 1) / splits;
  a.splits = (a.kb_total + a.kb_per_split - 1) / a.kb_per_split;
}

cudaError_t gemm_launch(const GemmArgs &a, cudaStream_t st) {
  const int m_tiles = (a.N + 127) / 128;
  const int token_tiles = (a.M + a.bn - 1) / a.bn;
  switch (a.bn) {
    case 16: return launch_bn<16>(a, m_tiles, token_tiles, st);
    case 32: return launch_bn<32>(a, m_tiles, token_tiles, st);
    case 64: return launch_bn<64>(a, m_tiles, token_tiles, st);
    case 128: return launch_bn<128>(a, m_tiles, token_tiles, st);
    default: return launch_bn<256>(a, m_tiles, token_tiles, st);
  }
}

}  // namespace sm
