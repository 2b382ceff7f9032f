// tp.cu -- tensor-parallel exchanges outside the residual path (north star a7/e):
// merging the vocabulary-parallel LM head statistics and the Medusa heads' top-K
// candidates across ranks over peer memory, and the per-call epoch advance.
// Protocol (see include/specmemo.h): a rank writes its payload into its own
// symmetric buffer (data slot = exchange parity), fences system-wide, raises its
// epoch flag in every peer's flags region, waits for the peers' flags, then reads
// the peers' payloads and merges in rank order -- all ranks compute identical
// results.  One CTA per exchange, so the waits can never depend on an unscheduled
// CTA.
#include <chrono>
#include <condition_variable>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace sm {

SM_DEV void tp_exchange(const TpArgs &tp, long long ep, int slot) {
  if (tp.phase != 0) return;  // host-ordered emulation: the launch function joins the ranks
  __threadfence_system();
  __syncthreads();
  const int q = threadIdx.x;
  if (q < tp.t && q != tp.rank) {
    st_release_sys(tp.flags[q] + (size_t)tp.rank * kTpFlagSlots + slot, ep);
    tp_wait_flag(tp.flags[tp.rank] + (size_t)q * kTpFlagSlots + slot, ep, tp.err);
  }
  __syncthreads();
}

// payload per row: amax, argmax (bits), m, s, t, cand, -, -
__global__ void __launch_bounds__(1024) tp_merge_logits_kernel(int rows, const float *amax, int32_t *argmax,
                                                               float *stats, const float *z_local, int Vl, int v0,
                                                               const int32_t *parent, int N, const int32_t *tok,
                                                               float *cand, TpArgs tp) {
  pdl_trigger();
  pdl_wait();
  const long long ep = 2 * (*tp.seq + tp.point + 1);  // even: see resid_norm_tp_kernel
  const int r = threadIdx.x;
  if (r < rows && tp.phase != 2) {  // publish (phase 2 of the emulation: already published)
    float c = __int_as_float(0x7fc00000);  // NaN: this rank does not own the candidate token
    if (tok) {
      const int n = r % N, base = r - n;
      if (n > 0) {
        const int tk = tok[r];
        if (tk >= v0 && tk < v0 + Vl) c = z_local[(size_t)(base + parent[n]) * Vl + (tk - v0)];
      }
    }
    float4 *dst = reinterpret_cast<float4 *>(tp.data[tp.rank] + (size_t)r * 8);
    __stcg(dst, make_float4(amax[r], __int_as_float(argmax[r]), stats[3 * r], stats[3 * r + 1]));
    __stcg(dst + 1, make_float4(stats[3 * r + 2], c, 0.f, 0.f));
  }
  tp_exchange(tp, ep, 0);
  if (r >= rows || tp.phase == 1) return;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  MST acc{-INFINITY, 0.f, 0.f};
  float c = __int_as_float(0x7fc00000);
  for (int q = 0; q < tp.t; ++q) {  // rank order (vocabulary order)
    const float4 *src = reinterpret_cast<const float4 *>(tp.data[q] + (size_t)r * 8);
    const float4 p0 = __ldcv(src), p1 = __ldcv(src + 1);
    argmax_merge(bv, bi, p0.x, __float_as_int(p0.y));
    acc = mst_merge(acc, MST{p0.z, p0.w, p1.x});
    if (p1.y == p1.y) c = p1.y;
  }
  argmax[r] = bi;
  stats[3 * r] = acc.m;
  stats[3 * r + 1] = acc.s;
  stats[3 * r + 2] = acc.t;
  if (cand) cand[r] = c;
}
cudaError_t tp_merge_logits_launch(int rows, const float *amax, int32_t *argmax, float *stats, const float *z_local,
                                   int Vl, int v0, const int32_t *parent, int N, const int32_t *tok, float *cand,
                                   const TpArgs &tp, cudaStream_t st) {
  if (rows > 1024) return cudaErrorInvalidValue;
  auto launch = [&](const TpArgs &a) {
    return launch_pdl(tp_merge_logits_kernel, dim3(1), dim3(1024), 0, st, rows, amax, argmax, stats, z_local, Vl, v0,
                      parent, N, tok, cand, a);
  };
  if (!tp.emu) return launch(tp);
  TpArgs a = tp;  // host-ordered emulation: publish, join every rank, merge
  a.phase = 1;
  cudaError_t e = launch(a);
  if (e == cudaSuccess) e = emu_exchange(a, 0, st);
  a.phase = 2;
  return e == cudaSuccess ? launch(a) : e;
}

// payload per entry (b, head): K values then K indices (bits)
__global__ void __launch_bounds__(256) tp_merge_topk_kernel(int entries, int K, const float *vals,
                                                            const int32_t *idx_local, int32_t *idx_out, TpArgs tp) {
  pdl_trigger();
  pdl_wait();
  const long long ep = 2 * (*tp.seq + tp.point + 1);  // even: see resid_norm_tp_kernel
  for (int e = threadIdx.x; e < entries && tp.phase != 2; e += blockDim.x) {
    float *dst = tp.data[tp.rank] + (size_t)e * 2 * K;
    for (int k = 0; k < K; ++k) {
      __stcg(dst + k, vals[(size_t)e * K + k]);
      __stcg(dst + K + k, __int_as_float(idx_local[(size_t)e * K + k]));
    }
  }
  tp_exchange(tp, ep, 0);
  for (int e = threadIdx.x; e < entries && tp.phase != 1; e += blockDim.x) {
    uint32_t taken[kMaxTP] = {0};  // K <= 32 candidates per rank
    for (int k = 0; k < K; ++k) {
      float bv = -INFINITY;
      int bi = 0x7fffffff, bq = -1, bk = -1;
      for (int q = 0; q < tp.t; ++q) {
        const float *src = tp.data[q] + (size_t)e * 2 * K;
        for (int j = 0; j < K; ++j) {
          if ((taken[q] >> j) & 1u) continue;
          const float v = __ldcv(src + j);
          const int ix = __float_as_int(__ldcv(src + K + j));
          if (v != v) continue;  // NaN never wins (as in the single-GPU top-k)
          if (bq < 0 || v > bv || (v == bv && ix < bi)) {
            bv = v;
            bi = ix;
            bq = q;
            bk = j;
          }
        }
      }
      if (bq >= 0) taken[bq] |= 1u << bk;
      idx_out[(size_t)e * K + k] = bi;
    }
  }
}
cudaError_t tp_merge_topk_launch(int entries, int K, const float *vals, const int32_t *idx_local, int32_t *idx_out,
                                 int nmed, int nb, const TpArgs &tp, cudaStream_t st) {
  (void)nmed;
  (void)nb;
  if (K > 32) return cudaErrorInvalidValue;
  auto launch = [&](const TpArgs &a) {
    return launch_pdl(tp_merge_topk_kernel, dim3(1), dim3(256), 0, st, entries, K, vals, idx_local, idx_out, a);
  };
  if (!tp.emu) return launch(tp);
  TpArgs a = tp;  // host-ordered emulation: publish, join every rank, merge
  a.phase = 1;
  cudaError_t e = launch(a);
  if (e == cudaSuccess) e = emu_exchange(a, 0, st);
  a.phase = 2;
  return e == cudaSuccess ? launch(a) : e;
}

__global__ void tp_advance_kernel(long long *seq, int n) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) *seq += n;
}
cudaError_t tp_advance_launch(long long *seq, int n, cudaStream_t st) {
  return launch_pdl(tp_advance_kernel, dim3(1), dim3(32), 0, st, seq, n);
}

// ------------------------------------------------------------------ layer-split pipeline (f4)
// One launch per hand-off on every participating rank, same grid everywhere: CTA c moves float4
// items [c * per, (c + 1) * per).  Flag slot c of the source row in each receiver's flags region.
constexpr int kPpThreads = 256;
__global__ void __launch_bounds__(kPpThreads) pp_xfer_kernel(float4 *x, int n4, int per, int src, unsigned dst_mask,
                                                             TpArgs tp) {
  pdl_trigger();
  pdl_wait();
  const long long ep = 2 * (*tp.seq + tp.point + 1);
  const int i0 = blockIdx.x * per, i1 = min(n4, i0 + per);
  if (tp.rank == src) {
    float4 *slot = reinterpret_cast<float4 *>(tp.data[src]);
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) __stcg(slot + i, x[i]);
    __threadfence_system();
    __syncthreads();
    const int q = threadIdx.x;
    if (q < tp.t && ((dst_mask >> q) & 1u)) st_release_sys(tp.flags[q] + (size_t)src * kTpFlagSlots + blockIdx.x, ep);
  } else if ((dst_mask >> tp.rank) & 1u) {
    if (threadIdx.x == 0 && tp.phase == 0)  // emulation: the host made this launch wait for the sender's
      tp_wait_flag(tp.flags[tp.rank] + (size_t)src * kTpFlagSlots + blockIdx.x, ep, tp.err);
    __syncthreads();
    const float4 *slot = reinterpret_cast<const float4 *>(tp.data[src]);
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) x[i] = __ldcv(slot + i);
  }
}
cudaError_t pp_xfer_launch(float *x, int n4, int src, unsigned dst_mask, const TpArgs &tp, cudaStream_t st) {
  const int per = 4 * kPpThreads;  // 16 KB per CTA
  const int grid = (n4 + per - 1) / per;
  if (grid > kTpFlagSlots || grid < 1) return cudaErrorInvalidValue;
  TpArgs a = tp;
  if (tp.emu) {  // host-ordered emulation: a receiver's launch waits for the sender's publish event
    a.phase = 1;
    if (tp.rank != src) {
      if (!((dst_mask >> tp.rank) & 1u)) return cudaSuccess;
      cudaError_t e = emu_wait(a, src, 0, st);
      if (e != cudaSuccess) return e;
    }
  }
  cudaError_t e = launch_pdl(pp_xfer_kernel, dim3(grid), dim3(kPpThreads), 0, st, reinterpret_cast<float4 *>(x), n4,
                             per, src, dst_mask, a);
  if (e == cudaSuccess && tp.emu && tp.rank == src) e = emu_publish(a, 0, st);
  return e;
}

// ------------------------------------------------------------------ host-ordered emulation
// Several ranks on ONE GPU (tests): no kernel may spin on a flag another rank's launch raises
// (nothing guarantees the two run at the same time), so each exchange runs as segment launches
// and the ranks' host threads join them with CUDA events: rank r records "segment sub of
// exchange gen published" on its stream; a rank that needs it makes its stream wait for that
// record before its next segment.  Each rank's records go round a 4-slot ring tagged by (gen, sub):
// a rank publishes at most two tags a peer has not consumed yet (to publish a third it must first
// have seen that peer's next publication, which the peer makes only after consuming the first).
struct EmuGroup {
  int t = 0;
  std::mutex mu;
  std::condition_variable cv;
  cudaEvent_t ev[kMaxTP][4] = {};
  long long tag[kMaxTP][4];
  unsigned next[kMaxTP] = {};
};
EmuGroup *emu_group_create(int t) {
  if (t < 2 || t > kMaxTP) return nullptr;
  EmuGroup *g = new EmuGroup();
  g->t = t;
  for (int r = 0; r < kMaxTP; ++r)
    for (int k = 0; k < 4; ++k) {
      g->tag[r][k] = -1;
      if (r < t && cudaEventCreateWithFlags(&g->ev[r][k], cudaEventDisableTiming) != cudaSuccess) {
        emu_group_destroy(g);
        return nullptr;
      }
    }
  return g;
}
void emu_group_destroy(EmuGroup *g) {
  if (!g) return;
  for (int r = 0; r < kMaxTP; ++r)
    for (int k = 0; k < 4; ++k)
      if (g->ev[r][k]) cudaEventDestroy(g->ev[r][k]);
  delete g;
}
static long long emu_tag(const TpArgs &tp, int sub) { return tp.gen * 4 + sub; }
cudaError_t emu_publish(const TpArgs &tp, int sub, cudaStream_t st) {
  EmuGroup *g = static_cast<EmuGroup *>(tp.emu);
  std::lock_guard<std::mutex> lk(g->mu);
  const int k = (int)(g->next[tp.rank]++ & 3u);
  cudaError_t e = cudaEventRecord(g->ev[tp.rank][k], st);
  g->tag[tp.rank][k] = emu_tag(tp, sub);
  g->cv.notify_all();
  return e;
}
cudaError_t emu_wait(const TpArgs &tp, int q, int sub, cudaStream_t st) {
  EmuGroup *g = static_cast<EmuGroup *>(tp.emu);
  const long long tg = emu_tag(tp, sub);
  int k = -1;
  std::unique_lock<std::mutex> lk(g->mu);
  auto found = [&] {
    for (int j = 0; j < 4; ++j)
      if (g->tag[q][j] == tg) k = j;
    return k >= 0;
  };
  if (!g->cv.wait_for(lk, std::chrono::seconds(60), found)) return cudaErrorTimeout;
  return cudaStreamWaitEvent(st, g->ev[q][k], 0);
}
cudaError_t emu_exchange(const TpArgs &tp, int sub, cudaStream_t st) {
  cudaError_t e = emu_publish(tp, sub, st);
  for (int q = 0; q < tp.t && e == cudaSuccess; ++q)
    if (q != tp.rank) e = emu_wait(tp, q, sub, st);
  return e;
}

void tp_preload() {  // force-load (see gemm_preload)
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, tp_merge_logits_kernel);
  cudaFuncGetAttributes(&fa, tp_merge_topk_kernel);
  cudaFuncGetAttributes(&fa, tp_advance_kernel);
  cudaFuncGetAttributes(&fa, pp_xfer_kernel);
}

}  // namespace sm
