// runtime.cu -- host runtime behind the C ABI (include/specmemo.h): tree, model
// and bounded-KV objects, step orchestration (propose -> verify -> accept ->
// compact -> next heads) entirely stream-ordered, captured once into a CUDA
// graph and replayed; lengths live on the device so no step syncs the host.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a profiler attaches

#include "../../include/specmemo.h"
#include "kernels.h"

namespace {
struct NvtxRange {  // host-side range around each public entry point (nsys / ncu --nvtx timelines)
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace sm;

static thread_local std::string g_err;
static sm_status fail(sm_status s, const std::string &msg) {
  g_err = msg;
  return s;
}
#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return fail(SM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define CKS(call)                       \
  do {                                  \
    sm_status s_ = (call);              \
    if (s_ != SM_OK) return s_;         \
  } while (0)

// ---------------------------------------------------------------- tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}
// 2D bf16 map over [rows][cols] (row-major), box [box_rows][box_cols].
static sm_status make_tmap(CUtensorMap *m, const void *base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                           uint32_t box_cols, bool sw128) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstride[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), gdim, gstride, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SM_ERR_INVALID_ARG, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rows=" +
                                        std::to_string(rows) + " cols=" + std::to_string(cols));
  return SM_OK;
}
static sm_status weight_map(CUtensorMap *m, const void *w, int N, int K) {
  if (K % 8) return fail(SM_ERR_INVALID_ARG, "GEMM K must be a multiple of 8");
  return make_tmap(m, w, (uint64_t)N, (uint64_t)K, 128, 64, true);
}
// activation maps of GEMM batch entry i: 16-row and 64-row boxes (BN < 64 / BN >= 64)
static sm_status act_map(GemmArgs &a, int i, const void *x, int rows, int K) {
  a.x_base[i] = x;
  a.x_rows[i] = rows;
  a.x_box = 64;
  CKS(make_tmap(&a.tmX[i], x, (uint64_t)rows, (uint64_t)K, 16, 64, true));
  return make_tmap(&a.tmX64[i], x, (uint64_t)rows, (uint64_t)K, 64, 64, true);
}
// BN >= 64: the kernel loads a stage's BN activation rows with one TMA box of BN rows
// (request count, not bytes, limits the L2 -> SM fill of small boxes).
static sm_status act_box(GemmArgs &a) {
  const int bn = a.plan.pair == 2 ? a.plan.bn / 2 : a.plan.bn;  // 2-SM: each CTA loads half the token rows
  if (a.plan.bn < 64 || bn == a.x_box) return SM_OK;
  for (int i = 0; i < a.batch; ++i)
    CKS(make_tmap(&a.tmX64[i], a.x_base[i], (uint64_t)a.x_rows[i], (uint64_t)a.K, (uint32_t)bn, 64, true));
  a.x_box = bn;
  return SM_OK;
}
static sm_status kv_map(CUtensorMap *m, const void *base, uint64_t rows, int hd) {
  const bool sw = hd >= 64;
  return make_tmap(m, base, rows, (uint64_t)hd, 64, sw ? 64 : (uint32_t)hd, sw);
}

template <typename T>
static sm_status dalloc(T **p, size_t n, const char *what) {
  *p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), n * sizeof(T));
  if (e != cudaSuccess) return fail(SM_ERR_DEVICE_OOM, std::string("Buffer: cudaMalloc ") + what);
  return SM_OK;
}

// ---------------------------------------------------------------- tree
struct sm_tree {
  int N = 1, S = 1, l = 0, topk = 1;
  std::vector<std::vector<int>> paths;  // canonical order, root = {}
  std::vector<int32_t> parent, depth, rank, dfs_pos, first_leaf, leaf_paths;
  std::vector<uint64_t> anc;  // [N][kAncWords]
  int32_t *d_parent = nullptr, *d_depth = nullptr, *d_rank = nullptr, *d_dfs = nullptr, *d_first_leaf = nullptr;
  uint64_t *d_anc = nullptr;
  bool on_device = false;
  TreeDev dev() const { return TreeDev{N, S, l, d_parent, d_depth, d_rank, d_dfs, d_first_leaf, d_anc}; }
};

static sm_status tree_finish(sm_tree *t) {
  const int N = (int)t->paths.size();
  t->N = N;
  std::map<std::vector<int>, int> id;
  for (int i = 0; i < N; ++i) id[t->paths[i]] = i;
  t->parent.assign(N, -1);
  t->depth.assign(N, 0);
  t->rank.assign(N, -1);
  t->anc.assign((size_t)N * kAncWords, 0ull);
  std::vector<int> nchild(N, 0);
  for (int i = 0; i < N; ++i) {
    const auto &p = t->paths[i];
    t->depth[i] = (int)p.size();
    if (!p.empty()) {
      t->rank[i] = p.back();
      t->parent[i] = id[std::vector<int>(p.begin(), p.end() - 1)];
      nchild[t->parent[i]]++;
    }
    for (int x = i; x >= 0; x = (x == 0 ? -1 : t->parent[x])) t->anc[(size_t)i * kAncWords + x / 64] |= 1ull << (x % 64);
  }
  t->l = N ? *std::max_element(t->depth.begin(), t->depth.end()) : 0;
  // DFS order = lexicographic order of rank paths
  std::vector<int> order(N);
  for (int i = 0; i < N; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return t->paths[a] < t->paths[b]; });
  t->dfs_pos.assign(N, 0);
  for (int i = 0; i < N; ++i) t->dfs_pos[order[i]] = i;
  std::vector<int> leaves;
  for (int i : order)
    if (nchild[i] == 0) leaves.push_back(i);
  t->S = (int)leaves.size();
  t->first_leaf.assign(N, 0);
  for (int n = 0; n < N; ++n) {
    const auto &pn = t->paths[n];
    for (int li = 0; li < t->S; ++li) {
      const auto &pl = t->paths[leaves[li]];
      if (pl.size() >= pn.size() && std::equal(pn.begin(), pn.end(), pl.begin())) {
        t->first_leaf[n] = li;
        break;
      }
    }
  }
  t->leaf_paths.assign((size_t)t->S * (t->l + 1), -1);
  for (int li = 0; li < t->S; ++li) {
    int x = leaves[li];
    for (int j = t->depth[x]; j >= 0; --j, x = t->parent[x]) t->leaf_paths[(size_t)li * (t->l + 1) + j] = x;
  }
  return SM_OK;
}

static sm_status tree_upload(sm_tree *t) {
  if (t->on_device) return SM_OK;
  const int N = t->N;
  CKS(dalloc(&t->d_parent, N, "tree"));
  CKS(dalloc(&t->d_depth, N, "tree"));
  CKS(dalloc(&t->d_rank, N, "tree"));
  CKS(dalloc(&t->d_dfs, N, "tree"));
  CKS(dalloc(&t->d_first_leaf, N, "tree"));
  CKS(dalloc(&t->d_anc, (size_t)N * kAncWords, "tree"));
  CK(cudaMemcpy(t->d_parent, t->parent.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t->d_depth, t->depth.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t->d_rank, t->rank.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t->d_dfs, t->dfs_pos.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t->d_first_leaf, t->first_leaf.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t->d_anc, t->anc.data(), (size_t)N * kAncWords * 8, cudaMemcpyHostToDevice));
  t->on_device = true;
  return SM_OK;
}

extern "C" sm_status sm_tree_create(const int32_t *ranks_flat, const int32_t *path_offsets, int n_paths, int topk,
                                    sm_tree **out) {
  if (!out || n_paths < 0 || topk < 1 || (n_paths > 0 && (!ranks_flat || !path_offsets)))
    return fail(SM_ERR_INVALID_ARG, "sm_tree_create: bad arguments");
  if (n_paths + 1 > kMaxTreeNodes) return fail(SM_ERR_INVALID_ARG, "sm_tree_create: more than 256 nodes");
  std::vector<std::vector<int>> ps;
  for (int i = 0; i < n_paths; ++i) {
    const int a = path_offsets[i], b = path_offsets[i + 1];
    if (b <= a) return fail(SM_ERR_INFEASIBLE_TREE, "empty path");
    std::vector<int> p(ranks_flat + a, ranks_flat + b);
    for (int r : p)
      if (r < 0 || r >= topk) return fail(SM_ERR_INFEASIBLE_TREE, "rank out of range");
    ps.push_back(p);
  }
  std::sort(ps.begin(), ps.end(), [](const std::vector<int> &a, const std::vector<int> &b) {
    return a.size() != b.size() ? a.size() < b.size() : a < b;
  });
  for (size_t i = 1; i < ps.size(); ++i)
    if (ps[i] == ps[i - 1]) return fail(SM_ERR_INFEASIBLE_TREE, "duplicate path");
  std::map<std::vector<int>, int> have;
  for (auto &p : ps) have[p] = 1;
  for (auto &p : ps)
    if (p.size() > 1 && !have.count(std::vector<int>(p.begin(), p.end() - 1)))
      return fail(SM_ERR_INFEASIBLE_TREE, "orphan path");
  sm_tree *t = new sm_tree();
  t->topk = topk;
  t->paths.push_back({});
  for (auto &p : ps) t->paths.push_back(p);
  tree_finish(t);
  *out = t;
  return SM_OK;
}

extern "C" sm_status sm_tree_create_chain(int n, sm_tree **out) {
  if (!out || n < 1 || n > kMaxTreeNodes) return fail(SM_ERR_INVALID_ARG, "sm_tree_create_chain: 1 <= n <= 256");
  sm_tree *t = new sm_tree();
  t->topk = 1;
  for (int i = 0; i < n; ++i) t->paths.push_back(std::vector<int>(i, 0));
  tree_finish(t);
  *out = t;
  return SM_OK;
}

// ---------------------------------------------------------------- tree construction (f1)
static sm_status tree_from_paths(std::vector<std::vector<int>> ps, int topk, sm_tree **out) {
  if ((int)ps.size() + 1 > kMaxTreeNodes) return fail(SM_ERR_INVALID_ARG, "tree construction: more than 256 nodes");
  std::sort(ps.begin(), ps.end(), [](const std::vector<int> &a, const std::vector<int> &b) {
    return a.size() != b.size() ? a.size() < b.size() : a < b;
  });
  sm_tree *t = new sm_tree();
  t->topk = topk;
  t->paths.push_back({});
  for (auto &p : ps) t->paths.push_back(p);
  tree_finish(t);
  *out = t;
  return SM_OK;
}

extern "C" sm_status sm_tree_create_full(int k, int l, sm_tree **out) {
  if (!out || k < 1 || l < 0) return fail(SM_ERR_INVALID_ARG, "sm_tree_create_full: k >= 1, l >= 0");
  double n = 0;
  for (int i = 1; i <= l; ++i) n += std::pow((double)k, i);
  if (n + 1 > kMaxTreeNodes) return fail(SM_ERR_INVALID_ARG, "sm_tree_create_full: more than 256 nodes");
  std::vector<std::vector<int>> ps, level{{}};
  for (int i = 0; i < l; ++i) {
    std::vector<std::vector<int>> next;
    for (auto &p : level)
      for (int r = 0; r < k; ++r) {
        auto q = p;
        q.push_back(r);
        next.push_back(q);
      }
    level = next;
    ps.insert(ps.end(), level.begin(), level.end());
  }
  return tree_from_paths(ps, k, out);
}

extern "C" sm_status sm_tree_prune(const sm_tree *t, int target_nodes, sm_tree **out) {
  if (!t || !out) return fail(SM_ERR_INVALID_ARG, "sm_tree_prune: null");
  if (target_nodes < 1 || target_nodes > t->N) return fail(SM_ERR_INFEASIBLE_TREE, "sm_tree_prune: target outside [1, N]");
  // R4 (Medusa's right-to-left pruning): drop the leaf with the lexicographically
  // largest rank path (the rightmost leaf in DFS order) until target_nodes remain.
  std::vector<std::vector<int>> cur(t->paths.begin() + 1, t->paths.end());
  while ((int)cur.size() + 1 > target_nodes) {
    int best = -1;
    for (int i = 0; i < (int)cur.size(); ++i) {
      bool leaf = true;
      for (const auto &q : cur)
        if (q.size() == cur[i].size() + 1 && std::equal(cur[i].begin(), cur[i].end(), q.begin())) {
          leaf = false;
          break;
        }
      if (leaf && (best < 0 || cur[i] > cur[best])) best = i;
    }
    cur.erase(cur.begin() + best);
  }
  return tree_from_paths(cur, t->topk, out);
}

extern "C" sm_status sm_tree_create_pruned_full(int k, int l, float r_min, float r_max, float mid, float steep,
                                                sm_tree **out) {
  if (!out || k < 1 || l < 1) return fail(SM_ERR_INVALID_ARG, "sm_tree_create_pruned_full: k >= 1, l >= 1");
  // scaled logistic rate r(i) = r_min + (r_max - r_min) / (1 + exp(-steep (i - mid))) (fig:prunefunc);
  // level 1 keeps all k nodes; level i keeps the first ceil((1 - r(i)) k^i) of its
  // full-tree nodes, left to right, whose parent was kept.
  std::vector<std::vector<int>> ps, prev;
  for (int r = 0; r < k; ++r) prev.push_back({r});
  ps = prev;
  for (int i = 2; i <= l && !prev.empty(); ++i) {
    const double rate = (double)r_min + ((double)r_max - (double)r_min) / (1.0 + std::exp(-(double)steep * (i - (double)mid)));
    const double want = std::ceil((1.0 - rate) * std::pow((double)k, i) - 1e-9);
    std::vector<std::vector<int>> level;
    for (auto &p : prev)
      for (int r = 0; r < k && (double)level.size() < want; ++r) {
        auto q = p;
        q.push_back(r);
        level.push_back(q);
      }
    if (ps.size() + level.size() + 1 > (size_t)kMaxTreeNodes)
      return fail(SM_ERR_INVALID_ARG, "sm_tree_create_pruned_full: more than 256 nodes");
    ps.insert(ps.end(), level.begin(), level.end());
    prev = level;
  }
  return tree_from_paths(ps, k, out);
}

extern "C" sm_status sm_tree_create_custom(int n_nodes, int n_leaves, int k, int l, sm_tree **out) {
  // Exact (N, S) features, reading Q30: level 1 = min(k, N-1, S) nodes; then
  // "deepening" additions (child of the first DFS leaf above depth l; leaves unchanged),
  // taking a "widening" step (next-rank child of the first BFS node with 1..k-1 children;
  // one more leaf) only when every leaf is at depth l; then the remaining widenings.
  if (!out || k < 1 || l < 0) return fail(SM_ERR_INVALID_ARG, "sm_tree_create_custom: bad arguments");
  const int N = n_nodes, S = n_leaves;
  if (N < 1 || S < 1 || (N == 1 && S != 1) || (N > 1 && S > N - 1))
    return fail(SM_ERR_INFEASIBLE_TREE, "sm_tree_create_custom: need 1 <= S <= N - 1 (or N = S = 1)");
  if (N > kMaxTreeNodes) return fail(SM_ERR_INVALID_ARG, "sm_tree_create_custom: more than 256 nodes");
  if (N == 1) return tree_from_paths({}, k, out);
  if (l < 1) return fail(SM_ERR_INFEASIBLE_TREE, "sm_tree_create_custom: N > 1 needs l >= 1");
  const int c1 = std::min({k, N - 1, S});
  std::vector<std::vector<int>> ps;
  std::map<std::vector<int>, int> nchild;
  for (int r = 0; r < c1; ++r) ps.push_back({r});
  nchild[{}] = c1;
  int widen = S - c1, deepen = (N - 1 - c1) - widen;
  if (widen < 0 || deepen < 0) return fail(SM_ERR_INFEASIBLE_TREE, "sm_tree_create_custom: too many leaves");
  auto widen_one = [&]() -> bool {
    std::vector<std::vector<int>> cand;
    if (nchild[{}] > 0 && nchild[{}] < k) cand.push_back({});
    for (auto &p : ps) {
      const int c = nchild.count(p) ? nchild[p] : 0;
      if (c > 0 && c < k) cand.push_back(p);
    }
    if (cand.empty()) return false;
    auto it = std::min_element(cand.begin(), cand.end(), [](const std::vector<int> &a, const std::vector<int> &b) {
      return a.size() != b.size() ? a.size() < b.size() : a < b;
    });
    auto q = *it;
    const int r = nchild[q];
    nchild[q] = r + 1;
    q.push_back(r);
    ps.push_back(q);
    return true;
  };
  while (deepen > 0) {
    const std::vector<int> *pick = nullptr;
    for (auto &p : ps)  // first leaf in DFS (lexicographic) order above depth l
      if ((int)p.size() < l && !(nchild.count(p) && nchild[p] > 0) && (!pick || p < *pick)) pick = &p;
    if (pick) {
      auto q = *pick;
      nchild[q] = 1;
      q.push_back(0);
      ps.push_back(q);
      --deepen;
    } else if (widen > 0) {
      if (!widen_one()) return fail(SM_ERR_INFEASIBLE_TREE, "sm_tree_create_custom: no node to widen");
      --widen;
    } else {
      return fail(SM_ERR_INFEASIBLE_TREE, "sm_tree_create_custom: no leaf above depth l to deepen");
    }
  }
  for (; widen > 0; --widen)
    if (!widen_one()) return fail(SM_ERR_INFEASIBLE_TREE, "sm_tree_create_custom: no node to widen");
  return tree_from_paths(ps, k, out);
}

// ---------------------------------------------------------------- tree-size selection (f1)
// E[tau] under SPEC's independent acceptance model: non-root node at level j, sibling
// rank r accepted with probability alpha_j rho^r; tau = depth of the longest all-accepted root path
// + 1.  E[tau] = 1 + sum_D f_D(root), f_D(n) = 1 if depth(n) >= D, else
// 1 - prod_children (1 - a(c) f_D(c)); children are visited in canonical order (same products, same
// order as oracle/tree.py expected_tau).
static double tree_expected_tau(const sm_tree *t, const float *alpha, float rho) {
  std::vector<double> a(t->N, 0.0), f(t->N, 0.0);
  std::vector<std::vector<int>> kids(t->N);
  for (int n = 1; n < t->N; ++n) {
    a[n] = (double)alpha[t->depth[n] - 1] * std::pow((double)rho, (double)t->rank[n]);
    kids[t->parent[n]].push_back(n);
  }
  double tau = 1.0;
  for (int D = 1; D <= t->l; ++D) {
    for (int n = t->N - 1; n >= 0; --n) {
      if (t->depth[n] >= D) {
        f[n] = 1.0;
      } else {
        double miss = 1.0;
        for (int c : kids[n]) miss *= 1.0 - a[c] * f[c];
        f[n] = 1.0 - miss;
      }
    }
    tau += f[0];
  }
  return tau;
}

extern "C" sm_status sm_tree_expected_tau(const sm_tree *t, const float *h_alpha, int n_alpha, float rho,
                                          double *tau) {
  if (!t || !h_alpha || !tau || n_alpha < t->l || !(rho > 0.f && rho <= 1.f))
    return fail(SM_ERR_INVALID_ARG, "sm_tree_expected_tau: need alpha[>= depth] in [0,1], 0 < rho <= 1");
  for (int j = 0; j < t->l; ++j)
    if (!(h_alpha[j] >= 0.f && h_alpha[j] <= 1.f)) return fail(SM_ERR_INVALID_ARG, "alpha outside [0, 1]");
  *tau = tree_expected_tau(t, h_alpha, rho);
  return SM_OK;
}

extern "C" sm_status sm_select_tree(const sm_tree *const *cands, int n, const double *h_step_ms, const float *h_alpha,
                                    int n_alpha, float rho, int batch, int *best, double *h_tokens_per_s) {
  if (!cands || n < 1 || !h_step_ms || !h_alpha || !best || batch < 1)
    return fail(SM_ERR_INVALID_ARG, "sm_select_tree: bad arguments");
  int b = -1;
  double bv = 0.0;
  for (int i = 0; i < n; ++i) {
    double tau;
    CKS(sm_tree_expected_tau(cands[i], h_alpha, n_alpha, rho, &tau));
    if (!(h_step_ms[i] > 0.0)) return fail(SM_ERR_INVALID_ARG, "sm_select_tree: step_ms must be > 0");
    const double v = batch * tau / h_step_ms[i] * 1e3;  // expected tokens/s
    if (h_tokens_per_s) h_tokens_per_s[i] = v;
    if (b < 0 || v > bv || (v == bv && cands[i]->N < cands[b]->N)) {
      b = i;
      bv = v;
    }
  }
  *best = b;
  return SM_OK;
}

extern "C" sm_status sm_alg2_select(int n, const double *h_acc_len, const double *h_speedup, int *best) {
  (void)h_acc_len;  // recorded by Algorithm 2, not part of its choice
  if (n < 1 || !h_speedup || !best) return fail(SM_ERR_INVALID_ARG, "sm_alg2_select: bad arguments");
  int b = 0;
  for (int i = 0; i < n; ++i) {
    if (!std::isfinite(h_speedup[i])) return fail(SM_ERR_INVALID_ARG, "sm_alg2_select: non-finite speedup");
    if (h_speedup[i] > h_speedup[b]) b = i;  // strict: ties keep the first configuration
  }
  *best = b;
  return SM_OK;
}
extern "C" sm_status sm_tree_query(const sm_tree *t, int *N, int *S, int *depth, int32_t *parent, int32_t *node_depth,
                                   int32_t *rank, uint64_t *anc_bits, int32_t *leaf_paths) {
  if (!t) return fail(SM_ERR_INVALID_ARG, "sm_tree_query: null tree");
  if (N) *N = t->N;
  if (S) *S = t->S;
  if (depth) *depth = t->l;
  if (parent) std::memcpy(parent, t->parent.data(), t->N * 4);
  if (node_depth) std::memcpy(node_depth, t->depth.data(), t->N * 4);
  if (rank) std::memcpy(rank, t->rank.data(), t->N * 4);
  if (anc_bits) std::memcpy(anc_bits, t->anc.data(), (size_t)t->N * kAncWords * 8);
  if (leaf_paths) std::memcpy(leaf_paths, t->leaf_paths.data(), t->leaf_paths.size() * 4);
  return SM_OK;
}

extern "C" void sm_tree_destroy(sm_tree *t) {
  if (!t) return;
  if (!t->on_device) {
    delete t;
    return;
  }
  cudaFree(t->d_parent);
  cudaFree(t->d_depth);
  cudaFree(t->d_rank);
  cudaFree(t->d_dfs);
  cudaFree(t->d_first_leaf);
  cudaFree(t->d_anc);
  delete t;
}

// ---------------------------------------------------------------- model
struct sm_model {
  sm_model_cfg cfg;
  int L, d, H, Hkv, hd, F, V, nmed, G, R, B, qkv_n;
  int P = 1;         // activation planes: 1 = bf16, 3 = fp32 parity mode (hi/mid/lo bf16 rows)
  bool f32 = false;  // fp32 parity mode (sm_model_cfg.dtype)
  int hdu = 0;       // K/V row length in bf16 units (hd, or 2 hd for fp32 K/V)
  const bf16 *embed, *final_norm, *lm_head;
  std::vector<const bf16 *> attn_norm, wqkv, wo, mlp_norm, wgu, wdown, mR, mb, mU;
  // workspace
  float *x = nullptr, *part = nullptr, *z = nullptr, *stats = nullptr;
  float *rs = nullptr;  // [R] deferred RMSNorm scale of the current GEMM input rows (R2)
  RsArgs rsa{};         // how the next consumer obtains it (see resid_norm)
  // fused tile epilogues (GemmArgs.epi): bf16, tp = 1, hd = 128, d % 128 == 0
  bool fused = false;
  int fuse_mask = 0;
  float *ss = nullptr;   // [R][d/64] sum-of-squares partials of kEpiResid
  int *tile_cnt = nullptr, *done_cnt = nullptr;
  int32_t *iota = nullptr;  // [R] 0, 1, 2, ...: node depths of a causal prefill chunk (f3)
  bf16 *h = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr, *hf = nullptr, *head_in = nullptr,
       *r_buf = nullptr;
  int32_t *argmax = nullptr;
  float2 *rope = nullptr;
  float *ws = nullptr;      // stream-K fp32 partial slots (shared by consecutive GEMMs)
  size_t ws_floats = 0;
  // GEMM prototypes (tensor maps prebuilt)
  std::vector<GemmArgs> g_qkv, g_o, g_gu, g_down;
  GemmArgs g_lm, g_R, g_U;
  sm_tree *chain = nullptr;
  cudaStream_t cap_stream = nullptr;
  // tensor parallelism (a7): local dims above are this rank's shard
  int tp = 1, tp_rank = 0, v0 = 0;
  int pp = 1, pp_rank = 0;       // layer-split pipeline (f4): this rank's layers are [pp_rank L, ..) of pp L
  void *sym[kMaxTP] = {};        // every rank's symmetric buffer, mapped on this device
  size_t sym_slot_floats = 0;
  long long *tp_seq = nullptr;   // device epoch base
  int *tp_err = nullptr;         // device: a wait timed out
  int tp_point = 0;              // host: exchange index within the current top-level call
  EmuGroup *emu = nullptr;       // host-ordered emulation group (several ranks on one GPU), borrowed
  long long emu_call = 0;        // host: top-level calls with exchanges so far (same on every rank)
  float *amax = nullptr, *cand = nullptr, *tk_val = nullptr;
  int32_t *tk_idx = nullptr;
  float *lean_part = nullptr;  // stream-K K1 partial slots (bf16 path, head_dim 128)
  int *lean_sync = nullptr;    // its grid-barrier counters (zero between launches)
};

// Most K1 units (sequence x kv head x 128-row block) one forward can have: nseq <= B sequences of
// Nq nodes with nseq Nq <= R rows, so nseq ceil(Nq G / 128) <= B + R G / 128.
static int lean_units_max(int Hkv, int G, int R, int B) { return Hkv * (B + (R * G + 127) / 128); }

static size_t tp_slot_floats(const sm_model_cfg &c) {
  return std::max({(size_t)c.max_rows * c.d_model, (size_t)c.max_rows * 8,
                   (size_t)c.max_batch * std::max(1, c.n_medusa) * 64});
}
static constexpr size_t kTpFlagBytes = (size_t)kMaxTP * kTpFlagSlots * sizeof(long long);
// Exchange descriptor for the next exchange point of the current call.
static TpArgs tp_next(sm_model *m) {
  TpArgs a;
  std::memset(&a, 0, sizeof(a));
  a.rank = m->tp_rank;
  a.t = m->tp;
  const int pt = m->tp_point++;
  for (int q = 0; q < m->tp; ++q) {
    char *b = static_cast<char *>(m->sym[q]);
    a.flags[q] = reinterpret_cast<long long *>(b);
    a.data[q] = reinterpret_cast<float *>(b + kTpFlagBytes + (size_t)(pt & 1) * m->sym_slot_floats * sizeof(float));
  }
  a.seq = m->tp_seq;
  a.point = pt;
  a.err = m->tp_err;
  a.emu = m->emu;
  a.gen = (m->emu_call << 16) + pt;
  return a;
}
static void tp_begin(sm_model *m) { m->tp_point = 0; }
// Exchange descriptor of pipeline hand-off `point` (absolute index within the current call).
static TpArgs pp_args(sm_model *m, int point) {
  TpArgs a;
  std::memset(&a, 0, sizeof(a));
  a.rank = m->pp_rank;
  a.t = m->pp;
  for (int q = 0; q < m->pp; ++q) {
    char *b = static_cast<char *>(m->sym[q]);
    a.flags[q] = reinterpret_cast<long long *>(b);
    a.data[q] = reinterpret_cast<float *>(b + kTpFlagBytes + (size_t)(point & 1) * m->sym_slot_floats * sizeof(float));
  }
  a.seq = m->tp_seq;
  a.point = point;
  a.err = m->tp_err;
  a.emu = m->emu;
  a.gen = (m->emu_call << 16) + point;
  return a;
}
// Advance the epoch base past this call's exchanges (kept even, so the data slot
// parity of an exchange is its index parity in every call).
static sm_status tp_end(sm_model *m, cudaStream_t st, int &nl) {
  if ((m->tp > 1 || m->pp > 1) && m->tp_point > 0) {
    CK(tp_advance_launch(m->tp_seq, (m->tp_point + 1) & ~1, st));
    ++nl;
    ++m->emu_call;
  }
  m->tp_point = 0;
  return SM_OK;
}

static GemmArgs gemm_proto(int N, int K, int batch) {
  GemmArgs a;
  std::memset(&a, 0, sizeof(a));
  a.N = N;
  a.K = K;
  a.batch = batch;
  return a;
}

// ---------------------------------------------------------------- in-graph kernel timing
struct ProfEvent {
  int kind;  // 0 = K2 GEMM, 1 = K1 tree attention (+ combine), 3 = whole step
  cudaEvent_t a, b;
  double bytes;
};
static thread_local std::vector<ProfEvent> *g_prof = nullptr;
static void prof_begin(cudaStream_t st, cudaEvent_t *ev) {
  if (!g_prof) return;
  cudaEventCreate(ev);
  cudaEventRecordWithFlags(*ev, st, cudaEventRecordExternal);
}
static void prof_end(cudaStream_t st, cudaEvent_t a, int kind, double bytes) {
  if (!g_prof) return;
  cudaEvent_t b;
  cudaEventCreate(&b);
  cudaEventRecordWithFlags(b, st, cudaEventRecordExternal);
  g_prof->push_back(ProfEvent{kind, a, b, bytes});
}

static int g_ablate_gemm = 0;  // set while enqueueing ablated per-layer GEMMs
static int g_epi_test = 0;     // experiments: sm_gemm_bf16(out = NULL) runs the fused SiLU epilogue
static int g_fused = 0;  // sm_set_option("fused_epilogue"): K2 tile epilogues instead of consumer kernels
                         // (bit 1 QKV/RoPE, bit 2 SiLU, bit 4 residual + deferred norm; 0 = consumers)
static constexpr int kMaxFusedTiles = 1 << 14;
// Launch one stream-K GEMM over rows [x_row0, x_row0 + M) of the prototype's
// activation map; its fp32 partials land in ws and are described by *pv.
// planes = 3 (fp32 parity mode): logical row m is GEMM rows 3m..3m+2.
static sm_status run_gemm(GemmArgs a, int M, int x_row0, float *ws, size_t ws_floats, cudaStream_t st, int &nl,
                          PartialView *pv, int planes = 1, int epi = kEpiPartial, const EpiArgs *ea = nullptr) {
  const int Mlog = M;
  M *= planes;
  a.no_pair = epi != kEpiPartial ? 1 : 0;  // the fused fixup addresses single-SM partial slots
  gemm_plan(a, a.N, a.K, M, a.batch);
  a.epi = epi;
  if (ea) a.e = *ea;
  if (epi != kEpiPartial && (a.batch != 1 || a.plan.tiles > kMaxFusedTiles || planes != 1))
    return fail(SM_ERR_INVALID_ARG, "fused GEMM epilogue: batch 1, bf16, <= 16384 tiles");
  CKS(act_box(a));
  a.x_row0 = x_row0 * planes;
  a.ws = ws;
  if (gemm_ws_floats(a) > ws_floats) return fail(SM_ERR_INVALID_ARG, "GEMM partial workspace too small");
  cudaEvent_t ev = nullptr;
  prof_begin(st, &ev);
  if (g_ablate_gemm == 0) CK(gemm_launch(a, st));
  // algorithmic bytes = the weight matrix (activations and the fp32 stream-K partial
  // slots are not part of the method's work)
  prof_end(st, ev, 0, (double)a.batch * ((double)a.N * a.K * 2));
  ++nl;
  *pv = PartialView{a.plan, ws, a.N, Mlog, planes};
  return SM_OK;
}
// Largest partial workspace a prototype can need for M in [1, max_m].
static size_t ws_need(const GemmArgs &proto, int max_m) {
  size_t need = 0;
  for (int M = 1; M <= max_m; M = (M < 16 ? 16 : M * 2)) {
    GemmArgs a = proto;
    gemm_plan(a, a.N, a.K, std::min(M, max_m), a.batch);
    need = std::max(need, gemm_ws_floats(a));
    if (M >= max_m) break;
  }
  GemmArgs a = proto;
  gemm_plan(a, a.N, a.K, max_m, a.batch);
  return std::max(need, gemm_ws_floats(a));
}

extern "C" sm_status sm_model_create(const sm_model_cfg *cfg, const sm_weights *w, const sm_dist *dist,
                                     sm_model **out) {
  if (!cfg || !w || !out) return fail(SM_ERR_INVALID_ARG, "sm_model_create: null argument");
  const sm_model_cfg &c = *cfg;
  const int tp = dist ? dist->tp_size : 1, tp_rank = dist ? dist->tp_rank : 0;
  const int pp = dist ? std::max(1, dist->pp_size) : 1, pp_rank = dist && dist->pp_size > 1 ? dist->pp_rank : 0;
  if (pp > 1) {  // layer-split pipeline (f4)
    if (pp > kMaxTP || tp != 1 || pp_rank < 0 || pp_rank >= pp || c.n_layers % pp || c.dtype != SM_DTYPE_BF16)
      return fail(SM_ERR_INVALID_ARG, "pipeline: pp_size in 2..8 with tp_size 1, bf16, pp_size dividing n_layers");
    for (int q = 0; q < pp; ++q)
      if (!dist->peer_sym[q]) return fail(SM_ERR_INVALID_ARG, "sm_dist.peer_sym[q] is null");
  }
  if (tp != 1 && tp != 2 && tp != 4 && tp != 8) return fail(SM_ERR_INVALID_ARG, "tp_size must be 1, 2, 4 or 8");
  if (tp_rank < 0 || tp_rank >= tp) return fail(SM_ERR_INVALID_ARG, "tp_rank out of range");
  if (tp > 1) {
    if (c.n_heads % tp || c.n_kv_heads % tp || c.d_ffn % (64 * tp) || c.vocab % (4 * tp))
      return fail(SM_ERR_INVALID_ARG, "tp_size must divide n_heads, n_kv_heads, d_ffn/64 and vocab/4");
    for (int q = 0; q < tp; ++q)
      if (!dist->peer_sym[q]) return fail(SM_ERR_INVALID_ARG, "sm_dist.peer_sym[q] is null");
  }
  if (c.n_layers < 1 || c.d_model % 64 || c.n_heads < 1 || c.n_kv_heads < 1 || c.n_heads % c.n_kv_heads ||
      (c.head_dim != 16 && c.head_dim != 32 && c.head_dim != 64 && c.head_dim != 128) || c.d_ffn % 64 ||
      c.vocab % 4 || c.n_medusa < 0 || c.n_medusa > kMaxGemmBatch || c.max_rows < 1 || c.max_rows > 1024 ||
      c.max_batch < 1 || c.max_seq_len < 1 || (c.n_heads * c.head_dim) % 64)
    return fail(SM_ERR_INVALID_ARG, "sm_model_create: unsupported shape (d, F multiple of 64; hd in {16,32,64,128}; "
                                    "max_rows <= 1024; n_medusa <= 5)");
  if (c.vocab / tp * 4 > 200 * 1024) return fail(SM_ERR_INVALID_ARG, "vocab too large for the shared-memory top-k");
  if (c.dtype != SM_DTYPE_BF16 && c.dtype != SM_DTYPE_FP32) return fail(SM_ERR_INVALID_ARG, "dtype must be 0 or 1");
  if (c.dtype == SM_DTYPE_FP32 && tp > 1) return fail(SM_ERR_UNSUPPORTED, "fp32 parity mode is single-GPU (tp_size 1)");
  if (c.dtype == SM_DTYPE_FP32 && 3 * c.max_rows > 1024)
    return fail(SM_ERR_INVALID_ARG, "fp32 parity mode: max_rows <= 341 (three GEMM rows per token row)");
  {  // every kernel resident before any work (see gemm_preload)
    static bool loaded = false;
    if (!loaded) {
      gemm_preload();
      attention_preload();
      attention_tc_preload();
      attention_f32_preload();
      decode_preload();
      epilogue_preload();
      tp_preload();
      loaded = true;
    }
  }
  sm_model *m = new sm_model();
  m->cfg = c;
  m->tp = tp;
  m->tp_rank = tp_rank;
  m->emu = (tp > 1 || pp > 1) ? static_cast<EmuGroup *>(dist->emu_group) : nullptr;
  m->pp = pp;
  m->pp_rank = pp_rank;
  m->L = c.n_layers / pp;  // this rank's layers
  m->d = c.d_model;
  m->H = c.n_heads / tp;  // this rank's shard
  m->Hkv = c.n_kv_heads / tp;
  m->hd = c.head_dim;
  m->F = c.d_ffn / tp;
  m->V = c.vocab / tp;
  m->v0 = tp_rank * m->V;
  m->nmed = c.n_medusa;
  m->G = c.n_heads / c.n_kv_heads;
  m->R = c.max_rows;
  m->B = c.max_batch;
  m->qkv_n = (m->H + 2 * m->Hkv) * c.head_dim;
  m->f32 = c.dtype == SM_DTYPE_FP32;
  m->P = m->f32 ? 3 : 1;
  m->hdu = c.head_dim * (m->f32 ? 2 : 1);
  m->fused = !m->f32 && tp == 1 && pp == 1 && c.head_dim == 128 && c.d_model % 128 == 0 && g_fused != 0;
  m->fuse_mask = m->fused ? g_fused : 0;
  m->embed = (const bf16 *)w->embed;
  m->final_norm = (const bf16 *)w->final_norm;
  m->lm_head = (const bf16 *)w->lm_head;
  for (int l = 0; l < m->L; ++l) {
    m->attn_norm.push_back((const bf16 *)w->attn_norm[l]);
    m->wqkv.push_back((const bf16 *)w->wqkv[l]);
    m->wo.push_back((const bf16 *)w->wo[l]);
    m->mlp_norm.push_back((const bf16 *)w->mlp_norm[l]);
    m->wgu.push_back((const bf16 *)w->wgate_up[l]);
    m->wdown.push_back((const bf16 *)w->wdown[l]);
  }
  for (int i = 0; i < m->nmed; ++i) {
    m->mR.push_back((const bf16 *)w->medusa_R[i]);
    m->mb.push_back((const bf16 *)w->medusa_b[i]);
    m->mU.push_back((const bf16 *)w->medusa_U[i]);
  }
  const int R = m->R, B = m->B, d = m->d, Hhd = m->H * m->hd, P = m->P;
  sm_status s;
#define ALLOC(p, n, what)                 \
  if ((s = dalloc(&p, n, what)) != SM_OK) { \
    sm_model_destroy(m);                  \
    return s;                             \
  }
  ALLOC(m->x, (size_t)R * d, "x");
  ALLOC(m->rs, (size_t)R, "rms scale");
  ALLOC(m->ss, (size_t)R * std::max(1, d / 64), "sum-of-squares partials");
  ALLOC(m->tile_cnt, (size_t)kMaxFusedTiles, "tile counters");
  ALLOC(m->done_cnt, 1, "tile counters");
  cudaMemset(m->tile_cnt, 0, (size_t)kMaxFusedTiles * sizeof(int));
  cudaMemset(m->done_cnt, 0, sizeof(int));
  ALLOC(m->h, (size_t)R * d * P, "h");
  ALLOC(m->q, (size_t)R * Hhd * (m->f32 ? 2 : 1), "q");  // fp32 q in the parity mode
  ALLOC(m->attn, (size_t)R * Hhd * P, "attn");
  ALLOC(m->act, (size_t)R * m->F * P, "act");
  ALLOC(m->hf, (size_t)R * d * P, "hf");
  ALLOC(m->z, (size_t)R * m->V, "logits");
  ALLOC(m->argmax, (size_t)R, "argmax");
  ALLOC(m->stats, (size_t)R * 3, "stats");
  ALLOC(m->head_in, (size_t)B * d * P, "head_in");
  ALLOC(m->r_buf, (size_t)std::max(1, m->nmed) * B * d * P, "r_buf");
  ALLOC(m->rope, (size_t)c.max_seq_len * (m->hd / 2), "rope");
  ALLOC(m->amax, (size_t)R, "amax");
  ALLOC(m->cand, (size_t)R, "cand");
  ALLOC(m->tk_val, (size_t)B * std::max(1, m->nmed) * 32, "topk values");
  ALLOC(m->tk_idx, (size_t)B * std::max(1, m->nmed) * 32, "topk indices");
  if (!m->f32 && m->hd == 128) {
    ALLOC(m->lean_part, attention_lean_part_floats(lean_units_max(m->Hkv, m->G, R, B)), "K1 partial slots");
    ALLOC(m->lean_sync, 4, "K1 barrier and unit counters");  // [0, 1] lean grid barrier, [2, 3] KSP work queue
    cudaMemset(m->lean_sync, 0, 4 * sizeof(int));
  }
  ALLOC(m->tp_seq, 1, "tp epoch");
  ALLOC(m->tp_err, 1, "tp error flag");
  cudaMemset(m->tp_seq, 0, sizeof(long long));
  cudaMemset(m->tp_err, 0, sizeof(int));
  if (tp > 1 || pp > 1) {
    const int nr = std::max(tp, pp), own = tp > 1 ? tp_rank : pp_rank;
    for (int q = 0; q < nr; ++q) m->sym[q] = dist->peer_sym[q];
    m->sym_slot_floats = tp_slot_floats(c);
    // own buffer: flags start below every epoch (the caller barriers before work)
    cudaMemset(m->sym[own], 0, kTpFlagBytes + 2 * m->sym_slot_floats * sizeof(float));
  }
  cudaMemset(m->x, 0, (size_t)R * d * 4);
  cudaMemset(m->h, 0, (size_t)R * d * 2 * P);
  cudaMemset(m->attn, 0, (size_t)R * Hhd * 2 * P);
  cudaMemset(m->act, 0, (size_t)R * m->F * 2 * P);
  cudaMemset(m->hf, 0, (size_t)R * d * 2 * P);
  cudaMemset(m->head_in, 0, (size_t)B * d * 2 * P);
  cudaMemset(m->r_buf, 0, (size_t)std::max(1, m->nmed) * B * d * 2 * P);
  // RoPE table: cos/sin built in fp64, stored fp32 (rounding contract R3)
  {
    const int half = m->hd / 2;
    std::vector<float2> tab((size_t)c.max_seq_len * half);
    for (int p = 0; p < c.max_seq_len; ++p)
      for (int i = 0; i < half; ++i) {
        const double ang = (double)p * std::pow((double)c.rope_theta, -2.0 * i / (double)m->hd);
        tab[(size_t)p * half + i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
    if (cudaMemcpy(m->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess) {
      sm_model_destroy(m);
      return fail(SM_ERR_CUDA, "rope upload");
    }
  }
  // GEMM prototypes
  auto mk = [&](const void *wp, int N, int K, const void *xp, int xrows, GemmArgs &a) -> sm_status {
    a = gemm_proto(N, K, 1);
    CKS(weight_map(&a.tmW[0], wp, N, K));
    CKS(act_map(a, 0, xp, xrows, K));
    return SM_OK;
  };
  for (int l = 0; l < m->L && s == SM_OK; ++l) {
    GemmArgs a;
    if ((s = mk(m->wqkv[l], m->qkv_n, d, m->h, R * P, a)) != SM_OK) break;
    m->g_qkv.push_back(a);
    if ((s = mk(m->wo[l], d, Hhd, m->attn, R * P, a)) != SM_OK) break;
    m->g_o.push_back(a);
    if ((s = mk(m->wgu[l], 2 * m->F, d, m->h, R * P, a)) != SM_OK) break;
    m->g_gu.push_back(a);
    if ((s = mk(m->wdown[l], d, m->F, m->act, R * P, a)) != SM_OK) break;
    m->g_down.push_back(a);
  }
  if (s == SM_OK) s = mk(m->lm_head, m->V, d, m->hf, R * P, m->g_lm);
  if (s != SM_OK) {
    sm_model_destroy(m);
    return s;
  }
  size_t need = 0;  // stream-K partial workspace: max over every GEMM the model runs
  for (int l = 0; l < m->L; ++l)
    need = std::max({need, ws_need(m->g_qkv[l], R * P), ws_need(m->g_o[l], R * P), ws_need(m->g_gu[l], R * P),
                     ws_need(m->g_down[l], R * P)});
  need = std::max(need, ws_need(m->g_lm, R * P));
  if (m->nmed > 0) {
    m->g_R = gemm_proto(d, d, m->nmed);
    m->g_U = gemm_proto(m->V, d, m->nmed);
    for (int i = 0; i < m->nmed && s == SM_OK; ++i) {
      if ((s = weight_map(&m->g_R.tmW[i], m->mR[i], d, d)) != SM_OK) break;
      if ((s = act_map(m->g_R, i, m->head_in, B * P, d)) != SM_OK) break;
      if ((s = weight_map(&m->g_U.tmW[i], m->mU[i], m->V, d)) != SM_OK) break;
      s = act_map(m->g_U, i, m->r_buf + (size_t)i * B * d * P, B * P, d);
    }
    if (s != SM_OK) {
      sm_model_destroy(m);
      return s;
    }
    need = std::max({need, ws_need(m->g_R, B * P), ws_need(m->g_U, B * P)});
  }
  ALLOC(m->ws, need, "stream-K partials");
  m->ws_floats = need;
  ALLOC(m->iota, (size_t)R, "prefill depths");  // last: the decode buffers keep their placement
  {
    std::vector<int32_t> io((size_t)R);
    for (int i = 0; i < R; ++i) io[(size_t)i] = i;
    if (cudaMemcpy(m->iota, io.data(), io.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      sm_model_destroy(m);
      return fail(SM_ERR_CUDA, "prefill depths upload");
    }
  }
#undef ALLOC
  if ((s = sm_tree_create_chain(std::min(R, kMaxTreeNodes), &m->chain)) != SM_OK ||
      (s = tree_upload(m->chain)) != SM_OK) {
    sm_model_destroy(m);
    return s;
  }
  if (cudaStreamCreateWithFlags(&m->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    sm_model_destroy(m);
    return fail(SM_ERR_CUDA, "stream create");
  }
  *out = m;
  return SM_OK;
}

extern "C" void sm_model_destroy(sm_model *m) {
  if (!m) return;
  cudaFree(m->lean_part);
  cudaFree(m->lean_sync);
  cudaFree(m->x);
  cudaFree(m->rs);
  cudaFree(m->ss);
  cudaFree(m->tile_cnt);
  cudaFree(m->iota);
  cudaFree(m->done_cnt);
  cudaFree(m->part);
  cudaFree(m->ws);
  cudaFree(m->z);
  cudaFree(m->stats);
  cudaFree(m->h);
  cudaFree(m->q);
  cudaFree(m->attn);
  cudaFree(m->act);
  cudaFree(m->hf);
  cudaFree(m->head_in);
  cudaFree(m->r_buf);
  cudaFree(m->argmax);
  cudaFree(m->rope);
  cudaFree(m->amax);
  cudaFree(m->cand);
  cudaFree(m->tk_val);
  cudaFree(m->tk_idx);
  cudaFree(m->tp_seq);
  cudaFree(m->tp_err);
  if (m->chain) sm_tree_destroy(m->chain);
  if (m->cap_stream) cudaStreamDestroy(m->cap_stream);
  delete m;
}

extern "C" sm_status sm_generate_bf16(void *dst, size_t numel, uint64_t seed, uint64_t stream_id, uint64_t start,
                                      int mode, void *stream) {
  if (!dst && numel) return fail(SM_ERR_INVALID_ARG, "sm_generate_bf16: null dst");
  CK(generate_bf16_launch(dst, numel, seed, stream_id, start, mode, (cudaStream_t)stream));
  return SM_OK;
}

extern "C" sm_status sm_generate_bf16_2d(void *dst, int rows, int cols, int full_cols, int row0, int col0,
                                         uint64_t seed, uint64_t stream_id, int mode, void *stream) {
  if ((!dst && rows * cols) || rows < 0 || cols < 0 || row0 < 0 || col0 < 0 || col0 + cols > full_cols)
    return fail(SM_ERR_INVALID_ARG, "sm_generate_bf16_2d: bad arguments");
  CK(generate_bf16_2d_launch(dst, rows, cols, full_cols, row0, col0, seed, stream_id, mode, (cudaStream_t)stream));
  return SM_OK;
}

// ---------------------------------------------------------------- tensor parallel plumbing
extern "C" sm_status sm_emu_group_create(int n_ranks, void **group) {
  if (!group || n_ranks < 2 || n_ranks > kMaxTP) return fail(SM_ERR_INVALID_ARG, "sm_emu_group_create: 2..8 ranks");
  *group = emu_group_create(n_ranks);
  if (!*group) return fail(SM_ERR_CUDA, "sm_emu_group_create: event creation failed");
  return SM_OK;
}
extern "C" void sm_emu_group_destroy(void *group) { emu_group_destroy(static_cast<EmuGroup *>(group)); }

extern "C" sm_status sm_tp_sym_bytes(const sm_model_cfg *cfg, size_t *bytes) {
  if (!cfg || !bytes || cfg->max_rows < 1 || cfg->d_model < 1 || cfg->max_batch < 1)
    return fail(SM_ERR_INVALID_ARG, "sm_tp_sym_bytes: bad arguments");
  *bytes = kTpFlagBytes + 2 * tp_slot_floats(*cfg) * sizeof(float);
  return SM_OK;
}
extern "C" sm_status sm_tp_status(const sm_model *m, int *timed_out) {
  if (!m || !timed_out) return fail(SM_ERR_INVALID_ARG, "sm_tp_status: null");
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(timed_out, m->tp_err, sizeof(int), cudaMemcpyDeviceToHost));
  return SM_OK;
}
extern "C" sm_status sm_ipc_get_handle(const void *d_ptr, unsigned char handle[64]) {
  if (!d_ptr || !handle) return fail(SM_ERR_INVALID_ARG, "sm_ipc_get_handle: null");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, const_cast<void *>(d_ptr)));
  std::memcpy(handle, &h, 64);
  return SM_OK;
}
extern "C" sm_status sm_ipc_open(const unsigned char handle[64], void **d_ptr) {
  if (!handle || !d_ptr) return fail(SM_ERR_INVALID_ARG, "sm_ipc_open: null");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  CK(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SM_OK;
}
extern "C" sm_status sm_ipc_close(void *d_ptr) {
  if (!d_ptr) return fail(SM_ERR_INVALID_ARG, "sm_ipc_close: null");
  CK(cudaIpcCloseMemHandle(d_ptr));
  return SM_OK;
}

// ---------------------------------------------------------------- memory-budget planner (f2)
// Algorithm 1 over Eqs. 1, 3-6; see include/specmemo.h and
// DESIGN.md reading Q31.  Integer arithmetic throughout (sizes in bytes).
namespace {
struct PlanCand {
  int N, S, kind;  // kind 0 default, 1 R4-pruned base tree, 2 custom
};
struct PlanCtx {
  const sm_plan_in *in;
  size_t mem_base(int p) const {
    const sm_model_cfg &c = in->cfg;
    const long long layer = (long long)(c.n_heads + 2 * c.n_kv_heads) * c.head_dim * c.d_model +
                            (long long)c.d_model * c.n_heads * c.head_dim + 3LL * c.d_ffn * c.d_model + 2LL * c.d_model;
    return (size_t)((c.n_layers * layer + 2LL * c.vocab * c.d_model + c.d_model) * p);  // Eq. 5
  }
  size_t mem_heads(int l, int p) const {  // Eq. 4 (paper) or the real Medusa-1 heads (b200)
    if (in->accounting == SM_ACCT_B200) {
      const long long d = in->cfg.d_model, V = in->cfg.vocab;
      return (size_t)(l * (d * d + d + V * d) * p);
    }
    return (size_t)(0.6e9 * l);
  }
  size_t mem_kv(int N, int p) const {  // Eq. 1 with d (+ N scratch slots, b200)
    const sm_model_cfg &c = in->cfg;
    const long long x = (long long)in->n_queries * in->max_tokens + (in->accounting == SM_ACCT_B200 ? N : 0);
    return (size_t)(2LL * c.n_layers * in->batch * c.n_kv_heads * c.head_dim * x * p);
  }
  size_t mem_buffers(int N, int S, int l, int p) const {  // Eq. 3 (paper) or fp32 node logits (b200)
    const long long b = in->batch, w = in->cfg.vocab;
    if (in->accounting == SM_ACCT_B200) return (size_t)(b * N * w * 4);
    return (size_t)((b * N * w + b * S * l * w + b * S * (long long)l * l * w) * p);
  }
  size_t total(int heads, int N, int S) const {  // Eq. 6
    const int p = in->prec_bytes;
    return mem_base(p) + mem_heads(heads, p) + mem_kv(N, p) + mem_buffers(N, S, heads, p);
  }
};
}  // namespace

extern "C" sm_status sm_workspace_bytes(const sm_model_cfg *cfg, size_t *bytes);

extern "C" sm_status sm_plan(const sm_plan_in *in, sm_plan_out *out) {
  if (!in || !out || !in->base_tree || in->batch < 1 || in->n_queries < 1 || in->max_tokens < 1 ||
      in->default_heads < 2 || in->prec_bytes < 1 || (in->accounting != SM_ACCT_PAPER && in->accounting != SM_ACCT_B200))
    return fail(SM_ERR_INVALID_ARG, "sm_plan: bad arguments");
  std::memset(out, 0, sizeof(*out));
  size_t budget = in->max_memory;
  if (budget == 0) {  // bound to the device: its free memory now
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    budget = fr;
  }
  PlanCtx P{in};
  const int p = in->prec_bytes;
  const sm_tree *bt = in->base_tree;
  const int N0 = bt->N, S0 = bt->S;
  out->max_memory = budget;
  out->x = (long long)in->n_queries * in->max_tokens;  // ComputeMinCache
  auto fill = [&](int status, int heads, const PlanCand &c) {
    out->status = status;
    out->heads = heads;
    out->N = c.N;
    out->S = c.S;
    out->kind = c.kind;
    out->base = P.mem_base(p);
    out->heads_bytes = P.mem_heads(heads, p);
    out->kv = P.mem_kv(c.N, p);
    out->buffers = P.mem_buffers(c.N, c.S, heads, p);
    out->total = P.total(heads, c.N, c.S);
  };
  int heads = in->default_heads;
  if (P.total(heads, N0, S0) <= budget) {  // AvailMemory(default config)
    fill(0, heads, PlanCand{N0, S0, 0});
    return SM_OK;
  }
  int status = 1;
  for (;;) {
    // ExploreTree: base tree cut to depth `heads`, R4-pruned to the mask sizes; custom trees at 4 heads
    std::vector<PlanCand> cands;
    std::vector<std::vector<int>> cut;
    for (size_t i = 1; i < bt->paths.size(); ++i)
      if ((int)bt->paths[i].size() <= heads) cut.push_back(bt->paths[i]);
    sm_tree *ct = nullptr;
    CKS(tree_from_paths(cut, bt->topk, &ct));
    for (int n : {64, 44, 31, 27, 16, 5}) {
      if (n > ct->N) continue;
      sm_tree *pt = nullptr;
      if (sm_tree_prune(ct, n, &pt) != SM_OK) continue;
      cands.push_back(PlanCand{pt->N, pt->S, 1});
      sm_tree_destroy(pt);
    }
    sm_tree_destroy(ct);
    if (heads == 4) {  // tab:treefeatures, C row, heads = 4
      cands.push_back(PlanCand{64, 56, 2});
      cands.push_back(PlanCand{44, 37, 2});
    }
    std::sort(cands.begin(), cands.end(), [](const PlanCand &a, const PlanCand &b) {
      return a.N != b.N ? a.N > b.N : (a.S != b.S ? a.S > b.S : a.kind > b.kind);
    });
    for (const auto &c : cands)
      if (P.total(heads, c.N, c.S) <= budget) {
        fill(status, heads, c);
        return SM_OK;
      }
    int nh = heads;
    for (int h = heads - 1; h >= 2; --h)
      if (P.total(h, N0, S0) <= budget) {
        nh = h;
        break;
      }
    if (nh == heads) {  // QuantizeBaseModel: not in this build
      out->status = 3;
      out->heads = heads;
      return SM_OK;
    }
    heads = nh;
    status = 2;
  }
}

extern "C" sm_status sm_workspace_bytes(const sm_model_cfg *cfg, size_t *bytes) {
  if (!cfg || !bytes) return fail(SM_ERR_INVALID_ARG, "sm_workspace_bytes: null");
  const sm_model_cfg &c = *cfg;
  const size_t R = c.max_rows, B = c.max_batch, d = c.d_model, P = c.dtype == SM_DTYPE_FP32 ? 3 : 1;
  const size_t Hhd = (size_t)c.n_heads * c.head_dim, nmed = std::max(1, c.n_medusa);
  size_t b = 0;
  b += R * d * 4 + R * 4 + R * std::max<size_t>(1, d / 64) * 4 + (size_t)kMaxFusedTiles * 4 + 4;  // x, rs, ss, counters
  b += R * 4;                                                                                        // prefill depths
  b += R * d * 2 * P + R * Hhd * 2 * (c.dtype == SM_DTYPE_FP32 ? 2 : 1) + R * Hhd * 2 * P;       // h, q, attn
  b += R * c.d_ffn * 2 * P + R * d * 2 * P + R * c.vocab * 4 + R * 4 + R * 3 * 4;                // act, hf, z, argmax, stats
  b += B * d * 2 * P + nmed * B * d * 2 * P + (size_t)c.max_seq_len * (c.head_dim / 2) * 8;       // head_in, r_buf, rope
  b += 2 * R * 4 + 2 * B * nmed * 32 * 4 + 16;                                                      // amax, cand, top-k
  if (c.dtype != SM_DTYPE_FP32 && c.head_dim == 128)                                                 // K1 partials
    b += attention_lean_part_floats(lean_units_max(c.n_kv_heads, c.n_heads / c.n_kv_heads, (int)R, (int)B)) * 4 + 16;
  // stream-K partial slots: the largest need over the model's GEMMs
  size_t need = 0;
  const int Rg = (int)(R * P);
  for (auto nk : {std::make_pair((c.n_heads + 2 * c.n_kv_heads) * c.head_dim, c.d_model),
                  std::make_pair(c.d_model, c.n_heads * c.head_dim), std::make_pair(2 * c.d_ffn, c.d_model),
                  std::make_pair(c.d_model, c.d_ffn), std::make_pair(c.vocab, c.d_model)})
    need = std::max(need, ws_need(gemm_proto(nk.first, nk.second, 1), Rg));
  if (c.n_medusa > 0)
    need = std::max({need, ws_need(gemm_proto(c.d_model, c.d_model, c.n_medusa), (int)(B * P)),
                     ws_need(gemm_proto(c.vocab, c.d_model, c.n_medusa), (int)(B * P))});
  *bytes = b + need * 4;
  return SM_OK;
}

// ---------------------------------------------------------------- bounded KV
// Bumped by sm_set_option / sm_reset_options: a graph captured under other launch knobs is stale
// (the knobs are process-wide and baked into the captured kernels).
static int g_opt_version = 0;
// True while sm_step captures its own per-step graph (the only place the commit may trigger early).
static thread_local bool g_lib_capture = false;

struct GraphKey {
  int ver;
  int prof;
  int mode;
  float T, eps, alpha;
  const void *max_new, *forced, *o0, *o1, *o2, *o3, *o4, *o5;
  bool operator<(const GraphKey &o) const {
    return std::tie(ver, prof, mode, T, eps, alpha, max_new, forced, o0, o1, o2, o3, o4, o5) <
           std::tie(o.ver, o.prof, o.mode, o.T, o.eps, o.alpha, o.max_new, o.forced, o.o0, o.o1, o.o2, o.o3, o.o4, o.o5);
  }
};

struct sm_kv {
  sm_model *m;
  sm_tree *t;  // private copy of the tree
  int b, x, cap, N;
  bf16 *base;
  size_t bytes;
  int32_t *len = nullptr, *root = nullptr, *topk = nullptr, *acc_row = nullptr, *root_next = nullptr,
          *emitted = nullptr, *tree_tok = nullptr;
  int att_nsplit_max = 32;
  // pad batching (f4): uniform cache advance, pad slots masked, positions count tokens
  int pad_mode = 0;
  int32_t *pos_len = nullptr;  // [b] tokens committed (the RoPE position base)
  uint32_t *pad = nullptr;     // [b][pad_words] masked cache slots
  int pad_words = 0;
  CUtensorMap tmKV;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  int32_t *h_sticky = nullptr, *d_sticky = nullptr;  // mapped host word: device-detected status
  int step_launches = 0;
  int prof = 0;
  std::vector<ProfEvent> prof_events;
  cudaStream_t last_stream = nullptr;
};

static size_t kv_elems_per_layer(const sm_model_cfg *c, int tp, int b, int cap) {
  return (size_t)2 * b * (c->n_kv_heads / tp) * (size_t)cap * c->head_dim;
}

extern "C" sm_status sm_kv_bytes(const sm_model_cfg *cfg, int tp_size, int batch, int max_seq_len, int tree_nodes,
                                 size_t *bytes) {
  if (!cfg || !bytes || tp_size < 1 || batch < 1 || max_seq_len < 1 || tree_nodes < 1 ||
      cfg->n_kv_heads % tp_size)
    return fail(SM_ERR_INVALID_ARG, "sm_kv_bytes: bad arguments");
  *bytes = kv_elems_per_layer(cfg, tp_size, batch, max_seq_len + tree_nodes) * cfg->n_layers *
           (cfg->dtype == SM_DTYPE_FP32 ? 4 : 2);
  return SM_OK;
}

extern "C" sm_status sm_kv_bind(sm_model *m, const sm_tree *tree, int batch, int max_seq_len, void *d_mem,
                                size_t bytes, sm_kv **out) {
  if (!m || !tree || !d_mem || !out || batch < 1 || batch > m->B || max_seq_len < 1)
    return fail(SM_ERR_INVALID_ARG, "sm_kv_bind: bad arguments");
  if (tree->l > m->nmed) return fail(SM_ERR_INFEASIBLE_TREE, "tree depth exceeds the number of Medusa heads");
  if (tree->topk > 32) return fail(SM_ERR_INVALID_ARG, "topk > 32");
  if (batch * tree->N > m->R) return fail(SM_ERR_INVALID_ARG, "batch * tree nodes exceeds max_rows");
  size_t need;
  sm_model_cfg lc = m->cfg;
  lc.n_layers = m->L;  // this rank's layers (pipeline)
  CKS(sm_kv_bytes(&lc, m->tp, batch, max_seq_len, tree->N, &need));
  if (bytes < need) return fail(SM_ERR_KV_CAPACITY, "Cache: KV memory smaller than sm_kv_bytes");
  if (max_seq_len + tree->N > m->cfg.max_seq_len)
    return fail(SM_ERR_INVALID_ARG, "max_seq_len + N exceeds the model's RoPE table (cfg.max_seq_len)");
  sm_kv *kv = new sm_kv();
  kv->m = m;
  kv->t = new sm_tree(*tree);
  kv->t->on_device = false;
  kv->b = batch;
  kv->x = max_seq_len;
  kv->N = tree->N;
  kv->cap = max_seq_len + tree->N;
  kv->base = (bf16 *)d_mem;
  kv->bytes = need;
  sm_status s;
  if ((s = tree_upload(kv->t)) != SM_OK || (s = dalloc(&kv->len, batch, "len")) != SM_OK ||
      (s = dalloc(&kv->root, batch, "root")) != SM_OK ||
      (s = dalloc(&kv->topk, (size_t)batch * std::max(1, m->nmed) * kv->t->topk, "topk")) != SM_OK ||
      (s = dalloc(&kv->acc_row, batch, "acc_row")) != SM_OK ||
      (s = dalloc(&kv->root_next, batch, "root_next")) != SM_OK ||
      (s = dalloc(&kv->emitted, batch, "emitted")) != SM_OK ||
      (s = dalloc(&kv->tree_tok, (size_t)batch * kv->N, "tree_tok")) != SM_OK ||
      (s = dalloc(&kv->pos_len, batch, "pos_len")) != SM_OK ||
      (s = dalloc(&kv->pad, (size_t)batch * (kv->cap / 32 + 2), "pad bitmap")) != SM_OK) {
    sm_kv_destroy(kv);
    return s;
  }
  if (cudaHostAlloc((void **)&kv->h_sticky, sizeof(int32_t), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void **)&kv->d_sticky, kv->h_sticky, 0) != cudaSuccess) {
    sm_kv_destroy(kv);
    return fail(SM_ERR_DEVICE_OOM, "Buffer: mapped status word");
  }
  *(volatile int32_t *)kv->h_sticky = 0;
  const uint64_t rows = (uint64_t)need / 2 / m->hd;
  if (!m->f32 && (s = kv_map(&kv->tmKV, d_mem, rows, m->hd)) != SM_OK) {  // bf16 kernels' TMA view
    sm_kv_destroy(kv);
    return s;
  }
  cudaMemset(d_mem, 0, need);  // finite contents everywhere (masked keys still meet P = 0 * V)
  cudaMemset(kv->len, 0, batch * 4);
  cudaMemset(kv->root, 0, batch * 4);
  cudaMemset(kv->topk, 0, (size_t)batch * std::max(1, m->nmed) * kv->t->topk * 4);
  cudaMemset(kv->emitted, 0, batch * 4);
  cudaMemset(kv->acc_row, 0, batch * 4);
  cudaMemset(kv->root_next, 0, batch * 4);
  kv->pad_words = kv->cap / 32 + 2;
  cudaMemset(kv->pos_len, 0, batch * 4);
  cudaMemset(kv->pad, 0, (size_t)batch * kv->pad_words * 4);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    sm_kv_destroy(kv);
    return fail(SM_ERR_CUDA, "kv bind memset");
  }
  *out = kv;
  return SM_OK;
}

extern "C" void sm_kv_destroy(sm_kv *kv) {
  if (!kv) return;
  for (auto &g : kv->graphs) cudaGraphExecDestroy(g.second);
  for (auto &pe : kv->prof_events) {
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  cudaFree(kv->len);
  cudaFree(kv->root);
  cudaFree(kv->topk);
  cudaFree(kv->acc_row);
  cudaFree(kv->root_next);
  cudaFree(kv->emitted);
  cudaFree(kv->tree_tok);
  cudaFree(kv->pos_len);
  cudaFree(kv->pad);
  if (kv->h_sticky) cudaFreeHost(kv->h_sticky);
  if (kv->t) sm_tree_destroy(kv->t);
  delete kv;
}

extern "C" sm_status sm_kv_lengths_device(const sm_kv *kv, int32_t **d_len) {
  if (!kv || !d_len) return fail(SM_ERR_INVALID_ARG, "null");
  *d_len = kv->len;
  return SM_OK;
}
extern "C" sm_status sm_kv_set_pad_mode(sm_kv *kv, int on) {
  if (!kv) return fail(SM_ERR_INVALID_ARG, "sm_kv_set_pad_mode: null");
  if (kv->m->tp > 1) return fail(SM_ERR_UNSUPPORTED, "pad batching: single GPU only");
  CK(cudaDeviceSynchronize());
  kv->pad_mode = on ? 1 : 0;
  CK(cudaMemcpy(kv->pos_len, kv->len, kv->b * 4, cudaMemcpyDeviceToDevice));  // positions = tokens so far
  CK(cudaMemset(kv->pad, 0, (size_t)kv->b * kv->pad_words * 4));
  for (auto &g : kv->graphs) cudaGraphExecDestroy(g.second);  // the step's kernel sequence changes
  kv->graphs.clear();
  return SM_OK;
}
extern "C" sm_status sm_kv_positions(const sm_kv *kv, int32_t *h_pos) {
  if (!kv || !h_pos) return fail(SM_ERR_INVALID_ARG, "null");
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h_pos, kv->pad_mode ? kv->pos_len : kv->len, kv->b * 4, cudaMemcpyDeviceToHost));
  return SM_OK;
}
extern "C" sm_status sm_kv_lengths(const sm_kv *kv, int32_t *h_len) {
  if (!kv || !h_len) return fail(SM_ERR_INVALID_ARG, "null");
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h_len, kv->len, kv->b * 4, cudaMemcpyDeviceToHost));
  return SM_OK;
}
extern "C" sm_status sm_state_device(const sm_kv *kv, int32_t **d_root, int32_t **d_topk) {
  if (!kv) return fail(SM_ERR_INVALID_ARG, "null");
  if (d_root) *d_root = kv->root;
  if (d_topk) *d_topk = kv->topk;
  return SM_OK;
}

// ---------------------------------------------------------------- forward (a2 + a3)
static int attn_splits(const sm_model *m, int nseq, int Nq, int cap) {
  return attention_nsplit(nseq * m->Hkv * attention_row_blocks(Nq, m->G, m->hd), m->hd, cap);
}

// Timing ablation (sm_set_option "ablate", experiments only -- results become
// meaningless): bit 1 skips K1 attention, bit 2 the per-layer GEMM consumers,
// bit 4 the per-layer GEMMs, bit 8 the Medusa heads.
static int g_ablate = 0;
#define KEEP(bit) ((g_ablate & (bit)) == 0)

// x += y (all-reduced across ranks under TP); deferred (per-layer norms, R2):
// h = bf16(x * g) and m->rs = 1/sqrt(mean(x^2) + eps) for the next GEMM's consumer;
// else (final norm, R8) h = bf16(rms(x) * g).
// The deferred scale reaches the next consumer as m->rsa: from the split kernel's per-slice sums
// of squares (single GPU, default), or precomputed in m->rs (TP exchange, fused epilogues).
static sm_status resid_norm(sm_model *m, const PartialView *pv, const bf16 *g, bf16 *h, int M, cudaStream_t st,
                            bool deferred) {
  float *rs = deferred ? m->rs : nullptr;
  if (m->tp > 1 && pv) {
    CK(resid_norm_tp_launch(*pv, m->x, g, h, M, m->d, m->cfg.rms_eps, tp_next(m), rs, st));
    m->rsa = RsArgs{m->rs, nullptr, 0, m->d, m->cfg.rms_eps};
  } else if (deferred && !m->fused) {
    CK(resid_norm_split_launch(pv, m->x, g, h, M, m->d, m->P, m->ss, st));
    m->rsa = RsArgs{nullptr, m->ss, resid_norm_slices(m->d), m->d, m->cfg.rms_eps};
  } else {
    CK(resid_norm_launch(pv, m->x, g, h, M, m->d, m->cfg.rms_eps, m->P, rs, st));
    m->rsa = RsArgs{m->rs, nullptr, 0, m->d, m->cfg.rms_eps};
  }
  return SM_OK;
}

// tokens d_tok [nseq * Nq] -> hf [nseq * Nq][d]; K/V rows of every layer written
static sm_status enqueue_forward(sm_model *m, sm_kv *kv, const int32_t *d_tok, int nseq, int seq_base, int Nq,
                                 const TreeDev &tree, cudaStream_t st, int &nl) {
  const int M = nseq * Nq;
  const int d = m->d;
  // layer-split pipeline (f4): hand-off k (rank k -> k + 1) is exchange point pt0 + k, the last
  // rank's final residual to every rank is point pt0 + pp - 1
  const int pt0 = m->tp_point;
  if (m->pp > 1) m->tp_point += m->pp;
  const int n4 = M * d / 4;
  if (m->pp_rank == 0) {
    CK(embed_launch(d_tok, m->embed, m->x, M, d, st));
    ++nl;
  } else {  // the previous stage's residual rows
    CK(pp_xfer_launch(m->x, n4, m->pp_rank - 1, 1u << m->pp_rank, pp_args(m, pt0 + m->pp_rank - 1), st));
    ++nl;
  }
  const int nsplit = attn_splits(m, nseq, Nq, kv->cap);
  const long long layer_rows = (long long)2 * kv->b * m->Hkv * kv->cap;
  const long long half_rows = (long long)kv->b * m->Hkv * kv->cap;
  RowCtx rc{M, Nq, seq_base, kv->len, tree.depth, kv->pad_mode ? kv->pos_len : nullptr};
  PartialView pv, pv_down{};
  bool have_down = false;
  g_ablate_gemm = (g_ablate & 4) ? 1 : 0;
  // Fused path (m->fused): the consumers below run inside the K2 GEMMs as tile
  // epilogues (kEpi*, gemm.cu); only the first layer's norm and the final norm
  // remain separate kernels.  Same rounding contract, same summation order.
  EpiArgs ea;
  std::memset(&ea, 0, sizeof(ea));
  ea.rope = m->rope;
  ea.rc = rc;
  ea.H = m->H;
  ea.Hkv = m->Hkv;
  ea.cap = kv->cap;
  ea.q = m->q;
  ea.act = m->act;
  ea.F = m->F;
  ea.x = m->x;
  ea.h = m->h;
  ea.ss = m->ss;
  ea.d = d;
  ea.eps = m->cfg.rms_eps;
  ea.tile_cnt = m->tile_cnt;
  ea.done_cnt = m->done_cnt;
  const int fm = (m->fused && KEEP(2)) ? m->fuse_mask : 0;
  const bool fq = fm & 1, fs = fm & 2, fr = fm & 4;
  for (int l = 0; l < m->L; ++l) {
    // x += down (previous layer, R7); h = bf16(x * g1), rs  (deferred R2)
    if (KEEP(2) && (!fr || l == 0)) {
      CKS(resid_norm(m, have_down ? &pv_down : nullptr, m->attn_norm[l], m->h, M, st, true));
      ++nl;
    }
    bf16 *kc = kv->base + (size_t)l * layer_rows * m->hdu;  // bf16 units (fp32 rows are 2 hd units)
    bf16 *vc = kc + (size_t)half_rows * m->hdu;
    if (fq) {  // QKV GEMM with the RoPE + cache-write epilogue
      ea.kc = kc;
      ea.vc = vc;
      ea.rs_in = m->rs;
      CKS(run_gemm(m->g_qkv[l], M, 0, m->ws, m->ws_floats, st, nl, &pv, 1, kEpiQKV, &ea));
    } else {
      CKS(run_gemm(m->g_qkv[l], M, 0, m->ws, m->ws_floats, st, nl, &pv, m->P));
    }
    // RoPE, q -> m->q, k/v -> cache slots Lc + node (R3)
    if (KEEP(2) && !fq) {
      CK(qkv_consumer_launch(pv, rc, m->H, m->Hkv, m->hd, m->rope, m->q, kc, vc, kv->cap, m->rsa, st));
      ++nl;
    }
    AttnArgs aa;
    std::memset(&aa, 0, sizeof(aa));
    aa.tmK = kv->tmKV;
    aa.tmV = kv->tmKV;
    aa.q = m->q;
    aa.out = m->attn;
    aa.len = kv->len;
    aa.anc = tree.anc;
    aa.k_row0 = (long long)l * layer_rows;
    aa.v_row0 = aa.k_row0 + half_rows;
    aa.seq_rows = (long long)m->Hkv * kv->cap;
    aa.cap = kv->cap;
    aa.Nq = Nq;
    aa.H = m->H;
    aa.Hkv = m->Hkv;
    aa.G = m->G;
    aa.nseq = nseq;
    aa.seq_base = seq_base;
    aa.nsplit = nsplit;
    aa.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)m->hd));
    aa.pad = kv->pad_mode ? kv->pad : nullptr;
    aa.pad_words = kv->pad_words;
    aa.causal = tree.anc == nullptr;  // causal prefill chunk (sm_prefill)
    aa.lean_part = m->lean_part;
    aa.lean_sync = m->lean_sync;
    aa.lean_min_tiles = attention_lean_min_tiles(Nq, m->G);
    aa.k_base = kv->base;
    aa.v_base = kv->base;
    aa.l2_pf = m->wo[l];  // o_proj weights stream into L2 while attention runs
    aa.l2_pf_bytes = (unsigned long long)d * m->H * m->hd * 2;
    cudaEvent_t ev = nullptr;
    prof_begin(st, &ev);
    if (KEEP(1)) {
      if (m->f32)
        CK(attention_f32_launch(reinterpret_cast<const float *>(m->q), reinterpret_cast<const float *>(kc),
                                reinterpret_cast<const float *>(vc), kv->len, tree.anc, Nq, m->H, m->Hkv, m->hd,
                                kv->cap, nseq, seq_base, aa.pad, kv->pad_words, m->attn, st));
      else
        CK(attention_launch(aa, m->hd, st));
      ++nl;
    }
    prof_end(st, ev, 1, 0.0);
    // x += o (R5); h = bf16(x * g2), rs  (deferred R2)
    if (fr) {
      ea.g = m->mlp_norm[l];
      ea.rs_out = m->rs;
      CKS(run_gemm(m->g_o[l], M, 0, m->ws, m->ws_floats, st, nl, &pv, 1, kEpiResid, &ea));
    } else {
      CKS(run_gemm(m->g_o[l], M, 0, m->ws, m->ws_floats, st, nl, &pv, m->P));
      if (KEEP(2)) {
        CKS(resid_norm(m, &pv, m->mlp_norm[l], m->h, M, st, true));
        ++nl;
      }
    }
    if (fs) {  // act = bf16(SiLU(rs g) * rs u) (R6) in the GEMM's tile epilogue
      ea.rs_in = m->rs;
      CKS(run_gemm(m->g_gu[l], M, 0, m->ws, m->ws_floats, st, nl, &pv, 1, kEpiSiLU, &ea));
    } else {
      CKS(run_gemm(m->g_gu[l], M, 0, m->ws, m->ws_floats, st, nl, &pv, m->P));
      if (KEEP(2)) {
        CK(silu_consumer_launch(pv, m->F, m->act, m->rsa, st));  // act = bf16(SiLU(rs g) * rs u) (R6)
        ++nl;
      }
    }
    if (fr && l + 1 < m->L) {  // x += down (R7); h = bf16(x * g1 of the next layer), rs
      ea.g = m->attn_norm[l + 1];
      ea.rs_out = m->rs;
      CKS(run_gemm(m->g_down[l], M, 0, m->ws, m->ws_floats, st, nl, &pv_down, 1, kEpiResid, &ea));
      have_down = false;  // already added into x
    } else {  // the final norm (R8, not deferred) needs the whole row: consumer kernel
      CKS(run_gemm(m->g_down[l], M, 0, m->ws, m->ws_floats, st, nl, &pv_down, m->P));
      have_down = true;
    }
  }
  g_ablate_gemm = 0;
  // x += down; hf = bf16(rms(x) * gf)   (R8)
  CKS(resid_norm(m, have_down ? &pv_down : nullptr, m->final_norm, m->hf, M, st, false));
  ++nl;
  if (m->pp > 1) {
    const int last = m->pp - 1;
    if (m->pp_rank < last) {  // to the next stage (hf above is unused), then the final rows back
      CK(pp_xfer_launch(m->x, n4, m->pp_rank, 1u << (m->pp_rank + 1), pp_args(m, pt0 + m->pp_rank), st));
      CK(pp_xfer_launch(m->x, n4, last, (1u << last) - 1u, pp_args(m, pt0 + last), st));
      CKS(resid_norm(m, nullptr, m->final_norm, m->hf, M, st, false));  // same kernel, same x: same hf
      nl += 3;
    } else {
      CK(pp_xfer_launch(m->x, n4, last, (1u << last) - 1u, pp_args(m, pt0 + last), st));
      ++nl;
    }
  }
  return SM_OK;
}

// heads at rows [row0, row0 + nb) of head_in -> topk rows [row0, row0 + nb)
static sm_status enqueue_heads(sm_model *m, sm_kv *kv, int row0, int nb, cudaStream_t st, int &nl) {
  if (m->nmed == 0 || kv->t->l == 0 || !KEEP(8)) return SM_OK;
  const int d = m->d, B = m->B, P = m->P;
  PartialView pv;
  CKS(run_gemm(m->g_R, nb, row0, m->ws, m->ws_floats, st, nl, &pv, P));
  CK(heads_r_consumer_launch(pv, m->nmed, nb, d, m->head_in + (size_t)row0 * d * P, m->mb.data(),
                             m->r_buf + (size_t)row0 * d * P, (long long)B * d * P, st));
  ++nl;
  CKS(run_gemm(m->g_U, nb, row0, m->ws, m->ws_floats, st, nl, &pv, P));
  const int K = kv->t->topk;
  int32_t *dst = kv->topk + (size_t)row0 * m->nmed * K;
  if (m->tp > 1) {  // vocabulary-parallel U: local top-K, then merge across ranks
    CK(topk_consumer_launch(pv, m->nmed, nb, m->V, K, m->tk_idx, m->v0, m->tk_val, st));
    CK(tp_merge_topk_launch(nb * m->nmed, K, m->tk_val, m->tk_idx, dst, m->nmed, nb, tp_next(m), st));
    nl += 2;
  } else {
    CK(topk_consumer_launch(pv, m->nmed, nb, m->V, K, dst, 0, nullptr, st));
    ++nl;
  }
  return SM_OK;
}

extern "C" sm_status sm_prefill(sm_model *m, sm_kv *kv, int seq, const int32_t *d_tokens, int n, void *stream) {
  NvtxRange nvtx_("sm_prefill");
  if (!m || !kv || seq < 0 || seq >= kv->b || (n > 0 && !d_tokens) || n < 0)
    return fail(SM_ERR_INVALID_ARG, "sm_prefill: bad arguments");
  if (n == 0) return SM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int32_t Lc = 0;  // stream-ordered read (no legacy-stream sync: TP peers may share the device)
  CK(cudaMemcpyAsync(&Lc, kv->len + seq, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (Lc + n > kv->x) return fail(SM_ERR_KV_CAPACITY, "Cache: prefill would exceed the KV bound x");
  int nl = 0;
  tp_begin(m);
  const TreeDev chain = m->chain->dev();
  const int R = m->R;
  // bf16, one GPU: causal chunks of up to max_rows tokens (the K1 kernels mask tree slot j for
  // node n by j <= n, no ancestor table); otherwise chain trees of <= 256 nodes (the fp32 K1
  // reads the ancestor table; the TP exchange flags are sized for 256-row chunks)
  const bool causal = !m->f32 && m->tp == 1;
  int done = 0, last = 0;
  while (done < n) {
    const int P = std::min(causal ? R : std::min(R, kMaxTreeNodes), n - done);
    TreeDev ct{};
    ct.N = P;
    ct.depth = m->iota;  // node n of the chunk sits at depth n: RoPE position Lc + n
    CKS(enqueue_forward(m, kv, d_tokens + done, 1, seq, P, causal ? ct : chain, st, nl));
    CK(advance_len_launch(kv->len, seq, P, kv->pad_mode ? kv->pos_len : nullptr, st));
    done += P;
    last = P;
  }
  // last token: LM head row, pending root, heads' top-k (reading Q8)
  PartialView pv;
  CKS(run_gemm(m->g_lm, 1, last - 1, m->ws, m->ws_floats, st, nl, &pv, m->P));
  CK(logits_consumer_launch(pv, 1.0f, m->z, m->argmax, m->stats, m->v0, m->amax, st));
  if (m->tp > 1)
    CK(tp_merge_logits_launch(1, m->amax, m->argmax, m->stats, m->z, m->V, m->v0, nullptr, 1, nullptr, nullptr,
                              tp_next(m), st));
  const int dP = m->d * m->P;  // a hidden row: d bf16, or its 3 planes (fp32 mode)
  CK(set_root_launch(kv->root, seq, m->argmax, m->hf + (size_t)(last - 1) * dP, dP, m->head_in + (size_t)seq * dP,
                     st));
  CKS(enqueue_heads(m, kv, seq, 1, st, nl));
  CKS(tp_end(m, st, nl));
  CK(cudaGetLastError());
  kv->last_stream = st;
  return SM_OK;
}

static sm_status enqueue_propose(sm_model *m, sm_kv *kv, int32_t *tree_tok, int32_t *pos, cudaStream_t st, int &nl) {
  CK(propose_launch(kv->t->dev(), kv->root, kv->topk, kv->t->topk, std::max(1, m->nmed), kv->b, tree_tok, pos,
                    kv->pad_mode ? kv->pos_len : kv->len, st));
  ++nl;
  return SM_OK;
}

static sm_status enqueue_verify(sm_model *m, sm_kv *kv, const int32_t *tree_tok, cudaStream_t st, int &nl) {
  const int M = kv->b * kv->N;
  CKS(enqueue_forward(m, kv, tree_tok, kv->b, 0, kv->N, kv->t->dev(), st, nl));
  PartialView pv;
  CKS(run_gemm(m->g_lm, M, 0, m->ws, m->ws_floats, st, nl, &pv, m->P));
  CK(logits_consumer_launch(pv, 1.0f, m->z, m->argmax, m->stats, m->v0, m->amax, st));
  ++nl;
  return SM_OK;
}

static sm_status enqueue_accept(sm_model *m, sm_kv *kv, const sm_accept_cfg *cfg, const sm_accept_out *o,
                                cudaStream_t st, int &nl) {
  const int M = kv->b * kv->N;
  float inv_temp = 1.0f;
  if (cfg->mode == SM_ACCEPT_TYPICAL) {
    inv_temp = 1.0f / cfg->temperature;
    // typical statistics at temperature T on the stored logits (one fp32 pass)
    CK(logits_finalize_launch(m->z, m->V, M, inv_temp, m->argmax, m->stats, m->v0, m->amax, st));
    ++nl;
  }
  const bool tp_cand = m->tp > 1 && cfg->mode == SM_ACCEPT_TYPICAL;
  if (m->tp > 1) {  // vocabulary-parallel LM head: merge (argmax, stats, candidate logits) across ranks
    CK(tp_merge_logits_launch(M, m->amax, m->argmax, m->stats, m->z, m->V, m->v0, kv->t->d_parent, kv->N,
                              kv->tree_tok, tp_cand ? m->cand : nullptr, tp_next(m), st));
    ++nl;
  }
  AcceptArgs a;
  std::memset(&a, 0, sizeof(a));
  a.t = kv->t->dev();
  a.b = kv->b;
  a.K = kv->t->topk;
  a.V = m->V;
  a.x_bound = kv->x;
  a.mode = cfg->mode == SM_ACCEPT_TYPICAL ? 1 : 0;
  a.inv_temp = inv_temp;
  a.eps = cfg->eps;
  a.alpha = cfg->alpha;
  a.tok = kv->tree_tok;
  a.argmax = m->argmax;
  a.stats = m->stats;
  a.z = m->z;
  a.cand = tp_cand ? m->cand : nullptr;
  a.len = kv->len;
  a.max_new = cfg->d_max_new;
  a.forced_path = cfg->d_forced_path;
  a.acc_len = o->acc_len;
  a.best_leaf = o->best_leaf;
  a.path = o->path;
  a.emit_tok = o->emit_tok;
  a.n_emit = o->n_emit;
  a.status = o->status;
  a.acc_row = kv->acc_row;
  a.root_next = kv->root_next;
  a.sticky = kv->d_sticky;
  CK(accept_launch(a, st));
  ++nl;
  CK(compact_launch(kv->base, m->L, kv->b, m->Hkv, kv->cap, m->hdu, kv->len, o->path, kv->t->l + 1, o->n_emit, st));
  ++nl;
  CK(commit_launch(kv->b, kv->pad_mode ? nullptr : kv->len, o->n_emit, kv->root, kv->root_next, kv->acc_row, m->hf,
                   m->d * m->P, m->head_in, kv->emitted, g_lib_capture, st));
  ++nl;
  if (kv->pad_mode) {  // every cache advances by the batch's longest acceptance; the rest are pads
    CK(pad_commit_launch(kv->b, kv->len, kv->pos_len, o->n_emit, kv->pad, kv->pad_words, st));
    ++nl;
  }
  CKS(enqueue_heads(m, kv, 0, kv->b, st, nl));
  return SM_OK;
}

static sm_status check_accept(const sm_accept_cfg *cfg, const sm_accept_out *o) {
  if (!cfg || !o || !o->acc_len || !o->best_leaf || !o->path || !o->emit_tok || !o->n_emit || !o->status)
    return fail(SM_ERR_INVALID_ARG, "accept: null cfg/out pointer");
  if (cfg->mode == SM_ACCEPT_TYPICAL && !(cfg->temperature > 0.f))
    return fail(SM_ERR_INVALID_ARG, "typical acceptance needs temperature > 0");
  return SM_OK;
}

// Device-detected conditions (accept kernel: status[b] = 3, a sequence reached the bound x) are
// latched in a mapped host word and returned, once, by the next sm_verify / sm_accept / sm_step
// whose host call runs after the detecting step completed (no synchronisation: a call enqueued
// while that step is still running reports it on a later call; sm_kv_status synchronises).
static sm_status kv_surface(sm_kv *kv) {
  // tensor parallel: every rank must issue the same calls, and ranks observe the word at different
  // times -- there only the synchronising sm_kv_status reports it
  if (kv->m->tp > 1) return SM_OK;
  volatile int32_t *w = (volatile int32_t *)kv->h_sticky;
  if (!w || *w == 0) return SM_OK;
  const int v = *w;
  *w = 0;
  if (v == 3)
    return fail(SM_ERR_KV_CAPACITY, "Cache: a sequence reached the KV bound x at an earlier step (status[b] = 3, "
                                    "nothing emitted for it); this call enqueued nothing");
  return fail(SM_ERR_CUDA, "device-detected status " + std::to_string(v));
}

extern "C" sm_status sm_kv_status(sm_kv *kv, int *h_status) {
  if (!kv || !h_status) return fail(SM_ERR_INVALID_ARG, "sm_kv_status: null");
  CK(cudaDeviceSynchronize());
  volatile int32_t *w = (volatile int32_t *)kv->h_sticky;
  *h_status = *w;
  *w = 0;
  return SM_OK;
}

extern "C" sm_status sm_propose(sm_model *m, sm_kv *kv, int32_t *d_tree_tok, int32_t *d_pos, void *stream) {
  NvtxRange nvtx_("sm_propose");
  if (!m || !kv || !d_tree_tok) return fail(SM_ERR_INVALID_ARG, "sm_propose: bad arguments");
  int nl = 0;
  CKS(enqueue_propose(m, kv, d_tree_tok, d_pos, (cudaStream_t)stream, nl));
  return SM_OK;
}

extern "C" sm_status sm_verify(sm_model *m, sm_kv *kv, const int32_t *d_tree_tok, float *d_logits, void *stream) {
  NvtxRange nvtx_("sm_verify");
  if (!m || !kv || !d_tree_tok) return fail(SM_ERR_INVALID_ARG, "sm_verify: bad arguments");
  CKS(kv_surface(kv));
  cudaStream_t st = (cudaStream_t)stream;
  int nl = 0;
  if (d_tree_tok != kv->tree_tok)
    CK(d2d_copy_launch(kv->tree_tok, d_tree_tok, (size_t)kv->b * kv->N * 4, st));
  tp_begin(m);
  CKS(enqueue_verify(m, kv, kv->tree_tok, st, nl));
  CKS(tp_end(m, st, nl));
  if (d_logits)
    CK(d2d_copy_launch(d_logits, m->z, (size_t)kv->b * kv->N * m->V * 4, st));
  kv->last_stream = st;
  return SM_OK;
}

extern "C" sm_status sm_accept(sm_model *m, sm_kv *kv, const sm_accept_cfg *cfg, const sm_accept_out *out,
                               void *stream) {
  NvtxRange nvtx_("sm_accept");
  if (!m || !kv) return fail(SM_ERR_INVALID_ARG, "sm_accept: bad arguments");
  CKS(check_accept(cfg, out));
  CKS(kv_surface(kv));
  int nl = 0;
  tp_begin(m);
  CKS(enqueue_accept(m, kv, cfg, out, (cudaStream_t)stream, nl));
  CKS(tp_end(m, (cudaStream_t)stream, nl));
  kv->last_stream = (cudaStream_t)stream;
  return SM_OK;
}

static sm_status enqueue_step(sm_model *m, sm_kv *kv, const sm_accept_cfg *cfg, const sm_accept_out *o,
                              cudaStream_t st, int &nl) {
  tp_begin(m);
  if (kv->pad_mode) {  // uniform cache lengths (after ragged prefills): pad the shorter ones
    CK(pad_align_launch(kv->b, kv->len, kv->pad, kv->pad_words, st));
    ++nl;
  }
  CKS(enqueue_propose(m, kv, kv->tree_tok, nullptr, st, nl));
  CKS(enqueue_verify(m, kv, kv->tree_tok, st, nl));
  CKS(enqueue_accept(m, kv, cfg, o, st, nl));
  CKS(tp_end(m, st, nl));
  return SM_OK;
}

extern "C" sm_status sm_step(sm_model *m, sm_kv *kv, const sm_accept_cfg *cfg, const sm_accept_out *out,
                             void *stream) {
  NvtxRange nvtx_("sm_step");
  if (!m || !kv) return fail(SM_ERR_INVALID_ARG, "sm_step: bad arguments");
  CKS(check_accept(cfg, out));
  CKS(kv_surface(kv));
  cudaStream_t st = (cudaStream_t)stream;
  GraphKey key{g_opt_version, kv->prof, (int)cfg->mode, cfg->temperature, cfg->eps, cfg->alpha, cfg->d_max_new, cfg->d_forced_path,
               out->acc_len, out->best_leaf, out->path, out->emit_tok, out->n_emit, out->status};
  auto it = kv->graphs.find(key);
  if (m->emu) {  // host-ordered emulation: the exchanges join the ranks' streams from their host threads
    int nl = 0;
    CKS(enqueue_step(m, kv, cfg, out, st, nl));
    kv->last_stream = st;
    return SM_OK;
  }
  if (it == kv->graphs.end()) {
    cudaStreamCaptureStatus cs;
    CK(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) {  // caller is capturing: enqueue directly
      int nl = 0;
      CKS(enqueue_step(m, kv, cfg, out, st, nl));
      return SM_OK;
    }
    cudaGraph_t g;
    int nl = 0;
    if (kv->prof) {
      for (auto &pe : kv->prof_events) {
        cudaEventDestroy(pe.a);
        cudaEventDestroy(pe.b);
      }
      kv->prof_events.clear();
      g_prof = &kv->prof_events;
    }
    CK(cudaStreamBeginCapture(m->cap_stream, cudaStreamCaptureModeRelaxed));
    cudaEvent_t ev_step = nullptr;
    prof_begin(m->cap_stream, &ev_step);  // kind 3: the whole (event-serialised) step
    g_lib_capture = true;
    sm_status s = enqueue_step(m, kv, cfg, out, m->cap_stream, nl);
    g_lib_capture = false;
    prof_end(m->cap_stream, ev_step, 3, 0.0);
    cudaError_t e = cudaStreamEndCapture(m->cap_stream, &g);
    g_prof = nullptr;
    if (s != SM_OK) return s;
    if (e != cudaSuccess) return fail(SM_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t ex;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(SM_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    it = kv->graphs.emplace(key, ex).first;
    if (!kv->prof) kv->step_launches = nl;
  }
  CK(cudaGraphLaunch(it->second, st));
  kv->last_stream = st;
  return SM_OK;
}

extern "C" sm_status sm_step_profile(sm_kv *kv, int enable) {
  if (!kv) return fail(SM_ERR_INVALID_ARG, "null");
  kv->prof = enable ? 1 : 0;
  return SM_OK;
}

extern "C" sm_status sm_profile_read(const sm_kv *kv, int kind, int *count, float *total_ms, double *alg_bytes) {
  if (!kv) return fail(SM_ERR_INVALID_ARG, "null");
  CK(cudaDeviceSynchronize());
  int n = 0;
  float tot = 0.f;
  double by = 0.0;
  for (const auto &pe : kv->prof_events) {
    if (pe.kind != kind) continue;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, pe.a, pe.b));
    tot += ms;
    by += pe.bytes;
    ++n;
  }
  if (count) *count = n;
  if (total_ms) *total_ms = tot;
  if (alg_bytes) *alg_bytes = by;
  return SM_OK;
}

extern "C" sm_status sm_step_launches(const sm_kv *kv, int *n) {
  if (!kv || !n) return fail(SM_ERR_INVALID_ARG, "null");
  *n = kv->step_launches;
  return SM_OK;
}

// ---------------------------------------------------------------- stage APIs (parity tests, K1 sweep)
// Stage entries (sm_gemm_bf16) keep their stream-K partial sums in scratch owned per stream, so
// calls on different streams never share it.  Growing it frees the old buffer after a device sync,
// which stream capture forbids: under capture the scratch must already be large enough (a first
// uncaptured call of the same size on that stream sizes it), else SM_ERR_UNSUPPORTED.
static std::map<cudaStream_t, std::pair<void *, size_t>> g_scratch;
static sm_status scratch(size_t bytes, cudaStream_t st, void **p) {
  auto &e = g_scratch[st];
  if (bytes > e.second) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(SM_ERR_UNSUPPORTED, "stage scratch must grow during stream capture: call once uncaptured first");
    CK(cudaDeviceSynchronize());  // earlier work on any stream may still read the old buffer
    cudaFree(e.first);
    e = {nullptr, 0};
    if (cudaMalloc(&e.first, bytes) != cudaSuccess) return fail(SM_ERR_DEVICE_OOM, "Buffer: stage scratch");
    e.second = bytes;
  }
  *p = e.first;
  return SM_OK;
}

// The stage K1's lean workspace: [256 B: barrier counters, zero between launches][partial slots],
// per stream (a growth re-zeroes the counters; same capture rule as scratch()).
static std::map<cudaStream_t, std::pair<void *, size_t>> g_lean_scratch;
static sm_status lean_scratch(size_t bytes, cudaStream_t st, void **p) {
  auto &e = g_lean_scratch[st];
  if (bytes + 256 > e.second) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(SM_ERR_UNSUPPORTED, "stage scratch must grow during stream capture: call once uncaptured first");
    CK(cudaDeviceSynchronize());
    cudaFree(e.first);
    e = {nullptr, 0};
    if (cudaMalloc(&e.first, bytes + 256) != cudaSuccess) return fail(SM_ERR_DEVICE_OOM, "Buffer: K1 stage scratch");
    CK(cudaMemset(e.first, 0, 256));
    e.second = bytes + 256;
  }
  *p = e.first;
  return SM_OK;
}

static sm_status attention_stage(const uint64_t *d_anc, int Nq, const void *d_q, const void *d_k, const void *d_v,
                                 const int32_t *d_len, int batch, int n_heads, int n_kv_heads, int head_dim, int cap,
                                 void *d_out, void *stream) {
  if (head_dim != 16 && head_dim != 32 && head_dim != 64 && head_dim != 128)
    return fail(SM_ERR_INVALID_ARG, "head_dim must be 16/32/64/128");
  const int G = n_heads / n_kv_heads;
  const int nsplit = attention_nsplit(batch * n_kv_heads * attention_row_blocks(Nq, G, head_dim), head_dim, cap);
  AttnArgs aa;
  std::memset(&aa, 0, sizeof(aa));
  const uint64_t rows = (uint64_t)batch * n_kv_heads * cap;
  CKS(kv_map(&aa.tmK, d_k, rows, head_dim));
  CKS(kv_map(&aa.tmV, d_v, rows, head_dim));
  aa.q = (const bf16 *)d_q;
  aa.out = (bf16 *)d_out;
  aa.len = d_len;
  aa.anc = d_anc;
  aa.causal = d_anc == nullptr;
  aa.k_row0 = 0;
  aa.v_row0 = 0;
  aa.k_base = (const bf16 *)d_k;
  aa.v_base = (const bf16 *)d_v;
  aa.seq_rows = (long long)n_kv_heads * cap;
  aa.cap = cap;
  aa.Nq = Nq;
  aa.H = n_heads;
  aa.Hkv = n_kv_heads;
  aa.G = G;
  aa.nseq = batch;
  aa.seq_base = 0;
  aa.nsplit = nsplit;
  aa.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)head_dim));
  if (head_dim == 128 && d_anc) {  // stream-K K1: per-stream partial slots + zeroed barrier counters
    const int units = batch * n_kv_heads * attention_row_blocks(Nq, G, head_dim);
    void *p = nullptr;
    CKS(lean_scratch(attention_lean_part_floats(units) * 4, (cudaStream_t)stream, &p));
    aa.lean_sync = reinterpret_cast<int *>(p);
    aa.lean_part = reinterpret_cast<float *>(reinterpret_cast<char *>(p) + 256);
    aa.lean_min_tiles = attention_lean_min_tiles(Nq, G);
  }
  CK(attention_launch(aa, head_dim, (cudaStream_t)stream));
  return SM_OK;
}

extern "C" sm_status sm_tree_attention(const sm_tree *t, const void *d_q, const void *d_k, const void *d_v,
                                       const int32_t *d_len, int batch, int n_heads, int n_kv_heads, int head_dim,
                                       int cap, void *d_out, void *stream) {
  if (!t || !d_q || !d_k || !d_v || !d_len || !d_out || batch < 1 || n_kv_heads < 1 || n_heads % n_kv_heads ||
      cap < t->N)
    return fail(SM_ERR_INVALID_ARG, "sm_tree_attention: bad arguments");
  sm_tree *tt = const_cast<sm_tree *>(t);
  CKS(tree_upload(tt));
  return attention_stage(tt->d_anc, t->N, d_q, d_k, d_v, d_len, batch, n_heads, n_kv_heads, head_dim, cap, d_out,
                         stream);
}

extern "C" sm_status sm_causal_attention(int n, const void *d_q, const void *d_k, const void *d_v,
                                         const int32_t *d_len, int batch, int n_heads, int n_kv_heads, int head_dim,
                                         int cap, void *d_out, void *stream) {
  if (n < 1 || n > 1024 || !d_q || !d_k || !d_v || !d_len || !d_out || batch < 1 || n_kv_heads < 1 ||
      n_heads % n_kv_heads || cap < n)
    return fail(SM_ERR_INVALID_ARG, "sm_causal_attention: bad arguments (1 <= n <= 1024)");
  return attention_stage(nullptr, n, d_q, d_k, d_v, d_len, batch, n_heads, n_kv_heads, head_dim, cap, d_out, stream);
}

extern "C" sm_status sm_gemm_bf16(const void *d_x, const void *d_w, float *d_out, int M, int N, int K,
                                  void *stream) {
  if (!d_x || !d_w || M < 1 || M > 1024 || N < 1 || K < 8 || K % 8)
    return fail(SM_ERR_INVALID_ARG, "sm_gemm_bf16: bad arguments (M <= 1024, K % 8 == 0)");
  GemmArgs a = gemm_proto(N, K, 1);
  CKS(weight_map(&a.tmW[0], d_w, N, K));
  CKS(act_map(a, 0, d_x, M, K));
  const size_t need = ws_need(a, M);
  void *scr = nullptr;
  CKS(scratch(need * 4, (cudaStream_t)stream, &scr));
  int nl = 0;
  PartialView pv;
  if (g_epi_test && !d_out) {  // experiments: the fused SiLU tile epilogue on scratch buffers
    static float *rs1 = nullptr;
    static bf16 *act = nullptr;
    static int *cnt = nullptr;
    static size_t act_n = 0;
    if (!rs1) {
      CKS(dalloc(&rs1, 1024, "epi test"));
      CKS(dalloc(&cnt, kMaxFusedTiles + 1, "epi test"));
      cudaMemset(cnt, 0, (kMaxFusedTiles + 1) * sizeof(int));
      std::vector<float> ones(1024, 1.0f);
      cudaMemcpy(rs1, ones.data(), 4096, cudaMemcpyHostToDevice);
    }
    if ((size_t)M * N / 2 > act_n) {
      cudaFree(act);
      act_n = (size_t)M * N / 2;
      CKS(dalloc(&act, act_n, "epi test"));
    }
    EpiArgs ea;
    std::memset(&ea, 0, sizeof(ea));
    ea.rs_in = rs1;
    ea.act = act;
    ea.F = N / 2;
    ea.tile_cnt = cnt;
    ea.done_cnt = cnt + kMaxFusedTiles;
    CKS(run_gemm(a, M, 0, (float *)scr, need, (cudaStream_t)stream, nl, &pv, 1, kEpiSiLU, &ea));
    return SM_OK;
  }
  CKS(run_gemm(a, M, 0, (float *)scr, need, (cudaStream_t)stream, nl, &pv));
  if (d_out) CK(plain_consumer_launch(pv, d_out, (cudaStream_t)stream));  // NULL: GEMM only (timing)
  return SM_OK;
}

extern "C" sm_status sm_topk_f32(const float *d_logits, int rows, int V, int k, int32_t *d_idx, void *stream) {
  if (!d_logits || !d_idx || rows < 1 || V < k || k < 1 || V * 4 > 200 * 1024 || V % 4)
    return fail(SM_ERR_INVALID_ARG, "sm_topk_f32: bad arguments (V % 4 == 0)");
  CK(topk_launch(d_logits, rows, V, k, d_idx, (cudaStream_t)stream));
  return SM_OK;
}

extern "C" sm_status sm_reset_options(void) {
  gemm_set_pdl(true);
  gemm_set_ctas(0);
  gemm_set_rep(1);
  gemm_set_l2_prefetch(0);
  gemm_set_bn(0);
  gemm_set_small(2);
  gemm_set_debug_mode(0);
  gemm_set_occ_smalln(0);
  gemm_set_pair(1);
  gemm_set_pre_stages(-2);
  consumer_set_threads(256);
  attention_set_tc(1);
  attention_set_l2pf(0);
  attention_set_splits(0);
  attention_set_lean(0);
  attention_set_ks(2);
  attention_set_l2ahead(2);
  attention_set_ksp(1);
  attention_set_split_model(1);
  attention_set_w2(1);
  attention_set_qearly(1);
  consumer_set_rpc(2);
  consumer_set_nm(4);
  resid_set_nm(8);
  attention_set_lean_div(16);
  tp_set_rsag(-1);
  g_fused = 0;
  g_epi_test = 0;
  g_ablate = 0;
  ++g_opt_version;
  return SM_OK;
}

extern "C" sm_status sm_set_option(const char *name, int value) {
  if (!name) return fail(SM_ERR_INVALID_ARG, "sm_set_option: null name");
  const std::string n(name);
  ++g_opt_version;
  if (n == "pdl") {
    gemm_set_pdl(value != 0);
  } else if (n == "gemm_ctas") {
    gemm_set_ctas(value);
  } else if (n == "gemm_rep") {  // token-tile CTA groups for M > one token tile (default 1)
    gemm_set_rep(value);
  } else if (n == "l2_prefetch") {
    gemm_set_l2_prefetch(value);
  } else if (n == "gemm_bn") {
    if (value != 0 && value != 16 && value != 32 && value != 64 && value != 80 && value != 96 && value != 128 &&
        value != 160 && value != 192 && value != 256)
      return fail(SM_ERR_INVALID_ARG, "gemm_bn must be 0 or one of 16 32 64 80 96 128 160 192 256");
    gemm_set_bn(value);
  } else if (n == "gemm_occ") {
    gemm_set_small(value);
  } else if (n == "gemm_mode") {
    gemm_set_debug_mode(value);
  } else if (n == "fused_epilogue") {  // takes effect for models created afterwards
    g_fused = value & 7;
  } else if (n == "gemm_occ_smalln") {
    gemm_set_occ_smalln(value);
  } else if (n == "gemm_pair") {
    gemm_set_pair(value);
  } else if (n == "gemm_pre") {
    gemm_set_pre_stages(value);
  } else if (n == "consumer_threads") {
    consumer_set_threads(value);
  } else if (n == "epi_test") {
    g_epi_test = value;
  } else if (n == "ablate") {
    g_ablate = value;
  } else if (n == "attn_tc") {
    attention_set_tc(value);
  } else if (n == "attn_l2pf") {
    attention_set_l2pf(value);
  } else if (n == "attn_splits") {
    attention_set_splits(value);
  } else if (n == "tp_rsag") {  // TP residual exchange: -1 auto (t >= 4 RS+AG), 0 one-shot, 1 RS+AG
    tp_set_rsag(value);
  } else if (n == "attn_lean") {  // tree-mode K1 (hd 128): stream-K kernel (1, default) or cluster splits (0)
    attention_set_lean(value);
  } else if (n == "attn_l2ahead") {  // K1 row-copy kernel: L2 prefetch ahead of the ring (bit 0 own range, bit 1 next wave)
    attention_set_l2ahead(value);
  } else if (n == "resid_nm") {  // one-row residual consumer: contributors loaded up front (16 or 8)
    resid_set_nm(value);
  } else if (n == "consumer_nm") {  // one-row QKV / SiLU consumers: contributors loaded up front (8 or 4)
    consumer_set_nm(value);
  } else if (n == "consumer_rpc") {  // token rows per CTA of the QKV / SiLU consumers for M >= 256 (experiments)
    consumer_set_rpc(value);
  } else if (n == "attn_qearly") {  // K1 row-copy kernel: Q loads before the CTA barrier (1) or after (0)
    attention_set_qearly(value);
  } else if (n == "attn_w2") {  // K1 row-copy kernel, 128 live rows: two softmax warps per row (1) or one (0)
    attention_set_w2(value);
  } else if (n == "attn_split_model") {  // K1 key splits: 1 occupancy-aware cost model (default), 0 round-1 rule
    attention_set_split_model(value);
  } else if (n == "attn_ksp") {  // K1: persistent row-copy kernel for one-split launches with > 148 units
    attention_set_ksp(value);
  } else if (n == "attn_ks") {  // K1 128-key-tile (row-copy) kernel on long key ranges: 0 off, 1 N G <= 64, 2 all (default)
    attention_set_ks(value);
  } else if (n == "attn_lean_div") {  // lean K1: minimum tiles per CTA = max(2, live rows / value)
    attention_set_lean_div(value);
  } else {
    return fail(SM_ERR_INVALID_ARG, "sm_set_option: unknown option " + n);
  }
  return SM_OK;
}

extern "C" const char *sm_last_error(void) { return g_err.c_str(); }
extern "C" const char *sm_version(void) {
  return "specmemo-b200 0.2 (sm_100a: tcgen05 GEMM and tree attention; bf16 and fp32 parity modes)";
}
