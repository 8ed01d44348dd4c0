// mlk_build_tree: level-synchronous median-split tree on the device (Algorithm 1 with
// ChooseRule RP / kD).  Per level: one projection kernel (x.v summed left to
// right without FMA, reading R6), one segmented sort of (segment, projection, original id)
// by a bitonic network (shared-memory tiles + global merge steps), one split kernel that
// writes the permutation and the median thresholds (reading R2).
#include <algorithm>
#include <climits>
#include <memory>
#include <cmath>

#include "api.cuh"

namespace mlk {
namespace {

struct SortKey {
  double p;    // projection (or the position, for frozen segments)
  int32_t s;   // segment ordinal (left to right)
  int32_t id;  // original point index
};

__device__ __forceinline__ bool key_less(const SortKey& a, const SortKey& b) {
  if (a.s != b.s) return a.s < b.s;
  if (a.p < b.p) return true;
  if (b.p < a.p) return false;
  return a.id < b.id;
}

constexpr int TILE = 2048;  // elements per shared-memory bitonic tile (1024 threads)

// Projection keys for every tree position k; pads to Npad with +inf segments.
__global__ void k_tree_keys(const double* __restrict__ X, int d, int64_t n, int64_t npad,
                            const int32_t* __restrict__ perm, const int64_t* __restrict__ seg_begin,
                            const int32_t* __restrict__ seg_node, const int8_t* __restrict__ seg_active,
                            int n_seg, const double* __restrict__ dirs, SortKey* __restrict__ keys) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= npad) return;
  SortKey out;
  if (k >= n) {
    out.p = 0.0;
    out.s = INT_MAX;
    out.id = INT_MAX;
    keys[k] = out;
    return;
  }
  // segment containing k: last seg_begin <= k
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (seg_begin[mid] <= k) lo = mid; else hi = mid - 1;
  }
  int32_t id = perm[k];
  out.s = lo;
  out.id = id;
  if (seg_active[lo]) {
    const double* x = X + (int64_t)id * d;
    const double* v = dirs + (int64_t)seg_node[lo] * d;
    double acc = __dmul_rn(x[0], v[0]);
    for (int j = 1; j < d; j++) acc = __dadd_rn(acc, __dmul_rn(x[j], v[j]));
    out.p = acc;
  } else {
    out.p = (double)k;  // frozen leaf: keep positional order
  }
  keys[k] = out;
}

__device__ __forceinline__ void cas(SortKey* a, int i, int l, bool asc) {
  SortKey x = a[i], y = a[l];
  bool sw = asc ? key_less(y, x) : key_less(x, y);
  if (sw) {
    a[i] = y;
    a[l] = x;
  }
}

// Bitonic network that sorts every aligned block of kfinal elements independently (kfinal =
// the whole padded array at the root; smaller below, where no segment straddles a block):
// merge stages k < kfinal alternate direction as usual, stage kfinal is ascending everywhere.
__device__ __forceinline__ bool bitonic_asc(int64_t i, int64_t k, int64_t kfinal) {
  return k == kfinal || (i & k) == 0;
}

// Bitonic steps inside one tile of `tile` elements: if full, stages k = 2..min(tile, kfinal);
// otherwise stage k (global) strides j0..1.
__global__ void k_bitonic_smem(SortKey* __restrict__ keys, int tile, int64_t k_stage, int j0, int full,
                               int64_t kfinal) {
  __shared__ SortKey sh[TILE];
  int64_t base = (int64_t)blockIdx.x * tile;
  for (int i = threadIdx.x; i < tile; i += blockDim.x) sh[i] = keys[base + i];
  __syncthreads();
  int half = tile >> 1;
  if (full) {
    const int kmax = (int)std::min<int64_t>(tile, kfinal);
    for (int k = 2; k <= kmax; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < half; t += blockDim.x) {
          int i = 2 * j * (t / j) + (t % j);
          cas(sh, i, i + j, bitonic_asc(base + i, k, kfinal));
        }
        __syncthreads();
      }
    }
  } else {
    for (int j = j0; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < half; t += blockDim.x) {
        int i = 2 * j * (t / j) + (t % j);
        cas(sh, i, i + j, bitonic_asc(base + i, k_stage, kfinal));
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < tile; i += blockDim.x) keys[base + i] = sh[i];
}

__global__ void k_bitonic_global(SortKey* __restrict__ keys, int64_t npad, int64_t k_stage, int64_t j,
                                 int64_t kfinal) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= npad / 2) return;
  int64_t i = 2 * j * (t / j) + (t % j);
  int64_t l = i + j;
  bool asc = bitonic_asc(i, k_stage, kfinal);
  SortKey x = keys[i], y = keys[l];
  bool sw = asc ? key_less(y, x) : key_less(x, y);
  if (sw) {
    keys[i] = y;
    keys[l] = x;
  }
}

__global__ void k_tree_perm(const SortKey* __restrict__ keys, int64_t n, int32_t* __restrict__ perm) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) perm[k] = keys[k].id;
}

// median threshold of every active node (reading R2)
__global__ void k_tree_thr(const SortKey* __restrict__ keys, const int64_t* __restrict__ nb,
                           const int64_t* __restrict__ ne, const int32_t* __restrict__ nodes, int cnt,
                           double* __restrict__ thr) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  int64_t b = nb[i], s = ne[i] - nb[i];
  int64_t h = (s + 1) / 2;
  double lo = keys[b + h - 1].p;
  double v = (s & 1) ? lo : __dmul_rn(__dadd_rn(lo, keys[b + h].p), 0.5);
  thr[nodes[i]] = v;
}

// Duplicate sites: after the root sort, equal projections form runs; compare coordinates
// of every pair inside a run (identical sites always share a run at the root).
__global__ void k_dup_runs(const SortKey* __restrict__ keys, int64_t n, const double* __restrict__ X, int d,
                           int* __restrict__ flag) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k == 0 || k >= n) return;
  if (!(keys[k].p == keys[k - 1].p)) return;
  const double* xk = X + (int64_t)keys[k].id * d;
  for (int64_t j = k - 1; j >= 0 && keys[j].p == keys[k].p; j--) {
    const double* xj = X + (int64_t)keys[j].id * d;
    bool same = true;
    for (int c = 0; c < d; c++) same = same && (xj[c] == xk[c]);
    if (same) atomicExch(flag, 1);
  }
}

__global__ void k_dup_pairwise(const double* __restrict__ X, int64_t n, int d, int* __restrict__ flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t j = i + 1; j < n; j++) {
    bool same = true;
    for (int c = 0; c < d; c++) same = same && (X[i * d + c] == X[j * d + c]);
    if (same) atomicExch(flag, 1);
  }
}

// tree-ordered, zero-padded coordinates and squared norms for the Gram identity
__global__ void k_tree_gather(const double* __restrict__ X, int d, int dp, int64_t n,
                              const int32_t* __restrict__ perm, double* __restrict__ Xt,
                              double* __restrict__ norm2) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double* x = X + (int64_t)perm[k] * d;
  double s = 0.0;
  for (int j = 0; j < dp; j++) {
    double v = j < d ? x[j] : 0.0;
    Xt[k * dp + j] = v;
    s = fma(v, v, s);
  }
  norm2[k] = s;
}

// Sort keys by (segment, projection, id) within aligned blocks of kfinal elements; every
// segment lies inside one block, so this equals the full sort of the array.
void bitonic_sort(Ctx& c, SortKey* keys, int64_t npad, int64_t kfinal) {
  TimedLaunch tl(c, "tree_sort");
  int tile = (int)std::min<int64_t>(TILE, npad);
  int threads = std::min(1024, std::max(1, tile / 2));
  k_bitonic_smem<<<(unsigned)(npad / tile), threads, 0, c.stream>>>(keys, tile, 0, 0, 1, kfinal);
  check_launch("k_bitonic_smem");
  for (int64_t k = 2 * (int64_t)tile; k <= kfinal; k <<= 1) {
    for (int64_t j = k >> 1; j >= tile; j >>= 1) {
      int64_t pairs = npad / 2;
      k_bitonic_global<<<(unsigned)ceil_div(pairs, 256), 256, 0, c.stream>>>(keys, npad, k, j, kfinal);
      check_launch("k_bitonic_global");
    }
    k_bitonic_smem<<<(unsigned)(npad / tile), threads, 0, c.stream>>>(keys, tile, k, tile / 2, 0, kfinal);
    check_launch("k_bitonic_smem");
  }
}

}  // namespace
}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_build_tree(mlk_ctx ctx, const double* X, int64_t n, int32_t d, int32_t leaf_size,
                          int32_t kind, const double* directions, int64_t n_dir_rows,
                          mlk_tree* out) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && out, "NULL ctx/out");
  *out = nullptr;
  MLK_REQUIRE(X != nullptr, "X is NULL");
  MLK_REQUIRE(n >= 1 && n < (int64_t)INT_MAX, "need 1 <= n < 2^31");
  MLK_REQUIRE(d >= 1 && d <= 4096, "need 1 <= d <= 4096");
  MLK_REQUIRE(leaf_size >= 1, "need leaf_size >= 1");
  MLK_REQUIRE(kind == MLK_TREE_KD || kind == MLK_TREE_RP, "unknown tree kind");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));

  // ---- shape (depends on n and leaf_size only)
  int t = 0;
  for (int64_t s = n; s > leaf_size; s = (s + 1) / 2) t++;
  MLK_REQUIRE(t <= 24, "tree deeper than 24 levels");
  if (kind == MLK_TREE_RP)
    MLK_REQUIRE(directions != nullptr && n_dir_rows >= ((int64_t)1 << t) - 1,
                "RP tree needs 2^t - 1 direction rows");
  auto tr = std::make_unique<mlk_tree_s>();
  tr->device = c.device;
  tr->n = n;
  tr->d = d;
  tr->d_pad = pad4(d);
  tr->leaf = leaf_size;
  tr->kind = kind;
  tr->t = t;
  int nn = (int)((1LL << (t + 1)) - 1);
  tr->n_nodes = nn;
  tr->state.assign(nn, -1);
  tr->begin.assign(nn, 0);
  tr->end.assign(nn, 0);
  tr->depth.assign(nn, 0);
  tr->thr.assign(nn, NAN);
  tr->dir.assign((size_t)nn * d, 0.0);
  tr->state[0] = 0;
  tr->end[0] = n;
  for (int q = 0; q < nn; q++) {
    if (tr->state[q] < 0) continue;
    int dep = 0;
    while (((int64_t)2 << dep) - 1 <= q) dep++;
    tr->depth[q] = dep;
    int64_t s = tr->end[q] - tr->begin[q];
    if (s <= leaf_size) {
      tr->state[q] = 1;
      continue;
    }
    tr->state[q] = 0;
    int64_t h = (s + 1) / 2;
    int l = 2 * q + 1, r = 2 * q + 2;
    tr->state[l] = tr->state[r] = 0;
    tr->begin[l] = tr->begin[q];
    tr->end[l] = tr->begin[q] + h;
    tr->begin[r] = tr->begin[q] + h;
    tr->end[r] = tr->end[q];
  }

  // ---- inputs on the device
  cudaStream_t st = c.stream;
  tr->X.alloc((size_t)n * d, st);
  if (is_device_ptr(X))
    CUDA_CHECK(cudaMemcpyAsync(tr->X.p, X, sizeof(double) * n * d, cudaMemcpyDeviceToDevice, st));
  else
    tr->X.upload(X, (size_t)n * d);
  if (kind == MLK_TREE_RP) {
    std::vector<double> dh((size_t)(((int64_t)1 << t) - 1) * d);
    if (!dh.empty()) {
      if (is_device_ptr(directions)) {
        CUDA_CHECK(cudaMemcpyAsync(dh.data(), directions, sizeof(double) * dh.size(), cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
      } else {
        std::copy(directions, directions + dh.size(), dh.begin());
      }
    }
    for (int q = 0; q < nn; q++)
      if (tr->state[q] == 0)
        for (int j = 0; j < d; j++) tr->dir[(size_t)q * d + j] = dh[(size_t)q * d + j];
  } else {
    for (int q = 0; q < nn; q++)
      if (tr->state[q] == 0) tr->dir[(size_t)q * d + (tr->depth[q] % d)] = 1.0;
  }
  tr->dir_d.alloc((size_t)nn * d, st);
  tr->dir_d.upload(tr->dir);
  tr->perm_d.alloc(n, st);
  {
    std::vector<int32_t> id(n);
    for (int64_t k = 0; k < n; k++) id[k] = (int32_t)k;
    tr->perm_d.upload(id);
  }
  tr->thr_d.alloc(nn, st);
  {
    std::vector<double> nanv(nn, NAN);
    tr->thr_d.upload(nanv);
  }
  DevBuf<int> flag(1, st);
  flag.zero();

  int64_t npad = 2;
  while (npad < n) npad <<= 1;
  DevBuf<SortKey> keys(npad, st);
  DevBuf<int64_t> seg_begin_d(1, st), nb_d(1, st), ne_d(1, st);
  DevBuf<int32_t> seg_node_d(1, st), nodes_d(1, st);
  DevBuf<int8_t> seg_active_d(1, st);

  HostTrace trace("tree");
  for (int dep = 0; dep < t; dep++) {
    // segments at this depth: nodes at depth dep and leaves above, left to right
    std::vector<std::pair<int64_t, int>> segs;
    for (int q = 0; q < nn; q++) {
      if (tr->state[q] < 0) continue;
      if (tr->depth[q] == dep || (tr->depth[q] < dep && tr->state[q] == 1)) segs.push_back({tr->begin[q], q});
    }
    std::sort(segs.begin(), segs.end());
    std::vector<int64_t> sb;
    std::vector<int32_t> sn, anodes;
    std::vector<int8_t> sa;
    std::vector<int64_t> ab, ae;
    for (auto& s : segs) {
      if (tr->end[s.second] == tr->begin[s.second]) continue;
      bool active = tr->depth[s.second] == dep && tr->state[s.second] == 0;
      sb.push_back(s.first);
      sn.push_back(s.second);
      sa.push_back(active ? 1 : 0);
      if (active) {
        anodes.push_back(s.second);
        ab.push_back(tr->begin[s.second]);
        ae.push_back(tr->end[s.second]);
      }
    }
    if (anodes.empty()) continue;
    seg_begin_d.upload(sb);
    seg_node_d.upload(sn);
    seg_active_d.upload(sa);
    nodes_d.upload(anodes);
    nb_d.upload(ab);
    ne_d.upload(ae);
    {
      TimedLaunch tl(c, "tree_project");
      k_tree_keys<<<(unsigned)ceil_div(npad, 256), 256, 0, st>>>(tr->X.p, d, n, npad, tr->perm_d.p, seg_begin_d.p,
                                                                seg_node_d.p, seg_active_d.p, (int)sb.size(),
                                                                tr->dir_d.p, keys.p);
      check_launch("k_tree_keys");
    }
    // smallest power-of-two block that no segment straddles (positions past n sort last)
    int64_t kfinal = 2;
    for (;;) {
      bool ok = kfinal >= npad;
      if (!ok) {
        ok = true;
        for (size_t i = 0; i < sb.size() && ok; i++) {
          const int64_t e = (i + 1 < sb.size() ? sb[i + 1] : n) - 1;
          ok = sb[i] / kfinal == e / kfinal;
        }
      }
      if (ok) break;
      kfinal <<= 1;
    }
    bitonic_sort(c, keys.p, npad, std::min(kfinal, npad));
    {
      TimedLaunch tl(c, "tree_split");
      k_tree_perm<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(keys.p, n, tr->perm_d.p);
      check_launch("k_tree_perm");
      k_tree_thr<<<(unsigned)ceil_div(anodes.size(), 128), 128, 0, st>>>(keys.p, nb_d.p, ne_d.p, nodes_d.p,
                                                                           (int)anodes.size(), tr->thr_d.p);
      check_launch("k_tree_thr");
      if (dep == 0) {
        k_dup_runs<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(keys.p, n, tr->X.p, d, flag.p);
        check_launch("k_dup_runs");
      }
    }
  }
  if (t == 0) {
    k_dup_pairwise<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(tr->X.p, n, d, flag.p);
    check_launch("k_dup_pairwise");
  }
  trace.mark("levels");
  auto fl = flag.download(1);
  trace.mark("sync");
  if (fl[0]) throw Error(MLK_ERR_DUPLICATE_POINTS, "duplicate observation sites");

  tr->Xt.alloc((size_t)n * tr->d_pad, st);
  tr->norm2.alloc(n, st);
  {
    TimedLaunch tl(c, "tree_gather");
    k_tree_gather<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(tr->X.p, d, tr->d_pad, n, tr->perm_d.p, tr->Xt.p,
                                                              tr->norm2.p);
    check_launch("k_tree_gather");
  }
  auto ph = tr->perm_d.download(n);
  tr->perm.assign(ph.begin(), ph.end());
  tr->thr = tr->thr_d.download(nn);
  keys.release();
  *out = tr.release();
  MLK_API_END
}

void mlk_tree_free(mlk_tree tree) {
  if (!tree) return;
  cudaSetDevice(tree->device);
  // the creating context's stream may already be gone: drain the device, free on stream 0
  cudaDeviceSynchronize();
  tree->perm_d.s = nullptr;
  tree->X.s = nullptr;
  tree->Xt.s = nullptr;
  tree->norm2.s = nullptr;
  tree->thr_d.s = nullptr;
  tree->dir_d.s = nullptr;
  delete tree;
}

mlk_status mlk_tree_info(mlk_tree tree, int32_t* t, int32_t* n_nodes, int64_t* n, int32_t* d) {
  MLK_API_BEGIN
  MLK_REQUIRE(tree, "tree is NULL");
  if (t) *t = tree->t;
  if (n_nodes) *n_nodes = tree->n_nodes;
  if (n) *n = tree->n;
  if (d) *d = tree->d;
  MLK_API_END
}

mlk_status mlk_tree_export(mlk_tree tree, int64_t* perm, int64_t* begin, int64_t* end, int32_t* depth,
                           int32_t* state, double* thr, double* dir) {
  MLK_API_BEGIN
  MLK_REQUIRE(tree, "tree is NULL");
  int nn = tree->n_nodes;
  if (perm) std::copy(tree->perm.begin(), tree->perm.end(), perm);
  if (begin) std::copy(tree->begin.begin(), tree->begin.end(), begin);
  if (end) std::copy(tree->end.begin(), tree->end.end(), end);
  if (depth) std::copy(tree->depth.begin(), tree->depth.end(), depth);
  if (state)
    for (int q = 0; q < nn; q++) state[q] = tree->state[q];
  if (thr) std::copy(tree->thr.begin(), tree->thr.end(), thr);
  if (dir) std::copy(tree->dir.begin(), tree->dir.end(), dir);
  MLK_API_END
}

}  // extern "C"
