// mlk_assemble_cw: admission (Algorithms 3-6 on the device), BSR structure, cost model and
// LPT partition (host), then the two contractions per admitted pair:
//   K5a (tile.cu)   U = C(X_a, X_b) W_b^T   fused tiles on FP64 DMMA
//   K5b (gemm.cu)   B = W_a U               batched FP64 DMMA GEMM, written into the BSR
// where b is the side contracted first (the cheaper order).
#include <algorithm>
#include <array>
#include <cmath>
#include <memory>
#include <set>

#include "api.cuh"
#include "tile.cuh"

namespace mlk {
void assemble_dd(Ctx& c, const mlk_tree_s* tree, const mlk_basis_s* B, const mlk_kernel& k,
                 const std::vector<std::array<int64_t, 8>>& jobs, double* values_base);
namespace {

struct SearchItem {
  int32_t a;      // searching cell (heap node)
  int32_t q;      // current node
  uint32_t mask;  // target depths still searched through q
};

// One CTA per item: emit (a, q) if depth(q) is a target, then min/max of the projections of
// a's points onto v_q and the symmetric rule of reading R12 for every remaining target depth.
__global__ void k_search_level(const SearchItem* __restrict__ cur, int n_cur, SearchItem* __restrict__ next,
                               int* __restrict__ n_next, int2* __restrict__ pairs, int* __restrict__ n_pairs,
                               const double* __restrict__ Xt, int dp, int d, const int64_t* __restrict__ nbeg,
                               const int64_t* __restrict__ nend, const int8_t* __restrict__ state,
                               const int32_t* __restrict__ depth, const double* __restrict__ thr,
                               const double* __restrict__ dirs, const double* __restrict__ tau_tab) {
  __shared__ double smn[32], smx[32];
  const SearchItem it = cur[blockIdx.x];
  const int dq = depth[it.q];
  if (threadIdx.x == 0 && ((it.mask >> dq) & 1u)) {
    int k = atomicAdd(n_pairs, 1);
    pairs[k] = make_int2(it.a, it.q);
  }
  const uint32_t rest = it.mask & ~((2u << dq) - 1u);
  if (rest == 0u || state[it.q] != 0) return;
  const double* v = dirs + (int64_t)it.q * d;
  double mn = INFINITY, mx = -INFINITY;
  for (int64_t k = nbeg[it.a] + threadIdx.x; k < nend[it.a]; k += blockDim.x) {
    const double* x = Xt + k * dp;
    double acc = __dmul_rn(x[0], v[0]);
    for (int j = 1; j < d; j++) acc = __dadd_rn(acc, __dmul_rn(x[j], v[j]));
    mn = fmin(mn, acc);
    mx = fmax(mx, acc);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    smn[warp] = mn;
    smx[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    const int i = depth[it.a];
    const double th = thr[it.q];
    uint32_t lm = 0, rm = 0;
    for (int j = 0; j < 32; j++) {
      if (!((rest >> j) & 1u)) continue;
      const double tau = tau_tab[i * 32 + j];
      if (__dsub_rn(mn, tau) <= th) lm |= 1u << j;
      if (__dadd_rn(mx, tau) > th) rm |= 1u << j;
    }
    if (lm) next[atomicAdd(n_next, 1)] = SearchItem{it.a, 2 * it.q + 1, lm};
    if (rm) next[atomicAdd(n_next, 1)] = SearchItem{it.a, 2 * it.q + 2, rm};
  }
}

// tau_{i,j} = tau 2^{t-(i+j)/2} exactly as ldexp(tau, floor(e/2)) * (sqrt 2 if e odd) (R15)
double tau_ij(double tau, int t, int i, int j) {
  int e = 2 * t - i - j;
  return std::ldexp(tau, e / 2) * ((e & 1) ? std::sqrt(2.0) : 1.0);
}

std::vector<std::pair<int, int>> admitted_pairs(Ctx& c, const mlk_tree_s* tree, const mlk_basis_s* B,
                                                const mlk_sparsity& sp) {
  const auto& cells = B->cells;
  std::set<std::pair<int, int>> S;
  auto add = [&](int a, int b) {
    if (B->cell_pos[a] < 0 || B->cell_pos[b] < 0) return;
    if (B->cell_pos[a] <= B->cell_pos[b]) S.insert({a, b});
    else S.insert({b, a});
  };
  if (sp.mode == MLK_PAIRS_ALL) {
    for (size_t x = 0; x < cells.size(); x++)
      for (size_t y = x; y < cells.size(); y++) S.insert({cells[x], cells[y]});
  } else {
    const int t = tree->t;
    std::vector<SearchItem> init;
    for (int a : cells) {
      add(a, a);  // self pairs (R14)
      if (tree->depth[a] == 0) {
        for (int b : cells) add(a, b);  // root row dense (R21)
        continue;
      }
      uint32_t mask = 0;
      for (int j = tree->depth[a]; j <= t; j++) mask |= 1u << j;
      init.push_back({a, 0, mask});
    }
    if (!init.empty()) {
      cudaStream_t st = c.stream;
      const int nn = tree->n_nodes;
      std::vector<double> tab(32 * 32, 0.0);
      for (int i = 1; i <= t; i++)
        for (int j = i; j <= t; j++) tab[i * 32 + j] = tau_ij(sp.tau, t, i, j);
      DevBuf<double> tab_d(tab.size(), st);
      tab_d.upload(tab);
      DevBuf<int64_t> nb(nn, st), ne(nn, st);
      nb.upload(tree->begin);
      ne.upload(tree->end);
      DevBuf<int8_t> state(nn, st);
      state.upload(tree->state);
      DevBuf<int32_t> dep(nn, st);
      dep.upload(tree->depth);
      DevBuf<SearchItem> cur(init.size(), st), nxt;
      cur.upload(init);
      int n_cur = (int)init.size();
      DevBuf<int> counts(2, st);
      std::vector<int2> all_pairs;
      TimedLaunch tl(c, "search");
      for (int level = 0; level <= t && n_cur > 0; level++) {
        nxt.alloc((size_t)2 * n_cur, st);
        DevBuf<int2> pr(n_cur, st);
        counts.zero();
        k_search_level<<<n_cur, 128, 0, st>>>(cur.p, n_cur, nxt.p, counts.p, pr.p, counts.p + 1, tree->Xt.p,
                                              tree->d_pad, tree->d, nb.p, ne.p, state.p, dep.p, tree->thr_d.p,
                                              tree->dir_d.p, tab_d.p);
        check_launch("k_search_level");
        auto cnt = counts.download(2);
        auto ph = pr.download(cnt[1]);
        all_pairs.insert(all_pairs.end(), ph.begin(), ph.end());
        std::swap(cur, nxt);
        n_cur = cnt[0];
      }
      for (auto& p : all_pairs) add(p.x, p.y);
    }
  }
  std::vector<std::pair<int, int>> out(S.begin(), S.end());
  std::sort(out.begin(), out.end(), [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
    int a = B->cell_pos[x.first], b = B->cell_pos[y.first];
    if (a != b) return a < b;
    return B->cell_pos[x.second] < B->cell_pos[y.second];
  });
  return out;
}

__global__ void k_unpack(const double* __restrict__ gathered, int64_t max_shard, const int32_t* __restrict__ owner,
                         const int64_t* __restrict__ shard_off, const int64_t* __restrict__ val_off,
                         double* __restrict__ values) {
  int64_t k = blockIdx.x;
  const double* src = gathered + owner[k] * max_shard + shard_off[k];
  int64_t len = val_off[k + 1] - val_off[k];
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) values[val_off[k] + e] = src[e];
}

}  // namespace
}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_assemble_cw(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel,
                           const mlk_sparsity* sparsity, int32_t precision, mlk_cw* out) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && tree && basis && kernel && sparsity && out, "NULL argument");
  *out = nullptr;
  MLK_REQUIRE(basis->tree == tree, "basis was built for another tree");
  MLK_REQUIRE(kernel->family >= MLK_MATERN_12 && kernel->family <= MLK_GAUSSIAN, "unknown covariance family");
  MLK_REQUIRE(kernel->rho > 0 && kernel->sigma2 > 0 && kernel->nugget >= 0, "need rho > 0, sigma2 > 0, nugget >= 0");
  MLK_REQUIRE(sparsity->mode == MLK_PAIRS_ALL || sparsity->mode == MLK_PAIRS_PAPER_TAU, "unknown sparsity mode");
  MLK_REQUIRE(sparsity->mode == MLK_PAIRS_ALL || (sparsity->tau >= 0 && !std::isnan(sparsity->tau)), "need tau >= 0");
  MLK_REQUIRE(precision == MLK_PREC_FP64 || precision == MLK_PREC_DD, "unknown precision");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  cudaStream_t st = c.stream;
  const mlk_basis_s* B = basis;
  const int dp = tree->d_pad, d = tree->d;

  auto pairs = admitted_pairs(c, tree, B, *sparsity);
  auto cw = std::make_unique<mlk_cw_s>();
  cw->device = c.device;
  cw->nranks = c.nranks;
  cw->rank = c.rank;
  cw->n_cells = (int32_t)B->cells.size();
  cw->n_blocks = (int64_t)pairs.size();
  const int64_t nb = cw->n_blocks;
  cw->brow_ptr.assign(cw->n_cells + 1, 0);
  cw->bcol.resize(nb);
  cw->brow.resize(nb);
  cw->val_off.assign(nb + 1, 0);
  std::vector<double> cost(nb), flops(nb), ent(nb);
  std::vector<int8_t> swap(nb);
  for (int64_t k = 0; k < nb; k++) {
    int r = pairs[k].first, cc = pairs[k].second;
    int pr = B->cell_pos[r], pc = B->cell_pos[cc];
    cw->brow[k] = pr;
    cw->bcol[k] = pc;
    cw->brow_ptr[pr + 1]++;
    double sr = (double)(tree->end[r] - tree->begin[r]), sc = (double)(tree->end[cc] - tree->begin[cc]);
    double qr = B->p[r], qc = B->p[cc];
    cw->val_off[k + 1] = cw->val_off[k] + (int64_t)B->p[r] * B->p[cc];
    double f1 = 2 * sr * sc * qc + 2 * qr * sr * qc;  // a = row, b = col (contract col first)
    double f2 = 2 * sc * sr * qr + 2 * qc * sc * qr;  // a = col, b = row
    swap[k] = f2 < f1;
    ent[k] = sr * sc;
    cw->f_gram += 2.0 * d * sr * sc;
    cw->f_c1 += swap[k] ? 2 * sc * sr * qr : 2 * sr * sc * qc;
    cw->f_c2 += swap[k] ? 2 * qc * sc * qr : 2 * qr * sr * qc;
    flops[k] = 2.0 * d * sr * sc + std::min(f1, f2);
    cost[k] = flops[k] + 60.0 * sr * sc;
  }
  for (int i = 0; i < cw->n_cells; i++) cw->brow_ptr[i + 1] += cw->brow_ptr[i];
  cw->nnz = cw->val_off[nb];
  cw->owner.assign(nb, 0);
  if (c.nranks > 1) partition_lpt(cost.data(), nb, c.nranks, cw->owner.data());
  std::vector<int64_t> shard_fill(c.nranks, 0);
  cw->shard_off.assign(nb, 0);
  shard_plan(cw->val_off.data(), cw->owner.data(), nb, c.nranks, cw->shard_off.data(), shard_fill.data());
  for (int64_t k = 0; k < nb; k++) {
    int o = cw->owner[k];
    cw->entries += ent[k];
    cw->flops += flops[k];
    if (o == c.rank) {
      cw->own_entries += ent[k];
      cw->own_flops += flops[k];
    }
  }
  cw->shard_len = shard_fill[c.rank];
  cw->max_shard_len = *std::max_element(shard_fill.begin(), shard_fill.end());
  cw->values.alloc(std::max<int64_t>(cw->nnz, 1), st);
  double* dst_base;
  if (c.nranks > 1) {
    cw->values.zero();
    cw->shard.alloc(std::max<int64_t>(cw->max_shard_len, 1), st);
    cw->shard.zero();
    dst_base = cw->shard.p;
  } else {
    dst_base = cw->values.p;
  }
  auto dst_of = [&](int64_t k) { return dst_base + (c.nranks > 1 ? cw->shard_off[k] : cw->val_off[k]); };

  // own pairs, processed in batches that bound the U scratch
  std::vector<int64_t> own;
  for (int64_t k = 0; k < nb; k++)
    if (cw->owner[k] == c.rank) own.push_back(k);

  if (precision == MLK_PREC_DD) {
    // jobs: a_node, b_node, dst offset, ld, trans
    std::vector<std::array<int64_t, 8>> jobs;
    for (int64_t k : own) {
      int r = pairs[k].first, cc = pairs[k].second;
      bool sw = swap[k];
      int a = sw ? cc : r, b = sw ? r : cc;
      jobs.push_back({a, b, (int64_t)(dst_of(k) - dst_base), (int64_t)B->p[cc], (int64_t)sw, 0, 0, 0});
    }
    assemble_dd(c, tree, B, *kernel, jobs, dst_base);
  } else {
    const KernelParams kp = make_kernel_params(*kernel);
    size_t freeb = 0, totalb = 0;
    CUDA_CHECK(cudaMemGetInfo(&freeb, &totalb));
    const int64_t budget = std::max<int64_t>((int64_t)(freeb / 3 / sizeof(double)), (int64_t)1 << 20);
    size_t pos = 0;
    while (pos < own.size()) {
      // batch
      int64_t need = 0;
      size_t end = pos;
      while (end < own.size()) {
        int64_t k = own[end];
        int r = pairs[k].first, cc = pairs[k].second;
        int a = swap[k] ? cc : r, b = swap[k] ? r : cc;
        int64_t u = (tree->end[a] - tree->begin[a]) * (int64_t)B->p[b];
        if (end > pos && need + u > budget) break;
        need += u;
        end++;
      }
      DevBuf<double> U(std::max<int64_t>(need, 1), st);
      std::vector<TileUnit> units;
      std::vector<GemmDesc> gd;
      int64_t uoff = 0;
      for (size_t i = pos; i < end; i++) {
        int64_t k = own[i];
        int r = pairs[k].first, cc = pairs[k].second;
        bool sw = swap[k];
        int a = sw ? cc : r, b = sw ? r : cc;
        int32_t sa = (int32_t)(tree->end[a] - tree->begin[a]), sb = (int32_t)(tree->end[b] - tree->begin[b]);
        int32_t pa = B->p[a], pb = B->p[b];
        double* Up = U.p + uoff;
        make_tile_units(units, tree->begin[a], sa, tree->begin[b], sb, B->W.p + B->w_off[b], sb, pb, Up, pb, 0, dp);
        // B = W_a U  (pa x pb), stored transposed when a is the column cell
        GemmDesc g{B->W.p + B->w_off[a], sa, Up, pb, dst_of(k), (int64_t)B->p[cc], pa, pb, sa, sw ? 1 : 0};
        gd.push_back(g);
        uoff += (int64_t)sa * pb;
      }
      run_tile_contract(c, tree, kp, units, "assemble_tile_contract");
      gemm_batched(c, gd, "assemble_wa_gemm");
      pos = end;
    }
  }
  CUDA_CHECK(cudaStreamSynchronize(st));
  cw->complete = c.nranks == 1;
  // device structure for the BSR matvec
  cw->brow_d.alloc(std::max<int64_t>(nb, 1), st);
  cw->brow_d.upload(cw->brow);
  cw->bcol_d.alloc(std::max<int64_t>(nb, 1), st);
  cw->bcol_d.upload(cw->bcol);
  cw->owner_d.alloc(std::max<int64_t>(nb, 1), st);
  cw->owner_d.upload(cw->owner);
  cw->val_off_d.alloc(nb + 1, st);
  cw->val_off_d.upload(cw->val_off);
  cw->shard_off_d.alloc(std::max<int64_t>(nb, 1), st);
  cw->shard_off_d.upload(cw->shard_off);
  {
    std::vector<int32_t> cptr(cw->n_cells + 1, 0), cblk;
    for (int64_t k = 0; k < nb; k++)
      if (cw->brow[k] != cw->bcol[k]) cptr[cw->bcol[k] + 1]++;
    for (int i = 0; i < cw->n_cells; i++) cptr[i + 1] += cptr[i];
    cblk.resize(cptr[cw->n_cells]);
    std::vector<int32_t> fill(cptr.begin(), cptr.end() - 1);
    for (int64_t k = 0; k < nb; k++)
      if (cw->brow[k] != cw->bcol[k]) cblk[fill[cw->bcol[k]]++] = (int32_t)k;
    cw->csc_ptr_d.alloc(cptr.size(), st);
    cw->csc_ptr_d.upload(cptr);
    cw->csc_blk_d.alloc(std::max<size_t>(cblk.size(), 1), st);
    cw->csc_blk_d.upload(cblk);
  }
  CUDA_CHECK(cudaStreamSynchronize(st));
  *out = cw.release();
  MLK_API_END
}

void mlk_cw_free(mlk_cw cw) {
  if (!cw) return;
  cudaSetDevice(cw->device);
  // the creating context's stream may already be gone: drain the device, free on stream 0
  cudaDeviceSynchronize();
  cw->values.s = nullptr;
  cw->shard.s = nullptr;
  cw->brow_d.s = nullptr;
  cw->bcol_d.s = nullptr;
  cw->owner_d.s = nullptr;
  cw->val_off_d.s = nullptr;
  cw->shard_off_d.s = nullptr;
  cw->csc_ptr_d.s = nullptr;
  cw->csc_blk_d.s = nullptr;
  delete cw;
}

mlk_status mlk_cw_info(mlk_cw cw, int32_t* n_cells, int64_t* n_blocks, int64_t* nnz, double* entries, double* flops,
                       double* own_entries, double* own_flops) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw, "cw is NULL");
  if (n_cells) *n_cells = cw->n_cells;
  if (n_blocks) *n_blocks = cw->n_blocks;
  if (nnz) *nnz = cw->nnz;
  if (entries) *entries = cw->entries;
  if (flops) *flops = cw->flops;
  if (own_entries) *own_entries = cw->own_entries;
  if (own_flops) *own_flops = cw->own_flops;
  MLK_API_END
}

mlk_status mlk_cw_export(mlk_cw cw, int32_t* brow_ptr, int32_t* bcol, int64_t* val_off, double* values) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw, "cw is NULL");
  CUDA_CHECK(cudaSetDevice(cw->device));
  if (brow_ptr) std::copy(cw->brow_ptr.begin(), cw->brow_ptr.end(), brow_ptr);
  if (bcol) std::copy(cw->bcol.begin(), cw->bcol.end(), bcol);
  if (val_off) std::copy(cw->val_off.begin(), cw->val_off.end(), val_off);
  if (values && cw->nnz > 0) CUDA_CHECK(cudaMemcpy(values, cw->values.p, sizeof(double) * cw->nnz, cudaMemcpyDefault));
  MLK_API_END
}

mlk_status mlk_cw_flops(mlk_cw cw, double* gram, double* contract1, double* contract2) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw, "cw is NULL");
  if (gram) *gram = cw->f_gram;
  if (contract1) *contract1 = cw->f_c1;
  if (contract2) *contract2 = cw->f_c2;
  MLK_API_END
}

mlk_status mlk_cw_owner(mlk_cw cw, int32_t* owner) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw && owner, "NULL argument");
  std::copy(cw->owner.begin(), cw->owner.end(), owner);
  MLK_API_END
}

mlk_status mlk_cw_shard_len(mlk_cw cw, int64_t* shard_len, int64_t* max_shard_len) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw, "cw is NULL");
  if (shard_len) *shard_len = cw->shard_len;
  if (max_shard_len) *max_shard_len = cw->max_shard_len;
  MLK_API_END
}

mlk_status mlk_cw_pack(mlk_ctx ctx, mlk_cw cw, double* dst) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && cw && dst, "NULL argument");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  MLK_REQUIRE(is_device_ptr(dst), "dst must be device memory");
  if (cw->max_shard_len == 0) return MLK_OK;
  CUDA_CHECK(cudaMemsetAsync(dst, 0, sizeof(double) * cw->max_shard_len, c.stream));
  const double* src = cw->nranks > 1 ? cw->shard.p : cw->values.p;
  if (cw->shard_len)
    CUDA_CHECK(cudaMemcpyAsync(dst, src, sizeof(double) * cw->shard_len, cudaMemcpyDeviceToDevice, c.stream));
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  MLK_API_END
}

mlk_status mlk_cw_unpack(mlk_ctx ctx, mlk_cw cw, const double* gathered) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && cw && gathered, "NULL argument");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  MLK_REQUIRE(is_device_ptr(gathered), "gathered must be device memory");
  if (cw->n_blocks == 0) return MLK_OK;
  {
    TimedLaunch tl(c, "cw_unpack");
    k_unpack<<<(unsigned)cw->n_blocks, 256, 0, c.stream>>>(gathered, cw->max_shard_len, cw->owner_d.p,
                                                           cw->shard_off_d.p, cw->val_off_d.p, cw->values.p);
    check_launch("k_unpack");
  }
  cw->complete = true;
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  MLK_API_END
}

mlk_status mlk_cw_values_device(mlk_cw cw, double** values) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw && values, "NULL argument");
  *values = cw->values.p;
  MLK_API_END
}

}  // extern "C"
