// mlk_assemble_cw: admission (Algorithms 3-6 on the device), BSR structure, cost model and
// LPT partition (host), then the two contractions per admitted pair:
//   K5a (tile.cu)   U = C(X_a, X_b) W_b^T   fused tiles on FP64 DMMA
//   K5b (gemm.cu)   B = W_a U               batched FP64 DMMA GEMM, written into the BSR
// where b is the side contracted first (the cheaper order).
#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <memory>
#include <set>

#include "api.cuh"
#include "tile.cuh"

namespace mlk {
// rows per work unit / per piece of a block: 4096 up to n = 2^18 (cfg1-4), then doubling with
// n up to 32768 -- a block's pieces are full p_a x p_b partials, so at cfg5 (n = 2^20, M = 1326)
// 4096-row pieces would hold 464 GB against 184 GB of final values (16384: 221 GB).  A function
// of n only, so the pieces (and the results) are the same for every rank count.
// cost model of the nested assembly against the direct units (K5a entries cost 2 dp + 16 rq + 60
// "units"): the nested leaf pass runs K5a ~15 % below the direct units' efficiency (shorter
// b streams, r02i), a transfer flop costs transfer_weight(M) units (the transfer kernel ran at
// 7-11 TFLOP/s against K5a's 26-28, r02j)
constexpr double kNestedK5aW = 1.15;
// 2M <= 112 (Q_c in <= 113 KB of shared memory, two transfer CTAs per SM): 3.5 units per flop
// (cfg4, M = 51); larger M one CTA per SM: 6 (cfg2, M = 66: 6.7 TFLOP/s, r02j)
inline double transfer_weight(int M) { return 2 * M <= 112 ? 3.5 : 6.0; }
int64_t row_chunk(int64_t n) {
  int64_t ch = 4096;
  while (ch < 32768 && (n >> 18) >= 2 * (ch / 4096)) ch *= 2;
  return ch;
}
void reduce_pieces(Ctx& c, mlk_cw_s* cw, const double* gathered);
// jobs: {a node, b node, destination pointer, ldc, store transposed, -, -, -}
void assemble_dd(Ctx& c, const mlk_tree_s* tree, const mlk_basis_s* B, const mlk_kernel& k,
                 const std::vector<std::array<int64_t, 8>>& jobs);
namespace {

struct SearchItem {
  int32_t a;      // searching cell (heap node)
  int32_t q;      // current node
  uint32_t mask;  // target depths still searched through q
};

// Projection extrema of every cell onto every internal node direction, mm[cell][q] =
// (min, max) of x . v_q over the cell's points with the R6 arithmetic (products and sums rounded
// separately, left to right).  Leaves: one CTA per (leaf, 8 directions); internal cells: the
// exact min / max of their children (k_minmax_up), so every entry equals the direct value.
constexpr int kMmQ = 8;
__global__ void k_proj_minmax(const double* __restrict__ Xt, int dp, int d, const int64_t* __restrict__ lbeg,
                              const int64_t* __restrict__ lend, const int32_t* __restrict__ lnode,
                              const int8_t* __restrict__ state, const double* __restrict__ dirs, int n_int,
                              double2* __restrict__ mm) {
  extern __shared__ double sv[];  // kMmQ x d directions
  __shared__ double smn[kMmQ][4], smx[kMmQ][4];
  const int leaf = blockIdx.x, q0 = blockIdx.y * kMmQ;
  const int nq = min(kMmQ, n_int - q0);
  for (int e = threadIdx.x; e < nq * d; e += blockDim.x) sv[e] = dirs[(int64_t)q0 * d + e];
  __syncthreads();
  double mn[kMmQ], mx[kMmQ];
#pragma unroll
  for (int i = 0; i < kMmQ; i++) {
    mn[i] = INFINITY;
    mx[i] = -INFINITY;
  }
  for (int64_t k = lbeg[leaf] + threadIdx.x; k < lend[leaf]; k += blockDim.x) {
    const double* x = Xt + k * dp;
    // the kMmQ projections advance together coordinate by coordinate (each x_j loaded once,
    // kMmQ independent add chains); every projection keeps its left-to-right order (R6)
    double acc[kMmQ];
    const double x0 = x[0];
#pragma unroll
    for (int i = 0; i < kMmQ; i++) acc[i] = i < nq ? __dmul_rn(x0, sv[i * d]) : 0.0;
    for (int j = 1; j < d; j++) {
      const double xj = x[j];
#pragma unroll
      for (int i = 0; i < kMmQ; i++)
        if (i < nq) acc[i] = __dadd_rn(acc[i], __dmul_rn(xj, sv[i * d + j]));
    }
#pragma unroll
    for (int i = 0; i < kMmQ; i++) {
      if (i < nq) {
        mn[i] = fmin(mn[i], acc[i]);
        mx[i] = fmax(mx[i], acc[i]);
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kMmQ; i++) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[i] = fmin(mn[i], __shfl_xor_sync(0xffffffffu, mn[i], o));
      mx[i] = fmax(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
    }
    if (lane == 0) {
      smn[i][warp] = mn[i];
      smx[i][warp] = mx[i];
    }
  }
  __syncthreads();
  if (threadIdx.x < nq) {
    const int i = threadIdx.x;
    double a = smn[i][0], b = smx[i][0];
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
      a = fmin(a, smn[i][w]);
      b = fmax(b, smx[i][w]);
    }
    if (state[q0 + i] == 0) mm[(int64_t)lnode[leaf] * n_int + q0 + i] = make_double2(a, b);
  }
}

__global__ void k_minmax_up(const int32_t* __restrict__ nodes, int cnt, int n_int, double2* __restrict__ mm) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)cnt * n_int) return;
  const int c = nodes[e / n_int], q = (int)(e % n_int);
  const double2 l = mm[(int64_t)(2 * c + 1) * n_int + q], r = mm[(int64_t)(2 * c + 2) * n_int + q];
  mm[(int64_t)c * n_int + q] = make_double2(fmin(l.x, r.x), fmax(l.y, r.y));
}

// One level of every search at once, one thread per item (grid-stride, count read on the
// device): emit (a, q) if depth(q) is a target, then the symmetric rule of reading R12 on the
// tabulated extrema for every remaining target depth; surviving children are appended to the
// next level's item region.  No host round trip between levels.
__global__ void k_search_level(const SearchItem* __restrict__ cur, const int* __restrict__ n_cur_p,
                               SearchItem* __restrict__ next, int* __restrict__ n_next, int2* __restrict__ pairs,
                               int* __restrict__ n_pairs, const double2* __restrict__ mm, int n_int,
                               const int8_t* __restrict__ state, const int32_t* __restrict__ depth,
                               const double* __restrict__ thr, const double* __restrict__ tau_tab) {
  const int n_cur = *n_cur_p;
  for (int item = blockIdx.x * blockDim.x + threadIdx.x; item < n_cur; item += gridDim.x * blockDim.x) {
    const SearchItem it = cur[item];
    const int dq = depth[it.q];
    if ((it.mask >> dq) & 1u) pairs[atomicAdd(n_pairs, 1)] = make_int2(it.a, it.q);
    const uint32_t rest = it.mask & ~((2u << dq) - 1u);
    if (rest == 0u || state[it.q] != 0) continue;
    const double2 e = mm[(int64_t)it.a * n_int + it.q];
    const int i = depth[it.a];
    const double th = thr[it.q];
    uint32_t lm = 0, rm = 0;
    for (int j = 0; j < 32; j++) {
      if (!((rest >> j) & 1u)) continue;
      const double tau = tau_tab[i * 32 + j];
      if (__dsub_rn(e.x, tau) <= th) lm |= 1u << j;
      if (__dadd_rn(e.y, tau) > th) rm |= 1u << j;
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
      DevBuf<int8_t> state(nn, st);
      state.upload(tree->state);
      DevBuf<int32_t> dep(nn, st);
      dep.upload(tree->depth);
      // level L holds items (a, q) with depth(q) = L: at most |init| 2^L of them
      std::vector<int64_t> off(t + 2, 0);
      for (int L = 0; L <= t; L++) off[L + 1] = off[L] + (int64_t)init.size() * ((int64_t)1 << L);
      DevBuf<SearchItem> items(off[t + 1], st);
      upload_async(items.p, init.data(), init.size() * sizeof(SearchItem), st);
      DevBuf<int2> pr(off[t + 1], st);
      std::vector<int> cnt0(t + 3, 0);
      cnt0[0] = (int)init.size();
      DevBuf<int> counts(t + 3, st);  // items per level, then the pair count
      counts.upload(cnt0);
      {
        TimedLaunch tl(c, "search");
        // projection extrema table: leaves directly, internal cells bottom-up
        const int n_int = (1 << t) - 1;
        DevBuf<double2> mm((size_t)nn * n_int, st);
        std::vector<int64_t> lb, le;
        std::vector<int32_t> ln;
        std::vector<std::vector<int32_t>> internal_at(t + 1);
        for (int q = 0; q < nn; q++) {
          if (tree->state[q] == 1) {
            lb.push_back(tree->begin[q]);
            le.push_back(tree->end[q]);
            ln.push_back(q);
          } else if (tree->state[q] == 0) {
            internal_at[tree->depth[q]].push_back(q);
          }
        }
        DevBuf<int64_t> lbd(lb.size(), st), led(le.size(), st);
        DevBuf<int32_t> lnd(ln.size(), st);
        lbd.upload(lb);
        led.upload(le);
        lnd.upload(ln);
        const int d = tree->d;
        const size_t vsm = sizeof(double) * kMmQ * d;
        if (vsm > 48 * 1024) CUDA_CHECK(cudaFuncSetAttribute(k_proj_minmax, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsm));
        k_proj_minmax<<<dim3((unsigned)ln.size(), (unsigned)ceil_div(n_int, kMmQ)), 128, vsm, st>>>(
            tree->Xt.p, tree->d_pad, d, lbd.p, led.p, lnd.p, state.p, tree->dir_d.p, n_int, mm.p);
        check_launch("k_proj_minmax");
        std::vector<DevBuf<int32_t>> lvl_nodes(t + 1);
        for (int L = t; L >= 1; L--) {
          if (internal_at[L].empty()) continue;
          lvl_nodes[L].alloc(internal_at[L].size(), st);
          lvl_nodes[L].upload(internal_at[L]);
          const int64_t cntL = (int64_t)internal_at[L].size() * n_int;
          k_minmax_up<<<(unsigned)ceil_div(cntL, 256), 256, 0, st>>>(lvl_nodes[L].p, (int)internal_at[L].size(), n_int,
                                                                    mm.p);
          check_launch("k_minmax_up");
        }
        for (int L = 0; L <= t; L++) {
          const int64_t cap = off[L + 1] - off[L];
          const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(cap, 128), 8 * (int64_t)num_sms(c.device));
          k_search_level<<<grid, 128, 0, st>>>(items.p + off[L], counts.p + L, items.p + off[std::min(L + 1, t)],
                                               counts.p + L + 1, pr.p, counts.p + t + 2, mm.p, n_int, state.p, dep.p,
                                               tree->thr_d.p, tab_d.p);
          check_launch("k_search_level");
        }
      }
      auto cnt = counts.download(t + 3);
      std::vector<int2> all_pairs = pr.download(cnt[t + 2]);
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

// values of the listed blocks = sum of their pieces in chunk order (pieces live in rank r's
// shard at gathered + r * max_shard + piece_off)
__global__ void k_reduce_pieces(const int32_t* __restrict__ blocks, const int64_t* __restrict__ piece_ptr,
                                const int64_t* __restrict__ piece_off, const int32_t* __restrict__ piece_owner,
                                const double* __restrict__ gathered, int64_t max_shard,
                                const int64_t* __restrict__ val_off, double* __restrict__ values) {
  const int64_t k = blocks[blockIdx.x];
  const int64_t len = val_off[k + 1] - val_off[k];
  const int64_t p0 = piece_ptr[k], p1 = piece_ptr[k + 1];
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    double s = 0.0;
    for (int64_t p = p0; p < p1; p++) s += gathered[piece_owner[p] * max_shard + piece_off[p] + e];
    values[val_off[k] + e] = s;
  }
}

// the leaves' Phi blocks (M x s_l each, at their phi offsets) as one M x n row-major matrix:
// column j = Phi_leaf(j)[:, j - begin(leaf)]
__global__ void k_phi_all(const double* __restrict__ Phi, const int64_t* __restrict__ off,
                          const int64_t* __restrict__ beg, const int32_t* __restrict__ sz, int M, int64_t n,
                          double* __restrict__ out) {
  const int l = blockIdx.y;
  const int64_t s = sz[l];
  const double* src = Phi + off[l];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * M; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / s, x = e - m * s;
    out[m * n + beg[l] + x] = src[e];
  }
}

}  // namespace

void reduce_pieces(Ctx& c, mlk_cw_s* cw, const double* gathered) {
  if (cw->reduce_blocks.empty()) return;
  const int64_t ms = cw->nranks > 1 ? cw->max_shard_len : 0;
  k_reduce_pieces<<<(unsigned)cw->reduce_blocks.size(), 256, 0, c.stream>>>(
      cw->reduce_d.p, cw->piece_ptr_d.p, cw->piece_off_d.p, cw->piece_owner_d.p, gathered, ms, cw->val_off_d.p,
      cw->vals());
  check_launch("k_reduce_pieces");
}

}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_assemble_cw(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel,
                           const mlk_sparsity* sparsity, int32_t precision, int32_t gather, mlk_cw* out) {
  MLK_API_BEGIN
  MLK_REQUIRE(gather >= MLK_GATHER_NONE && gather <= MLK_GATHER_HOST, "unknown gather mode");
  MLK_API_END_CALL(mlk_assemble_cw_ex(ctx, tree, basis, kernel, sparsity, precision,
                                      gather == MLK_GATHER_HOST ? MLK_VALUES_HOST : MLK_VALUES_DEVICE,
                                      gather == MLK_GATHER_NONE ? MLK_GATHER_NONE : MLK_GATHER_DEVICE, out));
}

mlk_status mlk_assemble_cw_ex(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel,
                              const mlk_sparsity* sparsity, int32_t precision, int32_t placement, int32_t gather,
                              mlk_cw* out) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && tree && basis && kernel && sparsity && out, "NULL argument");
  MLK_REQUIRE(placement == MLK_VALUES_DEVICE || placement == MLK_VALUES_HOST, "unknown value placement");
  MLK_REQUIRE(gather == MLK_GATHER_NONE || gather == MLK_GATHER_DEVICE, "mlk_assemble_cw_ex: gather is 0 or 1");
  MLK_REQUIRE(gather == MLK_GATHER_NONE || ctx->c.nranks == 1 || ctx->c.comm,
              "gather needs a context created with an NCCL unique id");
  *out = nullptr;
  MLK_REQUIRE(basis->tree == tree, "basis was built for another tree");
  MLK_REQUIRE(kernel->family >= MLK_MATERN_12 && kernel->family <= MLK_MATERN_NU, "unknown covariance family");
  MLK_REQUIRE(kernel->rho > 0 && kernel->sigma2 > 0 && kernel->nugget >= 0, "need rho > 0, sigma2 > 0, nugget >= 0");
  MLK_REQUIRE(kernel->family != MLK_MATERN_NU || (kernel->nu > 0 && kernel->nu <= 50),
              "MLK_MATERN_NU needs 0 < nu <= 50");
  MLK_REQUIRE(precision == MLK_PREC_FP64 || kernel->family != MLK_MATERN_NU,
              "the double-double mode covers the closed-form families only");
  MLK_REQUIRE(sparsity->mode == MLK_PAIRS_ALL || sparsity->mode == MLK_PAIRS_PAPER_TAU, "unknown sparsity mode");
  MLK_REQUIRE(sparsity->mode == MLK_PAIRS_ALL || (sparsity->tau >= 0 && !std::isnan(sparsity->tau)), "need tau >= 0");
  MLK_REQUIRE(precision == MLK_PREC_FP64 || precision == MLK_PREC_DD, "unknown precision");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  cudaStream_t st = c.stream;
  const mlk_basis_s* B = basis;
  const int dp = tree->d_pad, d = tree->d;

  HostTrace trace("assemble");
  auto pairs = admitted_pairs(c, tree, B, *sparsity);
  trace.mark("search");
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
  // ---- per block: orientation.  b = the cell contracted first (its W_b multiplies C first),
  // a = the other.  Ancestor pairs take b = the ancestor, so that U_ab = C(X_a, X_b) W_b^T is
  // a row slice of V_b = C(X_b, X_b) W_b^T (X_a is a subset of X_b): every such block reuses
  // the self-block intermediate of its ancestor.  Other pairs
  // take a = the smaller cell (its pieces are few, and b's V gains only |a| rows: at cfg5 this
  // cut the K5a / K5b flops by 6 % / 73 % and the pieces 3.5x against the cheaper-order rule),
  // and the cheaper order of the two contractions between cells of equal size.
  auto is_anc = [](int anc, int q) {
    while (q > anc) q = (q - 1) / 2;
    return q == anc;
  };
  std::vector<int32_t> A(nb), Bc(nb);
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
    cw->entries += sr * sc;
    bool sw;
    if (r == cc || is_anc(cc, r)) sw = false;
    else if (is_anc(r, cc)) sw = true;
    else if (sr != sc) sw = sc < sr;  // a = the smaller cell: fewer pieces, and its rows join R_b
    else sw = (2 * sc * sr * qr + 2 * qc * sc * qr) < (2 * sr * sc * qc + 2 * qr * sr * qc);
    swap[k] = sw;
    A[k] = sw ? cc : r;
    Bc[k] = sw ? r : cc;
  }
  for (int i = 0; i < cw->n_cells; i++) cw->brow_ptr[i + 1] += cw->brow_ptr[i];
  cw->nnz = cw->val_off[nb];
  trace.mark("orient");
  const bool dd = precision == MLK_PREC_DD;
  auto S = [&](int q) { return tree->end[q] - tree->begin[q]; };

  // ---- work units (column cell b, row chunk) and pieces (block, row chunk)
  const int64_t CH = row_chunk(tree->n);
  struct Unit {
    int b;            // the cell contracted first; -1: a nested unit (every internal b, one chunk)
    int64_t chunk;
    std::vector<std::pair<int64_t, int64_t>> rows;  // tree-position ranges inside the chunk
    int64_t nrows = 0;
    double cost = 0, flops_gram = 0, flops_c1 = 0, flops_c2 = 0, flops_tr = 0;
    int owner = 0;
    int64_t v_off = 0;  // offset of this unit's V rows in the V buffer (doubles)
  };
  std::vector<Unit> units;
  std::map<std::pair<int, int64_t>, int> unit_of;
  struct Piece {
    int64_t blk, chunk;
    int unit;
  };
  std::vector<Piece> pieces;
  std::vector<int64_t> piece_ptr(nb + 1, 0);
  // ---- nested evaluation (DESIGN.md section 6 "Nested assembly"): for every internal b,
  // V_b = C(X_R, X_b) W_b^T follows from the leaves' scaling sums S_l = C(X_R, X_l) Phi_l^T by the
  // merge factors of the basis, [S_c | V_c] = [S_cL S_cR] Q_c (W_c = Q_c[:, M:]^T (Phi_cL (+) Phi_cR),
  // Phi_c = Q_c[:, :M]^T (...), steps (c)-(e) of P:1427-1515), so each covariance entry is
  // evaluated once per row chunk instead of once per ancestor (and once per extra pair).  Taken
  // when its cost model beats the direct units of the internal cells (MLK_ASSEMBLY=direct /
  // nested forces a mode).
  const int64_t nn = tree->n_nodes;
  bool nested = false;
  if (!dd && B->Qm.p && !B->phi_dropped && tree->t >= 1) {
    const char* env = std::getenv("MLK_ASSEMBLY");
    const std::string mode = env ? env : "auto";
    if (mode == "nested") {
      nested = true;
    } else if (mode != "direct") {
      // per-entry K5a cost ~ (2 dp + 16 rq + 60) as in the unit costs below; transfers 8 M^2
      // flops per (row, internal cell) on the batched GEMM, weighted transfer_weight(M) per flop (it ran
      // at ~40 % of the FP64 peak against K5a's ~70 %: r02f)
      std::map<int, double> rows_b;
      std::map<int, std::vector<std::pair<int64_t, int64_t>>> rs;
      for (int64_t k = 0; k < nb; k++)
        if (tree->state[Bc[k]] == 0) rs[Bc[k]].push_back({tree->begin[A[k]], tree->end[A[k]]});
      double direct = 0.0;
      for (auto& kv : rs) {
        auto rg = kv.second;
        rg.push_back({tree->begin[kv.first], tree->end[kv.first]});
        std::sort(rg.begin(), rg.end());
        int64_t tot = 0, cur_lo = -1, cur_hi = -1;
        for (auto& x : rg) {
          if (x.first <= cur_hi) {
            cur_hi = std::max(cur_hi, x.second);
          } else {
            tot += cur_hi - cur_lo;
            cur_lo = x.first;
            cur_hi = x.second;
          }
        }
        tot += cur_hi - cur_lo;
        const int rq = tile_rq_class(std::min(B->p[kv.first], 8 * kTileMaxRQ));
        direct += (double)tot * (double)S(kv.first) * (2.0 * dp + 16.0 * rq + 60.0);
      }
      int64_t nint = 0;
      for (int64_t q = 0; q < nn; q++) nint += tree->state[q] == 0;
      const int rqm = tile_rq_class(std::min(B->M, 8 * kTileMaxRQ));
      // transfers: the S half (4 M^2 per row and internal cell) for every row, the V half only
      // for the rows of c's blocks (the same row sets the direct units would have evaluated)
      double vrows = 0.0;
      for (auto& kv : rs) {
        auto rg = kv.second;
        rg.push_back({tree->begin[kv.first], tree->end[kv.first]});
        std::sort(rg.begin(), rg.end());
        int64_t tot = 0, cur_lo = -1, cur_hi = -1;
        for (auto& x : rg) {
          if (x.first <= cur_hi) {
            cur_hi = std::max(cur_hi, x.second);
          } else {
            tot += cur_hi - cur_lo;
            cur_lo = x.first;
            cur_hi = x.second;
          }
        }
        vrows += (double)(tot + cur_hi - cur_lo);
      }
      const double nest = kNestedK5aW * (double)tree->n * (double)tree->n * (2.0 * dp + 16.0 * rqm + 60.0) +
                          transfer_weight(B->M) * 4.0 * B->M * B->M * ((double)tree->n * (double)nint + vrows);
      nested = nest < 0.9 * direct;
    }
  }
  cw->nested = nested;
  // the nested units cover CHN = m CH rows (m a power of two, CHN <= 16384): fewer, larger
  // K5a / transfer / K5b launches with fuller waves (r02v: the top transfer levels of a 4096-row
  // chunk ran < 1 wave of CTAs).  Pieces stay per CH rows, and every value is computed per row
  // or per piece, so the results do not depend on m; m depends only on (n, nodes, M) and the
  // device's total memory (the S and V buffers, 2 CHN n_nodes M doubles, <= 1/8 of it), so it
  // is the same on every rank.
  int64_t m_nest = 1;
  if (nested) {
    const double per_row = 2.0 * (double)tree->n_nodes * B->M * sizeof(double);
    while (CH * m_nest * 2 <= std::min<int64_t>(16384, tree->n) &&
           per_row * (double)(CH * m_nest * 2) <= (double)device_total_bytes(c.device) / 8)
      m_nest *= 2;
  }
  const int64_t CHN = CH * m_nest;
  std::vector<int> nested_unit;  // nested chunk -> unit
  std::map<int, std::vector<std::pair<int64_t, int64_t>>> nested_rows;  // internal c -> row ranges R_c
  if (!dd) {
    if (nested) {
      // the rows R_c whose V_c some block uses (X_c and the row cells of c's blocks), merged
      for (int64_t k = 0; k < nb; k++)
        if (tree->state[Bc[k]] == 0) nested_rows[Bc[k]].push_back({tree->begin[A[k]], tree->end[A[k]]});
      for (auto& kv : nested_rows) {
        auto& rg = kv.second;
        rg.push_back({tree->begin[kv.first], tree->end[kv.first]});
        std::sort(rg.begin(), rg.end());
        std::vector<std::pair<int64_t, int64_t>> merged;
        for (auto& x : rg) {
          if (!merged.empty() && x.first <= merged.back().second) merged.back().second = std::max(merged.back().second, x.second);
          else merged.push_back(x);
        }
        rg = merged;
      }
      const double n = (double)tree->n;
      int64_t nint = 0;
      for (int64_t q = 0; q < nn; q++) nint += tree->state[q] == 0;
      const int rqm = tile_rq_class(std::min(B->M, 8 * kTileMaxRQ));
      for (int64_t c0 = 0; c0 * CHN < tree->n; c0++) {
        Unit u;
        u.b = -1;
        u.chunk = c0;
        const int64_t lo = c0 * CHN, hi = std::min<int64_t>(tree->n, (c0 + 1) * CHN);
        u.rows.push_back({lo, hi});
        u.nrows = hi - lo;
        u.flops_gram = 2.0 * d * (hi - lo) * n;
        u.flops_c1 = 2.0 * (hi - lo) * n * B->M;
        // transfers: the S half for every row and internal cell (not the root), the V half for
        // the rows of R_c in this chunk
        double vr = 0.0;
        for (auto& kv : nested_rows)
          for (auto& rg : kv.second) vr += (double)std::max<int64_t>(0, std::min(rg.second, hi) - std::max(rg.first, lo));
        u.flops_tr = 4.0 * B->M * B->M * ((double)(hi - lo) * (double)(nint - 1) + vr);
        u.cost = kNestedK5aW * (hi - lo) * n * (2.0 * dp + 16.0 * rqm + 60.0) + transfer_weight(B->M) * u.flops_tr;
        nested_unit.push_back((int)units.size());
        units.push_back(u);
      }
    }
    auto direct_b = [&](int b) { return !nested || tree->state[b] != 0; };
    std::map<int, std::vector<std::pair<int64_t, int64_t>>> rowsets;
    for (int64_t k = 0; k < nb; k++)
      if (direct_b(Bc[k])) rowsets[Bc[k]].push_back({tree->begin[A[k]], tree->end[A[k]]});
    for (auto& kv : rowsets) {
      int b = kv.first;
      auto rg = kv.second;
      rg.push_back({tree->begin[b], tree->end[b]});
      std::sort(rg.begin(), rg.end());
      std::vector<std::pair<int64_t, int64_t>> merged;
      for (auto& x : rg) {
        if (!merged.empty() && x.first <= merged.back().second) merged.back().second = std::max(merged.back().second, x.second);
        else merged.push_back(x);
      }
      const double sb = (double)S(b);
      const int rq = tile_rq_class(std::min(B->p[b], 8 * kTileMaxRQ));
      for (auto& m : merged) {
        for (int64_t c0 = m.first / CH; c0 * CH < m.second; c0++) {
          int64_t lo = std::max(m.first, c0 * CH), hi = std::min(m.second, (c0 + 1) * CH);
          auto key = std::make_pair(b, c0);
          auto it = unit_of.find(key);
          int ui;
          if (it == unit_of.end()) {
            ui = (int)units.size();
            unit_of[key] = ui;
            Unit u;
            u.b = b;
            u.chunk = c0;
            units.push_back(u);
          } else {
            ui = it->second;
          }
          Unit& u = units[ui];
          u.rows.push_back({lo, hi});
          u.nrows += hi - lo;
          u.flops_gram += 2.0 * d * (hi - lo) * sb;
          u.flops_c1 += 2.0 * (hi - lo) * sb * B->p[b];
          u.cost += (hi - lo) * sb * (2.0 * dp + 16.0 * rq + 60.0);
        }
      }
    }
    for (int64_t k = 0; k < nb; k++) {
      int a = A[k], b = Bc[k];
      for (int64_t c0 = tree->begin[a] / CH; c0 * CH < tree->end[a]; c0++) {
        int ui = direct_b(b) ? unit_of.at({b, c0}) : nested_unit[c0 / m_nest];
        int64_t lo = std::max(tree->begin[a], c0 * CH), hi = std::min(tree->end[a], (c0 + 1) * CH);
        double f = 2.0 * B->p[a] * (double)(hi - lo) * B->p[b];
        units[ui].flops_c2 += f;
        units[ui].cost += f;
        pieces.push_back({k, c0, ui});
        piece_ptr[k + 1]++;
      }
    }
  } else {
    // DD mode: one unit and one piece per block
    for (int64_t k = 0; k < nb; k++) {
      Unit u;
      u.b = Bc[k];
      u.chunk = -1;
      double sa = (double)S(A[k]), sb = (double)S(Bc[k]);
      u.flops_gram = 3.0 * d * sa * sb;
      u.flops_c1 = 2.0 * sa * sb * B->p[Bc[k]];
      u.flops_c2 = 2.0 * B->p[A[k]] * sa * B->p[Bc[k]];
      u.cost = sa * sb * (300.0 + 20.0 * B->p[Bc[k]]);
      units.push_back(u);
      pieces.push_back({k, 0, (int)k});
      piece_ptr[k + 1] = 1;
    }
  }
  for (int64_t k = 0; k < nb; k++) piece_ptr[k + 1] += piece_ptr[k];
  const int64_t npc = (int64_t)pieces.size();
  // ---- ownership: LPT over units; a piece belongs to its unit's owner
  {
    std::vector<double> uc(units.size());
    for (size_t i = 0; i < units.size(); i++) uc[i] = units[i].cost;
    std::vector<int32_t> own(units.size(), 0);
    if (c.nranks > 1) partition_lpt(uc.data(), (int64_t)uc.size(), c.nranks, own.data());
    for (size_t i = 0; i < units.size(); i++) units[i].owner = own[i];
  }
  for (auto& u : units) {
    double f = u.flops_gram + u.flops_c1 + u.flops_c2 + u.flops_tr;
    cw->flops += f;
    cw->f_gram += u.flops_gram;
    cw->f_c1 += u.flops_c1;
    cw->f_tr += u.flops_tr;
    if (u.b < 0) cw->f_nested_k5a += u.flops_gram + u.flops_c1;
    cw->f_c2 += u.flops_c2;
    if (u.owner == c.rank) {
      cw->own_flops += f;
      cw->own_entries += (double)u.nrows * (double)S(u.b);
    }
  }
  cw->owner.assign(nb, 0);
  for (int64_t k = 0; k < nb; k++) cw->owner[k] = units[pieces[piece_ptr[k]].unit].owner;
  // a block computed by one rank in one piece is written straight into the BSR values when
  // nranks == 1; everything else goes through per-rank piece shards reduced in chunk order
  std::vector<int64_t> plen(npc + 1, 0);
  std::vector<int32_t> powner(npc);
  std::vector<int8_t> direct(nb, 0);
  for (int64_t k = 0; k < nb; k++) direct[k] = (c.nranks == 1 && piece_ptr[k + 1] - piece_ptr[k] == 1);
  for (int64_t i = 0; i < npc; i++) {
    int64_t k = pieces[i].blk;
    plen[i + 1] = plen[i] + (direct[k] ? 0 : cw->val_off[k + 1] - cw->val_off[k]);
    powner[i] = units[pieces[i].unit].owner;
  }
  std::vector<int64_t> shard_fill(c.nranks, 0);
  cw->piece_off.assign(npc, 0);
  shard_plan(plen.data(), powner.data(), npc, c.nranks, cw->piece_off.data(), shard_fill.data());
  cw->piece_ptr = piece_ptr;
  cw->piece_owner = powner;
  cw->shard_len = shard_fill[c.rank];
  cw->max_shard_len = *std::max_element(shard_fill.begin(), shard_fill.end());
  // the merge levels of the basis ran on the auxiliary stream during the search and planning;
  // wait for them before the large allocations, so that the pool can reuse the memory the
  // basis construction freed on that stream (cfg5: level buffers and QR scratch, ~50 GB)
  basis_wait(c, B);
  trace.mark("basis_wait");
  // the values: device memory now when nranks == 1 (ranks > 1 allocate at mlk_cw_unpack, so a
  // rank holds only its shard until the gather), or mapped pinned host memory (MLK_VALUES_HOST,
  // for matrices beyond HBM: the kernels store the blocks straight over the host link)
  if (placement == MLK_VALUES_HOST) {
    CUDA_CHECK(cudaHostAlloc((void**)&cw->hvals, sizeof(double) * std::max<int64_t>(cw->nnz, 1),
                             cudaHostAllocMapped | cudaHostAllocPortable));
  } else if (c.nranks == 1) {
    cw->values.alloc(std::max<int64_t>(cw->nnz, 1), st);
  }
  cw->shard.alloc(std::max<int64_t>(cw->max_shard_len, 1), st);
  for (int64_t k = 0; k < nb; k++)
    if (!direct[k]) cw->reduce_blocks.push_back((int32_t)k);
  auto piece_dst = [&](int64_t i) {
    int64_t k = pieces[i].blk;
    return direct[k] ? cw->vals() + cw->val_off[k] : cw->shard.p + cw->piece_off[i];
  };

  trace.mark("plan");
  if (dd) {
    std::vector<std::array<int64_t, 8>> jobs;
    for (int64_t i = 0; i < npc; i++) {
      int64_t k = pieces[i].blk;
      if (powner[i] != c.rank) continue;
      jobs.push_back({A[k], Bc[k], (int64_t)reinterpret_cast<uintptr_t>(piece_dst(i)),
                      (int64_t)B->p[pairs[k].second], (int64_t)swap[k], 0, 0, 0});
    }
    assemble_dd(c, tree, B, *kernel, jobs);
  } else {
    const KernelParams kp = make_kernel_params(*kernel);
    // own units in batches that bound the V scratch
    std::vector<int> mine;
    for (size_t i = 0; i < units.size(); i++)
      if (units[i].owner == c.rank && units[i].b >= 0) mine.push_back((int)i);
    std::vector<std::vector<int64_t>> unit_pieces(units.size());
    for (int64_t i = 0; i < npc; i++)
      if (powner[i] == c.rank) unit_pieces[pieces[i].unit].push_back(i);
    const int64_t budget = std::max<int64_t>(c.scratch_budget_bytes() / (int64_t)sizeof(double), (int64_t)1 << 22);
    size_t pos = 0;
    while (pos < mine.size()) {
      int64_t need = 0;
      size_t end = pos;
      while (end < mine.size()) {
        const Unit& u = units[mine[end]];
        int64_t v = u.nrows * (int64_t)B->p[u.b];
        if (end > pos && need + v > budget) break;
        units[mine[end]].v_off = need;
        need += v;
        end++;
      }
      DevBuf<double> V(std::max<int64_t>(need, 1), st);
      trace.mark("valloc");
      std::vector<TileUnit> tu;
      std::vector<GemmDesc> gd;
      for (size_t j = pos; j < end; j++) {
        const Unit& u = units[mine[j]];
        const int b = u.b;
        const int32_t sb = (int32_t)S(b), pb = B->p[b];
        int64_t roff = 0;
        for (auto& rg : u.rows) {
          make_tile_units(tu, rg.first, (int32_t)(rg.second - rg.first), tree->begin[b], sb, B->W.p + B->w_off[b],
                          sb, pb, V.p + u.v_off + roff * pb, pb, 0, dp);
          roff += rg.second - rg.first;
        }
        for (int64_t i : unit_pieces[mine[j]]) {
          int64_t k = pieces[i].blk;
          int a = A[k];
          int64_t lo = std::max(tree->begin[a], u.chunk * CH), hi = std::min(tree->end[a], (u.chunk + 1) * CH);
          // row offset of [lo, hi) inside this unit's compact V rows
          int64_t off = 0;
          for (auto& rg : u.rows) {
            if (lo >= rg.first && hi <= rg.second) {
              off += lo - rg.first;
              break;
            }
            off += rg.second - rg.first;
          }
          const int32_t pa = B->p[a];
          GemmDesc g{B->W.p + B->w_off[a] + (lo - tree->begin[a]), S(a), V.p + u.v_off + off * pb, pb, piece_dst(i),
                     (int64_t)B->p[pairs[k].second], pa, pb, (int32_t)(hi - lo), swap[k] ? 1 : 0};
          gd.push_back(g);
        }
      }
      trace.mark("units");
      run_tile_contract(c, tree, kp, tu, "assemble_tile_contract");
      trace.mark("k5a_launch");
      gemm_batched(c, gd, "assemble_wa_gemm");
      trace.mark("k5b_launch");
      pos = end;
    }
    // nested units, one row chunk at a time: (1) the leaves' scaling sums S_l = C(X_rows, X_l)
    // Phi_l^T on the fused tile kernel, (2) bottom-up [S_c | V_c] = [S_cL S_cR] Q_c on the batched
    // GEMM (level by level), (3) the pieces W_a V_b[rows] of every block with an internal b.
    // S and V hold one M-column slot per heap node (node q at column q M, ld = n_nodes M).
    if (nested) {
      const int M = B->M;
      const int64_t ld = nn * (int64_t)M;
      DevBuf<double> Sb, Vb;
      // leaf runs streamed by one unit each (segmented K5a: consecutive heap indices, equal sizes
      // that are multiples of 8, consecutive point ranges), G leaves per unit so a row chunk
      // still spreads over >= 4 x 148 x 4 tasks; the others one unit per leaf
      std::vector<int> leaves;
      for (int64_t q = 0; q < nn; q++)
        if (tree->state[q] == 1) leaves.push_back((int)q);
      std::sort(leaves.begin(), leaves.end(), [&](int x, int y) { return tree->begin[x] < tree->begin[y]; });
      DevBuf<double> phi_all;
      bool seg_ok = !leaves.empty();
      for (size_t i = 0; i < leaves.size() && seg_ok; i++) {
        seg_ok = S(leaves[i]) == S(leaves[0]) && S(leaves[0]) % 8 == 0 &&
                 (i == 0 || (leaves[i] == leaves[i - 1] + 1 && tree->begin[leaves[i]] == tree->end[leaves[i - 1]]));
      }
      if (seg_ok) {
        phi_all.alloc((size_t)M * tree->n, st);
        std::vector<int64_t> off, beg;
        std::vector<int32_t> sz;
        for (int q : leaves) {
          off.push_back(B->phi_off[q]);
          beg.push_back(tree->begin[q]);
          sz.push_back((int32_t)S(q));
        }
        DevBuf<int64_t> off_d(off.size(), st), beg_d(beg.size(), st);
        DevBuf<int32_t> sz_d(sz.size(), st);
        off_d.upload(off);
        beg_d.upload(beg);
        sz_d.upload(sz);
        k_phi_all<<<dim3(8, (unsigned)leaves.size()), 256, 0, st>>>(B->Phi.p, off_d.p, beg_d.p, sz_d.p, M, tree->n,
                                                                    phi_all.p);
        check_launch("k_phi_all");
      }
      for (size_t ui = 0; ui < units.size(); ui++) {
        const Unit& u = units[ui];
        if (u.b >= 0 || u.owner != c.rank) continue;
        const int64_t lo = u.rows[0].first, rows = u.nrows;
        if (Sb.n < (size_t)(rows * ld)) {
          Sb.alloc((size_t)(rows * ld), st);
          Vb.alloc((size_t)(rows * ld), st);
        }
        std::vector<TileUnit> tu;
        if (seg_ok) {
          const int64_t want = (int64_t)4 * num_sms(c.device) * 4;
          int64_t G = 1;
          while (2 * G <= (int64_t)leaves.size() && ceil_div(rows, 32) * ((int64_t)leaves.size() / (2 * G)) >= want)
            G *= 2;
          const int32_t sl = (int32_t)S(leaves[0]);
          for (size_t i = 0; i < leaves.size(); i += (size_t)G) {
            const int nl = (int)std::min<int64_t>(G, (int64_t)leaves.size() - (int64_t)i);
            const int64_t b0 = tree->begin[leaves[i]];
            const size_t first = tu.size();
            make_tile_units(tu, lo, (int32_t)rows, b0, sl * nl, phi_all.p + b0, tree->n, M, Sb.p + leaves[i] * M, ld,
                            0, dp);
            for (size_t j = first; j < tu.size(); j++) {
              tu[j].seg = sl;
              tu[j].seg_off = M;
              tu[j].w_cols = tree->n - b0;
            }
          }
        } else {
          for (int q : leaves) {
            const int32_t sl = (int32_t)S(q);
            make_tile_units(tu, lo, (int32_t)rows, tree->begin[q], sl, B->Phi.p + B->phi_off[q], sl, M, Sb.p + q * M,
                            ld, 0, dp);
          }
        }
        run_tile_contract(c, tree, kp, tu, "assemble_tile_nested");
        trace.mark("nested_k5a");
        // per internal cell and 64-row block of the chunk: does some row of it need V_c?
        const int64_t nblk = ceil_div(rows, 64);
        std::vector<uint8_t> vflag;
        std::vector<int64_t> vflag_off(nn, -1);
        for (int64_t q = 0; q < nn; q++) {
          if (tree->state[q] != 0) continue;
          vflag_off[q] = (int64_t)vflag.size();
          vflag.resize(vflag.size() + nblk, 0);
          auto it = nested_rows.find((int)q);
          if (it == nested_rows.end()) continue;
          for (auto& rg : it->second) {
            const int64_t a0 = std::max(rg.first, lo), a1 = std::min(rg.second, lo + rows);
            for (int64_t bk = (a0 - lo) / 64; a0 < a1 && bk <= (a1 - 1 - lo) / 64; bk++) vflag[vflag_off[q] + bk] = 1;
          }
        }
        DevBuf<uint8_t> vflag_d(std::max<size_t>(vflag.size(), 1), st);
        vflag_d.upload(vflag);
        if (trace.on && ui == 0) {  // V_c blocks per level (MLK_TRACE)
          for (int dep = 0; dep < tree->t; dep++) {
            int64_t on = 0, tot = 0;
            for (int64_t q = (1 << dep) - 1; q < (2 << dep) - 1 && q < nn; q++) {
              if (vflag_off[q] < 0) continue;
              for (int64_t bk = 0; bk < nblk; bk++) on += vflag[vflag_off[q] + bk];
              tot += nblk;
            }
            std::fprintf(stderr, "[mlk] nested chunk 0 level %d: V_c needed in %lld of %lld 64-row blocks\n", dep,
                         (long long)on, (long long)tot);
          }
        }
        for (int dep = tree->t - 1; dep >= 0; dep--) {
          std::vector<GemmDesc> gd;
          std::vector<std::array<const double*, 4>> tj;
          std::vector<const uint8_t*> tf;
          for (int64_t q = (1 << dep) - 1; q < (2 << dep) - 1 && q < nn; q++) {
            if (tree->state[q] != 0) continue;
            const double* Sch = Sb.p + (2 * q + 1) * M;  // [S_cL S_cR]: rows x 2M, adjacent slots
            const double* Q = B->Qm.p + B->q_off[q];      // 2M x 2M row-major
            if (transfer_kernel_ok(M)) {
              tj.push_back({Sch, Q, q > 0 ? Sb.p + q * M : nullptr, Vb.p + q * M});
              tf.push_back(vflag_d.p + vflag_off[q]);
            } else {
              if (q > 0) gd.push_back(GemmDesc{Sch, ld, Q, 2 * M, Sb.p + q * M, ld, (int32_t)rows, M, 2 * M, 0});
              gd.push_back(GemmDesc{Sch, ld, Q + M, 2 * M, Vb.p + q * M, ld, (int32_t)rows, M, 2 * M, 0});
            }
          }
          transfer_level(c, tj, tf, M, rows, ld);
          if (!gd.empty()) gemm_batched(c, gd, "assemble_transfer_gemm");
        }
        trace.mark("nested_transfer");
        std::vector<GemmDesc> gd;
        for (int64_t i = 0; i < npc; i++) {
          if (pieces[i].unit != (int)ui) continue;
          const int64_t k = pieces[i].blk;
          const int a = A[k], b = Bc[k];
          const int64_t ch = pieces[i].chunk;  // the piece's CH-row chunk inside this unit
          const int64_t plo = std::max(tree->begin[a], ch * CH), phi = std::min(tree->end[a], (ch + 1) * CH);
          GemmDesc g{B->W.p + B->w_off[a] + (plo - tree->begin[a]), S(a), Vb.p + (plo - lo) * ld + (int64_t)b * M, ld,
                     piece_dst(i), (int64_t)B->p[pairs[k].second], B->p[a], M, (int32_t)(phi - plo), swap[k] ? 1 : 0};
          gd.push_back(g);
        }
        gemm_batched(c, gd, "assemble_wa_gemm");
        trace.mark("nested_k5b");
      }
    }
  }
  // piece structure on the device; nranks == 1: reduce the multi-piece blocks now
  cw->val_off_d.alloc(nb + 1, st);
  cw->val_off_d.upload(cw->val_off);
  cw->piece_ptr_d.alloc(nb + 1, st);
  cw->piece_ptr_d.upload(cw->piece_ptr);
  cw->piece_off_d.alloc(std::max<int64_t>(npc, 1), st);
  cw->piece_off_d.upload(cw->piece_off);
  cw->piece_owner_d.alloc(std::max<int64_t>(npc, 1), st);
  cw->piece_owner_d.upload(cw->piece_owner);
  cw->reduce_d.alloc(std::max<size_t>(cw->reduce_blocks.size(), 1), st);
  cw->reduce_d.upload(cw->reduce_blocks);
  if (c.nranks == 1 && !cw->reduce_blocks.empty()) {
    TimedLaunch tl(c, "assemble_piece_reduce");
    reduce_pieces(c, cw.get(), cw->shard.p);
  }
  CUDA_CHECK(cudaStreamSynchronize(st));
  trace.mark("sync");
  cw->complete = c.nranks == 1;
  // device structure for the BSR matvec
  cw->brow_d.alloc(std::max<int64_t>(nb, 1), st);
  cw->brow_d.upload(cw->brow);
  cw->bcol_d.alloc(std::max<int64_t>(nb, 1), st);
  cw->bcol_d.upload(cw->bcol);
  cw->owner_d.alloc(std::max<int64_t>(nb, 1), st);
  cw->owner_d.upload(cw->owner);
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
  trace.mark("structure");
  if (gather != MLK_GATHER_NONE && c.nranks > 1) {
    gather_values(c, cw.get(), nullptr);
    trace.mark("gather");
  }
  *out = cw.release();
  MLK_API_END
}

void mlk_cw_free(mlk_cw cw) {
  if (!cw) return;
  cudaSetDevice(cw->device);
  // the creating context's stream may already be gone: drain the device, free on stream 0
  cudaDeviceSynchronize();
  cw->values.s = nullptr;
  if (cw->hvals) cudaFreeHost(cw->hvals);
  cw->hvals = nullptr;
  cw->shard.s = nullptr;
  cw->brow_d.s = nullptr;
  cw->bcol_d.s = nullptr;
  cw->owner_d.s = nullptr;
  cw->val_off_d.s = nullptr;
  cw->piece_ptr_d.s = nullptr;
  cw->piece_off_d.s = nullptr;
  cw->piece_owner_d.s = nullptr;
  cw->reduce_d.s = nullptr;
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
  MLK_REQUIRE(!values || cw->complete, "values are complete only after mlk_cw_unpack (nranks > 1)");
  if (values && cw->nnz > 0) CUDA_CHECK(cudaMemcpy(values, cw->vals(), sizeof(double) * cw->nnz, cudaMemcpyDefault));
  MLK_API_END
}

mlk_status mlk_cw_export_async(mlk_ctx ctx, mlk_cw cw, double* values) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && cw && values, "NULL argument");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  MLK_REQUIRE(cw->device == c.device, "cw lives on another device");
  if (!c.copy_stream) {
    CUDA_CHECK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&c.copy_ready, cudaEventDisableTiming));
  }
  CUDA_CHECK(cudaEventRecord(c.copy_ready, c.stream));
  CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, c.copy_ready, 0));
  if (cw->nnz > 0)
    CUDA_CHECK(cudaMemcpyAsync(values, cw->vals(), sizeof(double) * cw->nnz, cudaMemcpyDefault, c.copy_stream));
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

mlk_status mlk_cw_plan(mlk_cw cw, int32_t* nested, double* transfer_flops, double* nested_tile_flops) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw, "cw is NULL");
  if (nested) *nested = cw->nested ? 1 : 0;
  if (transfer_flops) *transfer_flops = cw->f_tr;
  if (nested_tile_flops) *nested_tile_flops = cw->f_nested_k5a;
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
  const double* src = cw->shard.p;
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
  if (cw->nranks > 1) gather_values(c, cw, gathered);
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  cw->complete = true;
  MLK_API_END
}

mlk_status mlk_cw_export_pieces(mlk_cw cw, int64_t* piece_ptr, int64_t* piece_off, int32_t* piece_owner,
                                double* shard) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw, "cw is NULL");
  CUDA_CHECK(cudaSetDevice(cw->device));
  if (piece_ptr) std::copy(cw->piece_ptr.begin(), cw->piece_ptr.end(), piece_ptr);
  if (piece_off) std::copy(cw->piece_off.begin(), cw->piece_off.end(), piece_off);
  if (piece_owner) std::copy(cw->piece_owner.begin(), cw->piece_owner.end(), piece_owner);
  if (shard && cw->shard_len > 0)
    CUDA_CHECK(cudaMemcpy(shard, cw->shard.p, sizeof(double) * cw->shard_len, cudaMemcpyDefault));
  MLK_API_END
}

mlk_status mlk_cw_values_device(mlk_cw cw, double** values) {
  MLK_API_BEGIN
  MLK_REQUIRE(cw && values, "NULL argument");
  *values = cw->vals();
  MLK_API_END
}

}  // extern "C"
