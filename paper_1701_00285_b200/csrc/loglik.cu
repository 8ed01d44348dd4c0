// mlk_loglik: the level-truncated multi-level log-likelihood of P:1954-1971 (the survey's
// NEXT-4),
//   l~^n_W = -N~/2 log(2 pi) - 1/2 log det C~^n_W - 1/2 (Z^n_W)^T (C~^n_W)^-1 Z^n_W,
// C~^n_W = the upper-left N~ x N~ block of the assembled sparse C~_W (the cells of levels
// t .. n, a prefix of the C_W order), through a Cholesky factor G G^T = C~^n_W with
// log det = 2 sum log G_ii and the quadratic form from the same factor.
//
// The factorisation is a block-sparse right-looking Cholesky over the BSR cells: symbolic fill
// on the host (block pattern of the factor's rows), then, for each wave of consecutive block
// rows none of which is in another's pattern (e.g. the leaves not joined by extra pairs),
//   1. L_jj = chol(A^_jj) and Linv_j = L_jj^-1                 (one CTA per row, batched)
//   2. T_jk = Linv_j A^_jk for the k in row j's pattern, y_j = Linv_j z^_j   (one GEMM batch)
//   3. partials T_jk^T T_jl (k <= l) and T_jk^T y_j             (one DMMA GEMM batch, TN mode)
//   4. A^_kl -= the partials of (k, l) summed in row order, z^_k likewise (one kernel)
// T_j* is the block row j of G^T and is discarded after its wave; y = G^-1 Z^n_W, so the
// quadratic form is |y|^2.  Fixed summation orders throughout: deterministic.  The paper reorders with nested dissection before a sparse Cholesky (SuiteSparse);
// the C_W order (finest level first, root last) already eliminates the leaves first, whose fill
// stays among their ancestors (mutually admitted) except for the extra pairs of the tau search.
#include <algorithm>
#include <cmath>
#include <map>
#include <set>

#include "api.cuh"

namespace mlk {
namespace {

constexpr int kLlThreads = 256;

struct DiagJob {
  double* A;      // p x p symmetric block (row-major), factored in place (lower)
  double* Linv;   // p x p output: L^-1
  int32_t p, row; // size; block row (index into logd)
};

// in-place lower Cholesky of one symmetric p x p block per CTA (row-major; the strict upper
// triangle is zeroed), non-positive pivot -> flag; logd[row] = sum log L_ii (fixed order).  The
// trailing update is spread over all threads (element-wise), three barriers per column.
__global__ void __launch_bounds__(kLlThreads) k_ll_chol(const DiagJob* __restrict__ jobs, int* __restrict__ flag,
                                                        double* __restrict__ logd) {
  const DiagJob jb = jobs[blockIdx.x];
  double* A = jb.A;
  const int p = jb.p, tid = threadIdx.x, nt = blockDim.x;
  __shared__ double s_d;
  for (int k = 0; k < p; k++) {
    if (tid == 0) {
      const double akk = A[(int64_t)k * p + k];
      if (!(akk > 0.0)) atomicExch(flag, 1);
      s_d = akk > 0.0 ? sqrt(akk) : 1.0;
      A[(int64_t)k * p + k] = s_d;
    }
    __syncthreads();
    const double inv = 1.0 / s_d;
    for (int i = k + 1 + tid; i < p; i += nt) A[(int64_t)i * p + k] *= inv;
    __syncthreads();
    // A[i][j] -= A[i][k] A[j][k] for k < j <= i < p: the (p-k-1)(p-k)/2 elements, row-major
    const int m = p - k - 1;
    for (int e = tid; e < m * (m + 1) / 2; e += nt) {
      int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);  // row of the packed lower triangle
      while (i * (i + 1) / 2 > e) i--;
      while ((i + 1) * (i + 2) / 2 <= e) i++;
      const int j = e - i * (i + 1) / 2;
      const int gi = k + 1 + i, gj = k + 1 + j;
      A[(int64_t)gi * p + gj] = fma(-A[(int64_t)gi * p + k], A[(int64_t)gj * p + k], A[(int64_t)gi * p + gj]);
    }
    __syncthreads();
  }
  for (int64_t e = tid; e < (int64_t)p * p; e += nt) {
    const int i = (int)(e / p), j = (int)(e - (int64_t)i * p);
    if (j > i) A[e] = 0.0;
  }
  if (tid == 0) {
    double s = 0.0;
    for (int i = 0; i < p; i++) s += log(A[(int64_t)i * p + i]);
    logd[jb.row] = s;
  }
}

// Linv = L^-1 for the lower-triangular L of each job (row-major): thread per column c, forward
// substitution of L x = e_c; the strict upper triangle of Linv is zero
__global__ void __launch_bounds__(kLlThreads) k_ll_trinv(const DiagJob* __restrict__ jobs) {
  const DiagJob jb = jobs[blockIdx.x];
  const double* L = jb.A;
  double* X = jb.Linv;
  const int p = jb.p;
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    for (int i = 0; i < c; i++) X[(int64_t)i * p + c] = 0.0;
    for (int i = c; i < p; i++) {
      double s = i == c ? 1.0 : 0.0;
      for (int k = c; k < i; k++) s = fma(-L[(int64_t)i * p + k], X[(int64_t)k * p + c], s);
      X[(int64_t)i * p + c] = s / L[(int64_t)i * p + i];
    }
  }
}

// target -= sum of its partials in row order (one CTA per target; partials of one target are
// consecutive in `part`, `len` doubles each)
struct RedJob {
  double* dst;
  int64_t first, len;
  int32_t count;
};
__global__ void k_ll_reduce(const RedJob* __restrict__ jobs, const double* __restrict__ part) {
  const RedJob jb = jobs[blockIdx.x];
  for (int64_t e = threadIdx.x; e < jb.len; e += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < jb.count; r++) s += part[jb.first + (int64_t)r * jb.len + e];
    jb.dst[e] -= s;
  }
}

struct CopyJob {
  int64_t src, dst, len;
};
__global__ void k_ll_copy(const CopyJob* __restrict__ jobs, const double* __restrict__ src, double* __restrict__ dst) {
  const CopyJob jb = jobs[blockIdx.x];
  for (int64_t e = threadIdx.x; e < jb.len; e += blockDim.x) dst[jb.dst + e] = src[jb.src + e];
}

// out = [loglik, logdet, quad]: fixed-order sums of the per-row log-diagonals and of y^2
__global__ void k_ll_finish(const double* __restrict__ logd, int K, const double* __restrict__ y, int64_t nt,
                            double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double ld = 0.0, q = 0.0;
  for (int j = 0; j < K; j++) ld += logd[j];
  for (int64_t i = 0; i < nt; i++) q = fma(y[i], y[i], q);
  ld *= 2.0;
  out[0] = -0.5 * (double)nt * 1.8378770664093454836 - 0.5 * ld - 0.5 * q;  // log(2 pi)
  out[1] = ld;
  out[2] = q;
}

}  // namespace
}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_loglik(mlk_ctx ctx, mlk_basis basis, mlk_cw cw, int32_t level, const double* z_w, double* loglik,
                      double* logdet, double* quad, int64_t* n_tilde) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && basis && cw && z_w, "NULL argument");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  MLK_REQUIRE(c.nranks == 1, "mlk_loglik needs nranks == 1");
  MLK_REQUIRE(cw->complete, "the likelihood needs the complete BSR values");
  MLK_REQUIRE(cw->n_cells == (int32_t)basis->cells.size(), "cw does not match the basis");
  const mlk_tree_s* tree = basis->tree;
  MLK_REQUIRE(level >= 0 && level <= tree->t, "need 0 <= level <= t");
  cudaStream_t st = c.stream;
  // truncation: the cells of depth >= level form a prefix of the C_W order
  int K = 0;
  while (K < cw->n_cells && tree->depth[basis->cells[K]] >= level) K++;
  const int64_t nt = basis->row_off[K];
  if (n_tilde) *n_tilde = nt;
  MLK_REQUIRE(K > 0 && nt > 0, "empty truncation");
  std::vector<int32_t> p(K);
  for (int j = 0; j < K; j++) p[j] = (int32_t)(basis->row_off[j + 1] - basis->row_off[j]);

  // ---- symbolic: block pattern of every row of the factor (columns k > j), with fill
  std::vector<std::set<int>> pat(K);
  std::vector<std::pair<int64_t, std::pair<int, int>>> stored;  // (value offset, (r, c)) of A's blocks
  for (int r = 0; r < K; r++)
    for (int32_t k = cw->brow_ptr[r]; k < cw->brow_ptr[r + 1]; k++) {
      const int cc = cw->bcol[k];
      if (cc >= K) continue;
      if (cc > r) pat[r].insert(cc);
      stored.push_back({cw->val_off[k], {r, cc}});
    }
  for (int j = 0; j < K; j++) {
    std::vector<int> row(pat[j].begin(), pat[j].end());
    for (size_t a = 0; a < row.size(); a++)
      for (size_t b = a + 1; b < row.size(); b++) pat[row[a]].insert(row[b]);
  }
  // storage of A^ (the working copy): diagonal blocks and the pattern blocks, row-major
  std::vector<int64_t> diag_off(K);
  std::vector<std::map<int, int64_t>> boff(K);
  int64_t tot = 0;
  for (int j = 0; j < K; j++) {
    diag_off[j] = tot;
    tot += (int64_t)p[j] * p[j];
    for (int k : pat[j]) {
      boff[j][k] = tot;
      tot += (int64_t)p[j] * p[k];
    }
  }
  DevBuf<double> Ah((size_t)std::max<int64_t>(tot, 1), st);
  Ah.zero();
  {
    std::vector<CopyJob> cj;
    for (auto& s : stored) {
      const int r = s.second.first, cc = s.second.second;
      cj.push_back({s.first, r == cc ? diag_off[r] : boff[r][cc], (int64_t)p[r] * p[cc]});
    }
    DevBuf<CopyJob> cjd(cj.size(), st);
    cjd.upload(cj);
    k_ll_copy<<<(unsigned)cj.size(), 256, 0, st>>>(cjd.p, cw->vals(), Ah.p);
    check_launch("k_ll_copy");
  }
  DevIn<double> zin(z_w, (size_t)basis->dim, st);
  DevBuf<double> zh((size_t)nt, st), y((size_t)nt, st), logd((size_t)K, st), res(3, st);
  CUDA_CHECK(cudaMemcpyAsync(zh.p, zin.p, sizeof(double) * nt, cudaMemcpyDeviceToDevice, st));
  DevBuf<int> flag(1, st);
  flag.zero();
  // ---- numeric, in waves: consecutive block rows none of which appears in another's pattern
  // (so no row of a wave updates another) are factored together; their updates go to per-row
  // partials that are subtracted from each target in row order (deterministic)
  std::vector<std::pair<int, int>> waves;  // [first, last) rows
  {
    int w0 = 0;
    std::set<int> touched;  // rows updated by the current wave
    const int64_t cap = std::max<int64_t>(c.scratch_budget_bytes() / 8 / 4, (int64_t)1 << 20);  // doubles
    int64_t wbytes = 0;
    for (int j = 0; j < K; j++) {
      int64_t need = (int64_t)p[j] * p[j];
      for (int k : pat[j]) need += (int64_t)p[j] * p[k] + (int64_t)p[k];
      for (int k : pat[j])
        for (int l : pat[j])
          if (k <= l) need += (int64_t)p[k] * p[l];
      if (j > w0 && (touched.count(j) || wbytes + need > cap)) {
        waves.push_back({w0, j});
        w0 = j;
        touched.clear();
        wbytes = 0;
      }
      wbytes += need;
      for (int k : pat[j]) touched.insert(k);
    }
    waves.push_back({w0, K});
  }
  for (auto& wv : waves) {
    const int j0 = wv.first, j1 = wv.second;
    // scratch layout: Linv per row, T_jk per (row, pattern column), partials per target
    std::vector<DiagJob> dj;
    std::vector<GemmDesc> g1, g2;
    std::map<std::pair<int, int>, std::vector<int64_t>> tpart;  // target (k, l) -> partial offsets
    std::map<int, std::vector<int64_t>> zpart;                  // k -> z partial offsets
    int64_t off = 0;
    std::vector<int64_t> linv_off(j1 - j0);
    std::vector<std::vector<std::pair<int, int64_t>>> trow(j1 - j0);
    for (int j = j0; j < j1; j++) {
      linv_off[j - j0] = off;
      off += (int64_t)p[j] * p[j];
      for (int k : pat[j]) {
        trow[j - j0].push_back({k, off});
        off += (int64_t)p[j] * p[k];
      }
    }
    const int64_t part0 = off;
    for (int j = j0; j < j1; j++)
      for (size_t a = 0; a < trow[j - j0].size(); a++) {
        const int k = trow[j - j0][a].first;
        for (size_t b = a; b < trow[j - j0].size(); b++) {
          const int l = trow[j - j0][b].first;
          tpart[{k, l}].push_back(off);
          off += (int64_t)p[k] * p[l];
        }
        zpart[k].push_back(off);
        off += p[k];
      }
    // partials of one target must be consecutive: lay them out target by target
    std::map<int64_t, int64_t> remap;  // provisional offset -> final offset
    {
      int64_t o2 = part0;
      for (auto& kv : tpart)
        for (int64_t x : kv.second) {
          remap[x] = o2;
          o2 += (int64_t)p[kv.first.first] * p[kv.first.second];
        }
      for (auto& kv : zpart)
        for (int64_t x : kv.second) {
          remap[x] = o2;
          o2 += p[kv.first];
        }
    }
    DevBuf<double> S((size_t)std::max<int64_t>(off, 1), st);
    for (int j = j0; j < j1; j++)
      dj.push_back({Ah.p + diag_off[j], S.p + linv_off[j - j0], p[j], j});
    DevBuf<DiagJob> djd(dj.size(), st);
    djd.upload(dj);
    {
      TimedLaunch tl(c, "loglik_diag_chol");
      k_ll_chol<<<(unsigned)dj.size(), kLlThreads, 0, st>>>(djd.p, flag.p, logd.p);
      check_launch("k_ll_chol");
      k_ll_trinv<<<(unsigned)dj.size(), kLlThreads, 0, st>>>(djd.p);
      check_launch("k_ll_trinv");
    }
    // 2. T_jk = Linv_j A^_jk, y_j = Linv_j z^_j
    for (int j = j0; j < j1; j++) {
      const int pj = p[j];
      const double* Lj = S.p + linv_off[j - j0];
      for (auto& tk : trow[j - j0])
        g1.push_back(GemmDesc{Lj, pj, Ah.p + boff[j][tk.first], p[tk.first], S.p + tk.second, p[tk.first], pj,
                              p[tk.first], pj, 0});
      g1.push_back(GemmDesc{Lj, pj, zh.p + basis->row_off[j], 1, y.p + basis->row_off[j], 1, pj, 1, pj, 0});
    }
    gemm_batched(c, g1, "loglik_rowsolve");
    // 3. partials T_jk^T T_jl (k <= l) and T_jk^T y_j, in the provisional (row-major) order
    {
      int64_t o = part0;
      for (int j = j0; j < j1; j++) {
        const int pj = p[j];
        auto& tr = trow[j - j0];
        for (size_t a = 0; a < tr.size(); a++) {
          const int k = tr[a].first;
          for (size_t b = a; b < tr.size(); b++) {
            const int l = tr[b].first;
            GemmDesc g{S.p + tr[a].second, p[k], S.p + tr[b].second, p[l], S.p + remap[o], p[l], p[k], p[l], pj, 0};
            g.trans_a = 1;
            g2.push_back(g);
            o += (int64_t)p[k] * p[l];
          }
          GemmDesc gz{S.p + tr[a].second, p[k], y.p + basis->row_off[j], 1, S.p + remap[o], 1, p[k], 1, pj, 0};
          gz.trans_a = 1;
          g2.push_back(gz);
          o += p[k];
        }
      }
    }
    gemm_batched(c, g2, "loglik_update");
    // 4. subtract the partials from their targets in row order
    std::vector<RedJob> rj;
    for (auto& kv : tpart) {
      const int k = kv.first.first, l = kv.first.second;
      double* dst = k == l ? Ah.p + diag_off[k] : Ah.p + boff[k][l];
      rj.push_back({dst, remap[kv.second.front()], (int64_t)p[k] * p[l], (int32_t)kv.second.size()});
    }
    for (auto& kv : zpart)
      rj.push_back({zh.p + basis->row_off[kv.first], remap[kv.second.front()], (int64_t)p[kv.first],
                    (int32_t)kv.second.size()});
    if (!rj.empty()) {
      DevBuf<RedJob> rjd(rj.size(), st);
      rjd.upload(rj);
      TimedLaunch tl(c, "loglik_reduce");
      k_ll_reduce<<<(unsigned)rj.size(), 256, 0, st>>>(rjd.p, S.p);
      check_launch("k_ll_reduce");
    }
  }
  k_ll_finish<<<1, 32, 0, st>>>(logd.p, K, y.p, nt, res.p);
  check_launch("k_ll_finish");
  double out[3];
  int fl = 0;
  CUDA_CHECK(cudaMemcpyAsync(out, res.p, sizeof(out), cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaMemcpyAsync(&fl, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaStreamSynchronize(st));
  if (fl) throw Error(MLK_ERR_RANK_DEFICIENT, "C~^n_W is not positive definite (non-positive Cholesky pivot)");
  if (loglik) *loglik = out[0];
  if (logdet) *logdet = out[1];
  if (quad) *quad = out[2];
  MLK_API_END
}

}  // extern "C"
