// mlk_loglik: the level-truncated multi-level log-likelihood of P:1954-1971 (the survey's
// NEXT-4),
//   l~^n_W = -N~/2 log(2 pi) - 1/2 log det C~^n_W - 1/2 (Z^n_W)^T (C~^n_W)^-1 Z^n_W,
// C~^n_W = the upper-left N~ x N~ block of the assembled sparse C~_W (the cells of levels
// t .. n, a prefix of the C_W order), through a Cholesky factor G G^T = C~^n_W with
// log det = 2 sum log G_ii and the quadratic form from the same factor.
//
// The factorisation is a block-sparse right-looking Cholesky over the BSR cells: symbolic fill
// on the host (block pattern of the factor's rows), then per block row j (in C_W order)
//   1. L_jj = chol(A^_jj) and Linv = L_jj^-1                   (one CTA each)
//   2. T_jk = Linv A^_jk for the k in the row's pattern, y_j = Linv z^_j   (one DMMA GEMM batch)
//   3. A^_kl -= T_jk^T T_jl (k <= l in the pattern), z^_k -= T_jk^T y_j   (one DMMA GEMM batch)
// T_j* is the block row j of G^T and is discarded after its step; y = G^-1 Z^n_W, so the
// quadratic form is |y|^2.  Every update of a block happens in its own step, in row order:
// deterministic.  The paper reorders with nested dissection before a sparse Cholesky (SuiteSparse);
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

// in-place lower Cholesky of one symmetric p x p block (row-major; the strict upper triangle is
// zeroed), non-positive pivot -> flag; logd = sum log L_ii (fixed order)
__global__ void __launch_bounds__(kLlThreads) k_ll_chol(double* __restrict__ A, int p, int* __restrict__ flag,
                                                        double* __restrict__ logd) {
  const int tid = threadIdx.x, nt = blockDim.x;
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
    for (int j = k + 1 + tid; j < p; j += nt) {
      const double ljk = A[(int64_t)j * p + k];
      for (int i = j; i < p; i++) A[(int64_t)i * p + j] = fma(-A[(int64_t)i * p + k], ljk, A[(int64_t)i * p + j]);
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
    *logd = s;
  }
}

// X = L^-1 for a lower-triangular p x p L (row-major): thread per column c, forward
// substitution of L x = e_c; X's strict upper triangle is zero
__global__ void __launch_bounds__(kLlThreads) k_ll_trinv(const double* __restrict__ L, int p,
                                                         double* __restrict__ X) {
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    for (int i = 0; i < c; i++) X[(int64_t)i * p + c] = 0.0;
    for (int i = c; i < p; i++) {
      double s = i == c ? 1.0 : 0.0;
      for (int k = c; k < i; k++) s = fma(-L[(int64_t)i * p + k], X[(int64_t)k * p + c], s);
      X[(int64_t)i * p + c] = s / L[(int64_t)i * p + i];
    }
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
  int pmax = 0;
  int64_t rowmax = 0;
  for (int j = 0; j < K; j++) {
    pmax = std::max(pmax, p[j]);
    int64_t r = 0;
    for (int k : pat[j]) r += (int64_t)p[j] * p[k];
    rowmax = std::max(rowmax, r);
  }
  DevBuf<double> Linv((size_t)pmax * pmax, st), T((size_t)std::max<int64_t>(rowmax, 1), st);

  for (int j = 0; j < K; j++) {
    const int pj = p[j];
    double* Ajj = Ah.p + diag_off[j];
    {
      TimedLaunch tl(c, "loglik_diag_chol");
      k_ll_chol<<<1, kLlThreads, 0, st>>>(Ajj, pj, flag.p, logd.p + j);
      check_launch("k_ll_chol");
      k_ll_trinv<<<1, kLlThreads, 0, st>>>(Ajj, pj, Linv.p);
      check_launch("k_ll_trinv");
    }
    const double* zj = zh.p + basis->row_off[j];
    double* yj = y.p + basis->row_off[j];
    std::vector<GemmDesc> g1, g2;
    std::vector<std::pair<int, int64_t>> trow;  // (k, offset of T_jk in T)
    int64_t to = 0;
    for (int k : pat[j]) {
      trow.push_back({k, to});
      to += (int64_t)pj * p[k];
    }
    // 2. T_jk = Linv A^_jk, y_j = Linv z^_j
    for (auto& tk : trow) {
      const int k = tk.first;
      g1.push_back(GemmDesc{Linv.p, pj, Ah.p + boff[j][k], p[k], T.p + tk.second, p[k], pj, p[k], pj, 0});
    }
    g1.push_back(GemmDesc{Linv.p, pj, zj, 1, yj, 1, pj, 1, pj, 0});
    gemm_batched(c, g1, "loglik_rowsolve");
    // 3. A^_kl -= T_jk^T T_jl (k <= l), z^_k -= T_jk^T y_j
    for (size_t a = 0; a < trow.size(); a++) {
      const int k = trow[a].first;
      for (size_t b = a; b < trow.size(); b++) {
        const int l = trow[b].first;
        double* dst = k == l ? Ah.p + diag_off[k] : Ah.p + boff[k][l];
        GemmDesc g{T.p + trow[a].second, p[k], T.p + trow[b].second, p[l], dst, p[l], p[k], p[l], pj, 0};
        g.sub = 1;
        g.trans_a = 1;
        g2.push_back(g);
      }
      GemmDesc gz{T.p + trow[a].second, p[k], yj, 1, zh.p + basis->row_off[k], 1, p[k], 1, pj, 0};
      gz.sub = 1;
      gz.trans_a = 1;
      g2.push_back(gz);
    }
    gemm_batched(c, g2, "loglik_update");
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
