// mlk_build_basis: the multi-level basis (steps (a)-(f)) as a tree QR.
//  leaves:   P(X_leaf) (s x M monomials, graded TD order, reading R8) -> complete Householder
//            QR (LAPACK convention, reading R7): Phi = Q_1^T, W = Q_2^T, R.
//  internal: [R_L; R_R] (2M x M) -> complete QR; Phi = Q_1^T (Phi_L (+) Phi_R),
//            W = Q_2^T (Phi_L (+) Phi_R) by four DMMA GEMMs per cell (gemm.cu).
// The QR kernel runs one CTA per matrix (batched over the cells of a level).
#include <algorithm>
#include <cmath>
#include <memory>

#include "api.cuh"

namespace mlk {
namespace {

// graded total-degree exponent set as factor lists (coordinate indices, nondecreasing),
// degree 0 first, then combinations with replacement in lexicographic order (R8)
std::vector<std::vector<int>> td_factors(int d, int w) {
  std::vector<std::vector<int>> out;
  out.push_back({});
  for (int deg = 1; deg <= w; deg++) {
    std::vector<int> cur(deg, 0);
    while (true) {
      out.push_back(cur);
      int i = deg - 1;
      while (i >= 0 && cur[i] == d - 1) i--;
      if (i < 0) break;
      cur[i]++;
      for (int j = i + 1; j < deg; j++) cur[j] = cur[i];
    }
  }
  return out;
}

struct LeafJob {
  int64_t pt_begin;  // first tree position
  int32_t s;         // points
  int64_t a_off;     // offset of the s x M column-major monomial matrix in scratch
};

// monomial matrix P (s x M, column-major) of each leaf; a monomial is the left-to-right
// product of its factors (factor table fac[m * w + j], -1 padded)
__global__ void k_monomials(const double* __restrict__ Xt, int dp, const LeafJob* __restrict__ jobs,
                            const int32_t* __restrict__ fac, int M, int w, double* __restrict__ A) {
  const LeafJob jb = jobs[blockIdx.y];
  int64_t total = (int64_t)jb.s * M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int m = (int)(e / jb.s);
    int i = (int)(e % jb.s);
    const double* x = Xt + (jb.pt_begin + i) * dp;
    double v = 1.0;
    bool first = true;
    for (int j = 0; j < w; j++) {
      int f = fac[m * w + j];
      if (f < 0) break;
      v = first ? x[f] : v * x[f];
      first = false;
    }
    A[jb.a_off + (int64_t)m * jb.s + i] = v;
  }
}

struct QrJob {
  double* A;      // m x nc column-major (lda = m), overwritten by the Householder vectors
  int32_t m, nc;
  double* R;      // nc x nc row-major output
  double* qlo;    // columns j < nc of Q (each a contiguous row of length m at qlo + j*ldq)
  double* qhi;    // columns j >= nc of Q at qhi + (j - nc)*ldq
  int64_t ldq;
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; i++) s += red[i];
  return s;
}

__device__ __forceinline__ double* qcol(const QrJob& jb, int j) {
  return j < jb.nc ? jb.qlo + (int64_t)j * jb.ldq : jb.qhi + (int64_t)(j - jb.nc) * jb.ldq;
}

// Complete Householder QR of one matrix per CTA (LAPACK dgeqr2 + dorg2r conventions:
// beta = -sign(alpha) ||(alpha, x)||, tau = (beta - alpha) / beta, v = x / (alpha - beta),
// tau = 0 when x = 0).  Q = H_0 H_1 ... H_{nc-1} is formed explicitly.
__global__ void __launch_bounds__(256) k_qr(const QrJob* __restrict__ jobs, int* __restrict__ rank_flag) {
  extern __shared__ double sh[];
  __shared__ double s_scal;
  const QrJob jb = jobs[blockIdx.x];
  const int m = jb.m, nc = jb.nc;
  double* taus = sh;              // nc
  double* red = sh + nc;          // 32
  double* A = jb.A;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;

  for (int k = 0; k < nc; k++) {
    double* ak = A + (int64_t)k * m;
    double part = 0.0;
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) part = fma(ak[i], ak[i], part);
    double xn2 = block_sum(part, red);
    if (threadIdx.x == 0) {
      double alpha = ak[k];
      double tau = 0.0, scal = 1.0, beta = alpha;
      if (xn2 > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, xn2)), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      taus[k] = tau;
      s_scal = scal;
      ak[k] = beta;
    }
    __syncthreads();
    double scal = s_scal, tau = taus[k];
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) ak[i] *= scal;
    __syncthreads();
    if (tau != 0.0) {
      for (int j = k + 1 + warp; j < nc; j += nw) {
        double* aj = A + (int64_t)j * m;
        const double akj = aj[k];  // read before the warp reduction (lane 0 writes it after)
        double s = 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) s = fma(ak[i], aj[i], s);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        s += akj;
        double f = tau * s;
        if (lane == 0) aj[k] -= f;
        for (int i = k + 1 + lane; i < m; i += 32) aj[i] = fma(-f, ak[i], aj[i]);
      }
    }
    __syncthreads();
  }
  // R and the rank test (reading R9)
  for (int e = threadIdx.x; e < nc * nc; e += blockDim.x) {
    int i = e / nc, j = e % nc;
    jb.R[e] = j >= i ? A[(int64_t)j * m + i] : 0.0;
  }
  if (threadIdx.x == 0) {
    double mx = 0.0, mn = INFINITY;
    for (int i = 0; i < nc; i++) {
      double v = fabs(A[(int64_t)i * m + i]);
      mx = fmax(mx, v);
      mn = fmin(mn, v);
    }
    if (!(mn > 1e-13 * mx)) atomicExch(rank_flag, 1);
  }
  __syncthreads();
  // Q = I, then apply H_k for k = nc-1 .. 0 to columns k..m-1 (columns j < k stay e_j)
  for (int j = warp; j < m; j += nw) {
    double* q = qcol(jb, j);
    for (int i = lane; i < m; i += 32) q[i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = nc - 1; k >= 0; k--) {
    double tau = taus[k];
    if (tau == 0.0) continue;
    const double* ak = A + (int64_t)k * m;
    for (int j = k + warp; j < m; j += nw) {
      double* q = qcol(jb, j);
      const double qk = q[k];
      double s = 0.0;
      for (int i = k + 1 + lane; i < m; i += 32) s = fma(ak[i], q[i], s);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      s += qk;
      double f = tau * s;
      if (lane == 0) q[k] -= f;
      for (int i = k + 1 + lane; i < m; i += 32) q[i] = fma(-f, ak[i], q[i]);
    }
    __syncthreads();
  }
}

// [R_L; R_R] (2M x M, column-major) for every internal cell of a level
struct StackJob {
  const double* RL;
  const double* RR;
  double* A;
};
__global__ void k_stack_r(const StackJob* __restrict__ jobs, int M) {
  const StackJob jb = jobs[blockIdx.x];
  for (int e = threadIdx.x; e < 2 * M * M; e += blockDim.x) {
    int j = e / (2 * M), i = e % (2 * M);
    jb.A[e] = i < M ? jb.RL[i * M + j] : jb.RR[(i - M) * M + j];
  }
}

void run_qr(Ctx& c, const std::vector<QrJob>& jobs, int nc, int* flag, const char* name) {
  if (jobs.empty()) return;
  DevBuf<QrJob> dj(jobs.size(), c.stream);
  dj.upload(jobs);
  size_t smem = (size_t)(nc + 32) * sizeof(double);
  TimedLaunch tl(c, name);
  k_qr<<<(unsigned)jobs.size(), 256, smem, c.stream>>>(dj.p, flag);
  check_launch("k_qr");
}

}  // namespace
}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_build_basis(mlk_ctx ctx, mlk_tree tree, int32_t w, mlk_basis* out) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && tree && out, "NULL argument");
  *out = nullptr;
  MLK_REQUIRE(w >= 0 && w <= 16, "need 0 <= w <= 16");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  cudaStream_t st = c.stream;
  const int d = tree->d, dp = tree->d_pad, nn = tree->n_nodes;
  auto fac = td_factors(d, w);
  const int M = (int)fac.size();
  MLK_REQUIRE(M < tree->n, "need n > M = C(d + w, w)");
  MLK_REQUIRE(M <= 4096, "M > 4096 not supported");

  auto B = std::make_unique<mlk_basis_s>();
  B->device = c.device;
  B->M = M;
  B->w = w;
  B->tree = tree;
  B->p.assign(nn, 0);
  B->cell_pos.assign(nn, -1);
  B->w_off.assign(nn, -1);
  B->phi_off.assign(nn, -1);
  for (int q = 0; q < nn; q++) {
    if (tree->state[q] < 0) continue;
    int64_t s = tree->end[q] - tree->begin[q];
    if (tree->state[q] == 1) {
      if (s < M) throw Error(MLK_ERR_RANK_DEFICIENT, "leaf with fewer points than monomials");
      B->p[q] = (int32_t)(s - M);
    } else {
      B->p[q] = M;
    }
  }
  // C_W order: levels t..0, heap order within a level (R11)
  std::vector<int> order;
  for (int dep = tree->t; dep >= 0; dep--)
    for (int q = (1 << dep) - 1; q < (2 << dep) - 1 && q < nn; q++)
      if (tree->state[q] >= 0) order.push_back(q);
  int64_t woff = 0, phioff = 0, row = 0;
  B->row_off.push_back(0);
  for (int q : order) {
    int64_t s = tree->end[q] - tree->begin[q];
    B->w_off[q] = woff;
    woff += (int64_t)B->p[q] * s;
    B->phi_off[q] = phioff;
    phioff += (int64_t)M * s;
    if (B->p[q] > 0) {
      B->cell_pos[q] = (int32_t)B->cells.size();
      B->cells.push_back(q);
      row += B->p[q];
      B->row_off.push_back(row);
    }
  }
  B->dim = row;
  B->W.alloc(std::max<int64_t>(woff, 1), st);
  B->Phi.alloc(std::max<int64_t>(phioff, 1), st);
  DevBuf<double> Rbuf((size_t)nn * M * M, st);
  DevBuf<int> flag(1, st);
  flag.zero();

  // factor table
  int wf = std::max(w, 1);
  std::vector<int32_t> fh((size_t)M * wf, -1);
  for (int m = 0; m < M; m++)
    for (size_t j = 0; j < fac[m].size(); j++) fh[(size_t)m * wf + j] = fac[m][j];
  DevBuf<int32_t> facd(fh.size(), st);
  facd.upload(fh);

  HostTrace trace("basis");
  // ---- leaves
  {
    std::vector<LeafJob> lj;
    std::vector<QrJob> qj;
    int64_t aoff = 0;
    int32_t smax = 0;
    for (int q : order) {
      if (tree->state[q] != 1) continue;
      int32_t s = (int32_t)(tree->end[q] - tree->begin[q]);
      lj.push_back({tree->begin[q], s, aoff});
      aoff += (int64_t)s * M;
      smax = std::max(smax, s);
    }
    DevBuf<double> A(std::max<int64_t>(aoff, 1), st);
    DevBuf<LeafJob> ljd(lj.size(), st);
    ljd.upload(lj);
    {
      TimedLaunch tl(c, "basis_monomials");
      dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(64, ceil_div((int64_t)smax * M, 256))),
                (unsigned)lj.size());
      k_monomials<<<grid, 256, 0, st>>>(tree->Xt.p, dp, ljd.p, facd.p, M, wf, A.p);
      check_launch("k_monomials");
    }
    size_t k = 0;
    for (int q : order) {
      if (tree->state[q] != 1) continue;
      int32_t s = (int32_t)(tree->end[q] - tree->begin[q]);
      QrJob jb;
      jb.A = A.p + lj[k].a_off;
      jb.m = s;
      jb.nc = M;
      jb.R = Rbuf.p + (int64_t)q * M * M;
      jb.qlo = B->Phi.p + B->phi_off[q];
      jb.qhi = B->W.p + B->w_off[q];
      jb.ldq = s;
      qj.push_back(jb);
      k++;
    }
    run_qr(c, qj, M, flag.p, "basis_leaf_qr");
  }
  trace.mark("leaves");
  // ---- internal levels, bottom-up
  DevBuf<double> Qt;
  DevBuf<double> Ast;
  for (int dep = tree->t - 1; dep >= 0; dep--) {
    std::vector<int> cellsq;
    for (int q = (1 << dep) - 1; q < (2 << dep) - 1; q++)
      if (tree->state[q] == 0) cellsq.push_back(q);
    if (cellsq.empty()) continue;
    size_t nc = cellsq.size();
    Ast.alloc(nc * 2 * M * M, st);
    Qt.alloc(nc * 4 * (size_t)M * M, st);
    std::vector<StackJob> sj;
    std::vector<QrJob> qj;
    for (size_t i = 0; i < nc; i++) {
      int q = cellsq[i];
      sj.push_back({Rbuf.p + (int64_t)(2 * q + 1) * M * M, Rbuf.p + (int64_t)(2 * q + 2) * M * M,
                    Ast.p + i * 2 * M * M});
      QrJob jb;
      jb.A = Ast.p + i * 2 * M * M;
      jb.m = 2 * M;
      jb.nc = M;
      jb.R = Rbuf.p + (int64_t)q * M * M;
      jb.qlo = Qt.p + i * 4 * (size_t)M * M;       // Q column-major == Q^T row-major
      jb.qhi = jb.qlo + (size_t)M * 2 * M;
      jb.ldq = 2 * M;
      qj.push_back(jb);
    }
    DevBuf<StackJob> sjd(nc, st);
    sjd.upload(sj);
    {
      TimedLaunch tl(c, "basis_stack");
      k_stack_r<<<(unsigned)nc, 256, 0, st>>>(sjd.p, M);
      check_launch("k_stack_r");
    }
    run_qr(c, qj, M, flag.p, "basis_merge_qr");
    // Phi_q / W_q = (Q^T)[rows, cols of child] x Phi_child
    std::vector<GemmDesc> gd;
    for (size_t i = 0; i < nc; i++) {
      int q = cellsq[i];
      int l = 2 * q + 1, r = 2 * q + 2;
      int64_t s = tree->end[q] - tree->begin[q];
      int32_t nl = (int32_t)(tree->end[l] - tree->begin[l]), nr = (int32_t)(tree->end[r] - tree->begin[r]);
      const double* Qrow = Qt.p + i * 4 * (size_t)M * M;  // (Q^T)[i][c] at Qrow[i*2M + c]
      for (int half = 0; half < 2; half++) {
        const double* Pc = B->Phi.p + B->phi_off[half ? r : l];
        int32_t ncol = half ? nr : nl;
        int64_t coff = half ? nl : 0;
        GemmDesc g1{Qrow + (half ? M : 0), 2 * M, Pc, ncol, B->Phi.p + B->phi_off[q] + coff, s, M, ncol, M, 0};
        GemmDesc g2{Qrow + (int64_t)M * 2 * M + (half ? M : 0), 2 * M, Pc, ncol, B->W.p + B->w_off[q] + coff, s, M,
                    ncol, M, 0};
        gd.push_back(g1);
        gd.push_back(g2);
      }
    }
    gemm_batched(c, gd, "basis_transfer_gemm");
  }
  trace.mark("levels");
  auto fl = flag.download(1);
  trace.mark("sync");
  if (fl[0]) throw Error(MLK_ERR_RANK_DEFICIENT, "moment matrix is rank deficient (|R_kk| <= 1e-13 max|R_ii|)");
  CUDA_CHECK(cudaStreamSynchronize(st));
  *out = B.release();
  MLK_API_END
}

void mlk_basis_free(mlk_basis basis) {
  if (!basis) return;
  cudaSetDevice(basis->device);
  // the creating context's stream may already be gone: drain the device, free on stream 0
  cudaDeviceSynchronize();
  basis->W.s = nullptr;
  basis->Phi.s = nullptr;
  delete basis;
}

mlk_status mlk_basis_info(mlk_basis basis, int32_t* M, int64_t* dim, int32_t* n_cells) {
  MLK_API_BEGIN
  MLK_REQUIRE(basis, "basis is NULL");
  if (M) *M = basis->M;
  if (dim) *dim = basis->dim;
  if (n_cells) *n_cells = (int32_t)basis->cells.size();
  MLK_API_END
}

mlk_status mlk_basis_export(mlk_basis basis, int32_t* cells, int64_t* cell_row_off, int32_t node, double* W_block,
                            double* Phi_block, double* L) {
  MLK_API_BEGIN
  MLK_REQUIRE(basis, "basis is NULL");
  CUDA_CHECK(cudaSetDevice(basis->device));
  const mlk_tree_s* tree = basis->tree;
  if (cells) std::copy(basis->cells.begin(), basis->cells.end(), cells);
  if (cell_row_off) std::copy(basis->row_off.begin(), basis->row_off.end(), cell_row_off);
  if (node >= 0) {
    MLK_REQUIRE(node < tree->n_nodes && tree->state[node] >= 0, "node out of range");
    int64_t s = tree->end[node] - tree->begin[node];
    if (W_block && basis->p[node] > 0)
      CUDA_CHECK(cudaMemcpy(W_block, basis->W.p + basis->w_off[node], sizeof(double) * basis->p[node] * s,
                            cudaMemcpyDefault));
    if (Phi_block)
      CUDA_CHECK(cudaMemcpy(Phi_block, basis->Phi.p + basis->phi_off[node], sizeof(double) * basis->M * s,
                            cudaMemcpyDefault));
  }
  if (L)
    CUDA_CHECK(cudaMemcpy(L, basis->Phi.p + basis->phi_off[0], sizeof(double) * basis->M * tree->n, cudaMemcpyDefault));
  MLK_API_END
}

}  // extern "C"
