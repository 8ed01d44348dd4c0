// mlk_pcg_solve: preconditioned conjugate gradient for C_W gamma_W = Z_W (the
// survey's NEXT-1).  The product C_W p is the EXACT three-step product of P:2146-2170 (K5a
// kernels, matvec.cu); the preconditioner P_W = diag(P^{i,k}) takes the self block of every
// cell from the assembled BSR, Cholesky-factored once per solve (one CTA per
// block) and applied by two block triangular solves per iteration.  Dot products are fixed-
// order two-level reductions, so the iteration is deterministic.
#include <algorithm>
#include <cmath>

#include "api.cuh"

namespace mlk {
namespace {

constexpr int kPcgThreads = 256;

struct PBlock {
  int64_t off;   // offset of the p x p block (row-major) in the factor buffer
  int64_t row;   // first C_W row of the cell
  int32_t p;
};

// copy the self blocks out of the BSR values
__global__ void k_gather_blocks(const PBlock* __restrict__ pb, const int64_t* __restrict__ src_off,
                                const double* __restrict__ values, double* __restrict__ L) {
  const PBlock b = pb[blockIdx.x];
  const int64_t len = (int64_t)b.p * b.p;
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) L[b.off + e] = values[src_off[blockIdx.x] + e];
}

// in-place lower Cholesky of every block (right-looking, thread per trailing column with
// register-staged updates); non-positive pivot -> flag
__global__ void __launch_bounds__(kPcgThreads) k_cholesky(const PBlock* __restrict__ pb, double* __restrict__ L,
                                                          int* __restrict__ flag) {
  const PBlock b = pb[blockIdx.x];
  double* A = L + b.off;
  const int p = b.p, tid = threadIdx.x, nt = blockDim.x;
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
    // trailing update of the lower triangle: A[i][j] -= A[i][k] A[j][k], j > k, i >= j
    for (int j = k + 1 + tid; j < p; j += nt) {
      const double ljk = A[(int64_t)j * p + k];
      for (int i = j; i < p; i++) A[(int64_t)i * p + j] = fma(-A[(int64_t)i * p + k], ljk, A[(int64_t)i * p + j]);
    }
    __syncthreads();
  }
  // zero the strict upper triangle (the block started as the full symmetric matrix)
  for (int64_t e = tid; e < (int64_t)p * p; e += nt) {
    const int i = (int)(e / p), j = (int)(e - (int64_t)i * p);
    if (j > i) A[e] = 0.0;
  }
}

// s = P_W^-1 r: per block L y = r (forward, column sweep), L^T s = y (backward); y lives in
// shared memory when it fits
__global__ void __launch_bounds__(kPcgThreads) k_block_solve(const PBlock* __restrict__ pb,
                                                             const double* __restrict__ L,
                                                             const double* __restrict__ r, double* __restrict__ s,
                                                             double* __restrict__ scratch) {
  extern __shared__ double y_sh[];
  const PBlock b = pb[blockIdx.x];
  const double* A = L + b.off;
  const int p = b.p, tid = threadIdx.x, nt = blockDim.x;
  double* y = y_sh;
  for (int i = tid; i < p; i += nt) y[i] = r[b.row + i];
  __syncthreads();
  // forward: y_i /= L_ii, then y_j -= L_ji y_i for j > i
  for (int i = 0; i < p; i++) {
    const double yi = y[i] / A[(int64_t)i * p + i];
    __syncthreads();
    if (tid == 0) y[i] = yi;
    for (int j = i + 1 + tid; j < p; j += nt) y[j] = fma(-A[(int64_t)j * p + i], yi, y[j]);
    __syncthreads();
  }
  // backward with L^T: y_i /= L_ii, then y_j -= L_ij y_i for j < i
  for (int i = p - 1; i >= 0; i--) {
    const double yi = y[i] / A[(int64_t)i * p + i];
    __syncthreads();
    if (tid == 0) y[i] = yi;
    for (int j = tid; j < i; j += nt) y[j] = fma(-A[(int64_t)i * p + j], yi, y[j]);
    __syncthreads();
  }
  for (int i = tid; i < p; i += nt) s[b.row + i] = y[i];
}

// two dot products at once (u.v, w.w), fixed-order: per-CTA partials then one CTA in order
constexpr int kDotBlocks = 256;
__global__ void k_dot2_partial(const double* __restrict__ u, const double* __restrict__ v,
                               const double* __restrict__ w, int64_t n, double* __restrict__ part) {
  __shared__ double sa[kPcgThreads], sb[kPcgThreads];
  double a = 0.0, b = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    a = fma(u[i], v[i], a);
    if (w) b = fma(w[i], w[i], b);
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sa[threadIdx.x] += sa[threadIdx.x + o];
      sb[threadIdx.x] += sb[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sa[0];
    part[2 * blockIdx.x + 1] = sb[0];
  }
}

__global__ void k_dot2_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < nb; i++) {
      a += part[2 * i];
      b += part[2 * i + 1];
    }
    out[0] = a;
    out[1] = b;
  }
}

// x += alpha p; r -= alpha q
__global__ void k_update_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                            const double* __restrict__ q, double alpha, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    r[i] = fma(-alpha, q[i], r[i]);
  }
}

// p = s + beta p
__global__ void k_update_p(double* __restrict__ p, const double* __restrict__ s, double beta, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], s[i]);
}

struct Dot2 {
  DevBuf<double> part, out;
  Dot2(cudaStream_t s) : part(2 * kDotBlocks, s), out(2, s) {}
  // returns (u.v, w.w) on the host (one synchronisation)
  std::pair<double, double> run(cudaStream_t st, const double* u, const double* v, const double* w, int64_t n) {
    k_dot2_partial<<<kDotBlocks, kPcgThreads, 0, st>>>(u, v, w, n, part.p);
    check_launch("k_dot2_partial");
    k_dot2_final<<<1, 32, 0, st>>>(part.p, kDotBlocks, out.p);
    check_launch("k_dot2_final");
    auto h = out.download(2);
    return {h[0], h[1]};
  }
};

}  // namespace
}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_pcg_solve(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel, mlk_cw cw,
                         int32_t precond, const double* z_w, double* gamma_w, double tol, int32_t max_iter,
                         int32_t* iters, double* rel_residual) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && tree && basis && z_w && gamma_w, "NULL argument");
  MLK_REQUIRE(basis->tree == tree, "basis was built for another tree");
  check_kernel(kernel);
  MLK_REQUIRE(precond == 0 || precond == 1, "precond must be 0 (none) or 1 (block diagonal P_W)");
  MLK_REQUIRE(precond == 0 || cw != nullptr, "the block-diagonal preconditioner needs the assembled matrix");
  MLK_REQUIRE(tol > 0 && max_iter >= 1, "need tol > 0 and max_iter >= 1");
  Ctx& c = ctx->c;
  if (c.nranks != 1) throw Error(MLK_ERR_UNSUPPORTED, "mlk_pcg_solve runs on one rank (nranks == 1)");
  CUDA_CHECK(cudaSetDevice(c.device));
  cudaStream_t st = c.stream;
  const int64_t dim = basis->dim, n = tree->n;
  basis_wait(c, basis);
  DevIn<double> zin(z_w, (size_t)dim, st);
  DevOut<double> xout(gamma_w, (size_t)dim, st);
  DevBuf<double> r(dim, st), s(dim, st), p(dim, st), q(dim, st), a(n, st), b(n, st);
  CUDA_CHECK(cudaMemsetAsync(xout.p, 0, sizeof(double) * dim, st));
  CUDA_CHECK(cudaMemcpyAsync(r.p, zin.p, sizeof(double) * dim, cudaMemcpyDeviceToDevice, st));
  auto cw_apply = [&](const double* v, double* y) {  // y = C_W v (EXACT)
    apply_wt_dev(c, tree, basis, v, a.p, 1);
    cov_matvec_dev(c, tree, *kernel, a.p, b.p, 1);
    apply_w_dev(c, tree, basis, b.p, y, 1);
  };
  // ---- preconditioner: Cholesky factors of the self blocks
  std::vector<PBlock> blocks;
  DevBuf<double> Lf;
  DevBuf<PBlock> pb_d;
  size_t solve_smem = 0;
  if (precond) {
    MLK_REQUIRE(cw->complete, "the preconditioner needs the complete BSR values (mlk_cw_unpack first)");
    MLK_REQUIRE(cw->n_cells == (int32_t)basis->cells.size(), "cw does not match the basis");
    std::vector<int64_t> src;
    int64_t off = 0;
    for (int32_t cpos = 0; cpos < cw->n_cells; cpos++) {
      const int32_t k = cw->brow_ptr[cpos];  // blocks of a row are sorted by column: first is the self block
      MLK_REQUIRE(k < cw->brow_ptr[cpos + 1] && cw->bcol[k] == cpos, "self block missing from the BSR");
      const int32_t pc = (int32_t)(basis->row_off[cpos + 1] - basis->row_off[cpos]);
      blocks.push_back({off, basis->row_off[cpos], pc});
      src.push_back(cw->val_off[k]);
      off += (int64_t)pc * pc;
      solve_smem = std::max(solve_smem, sizeof(double) * (size_t)pc);
    }
    MLK_REQUIRE(solve_smem <= 200 * 1024, "block too large for the shared-memory triangular solve");
    Lf.alloc(std::max<int64_t>(off, 1), st);
    pb_d.alloc(blocks.size(), st);
    pb_d.upload(blocks);
    DevBuf<int64_t> src_d(src.size(), st);
    src_d.upload(src);
    DevBuf<int> flag(1, st);
    flag.zero();
    {
      TimedLaunch tl(c, "pcg_factor");
      k_gather_blocks<<<(unsigned)blocks.size(), kPcgThreads, 0, st>>>(pb_d.p, src_d.p, cw->vals(), Lf.p);
      check_launch("k_gather_blocks");
      k_cholesky<<<(unsigned)blocks.size(), kPcgThreads, 0, st>>>(pb_d.p, Lf.p, flag.p);
      check_launch("k_cholesky");
    }
    if (flag.download(1)[0]) throw Error(MLK_ERR_RANK_DEFICIENT, "a preconditioner block is not positive definite");
    if (solve_smem > 48 * 1024)
      CUDA_CHECK(cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_smem));
  }
  auto precondition = [&](const double* rin, double* sout) {
    if (!precond) {
      CUDA_CHECK(cudaMemcpyAsync(sout, rin, sizeof(double) * dim, cudaMemcpyDeviceToDevice, st));
      return;
    }
    TimedLaunch tl(c, "pcg_precond");
    k_block_solve<<<(unsigned)blocks.size(), kPcgThreads, solve_smem, st>>>(pb_d.p, Lf.p, rin, sout, nullptr);
    check_launch("k_block_solve");
  };
  const unsigned vgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(4 * num_sms(c.device), ceil_div(dim, 256)));
  Dot2 dot(st);
  // ---- PCG (oracle/pcg.py): x = 0, r = z, s = M^-1 r, p = s, rs = r.s
  const double nz = std::sqrt(dot.run(st, r.p, r.p, nullptr, dim).first);
  int it = 0;
  double res = 0.0;
  if (nz > 0.0) {
    precondition(r.p, s.p);
    CUDA_CHECK(cudaMemcpyAsync(p.p, s.p, sizeof(double) * dim, cudaMemcpyDeviceToDevice, st));
    double rs = dot.run(st, r.p, s.p, nullptr, dim).first;
    while (it < max_iter) {
      {
        TimedLaunch tl(c, "pcg_matvec");
        cw_apply(p.p, q.p);
      }
      const double pq = dot.run(st, p.p, q.p, nullptr, dim).first;
      const double alpha = rs / pq;
      k_update_xr<<<vgrid, 256, 0, st>>>(xout.p, r.p, p.p, q.p, alpha, dim);
      check_launch("k_update_xr");
      it++;
      precondition(r.p, s.p);
      const auto rs_rr = dot.run(st, r.p, s.p, r.p, dim);  // (r.s, r.r) in one pass
      res = std::sqrt(rs_rr.second) / nz;
      if (res <= tol) break;
      const double beta = rs_rr.first / rs;
      rs = rs_rr.first;
      k_update_p<<<vgrid, 256, 0, st>>>(p.p, s.p, beta, dim);
      check_launch("k_update_p");
    }
    // the unpreconditioned accuracy: true residual ||z - C_W x|| / ||z||
    cw_apply(xout.p, q.p);
    k_update_p<<<vgrid, 256, 0, st>>>(q.p, zin.p, -1.0, dim);  // q = z - C_W x
    check_launch("k_update_p");
    res = std::sqrt(dot.run(st, q.p, q.p, nullptr, dim).first) / nz;
  }
  xout.finish();
  if (iters) *iters = it;
  if (rel_residual) *rel_residual = res;
  MLK_API_END
}

}  // extern "C"
