// MLK_PREC_DD: double-double (~106-bit) evaluation of the blocks B = W_a C W_b^T for
// workloads at the FP64 floor (cfg1 blocks whose norm is ~1e-6 of
// |W_a| |C| |W_b| lose ~1e-11 relative accuracy in plain FP64).  Distances by direct
// differences, the covariance closed forms and both contractions are carried in
// double-double; the W blocks are the FP64 basis.  Scalar FP64 arithmetic (error-free
// transformations with FMA), one thread per output entry.
#include <algorithm>
#include <array>
#include <cmath>

#include "api.cuh"

namespace mlk {
namespace {

struct dd {
  double hi, lo;
};

__host__ __device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__host__ __device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = fma(a.hi, b.lo, fma(a.lo, b.hi, p.lo));
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = fma(a.lo, b, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd sqrt_dd(dd a) {
  if (a.hi <= 0.0) return {0.0, 0.0};
  double s = sqrt(a.hi);
  dd p = two_prod(s, s);
  double e = ((a.hi - p.hi) - p.lo + a.lo) / (2.0 * s);
  return quick_two_sum(s, e);
}

__constant__ double c_inv_fact[10] = {1.0, 1.0, 1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040,
                                      1.0 / 40320, 1.0 / 362880};
__constant__ double c_inv_fact_lo[10];

// e^x for x <= 0 in double-double: x = k ln2 + r, e^r = (e^{r/1024})^1024 via expm1 squaring
__device__ dd exp_dd(dd x) {
  const dd ln2 = {6.931471805599452862e-01, 2.319046813846299558e-17};
  if (x.hi < -700.0) return {0.0, 0.0};
  double k = rint(x.hi / ln2.hi);
  dd r = add(x, mul_d(ln2, -k));
  r.hi = ldexp(r.hi, -10);
  r.lo = ldexp(r.lo, -10);
  // s = expm1(r) by Taylor to r^9/9!
  dd s = {0.0, 0.0};
  for (int i = 9; i >= 1; i--) {
    dd f = {c_inv_fact[i], c_inv_fact_lo[i]};
    s = mul(add(s, f), r);
  }
  for (int i = 0; i < 10; i++) s = add(mul_d(s, 2.0), mul(s, s));  // expm1(2a) = 2 expm1(a) + expm1(a)^2
  dd e = add(s, dd{1.0, 0.0});
  int ki = (int)k;
  return {ldexp(e.hi, ki), ldexp(e.lo, ki)};
}

struct DDKernel {
  int family;
  dd c1;         // sqrt(2 nu)/rho or 1/rho^2
  dd third;      // 1/3
  double sigma2, nugget;
};

__device__ dd cov_dd(const double* x, const double* y, int d, bool same, const DDKernel& k) {
  dd r2 = {0.0, 0.0};
  for (int j = 0; j < d; j++) {
    dd df = two_sum(x[j], -y[j]);
    dd sq = two_prod(df.hi, df.hi);
    sq.lo = fma(2.0 * df.hi, df.lo, sq.lo);
    r2 = add(r2, quick_two_sum(sq.hi, sq.lo));
  }
  if (same) r2 = {0.0, 0.0};
  dd phi;
  if (k.family == MLK_GAUSSIAN) {
    dd a = mul(r2, k.c1);
    phi = exp_dd({-a.hi, -a.lo});
  } else {
    dd z = mul(sqrt_dd(r2), k.c1);
    dd e = exp_dd({-z.hi, -z.lo});
    if (k.family == MLK_MATERN_12) phi = e;
    else if (k.family == MLK_MATERN_32) phi = mul(add(dd{1.0, 0.0}, z), e);
    else phi = mul(add(add(dd{1.0, 0.0}, z), mul(mul(z, z), k.third)), e);
  }
  dd v = mul_d(phi, k.sigma2);
  if (same && k.nugget != 0.0) v = add(v, dd{k.nugget, 0.0});
  return v;
}

struct DDJob {
  int64_t a_begin, b_begin;
  int32_t s_a, s_b, p_a, p_b;
  const double* Wa;  // p_a x s_a
  const double* Wb;  // p_b x s_b
  int64_t u_off;     // U scratch offset (s_a x p_b)
  int64_t e_u;       // prefix of U entries
  int64_t e_b;       // prefix of B entries
  double* dst;
  int64_t ldc;
  int32_t trans;
};

__device__ __forceinline__ int find_job(const int64_t* pre, int n, int64_t e) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void k_dd_u(const DDJob* __restrict__ jobs, const int64_t* __restrict__ pre, int nj, int64_t total,
                       const double* __restrict__ Xt, int dp, int d, DDKernel kk, double* __restrict__ Uh,
                       double* __restrict__ Ul) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  const DDJob jb = jobs[find_job(pre, nj, e)];
  int64_t le = e - jb.e_u;
  int r = (int)(le % jb.s_a), l = (int)(le / jb.s_a);  // consecutive threads: consecutive rows
  const double* x = Xt + (jb.a_begin + r) * dp;
  dd acc = {0.0, 0.0};
  for (int y = 0; y < jb.s_b; y++) {
    bool same = (jb.a_begin + r) == (jb.b_begin + y);
    dd cv = cov_dd(x, Xt + (jb.b_begin + y) * dp, d, same, kk);
    acc = add(acc, mul_d(cv, jb.Wb[(int64_t)l * jb.s_b + y]));
  }
  Uh[jb.u_off + (int64_t)r * jb.p_b + l] = acc.hi;
  Ul[jb.u_off + (int64_t)r * jb.p_b + l] = acc.lo;
}

__global__ void k_dd_b(const DDJob* __restrict__ jobs, const int64_t* __restrict__ pre, int nj, int64_t total,
                       const double* __restrict__ Uh, const double* __restrict__ Ul) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  const DDJob jb = jobs[find_job(pre, nj, e)];
  int64_t le = e - jb.e_b;
  int i = (int)(le / jb.p_b), l = (int)(le % jb.p_b);
  dd acc = {0.0, 0.0};
  for (int r = 0; r < jb.s_a; r++) {
    dd u = {Uh[jb.u_off + (int64_t)r * jb.p_b + l], Ul[jb.u_off + (int64_t)r * jb.p_b + l]};
    acc = add(acc, mul_d(u, jb.Wa[(int64_t)i * jb.s_a + r]));
  }
  double v = acc.hi + acc.lo;
  if (jb.trans) jb.dst[(int64_t)l * jb.ldc + i] = v;
  else jb.dst[(int64_t)i * jb.ldc + l] = v;
}

dd host_div(dd a, double b) {
  double q1 = a.hi / b;
  double ph = q1 * b;
  double pl = std::fma(q1, b, -ph);
  double r = ((a.hi - ph) - pl + a.lo) / b;
  return quick_two_sum(q1, r);
}
dd host_sqrt(double x) {
  double s = std::sqrt(x);
  double e = std::fma(-s, s, x) / (2.0 * s);
  return quick_two_sum(s, e);
}

}  // namespace

void assemble_dd(Ctx& c, const mlk_tree_s* tree, const mlk_basis_s* B, const mlk_kernel& k,
                 const std::vector<std::array<int64_t, 8>>& in) {
  if (in.empty()) return;
  cudaStream_t st = c.stream;
  // 1/k! in double-double
  double lo[10];
  for (int i = 0; i < 10; i++) {
    double f = 1.0;
    for (int j = 2; j <= i; j++) f *= j;  // exact for i <= 9
    dd q = host_div(dd{1.0, 0.0}, f);
    lo[i] = q.lo;
  }
  CUDA_CHECK(cudaMemcpyToSymbolAsync(c_inv_fact_lo, lo, sizeof(lo), 0, cudaMemcpyHostToDevice, st));
  DDKernel kk;
  kk.family = k.family;
  kk.sigma2 = k.sigma2;
  kk.nugget = k.nugget;
  kk.third = host_div(dd{1.0, 0.0}, 3.0);
  dd one_over_rho = host_div(dd{1.0, 0.0}, k.rho);
  switch (k.family) {
    case MLK_MATERN_12: kk.c1 = one_over_rho; break;
    case MLK_MATERN_32: kk.c1 = host_div(host_sqrt(3.0), k.rho); break;
    case MLK_MATERN_52: kk.c1 = host_div(host_sqrt(5.0), k.rho); break;
    default: {
      dd t = host_div(one_over_rho, k.rho);
      kk.c1 = t;
      break;
    }
  }
  std::vector<DDJob> jobs;
  std::vector<int64_t> pre_u, pre_b;
  int64_t eu = 0, eb = 0, uo = 0;
  for (auto& j : in) {
    int a = (int)j[0], b = (int)j[1];
    DDJob x;
    x.a_begin = tree->begin[a];
    x.b_begin = tree->begin[b];
    x.s_a = (int32_t)(tree->end[a] - tree->begin[a]);
    x.s_b = (int32_t)(tree->end[b] - tree->begin[b]);
    x.p_a = B->p[a];
    x.p_b = B->p[b];
    x.Wa = B->W.p + B->w_off[a];
    x.Wb = B->W.p + B->w_off[b];
    x.u_off = uo;
    x.e_u = eu;
    x.e_b = eb;
    x.dst = reinterpret_cast<double*>(static_cast<uintptr_t>(j[2]));
    x.ldc = j[3];
    x.trans = (int32_t)j[4];
    pre_u.push_back(eu);
    pre_b.push_back(eb);
    uo += (int64_t)x.s_a * x.p_b;
    eu += (int64_t)x.s_a * x.p_b;
    eb += (int64_t)x.p_a * x.p_b;
    jobs.push_back(x);
  }
  DevBuf<DDJob> dj(jobs.size(), st);
  dj.upload(jobs);
  DevBuf<int64_t> pu(pre_u.size(), st), pb(pre_b.size(), st);
  pu.upload(pre_u);
  pb.upload(pre_b);
  DevBuf<double> Uh(std::max<int64_t>(uo, 1), st), Ul(std::max<int64_t>(uo, 1), st);
  TimedLaunch tl(c, "assemble_dd");
  k_dd_u<<<(unsigned)ceil_div(eu, 128), 128, 0, st>>>(dj.p, pu.p, (int)jobs.size(), eu, tree->Xt.p, tree->d_pad,
                                                       tree->d, kk, Uh.p, Ul.p);
  check_launch("k_dd_u");
  k_dd_b<<<(unsigned)ceil_div(eb, 128), 128, 0, st>>>(dj.p, pb.p, (int)jobs.size(), eb, Uh.p, Ul.p);
  check_launch("k_dd_b");
}

}  // namespace mlk
