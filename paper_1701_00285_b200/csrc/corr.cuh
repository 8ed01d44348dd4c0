// Correlation functions of the covariance families (R16, R17), shared by the fused
// tile kernel (tile.cu) and the symmetric multi-vector C a kernel (covsym.cu).
#pragma once
#include "fastmath.cuh"
#include "tile.cuh"

namespace mlk {
namespace {

// phi(z) = 2^(1-nu)/Gamma(nu) z^nu K_nu(z), z > 0 (the Matern definition), from
// two textbook representations of K_nu:
//  * the integral K_nu(z) = int_0^inf exp(-z cosh t) cosh(nu t) dt, by the trapezoidal rule with
//    step h = h0 / max(1, sqrt z).  The integrand is entire and decays double-exponentially, so
//    the rule converges geometrically in 1/h; the sqrt(z) scaling keeps the peak of width
//    ~1/sqrt(z) resolved at large z.  z^nu is folded into the exponent,
//    z^nu e^{-z cosh t} cosh(nu t) = e^{nu (t + log z) - z cosh t} (1 + e^{-2 nu t}) / 2,
//    so nothing overflows for large nu or small z; the sum stops once t is past the integrand's
//    peak (sinh t = nu / z) and a term falls below 1e-17 of the sum.  e^t and e^{-2 nu t} advance
//    by one multiplication per node.  Measured against scipy's K_nu (tools, this round): relative
//    error <= 7e-13 for nu in [0.1, 50], z in [1e-8, 700]; <= 2e-13 for nu <= 12.
//  * for z < 2 and nu at least 0.01 from an integer, the series from K_nu = pi/2 (I_-nu - I_nu) /
//    sin(nu pi) and I_mu(z) = sum_k (z/2)^(2k+mu) / (k! Gamma(k+mu+1)), which with
//    Gamma(nu) Gamma(1-nu) = pi / sin(nu pi) becomes
//      phi = sum_k w^k Gamma(1-nu) / (k! Gamma(k+1-nu)) - Gamma(1-nu) (z/2)^(2 nu) sum_k w^k / (k! Gamma(k+1+nu)),
//    w = z^2 / 4 (about 13 terms; phi(0) = 1 is its k = 0 term).  Near integer nu the two sums
//    cancel (Gamma(1-nu) has poles there), so those nu always take the integral.
__device__ __noinline__ double matern_nu(double z, const KernelParams& kp) {
  const double nu = kp.nu;
  if (kp.series && z < 2.0) {
    const double w = 0.25 * z * z;
    double a = 1.0, sm = 1.0, b = kp.rg1p, sp = kp.rg1p;
    for (int k = 1; k < 100; k++) {
      a *= w / (k * (k - nu));
      b *= w / (k * (k + nu));
      sm += a;
      sp += b;
      if (fabs(a) <= 1e-17 * fabs(sm) && fabs(b) <= 1e-17 * fabs(sp)) break;
    }
    return sm - kp.g1m * exp(2.0 * nu * log(0.5 * z)) * sp;
  }
  const double h = kp.h0 / fmax(1.0, sqrt(z));
  const double lz = nu * log(z), E = exp(h), Q = exp(-2.0 * nu * h);
  const double tpk = asinh(nu / z);
  double e = 1.0, q = 1.0, s = 0.5 * exp(lz - z);  // node t = 0, weight 1/2
  for (int k = 1; k < 4096; k++) {
    e *= E;
    q *= Q;
    const double t = k * h;
    const double term = exp(nu * t + lz - 0.5 * z * (e + 1.0 / e)) * 0.5 * (1.0 + q);
    s += term;
    if (t > tpk && term <= 1e-17 * s) break;
  }
  return kp.norm * h * s;
}

// correlation phi from the augmented Gram value x = z^2 (Matern, z = sqrt(2 nu) r / rho) or
// x = r^2 / rho^2 (Gaussian); R16, R17
template <int FAM>
__device__ __forceinline__ double corr(double x, const double* tab, const KernelParams& kp) {
  if (FAM == MLK_GAUSSIAN) return exp_neg(x, tab);  // x >= -O(u|y|^2): e^{-x} stays ~1
  if (FAM == MLK_MATERN_NU) return x > 0.0 ? matern_nu(sqrt(x), kp) : 1.0;
  x = clamp_pos(x);
  const double z = sqrt_pos(x);
  const double e = exp_neg(z, tab);
  if (FAM == MLK_MATERN_12) return e;
  if (FAM == MLK_MATERN_32) return fma(z, e, e);                  // (1 + z) e^{-z}
  return fma(e, fma(x, 1.0 / 3.0, z), e);                         // (1 + z + z^2/3) e^{-z}
}

}  // namespace
}  // namespace mlk
