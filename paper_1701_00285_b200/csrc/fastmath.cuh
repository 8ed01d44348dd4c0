// FP64 elementary functions for the covariance closed forms, cheaper on the FP64 pipe than
// the general libdevice versions (their argument ranges are restricted here):
//   exp_neg(x), x <= 0:  x = (k/16) ln 2 + r, |r| <= ln2/32, e^r by a degree-7 Taylor
//                        polynomial (truncation < 1.2e-18), 2^(j/16) from a 16-entry shared
//                        table (one double per bank pair: conflict-free), 2^(k>>4) by an
//                        exponent-field add.  ~13 FP64 instructions, <= ~2 ulp.
//   sqrt_pos(x), x >= 0: rsqrt.approx.f64 + two Newton steps, <= ~2 ulp (x = 0 -> ~1e-150).
#pragma once
#include <cuda_runtime.h>

namespace mlk {

// 2^(j/16), j = 0..15, correctly rounded
static __constant__ double kExp2Tab16[16] = {
    1.0,                1.0442737824274138, 1.0905077326652577, 1.1387886347566916,
    1.189207115002721,  1.241857812073484,  1.2968395546510096, 1.3542555469368927,
    1.4142135623730951, 1.4768261459394993, 1.5422108254079407, 1.6104903319492543,
    1.681792830507429,  1.7562521603732995, 1.8340080864093424, 1.9152065613971474};

__device__ __forceinline__ double exp_neg(double x, const double* __restrict__ tab) {
  const double kShift = 6755399441055744.0;          // 1.5 * 2^52
  const double kInvLn2x16 = 23.083120654223414518;   // 16 / ln 2
  const double kLn2d16Hi = 0.04332169878489367;      // ln2/16 split: hi has 36 bits, so
  const double kLn2d16Lo = 1.0291218489310676e-13;    // kd * hi is exact for |kd| < 2^17
  x = fmax(x, -708.0);
  double t = fma(x, kInvLn2x16, kShift);
  int k = __double2loint(t);
  double kd = t - kShift;
  double r = fma(kd, -kLn2d16Hi, x);
  r = fma(kd, -kLn2d16Lo, r);
  double p = fma(r, 1.0 / 5040.0, 1.0 / 720.0);
  p = fma(r, p, 1.0 / 120.0);
  p = fma(r, p, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = p * r;                                          // expm1(r)
  double tj = tab[k & 15];
  double v = fma(tj, p, tj);                          // 2^(j/16) e^r
  int hi = __double2hiint(v) + ((k >> 4) << 20);      // times 2^(k >> 4)
  return __hiloint2double(hi, __double2loint(v));
}

__device__ __forceinline__ double sqrt_pos(double x) {
  x = fmax(x, 1e-300);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  return x * y;
}

}  // namespace mlk
