// FP64 elementary functions for the covariance closed forms (R16, R17), cheaper on the FP64
// pipe than the general libdevice versions because their argument ranges are restricted.
// On sm_100a DFMA and DMMA share one pipe, so every instruction here
// is paid out of the contraction's budget.
//   exp_neg(z), z >= 0:  e^{-z} = 2^{k/64} e^r, k = round(-64 z / ln 2), r = -z - k ln2/64
//                        (single-constant reduction: |error| <= 0.7 ulp of z), |r| <= ln2/128,
//                        expm1(r) by a degree-5 Taylor polynomial (truncation < 3.5e-17),
//                        2^{(k mod 64)/64} from a 64-entry shared table, 2^{floor(k/64)} by an
//                        exponent-field add.  z is clamped to <= ~704 by an integer min on
//                        its high word (e^{-704} ~ 1e-306 stands in for smaller values).
//                        9 FP64 instructions.
//   sqrt_pos(x), x > 0 normal: rsqrt.approx.f64, one coupled Newton (Goldschmidt) step and a
//                        final residual correction.  7 FP64 instructions, <= ~1 ulp.
#pragma once
#include <cuda_runtime.h>

namespace mlk {

// 2^(j/64), j = 0..63, correctly rounded (generated with Python's decimal module at 60 digits)
static __constant__ double kExp2Tab64[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284,
    1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199,
    1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
    1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
    1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687,
    1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
    1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303,
    1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
    1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
    1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384,
    1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267,
    1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
    1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
    1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989,
    1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
    1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951};

__device__ __forceinline__ double exp_neg(double z, const double* __restrict__ tab) {
  const double kShift = 6755399441055744.0;          // 1.5 * 2^52
  const double kInvLn2x64 = 92.33248261689366;       // 64 / ln 2
  const double kLn2d64 = 0.010830424696249145;       // ln 2 / 64
  z = __hiloint2double(min(__double2hiint(z), 0x40860000), __double2loint(z));  // z <= 704
  const double t = fma(z, -kInvLn2x64, kShift);
  const int k = __double2loint(t);                   // round(-64 z / ln 2)
  const double kd = t - kShift;
  const double r = fma(kd, -kLn2d64, -z);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = p * r;                                         // expm1(r)
  const double tj = tab[k & 63];
  const double v = fma(tj, p, tj);                   // 2^((k mod 64)/64) e^r, in [0.99, 2)
  return __hiloint2double(__double2hiint(v) + ((k >> 6) << 20), __double2loint(v));
}

__device__ __forceinline__ double sqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double s = x * y, h = 0.5 * y;
  const double r = fma(-s, h, 0.5);
  s = fma(s, r, s);
  h = fma(h, r, h);
  const double e = fma(-s, s, x);
  return fma(e, h, s);
}

// x if x is a positive normal number, else 2^-997 (a stand-in for 0 that keeps sqrt_pos
// finite); integer ops only, so the FP64 pipe is not used
__device__ __forceinline__ double clamp_pos(double x) {
  int hi = __double2hiint(x);
  hi = hi < 0x00100000 ? 0x01a00000 : hi;
  return __hiloint2double(hi, __double2loint(x));
}

}  // namespace mlk
