// K5a: fused covariance-tile generation + first contraction on FP64 DMMA (see tile.cuh).
//
// CTA = 4 warps, 32 rows of the a range (8 per warp).  Coordinates enter as augmented,
// pre-scaled rows (k_tile_aug): Pa = [u, |u|^2, 1], Pb = [-2u, 1, |u|^2] with u = scale * x, so
// the Gram DMMAs produce z^2 = |u_a - u_b|^2 directly (no norm loads, no FP64 fix-up).  The
// b range is streamed in stages of BN points (cp.async double buffering): the stage holds the
// b rows (BN x dpa) and the W_b columns (8 RQ rows x BN, 16-byte chunks XOR-swizzled so the
// B-fragment loads are bank-conflict free).  Per 8-point sub-tile a warp
//   1. forms z^2 with dpa/4 DMMA.8x8x4,
//   2. turns its two accumulator entries into correlations in registers (fastmath.cuh; the
//      same-site entry is set to 1 + nugget/sigma2 exactly, sigma2 is applied once in the
//      epilogue),
//   3. feeds them straight back as DMMA A-fragments: accumulator column 2(lane%4)+s is the
//      A element k = lane%4 of k-step s, provided W_b is read with the same point
//      permutation -- no shuffles between the two products,
//   4. accumulates U (8 rows x 8 RQ columns) with 2 RQ DMMAs.
// A persistent grid pulls units (largest first) from an atomic counter.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <array>
#include <string>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "dmma.cuh"
#include "corr.cuh"
#include "fastmath.cuh"
#include "tile.cuh"

namespace mlk {

KernelParams make_kernel_params(const mlk_kernel& k) {
  KernelParams p;
  p.family = k.family;
  p.sigma2 = k.sigma2;
  p.nugget = k.nugget;
  p.same_val = 1.0 + k.nugget / k.sigma2;
  switch (k.family) {
    case MLK_MATERN_12: p.c1 = 1.0 / k.rho; break;
    case MLK_MATERN_32: p.c1 = std::sqrt(3.0) / k.rho; break;
    case MLK_MATERN_52: p.c1 = std::sqrt(5.0) / k.rho; break;
    case MLK_MATERN_NU: p.c1 = std::sqrt(2.0 * k.nu) / k.rho; break;
    default: p.c1 = 1.0 / (k.rho * k.rho); break;
  }
  if (k.family == MLK_MATERN_NU) {
    // constants of matern_nu (computed once, in long double)
    const long double nu = k.nu;
    p.nu = k.nu;
    p.norm = (double)(std::pow(2.0L, 1.0L - nu) / std::tgamma(nu));
    p.h0 = std::min(0.2, 0.5 / std::sqrt(k.nu + 1.0));
    p.series = std::fabs(k.nu - std::nearbyint(k.nu)) >= 0.01 ? 1 : 0;
    p.g1m = p.series ? (double)std::tgamma(1.0L - nu) : 0.0;
    p.rg1p = (double)(1.0L / std::tgamma(1.0L + nu));
  } else {
    p.nu = p.norm = p.h0 = p.g1m = p.rg1p = 0.0;
    p.series = 0;
  }
  // coordinates are pre-scaled so that the augmented Gram product is z^2 = (c1 r)^2
  // (Matern) or r^2 / rho^2 (Gaussian)
  p.scale = k.family == MLK_GAUSSIAN ? 1.0 / k.rho : p.c1;
  return p;
}

static const int kRQ[] = {1, 2, 3, 4, 6, 7, 8, 9, 12, 16, 20, 24};

int tile_rq_class(int qc) {
  for (int r : kRQ)
    if (8 * r >= qc) return r;
  return kTileMaxRQ;
}

// (rq, nr) for a chunk of qc columns: 8 rq DMMA columns plus nr <= tile_max_nr(rq) DFMA columns when
// qc = 8 rq + nr with rq a class, else rq = the padding class and nr = 0
static void tile_split(int qc, int& rq, int& nr) {
  const int lo = qc / 8, rem = qc % 8;
  if (lo >= 1 && lo <= 12 && rem >= 1 && rem <= tile_max_nr(lo) && tile_rq_class(8 * lo) == lo) {
    rq = lo;
    nr = rem;
  } else {
    rq = tile_rq_class(qc);
    nr = 0;
  }
}

void make_tile_units(std::vector<TileUnit>& out, int64_t a_begin, int32_t s_a, int64_t b_begin, int32_t s_b,
                     const double* Wb, int64_t ldw, int32_t p_b, double* U, int64_t ldu, int32_t trans, int dp) {
  int nch = (int)ceil_div(p_b, 8 * kTileMaxRQ);
  int width = (int)ceil_div(ceil_div(p_b, nch), 8) * 8;
  for (int c0 = 0; c0 < p_b; c0 += width) {
    int qc = std::min(width, p_b - c0);
    int rq, nr;
    tile_split(qc, rq, nr);
    TileUnit u;
    u.a_begin = a_begin;
    u.b_begin = b_begin;
    u.s_a = s_a;
    u.s_b = s_b;
    u.row0 = 0;
    u.n_tasks = (int32_t)ceil_div(s_a, 32);
    u.c0 = c0;
    u.qc = qc;
    u.p_b = p_b;
    u.trans = trans;
    u.rq = rq;
    u.nr = nr;
    u.Wb = Wb;
    u.ldw = ldw;
    u.U = U;
    u.ldu = ldu;
    // a tensor map needs a 16-byte aligned base and a row stride that is a multiple of 16 bytes
    u.bulk = (ldw % 2 == 0) && ((reinterpret_cast<uintptr_t>(Wb) & 15) == 0);
    u.xmap = u.wmap = -1;
    u.w_col0 = 0;
    u.w_cols = s_b;
    u.cp_off = 0;
    u.seg = 0;
    u.seg_off = 0;
    // FP64-slot estimate per 32-row task: Gram dp + evaluation ~20 + contraction per entry
    u.cost = 32.0 * s_b * (dp + 20 + 8.0 * rq + nr);
    out.push_back(u);
  }
}

namespace {

// A/B switches (tools/build_variant.py): occupancy target and stage width of the 2-4 group classes
#ifndef MLK_MINCTAS_SMALL
#define MLK_MINCTAS_SMALL 5  // 5 CTAs: cfg3 K5a 250.6 -> 246.3 ms (r02d)
#endif
#ifndef MLK_BN_ONE
#define MLK_BN_ONE 56
#endif
#ifndef MLK_BN_SMALL
#define MLK_BN_SMALL 40
#endif
template <int RQ>
struct TileCfg {
  // b points per stage.  BN = 8 (mod 16) makes a W row 8 BN doubles = 64 (mod 128) bytes, so
  // the 16-byte B-fragment loads of a quarter-warp (2 rows x 4 chunks) hit distinct banks
  // without any swizzle -- which a 1-D bulk copy could not apply
  static constexpr int BN = RQ >= 6 ? 24 : (RQ == 1 ? MLK_BN_ONE : MLK_BN_SMALL);  // 40 for RQ 6-9 measured 13 % slower on cfg4
  // maximum stages in the smem ring (the launch uses the deepest ring that keeps the target
  // occupancy, >= 2): the one-group class (C a, tiny cells) has short stages, so it wants a
  // deeper ring to cover the TMA latency
  static constexpr int NST = RQ == 1 ? 6 : (RQ >= 16 ? 2 : 3);
  static constexpr int MIN_CTAS = RQ >= 20 ? 3 : ((RQ == 2 || RQ == 3) ? MLK_MINCTAS_SMALL : 4);  // (5 CTAs with 4
                                                     // held W fragments measured 1.7 % slower)
  static constexpr int G = RQ <= 12 ? RQ : 8;    // W_b fragments held per DMMA group
  static constexpr int NACC = 1;                 // accumulator sets (2 measured no faster)
};

// stage size rounded to 128 bytes: 2-D TMA writes need 128-byte aligned shared destinations
// (the W part starts BN sdp doubles in, a multiple of 128 bytes since sdp is a multiple of 4)
// W_b rows a stage holds: 8 rq + the DFMA remainder rows, or NV for the C a variants (their
// tensor map box covers only the vector rows)
__host__ __device__ constexpr int stage_wrows(int rq, int nv) { return nv > 0 ? nv : 8 * rq + tile_max_nr(rq); }
__host__ __device__ constexpr int stage_doubles(int rq, int bn, int sdp, int red = 0, int nv = 0) {
  return (bn * sdp + stage_wrows(rq, nv) * bn + red + 15) / 16 * 16;
}
// SYM: per stage, the four warps' column partials (4 x NV x BN doubles) for the last warp's
// fixed-order sum
__host__ __device__ constexpr int sym_red_doubles(bool sym, int nv, int bn) { return sym ? 4 * nv * bn : 0; }

// Augmented, pre-scaled coordinates (x in tree order, s = kp.scale, u = s x), dpa doubles per row.
// Augmented mode (dk == dpa = pad4(d + 2)):
//   Pa[i] = [u_i, |u_i|^2, 1, 0...],  Pb[i] = [-2 u_i, 1, |u_i|^2, 0...]
// so that one DMMA dot product gives Pa[i].Pb[j] = |u_i - u_j|^2 (the Gram identity) directly.
// Norm mode (dk = pad4(d) < pad4(d + 2), e.g. d = 20: 5 instead of 6 DMMA k-steps; dpa = dk + 4):
//   Pa[i] = [u_i, 0.., |u_i|^2 at column dk, 0..],  Pb[i] = [-2 u_i, 0.., |u_i|^2 at column dk, 0..]
// and the kernel starts the Gram accumulator at |u_i|^2 + |u_j|^2 (the DMMA adds -2 u_i.u_j).
__global__ void k_tile_aug(const double* __restrict__ Xt, int dpt, int d, int64_t n, double s,
                           double* __restrict__ Pa, double* __restrict__ Pb, int dpa, int dk) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* x = Xt + i * dpt;
  double* pa = Pa + i * dpa;
  double* pb = Pb + i * dpa;
  double nn = 0.0;
  for (int k = 0; k < d; k++) {
    const double u = s * x[k];
    nn = fma(u, u, nn);
    pa[k] = u;
    pb[k] = -2.0 * u;
  }
  for (int k = d; k < dpa; k++) pa[k] = pb[k] = 0.0;
  if (dk < dpa) {
    pa[dk] = nn;
    pb[dk] = nn;
  } else {
    pa[d] = nn;
    pa[d + 1] = 1.0;
    pb[d] = 1.0;
    pb[d + 1] = nn;
  }
}

// NV > 0 (with RQ = 1): the contraction has NV <= 4 columns (C a for a few vectors) and is done
// with DFMAs per lane instead of 8-column DMMAs; the four lanes of a quad hold disjoint column
// subsets of a row and are summed by two shuffles in the epilogue (fixed order).
//
// Staging: a ring of nring <= NST stages, each {BN rows of Pb, 8 RQ rows x BN columns of W_b}, filled by
// two 2-D TMA box loads (tensor maps built by run_tile_contract) that complete on the stage's
// mbarrier; out-of-range rows / columns arrive zero-filled.  Units whose W_b cannot be described
// by a tensor map (odd row stride or unaligned base) use 8-byte cp.async instead.  The last
// warp to finish a stage (a shared counter) refills it with the stage nring ahead, so warps never
// wait on a CTA barrier inside a unit.
// SYM (with NV > 0): symmetric C a.  A task (32-row tile I) covers the points j >= its first
// row; the row part b_i += C_ij a_j keeps j >= i, the column part b_j += C_ij a_i (j > i) is
// reduced over each warp's 8 rows by shuffles and written to colpart (one row per warp and
// vector); k_colpart_sum adds them in (tile, warp) order.  Half the covariance evaluations,
// deterministic.
template <int RQ, int FAM, int NV, bool SYM = false, bool SEG = false>
__global__ void __launch_bounds__(128, TileCfg<RQ>::MIN_CTAS)
    k_tile_contract(const TileUnit* __restrict__ units, const int32_t* __restrict__ task_range,
                    const int32_t* __restrict__ task_first, int n_units, int* __restrict__ counter,
                    const double* __restrict__ Pa, const double* __restrict__ Pb, int dpa, int dk, int sdp, int nring,
                    KernelParams kp, const CUtensorMap* __restrict__ maps, double* __restrict__ colpart) {
  constexpr int BN = TileCfg<RQ>::BN;
  constexpr int G = TileCfg<RQ>::G;
  constexpr int NST = TileCfg<RQ>::NST;
  constexpr int T = BN / 8;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[NST];
  __shared__ int cnt[NST];
  __shared__ int s_unit;
  __shared__ double s_tab[kExpTabN];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int RED = sym_red_doubles(SYM, NV, BN);
  const int sd = stage_doubles(RQ, BN, sdp, RED, NV);
  const int red_off = stage_doubles(RQ, BN, sdp, 0, NV);  // the stage's reduction area (SYM)
  double* As = sm;                  // 32 x sdp
  double* St = sm + 32 * sdp;       // nring stages
  for (int i = tid; i < kExpTabN; i += blockDim.x) s_tab[i] = kExp2Tab[i];
  if (tid == 0) {
    for (int i = 0; i < nring; i++) {
      mbar_init(&full[i], 1);
      cnt[i] = 0;
    }
    fence_mbar_init();
  }
  // stale stage contents are only ever multiplied by zeroed covariances: keep them finite
  for (int e = tid; e < nring * sd; e += 128) St[e] = 0.0;
  fence_proxy_async_smem();
  const int ks_n = dk >> 2;
  const bool nmode = dk < dpa;  // norm mode: Gram accumulators start at |u_a|^2 + |u_b|^2
  int gs = 0;  // stages consumed so far by this CTA (ring position and mbarrier phases)

  while (true) {
    __syncthreads();
    if (tid == 0) s_unit = atomicAdd(counter, 1);
    __syncthreads();
    const int ui = s_unit;
    if (ui >= n_units) break;
    const int ri = task_range[ui];
    TileUnit u = units[ri];
    u.row0 += 32 * (ui - task_first[ri]);
    const int64_t a0 = u.a_begin + u.row0;
    const int rows = min(32, u.s_a - u.row0);
    // a tile (rows x dpa); rows past the range are zero (their outputs are discarded)
    {
      const int cpr = dpa >> 1;
      for (int e = tid; e < 32 * cpr; e += 128) {
        const int r = e / cpr, ch = e - r * cpr;
        const bool ok = r < rows;
        cp_async16(As + r * sdp + 2 * ch, ok ? Pa + (a0 + r) * dpa + 2 * ch : Pa, ok);
      }
      cp_async_commit();
    }
    const int nst = (u.s_b + BN - 1) / BN;

    // fill the ring slot of stage s (called by one whole warp)
    // ring position of this task's first stage (one division per task; per stage the slot and
    // the mbarrier parity advance incrementally)
    const int slot0 = gs % nring;
    const unsigned par0 = (unsigned)((gs / nring) & 1);
    auto issue = [&](int s, int slot) {
      double* Xs = St + slot * sd;
      double* Ws = Xs + BN * sdp;
      const int b0 = s * BN, nb = min(BN, u.s_b - b0);
      const double* pb = Pb + (u.b_begin + b0) * dpa;
      if (u.bulk) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[slot], 8u * BN * (sdp + u.wrows));
          tma_2d_g2s(Xs, maps + u.xmap, 0, (int)(u.b_begin + b0), &full[slot]);
          tma_2d_g2s(Ws, maps + u.wmap, (int)(u.w_col0 + b0), u.c0, &full[slot]);
        }
      } else {
        const int cpr = dpa >> 1;
        for (int e = lane; e < nb * cpr; e += 32) {
          const int y = e / cpr, ch = e - y * cpr;
          cp_async16(Xs + y * sdp + 2 * ch, pb + y * dpa + 2 * ch, true);
        }
        for (int e = lane; e < u.qc * nb; e += 32) {
          const int rho = e / nb, y = e - rho * nb;
          cp_async8(Ws + rho * BN + y, u.Wb + (int64_t)(u.c0 + rho) * u.ldw + u.w_col0 + b0 + y, true);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[slot]);
      }
    };

    if (warp == 0)
      for (int s = 0, sl = slot0; s < min(nring, nst); s++, sl = sl + 1 == nring ? 0 : sl + 1) issue(s, sl);
    cp_async_wait<0>();
    __syncthreads();  // As visible

    constexpr int NACC = TileCfg<RQ>::NACC;
    double acc[NACC][RQ][2];
#pragma unroll
    for (int h = 0; h < NACC; h++)
#pragma unroll
      for (int i = 0; i < RQ; i++) acc[h][i][0] = acc[h][i][1] = 0.0;
    double accv[NV > 0 ? NV : 1];
#pragma unroll
    for (int i = 0; i < (NV > 0 ? NV : 1); i++) accv[i] = 0.0;
    // DFMA remainder columns 8 RQ .. 8 RQ + nr - 1 (lane-partial sums); classes above 12 have
    // no remainder (tile_split), which keeps their register budget
    constexpr int NRMAX = (NV > 0 || RQ > 12) ? 0 : tile_max_nr(RQ);
    double accr[NRMAX > 0 ? NRMAX : 1];
#pragma unroll
    for (int i = 0; i < (NRMAX > 0 ? NRMAX : 1); i++) accr[i] = 0.0;
    const int nr = NRMAX > 0 ? u.nr : 0;

    const int ar = warp * 8 + (lane >> 2);
    const int64_t ga = a0 + ar;
    int seg_k = 0, seg_next = SEG ? u.seg : 0;  // SEG: current segment, first point of the next
    // store sigma2 x the accumulators of the current output (segment kseg of a segmented unit,
    // else the unit's U) and clear them; the lane-partial DFMA columns are summed over the quad
    auto flush = [&](int kseg) {
      double* Uo = u.U + (int64_t)kseg * u.seg_off;
      const int r = u.row0 + ar;
      if constexpr (NV == 0) {
        if (NRMAX > 0 && nr > 0) {
#pragma unroll
          for (int l = 0; l < NRMAX; l++) {
            double v = accr[l];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            if ((lane & 3) == 0 && r < u.s_a && l < nr) {
              v *= kp.sigma2;
              const int col = u.c0 + 8 * RQ + l;
              if (u.trans) Uo[(int64_t)col * u.ldu + r] = v;
              else Uo[(int64_t)r * u.ldu + col] = v;
            }
            accr[l] = 0.0;
          }
        }
        if (r < u.s_a) {
#pragma unroll
          for (int q = 0; q < RQ; q++) {
#pragma unroll
            for (int e = 0; e < 2; e++) {
              const int l = 8 * q + 2 * (lane & 3) + e;
              if (l < u.qc) {
                const double v = kp.sigma2 * (NACC == 2 ? acc[0][q][e] + acc[NACC - 1][q][e] : acc[0][q][e]);
                if (u.trans) Uo[(int64_t)(u.c0 + l) * u.ldu + r] = v;
                else Uo[(int64_t)r * u.ldu + u.c0 + l] = v;
              }
            }
          }
        }
#pragma unroll
        for (int h = 0; h < NACC; h++)
#pragma unroll
          for (int i = 0; i < RQ; i++) acc[h][i][0] = acc[h][i][1] = 0.0;
      }
    };
    const double na = nmode ? As[ar * sdp + dk] : 0.0;  // |u_a|^2 of the lane's row (norm mode)
    // the lane's row as a local b index (dga) and the CTA's rows' range [dga_lo, dga_hi], clamped
    // to int: b points are local indices 0 .. s_b - 1, so a far-away row never matches
    auto clamp_i = [](int64_t x) { return (int)max((int64_t)INT_MIN / 2, min((int64_t)INT_MAX / 2, x)); };
    const int dga = clamp_i(ga - u.b_begin);
    const int dga_lo = clamp_i(a0 - u.b_begin), dga_hi = clamp_i(a0 + rows - 1 - u.b_begin);
    double arow[SYM ? NV : 1];  // a_i of the lane's row (column part of the symmetric product)
    if constexpr (SYM) {
#pragma unroll
      for (int l = 0; l < NV; l++)  // sigma2 folded in here (the row part gets it in the epilogue)
        arow[l] = (ar < rows && l < u.qc) ? kp.sigma2 * u.Wb[(int64_t)l * u.ldw + ga] : 0.0;
    }
    int slot = slot0;
    unsigned par = par0;
    // 1. Gram: g = |u_a - u_b|^2 for the T sub-tiles of a stage (independent chains); norm mode
    //    starts the accumulators at |u_a|^2 + |u_b|^2
    const double* ap = As + ar * sdp + (lane & 3);
    auto gram = [&](const double* Xs, double (&g)[T][2]) {
      if (nmode) {
#pragma unroll
        for (int t = 0; t < T; t++) {
          const double* nb = Xs + (8 * t + 2 * (lane & 3)) * sdp + dk;
          g[t][0] = na + nb[0];
          g[t][1] = na + nb[sdp];
        }
      } else {
#pragma unroll
        for (int t = 0; t < T; t++) g[t][0] = g[t][1] = 0.0;
      }
      const double* bp = Xs + (lane >> 2) * sdp + (lane & 3);
#pragma unroll 4
      for (int ks = 0; ks < ks_n; ks++) {
        const double a = ap[4 * ks];
#pragma unroll
        for (int t = 0; t < T; t++) dmma_8x8x4(g[t][0], g[t][1], a, bp[8 * t * sdp + 4 * ks]);
      }
    };
    for (int s = 0; s < nst; s++) {
      const double* Xs = St + slot * sd;
      const double* Ws = Xs + BN * sdp;
      const int yb = s * BN;                       // first b point of the stage (local index)
      double gr[T][2];
      mbar_wait(&full[slot], par);
      gram(Xs, gr);
      // 2. covariances in registers: closed form, same-site entries exactly 1 + nugget/sigma2,
      //    points past the range exactly 0 (their stage rows are stale)
      // masks only where a stage can need them (warp-uniform tests): the CTA's rows inside the
      // stage's b range (same-site entries; for SYM the diagonal j vs i), and the range end
      // (SYM: any stage starting at or before the last row needs the j <= i masks)
      const bool diag = SYM ? yb <= dga_hi : (dga_lo < yb + BN && yb <= dga_hi);
      const bool tail = yb + BN > u.s_b;
      double cv[T][2];
#pragma unroll
      for (int t = 0; t < T; t++) {
#pragma unroll
        for (int e = 0; e < 2; e++) cv[t][e] = corr<FAM>(gr[t][e], s_tab, kp);
      }
      if (diag || tail) {
#pragma unroll
        for (int t = 0; t < T; t++) {
          const int y = yb + 8 * t + 2 * (lane & 3);
#pragma unroll
          for (int e = 0; e < 2; e++) {
            if (y + e == dga) cv[t][e] = kp.same_val;
            if (y + e >= u.s_b) cv[t][e] = 0.0;
          }
        }
      }
      double cvc[SYM ? T : 1][2];  // column-part weights: j > i only (arow is 0 past the rows)
      if constexpr (SYM) {
#pragma unroll
        for (int t = 0; t < T; t++) {
#pragma unroll
          for (int e = 0; e < 2; e++) cvc[t][e] = cv[t][e];
        }
        if (diag) {
#pragma unroll
          for (int t = 0; t < T; t++) {
            const int y = yb + 8 * t + 2 * (lane & 3);
#pragma unroll
            for (int e = 0; e < 2; e++) {
              if (y + e <= dga) cvc[t][e] = 0.0;
              if (y + e < dga) cv[t][e] = 0.0;  // row part: j >= i only
            }
          }
        }
      }
      if constexpr (NV > 0) {
        // 3'. C a for NV vectors: lane-local DFMAs over the lane's two columns per sub-tile
#pragma unroll
        for (int t = 0; t < T; t++) {
          const int ch = 4 * t + (lane & 3);
#pragma unroll
          for (int l = 0; l < NV; l++) {
            const double2 wv = *reinterpret_cast<const double2*>(Ws + l * BN + 2 * ch);
            accv[l] = fma(cv[t][0], wv.x, accv[l]);
            accv[l] = fma(cv[t][1], wv.y, accv[l]);
          }
        }
        if constexpr (SYM && NV == 1) {
          // column part, one vector: the 2T values of a lane (its two columns per sub-tile) are
          // summed over the warp's 8 rows (the lanes with equal lane & 3) by a reduce-scatter
          // (recursive halving over the row bits: 2T - 2 adds per lane instead of 3 x 2T for an
          // all-reduce, and each lane stores its own 2T/8 sums -- the kernel was issue-bound);
          // lane row r ends with the values r Q .. r Q + Q - 1
          constexpr int NVAL = 2 * T, P8 = (NVAL + 7) / 8 * 8, Q = P8 / 8;
          double v[P8];
#pragma unroll
          for (int t = 0; t < T; t++) {
            v[2 * t] = cvc[t][0] * arow[0];
            v[2 * t + 1] = cvc[t][1] * arow[0];
          }
#pragma unroll
          for (int i = NVAL; i < P8; i++) v[i] = 0.0;
          const int r = lane >> 2;
#pragma unroll
          for (int step = 0; step < 3; step++) {
            const int half = P8 >> (step + 1);
            const int mask = 16 >> step;       // lane bits 4, 3, 2 = row bits 2, 1, 0
            const bool up = (r & (4 >> step)) != 0;
#pragma unroll
            for (int i = 0; i < half; i++) {
              const double keep = up ? v[i + half] : v[i];
              const double send = up ? v[i] : v[i + half];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
            }
          }
#pragma unroll
          for (int q = 0; q < Q; q++) {
            const int idx = r * Q + q;
            const int y = yb + 8 * (idx >> 1) + 2 * (lane & 3) + (idx & 1);
            if (idx < NVAL) const_cast<double*>(Xs)[red_off + warp * BN + (y - yb)] = v[q];
          }
        } else if constexpr (SYM) {
          // column part: sum over the warp's 8 rows (lanes with equal lane & 3), lanes 0..3
          // keep the sums of their columns
#pragma unroll
          for (int t = 0; t < T; t++) {
#pragma unroll
            for (int e = 0; e < 2; e++) {
#pragma unroll
              for (int l = 0; l < NV; l++) {
                double v = cvc[t][e] * arow[l];
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                const int y = yb + 8 * t + 2 * lane + e;
                if (lane < 4) const_cast<double*>(Xs)[red_off + (warp * NV + l) * BN + (y - yb)] = v;
              }
            }
          }
        }
      } else {
        // 3./4. the accumulator entries are the A fragments of k-steps 0, 1 (no shuffles); W_b
        // fragments for G n-tiles are held in registers
#pragma unroll
        for (int t = 0; t < T; t++) {
          if constexpr (SEG) {  // warp-uniform: a segment ends before this sub-tile
            if (yb + 8 * t == seg_next && seg_next < u.s_b) {
              flush(seg_k++);
              seg_next += u.seg;
            }
          }
#pragma unroll
          for (int q0 = 0; q0 < RQ; q0 += G) {
            double2 w[G];
#pragma unroll
            for (int qq = 0; qq < G; qq++) {
              if (q0 + qq < RQ) {
                const int rho = 8 * (q0 + qq) + (lane >> 2);
                w[qq] = *reinterpret_cast<const double2*>(Ws + rho * BN + 2 * (4 * t + (lane & 3)));
              }
            }
#pragma unroll
            for (int qq = 0; qq < G; qq++)
              if (q0 + qq < RQ) dmma_8x8x4(acc[0][q0 + qq][0], acc[0][q0 + qq][1], cv[t][0], w[qq].x);
#pragma unroll
            for (int qq = 0; qq < G; qq++)
              if (q0 + qq < RQ)
                dmma_8x8x4(acc[NACC - 1][q0 + qq][0], acc[NACC - 1][q0 + qq][1], cv[t][1], w[qq].y);
          }
          // remainder columns on DFMA: every lane of a quad reads the same W row (broadcast)
          if (NRMAX > 0 && nr > 0) {
#pragma unroll
            for (int l = 0; l < NRMAX; l++) {
              if (l < nr) {
                const double2 wv =
                    *reinterpret_cast<const double2*>(Ws + (8 * RQ + l) * BN + 2 * (4 * t + (lane & 3)));
                accr[l] = fma(cv[t][0], wv.x, accr[l]);
                accr[l] = fma(cv[t][1], wv.y, accr[l]);
              }
            }
          }
        }
      }
      // release the slot: the last of the four warps refills it with stage s + nring
      if constexpr (SYM) __threadfence_block();  // the column partials, before the count
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(&cnt[slot], 1) == 3;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        if constexpr (SYM) {
          // the stage's column partials of the CTA's 32 rows: warps 0..3 summed in order
          __threadfence_block();
          const double* rd = Xs + red_off;
          for (int e = lane; e < NV * BN; e += 32) {
            const int l = e / BN, y = e - l * BN;
            if (yb + y < u.s_b && l < u.qc)
              colpart[u.cp_off + (int64_t)l * u.s_b + yb + y] =
                  ((rd[(0 * NV + l) * BN + y] + rd[(1 * NV + l) * BN + y]) + rd[(2 * NV + l) * BN + y]) +
                  rd[(3 * NV + l) * BN + y];
          }
          __syncwarp();
        }
        if (lane == 0) cnt[slot] = 0;
        if (s + nring < nst) issue(s + nring, slot);  // stage s + nring reuses this slot
      }
      if (++slot == nring) {
        slot = 0;
        par ^= 1u;
      }
    }
    gs += nst;
    // epilogue: U = sigma2 * acc
    const int r = u.row0 + ar;
    if constexpr (NV > 0) {
#pragma unroll
      for (int l = 0; l < NV; l++) {
        double v = accv[l];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if ((lane & 3) == 0 && r < u.s_a && l < u.qc) {
          v *= kp.sigma2;
          if (u.trans) u.U[(int64_t)(u.c0 + l) * u.ldu + r] = v;
          else u.U[(int64_t)r * u.ldu + u.c0 + l] = v;
        }
      }
    } else {
      flush(seg_k);
    }
  }
}

struct AugArgs {
  const double* Pa;
  const double* Pb;
  int dpa, dk, sdp;
  const CUtensorMap* maps;
  const int32_t* task_range;  // task -> range (relative to the class), per class
  const int32_t* task_first;  // range -> first task (relative to the class)
  double* colpart = nullptr;  // symmetric C a column partials (nullptr: ordinary product)
  bool seg = false;           // segmented units (the nested assembly's leaf runs; rq <= 9)
};

// task -> range map of one class: ranges r own tasks first[r] .. first[r] + n_tasks[r] - 1
__global__ void k_expand_tasks(const int32_t* __restrict__ first, const int32_t* __restrict__ ntask, int n_ranges,
                               int32_t* __restrict__ task_range) {
  const int r = blockIdx.x;
  if (r >= n_ranges) return;
  for (int t = threadIdx.x; t < ntask[r]; t += blockDim.x) task_range[first[r] + t] = r;
}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw Error(MLK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// row-major FP64 matrix (rows x cols, row stride ld elements) read in boxes of box_rows x box_cols
CUtensorMap make_map_2d(const double* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows,
                        uint32_t box_cols) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * sizeof(double)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(MLK_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

namespace {

int class_bn(int rq) {
  switch (rq) {
    case 1: case -1: case -2: case -4: return TileCfg<1>::BN;
    case 2: case 3: case 4: return TileCfg<2>::BN;
    case 6: return TileCfg<6>::BN;
    case 7: return TileCfg<7>::BN;
    case 8: return TileCfg<8>::BN;
    case 9: return TileCfg<9>::BN;
    default: return TileCfg<24>::BN;
  }
}

template <int RQ, int FAM, int NV = 0, bool SYM = false, bool SEG = false>
void launch_class(Ctx& c, const AugArgs& ag, const KernelParams& kp, const TileUnit* units, int n, int* counter) {
  // units = this class's ranges; n = its tasks (ag.task_range / ag.task_first are class-relative)
  constexpr int BN = TileCfg<RQ>::BN;
  auto fn = k_tile_contract<RQ, FAM, NV, SYM, SEG>;
  // ring depth: the deepest ring (<= NST, >= 2) that keeps MIN_CTAS resident CTAs per SM (the
  // stage size grows with d: a fixed depth cut cfg3 / cfg4 to 1-2 CTAs per SM).  Attribute and
  // occupancy queries are driver round trips: once per instantiation, device and row stride
  // (the dynamic shared-memory attribute is per device), under a lock.
  struct Cfg {
    int nring = 0, occ = 0;
    size_t smem = 0;
  };
  static std::mutex mu;
  static std::map<std::pair<int, int>, Cfg> cache;
  static std::map<int, size_t> attr;  // per device: the MaxDynamicSharedMemorySize now set
  std::lock_guard<std::mutex> lock(mu);
  Cfg& cf = cache[{c.device, ag.sdp}];
  if (cf.nring == 0) {
    for (int ns = TileCfg<RQ>::NST; ns >= 2; ns--) {
      const size_t sm_ns =
          sizeof(double) * (size_t)(32 * ag.sdp + ns * stage_doubles(RQ, BN, ag.sdp, sym_red_doubles(SYM, NV, BN), NV));
      if (sm_ns > 227 * 1024) continue;
      CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_ns));
      attr[c.device] = sm_ns;
      int o = 0;
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 128, sm_ns));
      if (cf.nring == 0 || o > cf.occ) {  // deepest ring at the best occupancy seen
        cf.nring = ns;
        cf.occ = o;
        cf.smem = sm_ns;
      }
      if (o >= TileCfg<RQ>::MIN_CTAS) break;
    }
    if (cf.nring == 0) throw Error(MLK_ERR_UNSUPPORTED, "tile stages do not fit shared memory");
    cf.occ = std::max(cf.occ, 1);
  }
  // the attribute is an upper bound: raise it when this row stride needs more than the last
  // configuration set on this device (a smaller launch is always allowed)
  if (attr[c.device] < cf.smem) {
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf.smem));
    attr[c.device] = cf.smem;
  }
  int grid = std::min<int64_t>(n, (int64_t)num_sms(c.device) * cf.occ);
  fn<<<grid, 128, cf.smem, c.stream>>>(units, ag.task_range, ag.task_first, n, counter, ag.Pa, ag.Pb, ag.dpa, ag.dk,
                                       ag.sdp, cf.nring, kp, ag.maps, ag.colpart);
  check_launch("k_tile_contract");
}

template <int FAM>
void launch_fam(Ctx& c, const AugArgs& ag, const KernelParams& kp, int rq, const TileUnit* units, int n,
                int* counter) {
  switch (rq) {
    case -1:
      if (ag.colpart) launch_class<1, FAM, 1, true>(c, ag, kp, units, n, counter);
      else launch_class<1, FAM, 1>(c, ag, kp, units, n, counter);
      break;
    case -2:
      if (ag.colpart) launch_class<1, FAM, 2, true>(c, ag, kp, units, n, counter);
      else launch_class<1, FAM, 2>(c, ag, kp, units, n, counter);
      break;
    case -4:
      if (ag.colpart) launch_class<1, FAM, 4, true>(c, ag, kp, units, n, counter);
      else launch_class<1, FAM, 4>(c, ag, kp, units, n, counter);
      break;
#define MLK_SEG_CASE(K)                                                            \
  case K:                                                                          \
    if (ag.seg) launch_class<K, FAM, 0, false, true>(c, ag, kp, units, n, counter); \
    else launch_class<K, FAM>(c, ag, kp, units, n, counter);                        \
    break;
    MLK_SEG_CASE(1) MLK_SEG_CASE(2) MLK_SEG_CASE(3) MLK_SEG_CASE(4) MLK_SEG_CASE(6) MLK_SEG_CASE(7)
    MLK_SEG_CASE(8) MLK_SEG_CASE(9)
#undef MLK_SEG_CASE
    case 12: launch_class<12, FAM>(c, ag, kp, units, n, counter); break;
    case 16: launch_class<16, FAM>(c, ag, kp, units, n, counter); break;
    case 20: launch_class<20, FAM>(c, ag, kp, units, n, counter); break;
    case 24: launch_class<24, FAM>(c, ag, kp, units, n, counter); break;
    default: throw Error(MLK_ERR_INVALID_ARG, "bad rq class");
  }
}

}  // namespace

// Gram columns: augmented [u, |u|^2, 1] rows when d + 2 pads to the same multiple of 4 as d,
// else (d = 3, 4 mod 4, e.g. cfg3's d = 20) the norm mode: one DMMA k-step fewer per sub-tile.
// The shared-memory row stride avoids 2-way bank conflicts of the fragment loads when dpa/4 is
// even.
void tile_aug_layout(int d, AugCoords& a) {
#ifndef MLK_NO_NORM_MODE  // A/B switch (tools/build_variant.py)
  const bool norm_mode = pad4(d + 2) > pad4(d);
#else
  const bool norm_mode = false;
#endif
  if (norm_mode) {
    a.dk = pad4(d);
    a.dpa = a.dk + 4;
  } else {
    a.dk = a.dpa = pad4(d + 2);
  }
  a.sdp = ((a.dpa >> 2) & 1) ? a.dpa : a.dpa + 4;
}

const double* tile_aug_get(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, const AugCoords& a) {
  const size_t need = (size_t)2 * tree->n * a.dpa;
  if (tree->aug.p && tree->aug.n == need && tree->aug_scale == kp.scale && tree->aug_dpa == a.dpa)
    return tree->aug.p;
  if (tree->aug.n != need) tree->aug.alloc(need, c.stream);
  k_tile_aug<<<(unsigned)ceil_div(tree->n, 256), 256, 0, c.stream>>>(tree->Xt.p, tree->d_pad, tree->d, tree->n,
                                                                     kp.scale, tree->aug.p,
                                                                     tree->aug.p + (size_t)tree->n * a.dpa, a.dpa, a.dk);
  check_launch("k_tile_aug");
  tree->aug_scale = kp.scale;
  tree->aug_dpa = a.dpa;
  return tree->aug.p;
}

void run_tile_contract(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, std::vector<TileUnit>& units,
                       const char* name, double* colpart) {
  if (units.empty()) return;
  // ranges grouped by class, largest per-task cost first inside a class
  std::vector<int32_t> order(units.size());
  for (size_t i = 0; i < units.size(); i++) order[i] = (int32_t)i;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    const TileUnit& a = units[x];
    const TileUnit& b = units[y];
    if (a.rq != b.rq) return a.rq > b.rq;
    return a.cost > b.cost;
  });
  std::vector<TileUnit> ranges(units.size());
  for (size_t i = 0; i < order.size(); i++) ranges[i] = units[order[i]];
  // classes, task prefixes (class-relative)
  std::vector<int> starts;
  for (size_t i = 0; i < ranges.size(); i++)
    if (i == 0 || ranges[i].rq != ranges[i - 1].rq) starts.push_back((int)i);
  starts.push_back((int)ranges.size());
  std::vector<int32_t> first(ranges.size()), ntask(ranges.size());
  std::vector<int64_t> class_task0(starts.size(), 0);
  int64_t tasks_total = 0;
  for (size_t g = 0; g + 1 < starts.size(); g++) {
    class_task0[g] = tasks_total;
    int32_t acc = 0;
    for (int i = starts[g]; i < starts[g + 1]; i++) {
      first[i] = acc;
      ntask[i] = ranges[i].n_tasks;
      acc += ranges[i].n_tasks;
    }
    tasks_total += acc;
  }
  class_task0.back() = tasks_total;
  DevBuf<int> counters(starts.size(), c.stream);
  counters.zero();
  // augmented, pre-scaled coordinates (k_tile_aug); the smem row stride avoids 2-way bank
  // conflicts of the fragment loads when dpa/4 is even
  AugArgs ag;
  ag.colpart = colpart;
  ag.seg = units.front().seg > 0;
  for (const auto& u : units)
    MLK_REQUIRE((u.seg > 0) == ag.seg && (!ag.seg || (u.rq >= 1 && u.rq <= 9)),
                "run_tile_contract: segmented and plain units cannot share a call");
  AugCoords aug;
  tile_aug_layout(tree->d, aug);
  ag.dk = aug.dk;
  ag.dpa = aug.dpa;
  ag.sdp = aug.sdp;
  ag.Pa = tile_aug_get(c, tree, kp, aug);  // formed on the stream here unless cached
  ag.Pb = ag.Pa + (size_t)tree->n * ag.dpa;
  // tensor maps: one for the b rows per stage width, one per distinct W_b (base, shape, box)
  std::vector<CUtensorMap> maps;
  {
    std::map<std::array<int64_t, 6>, int> idx;
    auto get = [&](const double* base, int64_t rows, int64_t cols, int64_t ld, int br, int bc) {
      std::array<int64_t, 6> key{(int64_t)reinterpret_cast<uintptr_t>(base), rows, cols, ld, br, bc};
      auto it = idx.find(key);
      if (it != idx.end()) return it->second;
      int k = (int)maps.size();
      maps.push_back(make_map_2d(base, rows, cols, ld, br, bc));
      idx[key] = k;
      return k;
    };
    const TileUnit* prev = nullptr;  // consecutive ranges mostly share W_b: skip the lookup
    for (auto& u : ranges) {
      // C a (rq < 0): stage only the qc real vector rows (the kernel never reads rows >= qc)
      u.wrows = u.rq > 0 ? 8 * u.rq + u.nr : u.qc;
      if (!u.bulk) continue;
      if (prev && prev->Wb == u.Wb && prev->rq == u.rq && prev->nr == u.nr && prev->p_b == u.p_b &&
          prev->w_cols == u.w_cols && prev->ldw == u.ldw) {
        u.xmap = prev->xmap;
        u.wmap = prev->wmap;
      } else {
        const int bn = class_bn(u.rq);
        u.xmap = get(ag.Pb, tree->n, ag.dpa, ag.dpa, bn, ag.sdp);
        u.wmap = get(u.Wb, u.p_b, u.w_cols, u.ldw, u.wrows, bn);
      }
      prev = &u;
    }
  }
  DevBuf<CUtensorMap> maps_d(std::max<size_t>(maps.size(), 1), c.stream);
  maps_d.upload(maps);
  ag.maps = maps_d.p;
  DevBuf<TileUnit> du(ranges.size(), c.stream);
  du.upload(ranges);
  DevBuf<int32_t> first_d(ranges.size(), c.stream), ntask_d(ranges.size(), c.stream);
  first_d.upload(first);
  ntask_d.upload(ntask);
  DevBuf<int32_t> task_range((size_t)std::max<int64_t>(tasks_total, 1), c.stream);
  TimedLaunch tl(c, name);
  for (size_t g = 0; g + 1 < starts.size(); g++) {
    const int s0 = starts[g], nr_ = starts[g + 1] - starts[g];
    k_expand_tasks<<<(unsigned)nr_, 128, 0, c.stream>>>(first_d.p + s0, ntask_d.p + s0, nr_,
                                                        task_range.p + class_task0[g]);
    check_launch("k_expand_tasks");
  }
  for (size_t g = 0; g + 1 < starts.size(); g++) {
    const int s0 = starts[g];
    const int n = (int)(class_task0[g + 1] - class_task0[g]);
    const int rq = ranges[s0].rq;
    ag.task_range = task_range.p + class_task0[g];
    ag.task_first = first_d.p + s0;
    switch (kp.family) {
      case MLK_MATERN_12: launch_fam<MLK_MATERN_12>(c, ag, kp, rq, du.p + s0, n, counters.p + g); break;
      case MLK_MATERN_32: launch_fam<MLK_MATERN_32>(c, ag, kp, rq, du.p + s0, n, counters.p + g); break;
      case MLK_MATERN_52: launch_fam<MLK_MATERN_52>(c, ag, kp, rq, du.p + s0, n, counters.p + g); break;
      case MLK_MATERN_NU: launch_fam<MLK_MATERN_NU>(c, ag, kp, rq, du.p + s0, n, counters.p + g); break;
      default: launch_fam<MLK_GAUSSIAN>(c, ag, kp, rq, du.p + s0, n, counters.p + g); break;
    }
  }
}

}  // namespace mlk
