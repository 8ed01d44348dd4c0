// K5a: fused covariance-tile generation + first contraction on FP64 DMMA (see tile.cuh).
//
// CTA = 4 warps, 32 rows of the a range (8 per warp).  The b range is streamed in stages of
// BN points (cp.async double buffering): the stage holds the b coordinates (BN x dp), their
// squared norms and the W_b columns (8 RQ rows x BN, 16-byte chunks XOR-swizzled so the
// B-fragment loads are bank-conflict free).  Per 8-point sub-tile a warp
//   1. forms S = X_a X_b^T with dp/4 DMMA.8x8x4 (k = coordinates),
//   2. turns its two accumulator entries into covariances in registers,
//   3. feeds them straight back as DMMA A-fragments: accumulator column 2(lane%4)+s is the
//      A element k = lane%4 of k-step s, provided W_b is read with the same point
//      permutation -- no shuffles between the two products,
//   4. accumulates U (8 rows x 8 RQ columns) with 2 RQ DMMAs.
// A persistent grid pulls units (largest first) from an atomic counter.
#include <algorithm>
#include <cmath>

#include "dmma.cuh"
#include "fastmath.cuh"
#include "tile.cuh"

namespace mlk {

KernelParams make_kernel_params(const mlk_kernel& k) {
  KernelParams p;
  p.family = k.family;
  p.sigma2 = k.sigma2;
  p.nugget = k.nugget;
  switch (k.family) {
    case MLK_MATERN_12: p.c1 = 1.0 / k.rho; break;
    case MLK_MATERN_32: p.c1 = std::sqrt(3.0) / k.rho; break;
    case MLK_MATERN_52: p.c1 = std::sqrt(5.0) / k.rho; break;
    default: p.c1 = 1.0 / (k.rho * k.rho); break;
  }
  return p;
}

static const int kRQ[] = {1, 2, 3, 4, 6, 7, 9, 12, 16, 20, 24};

int tile_rq_class(int qc) {
  for (int r : kRQ)
    if (8 * r >= qc) return r;
  return kTileMaxRQ;
}

void make_tile_units(std::vector<TileUnit>& out, int64_t a_begin, int32_t s_a, int64_t b_begin, int32_t s_b,
                     const double* Wb, int64_t ldw, int32_t p_b, double* U, int64_t ldu, int32_t trans, int dp) {
  int nch = (int)ceil_div(p_b, 8 * kTileMaxRQ);
  int width = (int)ceil_div(ceil_div(p_b, nch), 8) * 8;
  for (int c0 = 0; c0 < p_b; c0 += width) {
    int qc = std::min(width, p_b - c0);
    int rq = tile_rq_class(qc);
    for (int32_t r0 = 0; r0 < s_a; r0 += 32) {
      TileUnit u;
      u.a_begin = a_begin;
      u.b_begin = b_begin;
      u.s_a = s_a;
      u.s_b = s_b;
      u.row0 = r0;
      u.c0 = c0;
      u.qc = qc;
      u.p_b = p_b;
      u.trans = trans;
      u.rq = rq;
      u.Wb = Wb;
      u.ldw = ldw;
      u.U = U;
      u.ldu = ldu;
      // FP64-slot estimate: Gram dp + kernel ~50 + contraction 8 rq per entry
      u.cost = 32.0 * s_b * (dp + 50 + 8.0 * rq);
      out.push_back(u);
    }
  }
}

namespace {

template <int FAM>
__device__ __forceinline__ double corr(double r2, double c1, const double* tab) {
  if (FAM == MLK_GAUSSIAN) return exp_neg(-r2 * c1, tab);
  double z = sqrt_pos(r2) * c1;
  double e = exp_neg(-z, tab);
  if (FAM == MLK_MATERN_12) return e;
  if (FAM == MLK_MATERN_32) return fma(z, e, e);                  // (1 + z) e^{-z}
  return fma(z, fma(z, 1.0 / 3.0, 1.0), 1.0) * e;                // (1 + z + z^2/3) e^{-z}
}

template <int RQ>
struct TileCfg {
  static constexpr int BN = RQ >= 6 ? 16 : 32;  // b points per stage
  static constexpr int WROWS = 8 * RQ;
};

__host__ __device__ constexpr int stage_doubles(int rq, int bn, int dp) { return bn * dp + bn + 8 * rq * bn; }

template <int RQ, int FAM>
__global__ void __launch_bounds__(128, RQ >= 20 ? 3 : 4) k_tile_contract(const TileUnit* __restrict__ units, int n_units,
                                                       int* __restrict__ counter, const double* __restrict__ Xt,
                                                       const double* __restrict__ norm2, int dp, KernelParams kp) {
  constexpr int BN = TileCfg<RQ>::BN;
  constexpr int WROWS = TileCfg<RQ>::WROWS;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_unit;
  __shared__ double s_tab[16];
  if (threadIdx.x < 16) s_tab[threadIdx.x] = kExp2Tab16[threadIdx.x];
  const int sd = stage_doubles(RQ, BN, dp);
  double* As = sm;                  // 32 x dp
  double* An = sm + 32 * dp;        // 32
  double* St = sm + 32 * dp + 32;   // 2 stages
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  while (true) {
    __syncthreads();
    if (tid == 0) s_unit = atomicAdd(counter, 1);
    __syncthreads();
    const int ui = s_unit;
    if (ui >= n_units) break;
    const TileUnit u = units[ui];
    const int64_t a0 = u.a_begin + u.row0;
    const int rows = min(32, u.s_a - u.row0);
    // a tile (rows x dp) + norms
    for (int e = tid; e < 32 * dp; e += 128) {
      int r = e / dp;
      As[e] = r < rows ? Xt[(a0 + r) * dp + (e - r * dp)] : 0.0;
    }
    if (tid < 32) An[tid] = tid < rows ? norm2[a0 + tid] : 0.0;

    auto load_stage = [&](int st, int b0) {
      double* Xs = St + st * sd;
      double* Ns = Xs + BN * dp;
      double* Ws = Ns + BN;
      const int nb = min(BN, u.s_b - b0);
      // coordinates: rows of dp doubles, 16-byte chunks
      const int cpr = dp / 2;
      for (int e = tid; e < BN * cpr; e += 128) {
        int y = e / cpr, ch = e - y * cpr;
        bool ok = y < nb;
        const double* src = ok ? Xt + (u.b_begin + b0 + y) * dp + 2 * ch : Xt;
        cp_async16(Xs + y * dp + 2 * ch, src, ok);
      }
      for (int y = tid; y < BN; y += 128) {
        bool ok = y < nb;
        cp_async8(Ns + y, ok ? norm2 + u.b_begin + b0 + y : norm2, ok);
      }
      // W_b columns b0..b0+BN of rows c0..c0+8RQ, chunk c of row rho at (c ^ 4(rho&1))
      constexpr int CH = BN / 2;
      for (int e = tid; e < WROWS * CH; e += 128) {
        int rho = e / CH, ch = e - rho * CH;
        int phys = ch ^ ((rho & 1) << 2);
        double* dst = Ws + rho * BN + 2 * phys;
        int y = b0 + 2 * ch;
        bool rowok = rho < u.qc;
        const double* src = u.Wb + (int64_t)(u.c0 + rho) * u.ldw + y;
        bool ok0 = rowok && (y < u.s_b), ok1 = rowok && (y + 1 < u.s_b);
        if (ok0 && ok1 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
          cp_async16(dst, src, true);
        } else {
          cp_async8(dst, ok0 ? src : u.Wb, ok0);
          cp_async8(dst + 1, ok1 ? src + 1 : u.Wb, ok1);
        }
      }
    };

    double acc[RQ][2];
#pragma unroll
    for (int i = 0; i < RQ; i++) acc[i][0] = acc[i][1] = 0.0;

    const int nst = (u.s_b + BN - 1) / BN;
    load_stage(0, 0);
    cp_async_commit();
    __syncthreads();  // As/An visible
    const int ar = warp * 8 + (lane >> 2);
    const double na = An[ar];
    const int64_t ga = a0 + ar;
    const int ks_n = dp >> 2;
    for (int s = 0; s < nst; s++) {
      if (s + 1 < nst) load_stage((s + 1) & 1, (s + 1) * BN);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      const double* Xs = St + (s & 1) * sd;
      const double* Ns = Xs + BN * dp;
      const double* Ws = Ns + BN;
      const int b0 = s * BN;
      constexpr int T = BN / 8;
      // 1. Gram S = X_a X_b^T for the T sub-tiles (independent accumulator chains)
      double g[T][2];
#pragma unroll
      for (int t = 0; t < T; t++) g[t][0] = g[t][1] = 0.0;
      for (int ks = 0; ks < ks_n; ks++) {
        const double a = As[ar * dp + 4 * ks + (lane & 3)];
#pragma unroll
        for (int t = 0; t < T; t++) {
          const double b = Xs[(8 * t + (lane >> 2)) * dp + 4 * ks + (lane & 3)];
          dmma_8x8x4(g[t][0], g[t][1], a, b);
        }
      }
      // 2. covariances in registers (Gram identity, clamp, same-site fix, closed form)
      double cv[T][2];
#pragma unroll
      for (int t = 0; t < T; t++) {
        const int col = 8 * t + 2 * (lane & 3);
#pragma unroll
        for (int e = 0; e < 2; e++) {
          double r2 = fmax(fma(-2.0, g[t][e], na + Ns[col + e]), 0.0);
          const bool same = (u.b_begin + b0 + col + e) == ga;
          if (same) r2 = 0.0;
          double v = kp.sigma2 * corr<FAM>(r2, kp.c1, s_tab);
          cv[t][e] = same ? v + kp.nugget : v;
        }
      }
      // 3./4. accumulator entries are the A fragments of k-steps s = 0, 1; W_b fragments
      // are loaded 4 n-tiles at a time so consecutive DMMAs are independent
#pragma unroll
      for (int t = 0; t < T; t++) {
#pragma unroll
        for (int q0 = 0; q0 < RQ; q0 += 4) {
          double2 w[4];
#pragma unroll
          for (int qq = 0; qq < 4; qq++) {
            if (q0 + qq < RQ) {
              const int rho = 8 * (q0 + qq) + (lane >> 2);
              const int ch = 4 * t + (lane & 3);
              w[qq] = *reinterpret_cast<const double2*>(Ws + rho * BN + 2 * (ch ^ ((rho & 1) << 2)));
            }
          }
#pragma unroll
          for (int qq = 0; qq < 4; qq++)
            if (q0 + qq < RQ) dmma_8x8x4(acc[q0 + qq][0], acc[q0 + qq][1], cv[t][0], w[qq].x);
#pragma unroll
          for (int qq = 0; qq < 4; qq++)
            if (q0 + qq < RQ) dmma_8x8x4(acc[q0 + qq][0], acc[q0 + qq][1], cv[t][1], w[qq].y);
        }
      }
      __syncthreads();
    }
    // epilogue
    const int r = u.row0 + ar;
    if (r < u.s_a) {
#pragma unroll
      for (int q = 0; q < RQ; q++) {
#pragma unroll
        for (int e = 0; e < 2; e++) {
          int l = 8 * q + 2 * (lane & 3) + e;
          if (l < u.qc) {
            if (u.trans) u.U[(int64_t)(u.c0 + l) * u.ldu + r] = acc[q][e];
            else u.U[(int64_t)r * u.ldu + u.c0 + l] = acc[q][e];
          }
        }
      }
    }
  }
}

template <int RQ, int FAM>
void launch_class(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, const TileUnit* units, int n, int* counter) {
  constexpr int BN = TileCfg<RQ>::BN;
  const int dp = tree->d_pad;
  size_t smem = sizeof(double) * (size_t)(32 * dp + 32 + 2 * stage_doubles(RQ, BN, dp));
  auto fn = k_tile_contract<RQ, FAM>;
  CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 128, smem));
  occ = std::max(occ, 1);
  int grid = std::min<int64_t>(n, (int64_t)num_sms(c.device) * occ);
  fn<<<grid, 128, smem, c.stream>>>(units, n, counter, tree->Xt.p, tree->norm2.p, dp, kp);
  check_launch("k_tile_contract");
}

template <int FAM>
void launch_fam(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, int rq, const TileUnit* units, int n,
                int* counter) {
  switch (rq) {
    case 1: launch_class<1, FAM>(c, tree, kp, units, n, counter); break;
    case 2: launch_class<2, FAM>(c, tree, kp, units, n, counter); break;
    case 3: launch_class<3, FAM>(c, tree, kp, units, n, counter); break;
    case 4: launch_class<4, FAM>(c, tree, kp, units, n, counter); break;
    case 6: launch_class<6, FAM>(c, tree, kp, units, n, counter); break;
    case 7: launch_class<7, FAM>(c, tree, kp, units, n, counter); break;
    case 9: launch_class<9, FAM>(c, tree, kp, units, n, counter); break;
    case 12: launch_class<12, FAM>(c, tree, kp, units, n, counter); break;
    case 16: launch_class<16, FAM>(c, tree, kp, units, n, counter); break;
    case 20: launch_class<20, FAM>(c, tree, kp, units, n, counter); break;
    case 24: launch_class<24, FAM>(c, tree, kp, units, n, counter); break;
    default: throw Error(MLK_ERR_INVALID_ARG, "bad rq class");
  }
}

}  // namespace

void run_tile_contract(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, std::vector<TileUnit>& units,
                       const char* name) {
  if (units.empty()) return;
  // group by class, largest cost first inside a class
  std::stable_sort(units.begin(), units.end(), [](const TileUnit& a, const TileUnit& b) {
    if (a.rq != b.rq) return a.rq > b.rq;
    return a.cost > b.cost;
  });
  DevBuf<TileUnit> du(units.size(), c.stream);
  du.upload(units);
  std::vector<int> starts;
  for (size_t i = 0; i < units.size(); i++)
    if (i == 0 || units[i].rq != units[i - 1].rq) starts.push_back((int)i);
  starts.push_back((int)units.size());
  DevBuf<int> counters(starts.size(), c.stream);
  counters.zero();
  TimedLaunch tl(c, name);
  for (size_t g = 0; g + 1 < starts.size(); g++) {
    int s0 = starts[g], n = starts[g + 1] - starts[g];
    int rq = units[s0].rq;
    switch (kp.family) {
      case MLK_MATERN_12: launch_fam<MLK_MATERN_12>(c, tree, kp, rq, du.p + s0, n, counters.p + g); break;
      case MLK_MATERN_32: launch_fam<MLK_MATERN_32>(c, tree, kp, rq, du.p + s0, n, counters.p + g); break;
      case MLK_MATERN_52: launch_fam<MLK_MATERN_52>(c, tree, kp, rq, du.p + s0, n, counters.p + g); break;
      default: launch_fam<MLK_GAUSSIAN>(c, tree, kp, rq, du.p + s0, n, counters.p + g); break;
    }
  }
}

}  // namespace mlk
