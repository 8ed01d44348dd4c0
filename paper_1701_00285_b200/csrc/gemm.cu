// Batched variable-size FP64 GEMM on DMMA.8x8x4 (row-major NN or TN, optional transposed store).
// Used for the basis transfers Phi_q/W_q = Q^T (Phi_L (+) Phi_R), the blocked QR's trailing
// updates and the second contraction B = W_a U of the assembly.  Three tilings, chosen per
// product by the smallest padded volume: 64 x 64 (2 x 2 warps of 32 x 32), 72 x 72 (3 x 3
// warps of 24 x 24; the p = 66 products of cfg2 pad to 72 instead of 128) and 64 x 32 (the
// 32-column panel products of the blocked QR).  Every output element accumulates over k in the
// same order under every tiling, so the choice does not change results.  k steps of 16 with cp.async double
// buffering; k > KCHUNK is split into fixed chunks reduced in order (deterministic).
#include <algorithm>

#include "api.cuh"
#include "dmma.cuh"

namespace mlk {
namespace {

constexpr int BK = 16;
constexpr int64_t KCHUNK = 8192;

template <int WTM, int WTN, int WM, int WN>  // 8x8 tiles per warp (m, n), warps (m, n)
struct GemmCfg {
  static constexpr int BM = 8 * WTM * WM, BN = 8 * WTN * WN;
  static constexpr int NT = 32 * WM * WN;
  static constexpr int AS = BK + 4;   // A tile row stride (doubles): conflict-free fragment reads
  static constexpr int BS = BN + 4;   // B tile row stride: 2 BS = 8 (mod 32) words -> conflict-free
};
using Cfg64 = GemmCfg<4, 4, 2, 2>;
using Cfg72 = GemmCfg<3, 3, 3, 3>;
using Cfg32 = GemmCfg<4, 2, 2, 2>;

struct GemmJob {
  int32_t desc;
  int32_t m0, n0;
  int32_t part;  // -1: final store; else partial slot index
  int64_t k0, k1;
};

template <class CF>
__device__ __forceinline__ void load_tiles(const GemmDesc& g, int m0, int n0, int64_t kk, int64_t k1, double* As,
                                           double* Bs) {
  const int tid = threadIdx.x;
  if (g.trans_a) {  // A(m, k) at A[k lda + m]: rows of the tile fastest, coalesced along m
    for (int e = tid; e < CF::BM * BK; e += CF::NT) {
      const int row = e % CF::BM, col = e / CF::BM;
      const int gm = m0 + row;
      const int64_t gk = kk + col;
      const bool ok = gm < g.m && gk < k1;
      cp_async8(As + row * CF::AS + col, ok ? g.A + gk * g.lda + gm : g.A, ok);
    }
  } else {
    for (int e = tid; e < CF::BM * BK; e += CF::NT) {
      const int row = e / BK, col = e % BK;
      const int gm = m0 + row;
      const int64_t gk = kk + col;
      const bool ok = gm < g.m && gk < k1;
      cp_async8(As + row * CF::AS + col, ok ? g.A + (int64_t)gm * g.lda + gk : g.A, ok);
    }
  }
  for (int e = tid; e < BK * CF::BN; e += CF::NT) {
    const int row = e / CF::BN, col = e % CF::BN;
    const int64_t gk = kk + row;
    const int gn = n0 + col;
    const bool ok = gk < k1 && gn < g.n;
    cp_async8(Bs + row * CF::BS + col, ok ? g.B + gk * g.ldb + gn : g.B, ok);
  }
}

template <int WTM, int WTN, int WM, int WN>
__global__ void __launch_bounds__(32 * WM * WN) k_gemm(const GemmDesc* __restrict__ descs,
                                                       const GemmJob* __restrict__ jobs,
                                                       double* __restrict__ partials) {
  using CF = GemmCfg<WTM, WTN, WM, WN>;
  constexpr int BM = CF::BM, BN = CF::BN, AS = CF::AS, BS = CF::BS;
  __shared__ __align__(16) double As[2][BM * AS];
  __shared__ __align__(16) double Bs[2][BK * BS];
  const GemmJob job = jobs[blockIdx.x];
  const GemmDesc g = descs[job.desc];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp / WN) * 8 * WTM, wn = (warp % WN) * 8 * WTN;
  double acc[WTM][WTN][2];
#pragma unroll
  for (int i = 0; i < WTM; i++)
#pragma unroll
    for (int j = 0; j < WTN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t nk = (job.k1 - job.k0 + BK - 1) / BK;
  if (nk > 0) load_tiles<CF>(g, job.m0, job.n0, job.k0, job.k1, As[0], Bs[0]);
  cp_async_commit();
  for (int64_t it = 0; it < nk; it++) {
    const int cur = it & 1;
    if (it + 1 < nk) load_tiles<CF>(g, job.m0, job.n0, job.k0 + (it + 1) * BK, job.k1, As[cur ^ 1], Bs[cur ^ 1]);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* A = As[cur];
    const double* B = Bs[cur];
#pragma unroll
    for (int ks = 0; ks < BK / 4; ks++) {
      double af[WTM], bf[WTN];
#pragma unroll
      for (int i = 0; i < WTM; i++) af[i] = A[(wm + i * 8 + (lane >> 2)) * AS + ks * 4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < WTN; j++) bf[j] = B[(ks * 4 + (lane & 3)) * BS + wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < WTM; i++)
#pragma unroll
        for (int j = 0; j < WTN; j++) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < WTM; i++) {
#pragma unroll
    for (int j = 0; j < WTN; j++) {
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int r = wm + i * 8 + (lane >> 2);
        const int cc = wn + j * 8 + 2 * (lane & 3) + e;
        if (job.part >= 0) {
          partials[(int64_t)job.part * BM * BN + r * BN + cc] = acc[i][j][e];
        } else {
          const int gm = job.m0 + r, gn = job.n0 + cc;
          if (gm < g.m && gn < g.n) {
            double v = acc[i][j][e];
            if (g.diag >= 0) v = ((int64_t)gm + g.diag == gn ? 1.0 : 0.0) - v;
            double* cp = g.trans_c ? g.C + (int64_t)gn * g.ldc + gm : g.C + (int64_t)gm * g.ldc + gn;
            if (g.sub) v = *cp - v;
            *cp = v;
          }
        }
      }
    }
  }
}

struct ReduceJob {
  int32_t desc, m0, n0, nparts;
  int64_t first;  // first partial slot
};

template <int BM, int BN>
__global__ void k_gemm_reduce(const GemmDesc* __restrict__ descs, const ReduceJob* __restrict__ jobs,
                              const double* __restrict__ partials) {
  const ReduceJob job = jobs[blockIdx.x];
  const GemmDesc g = descs[job.desc];
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    const int r = e / BN, cc = e % BN;
    const int gm = job.m0 + r, gn = job.n0 + cc;
    if (gm >= g.m || gn >= g.n) continue;
    double s = 0.0;
    for (int p = 0; p < job.nparts; p++) s += partials[(job.first + p) * BM * BN + e];
    if (g.diag >= 0) s = ((int64_t)gm + g.diag == gn ? 1.0 : 0.0) - s;
    double* cp = g.trans_c ? g.C + (int64_t)gn * g.ldc + gm : g.C + (int64_t)gm * g.ldc + gn;
    if (g.sub) s = *cp - s;
    *cp = s;
  }
}

// padded volume of a product under a tiling
int64_t padded(const GemmDesc& g, int bm, int bn) { return ceil_div(g.m, bm) * bm * ceil_div(g.n, bn) * bn; }

template <class CF, int WTM, int WTN, int WM, int WN>
void run_tiling(Ctx& c, const GemmDesc* dd, const std::vector<GemmDesc>& descs, const std::vector<int32_t>& sel) {
  constexpr int BM = CF::BM, BN = CF::BN;
  std::vector<GemmJob> jobs;
  std::vector<ReduceJob> red;
  int64_t slots = 0;
  for (int32_t di : sel) {
    const GemmDesc& g = descs[di];
    const int64_t nchunks = g.k <= KCHUNK ? 1 : ceil_div(g.k, KCHUNK);
    for (int m0 = 0; m0 < g.m; m0 += BM)
      for (int n0 = 0; n0 < g.n; n0 += BN) {
        if (nchunks == 1) {
          jobs.push_back({di, m0, n0, -1, 0, (int64_t)g.k});
        } else {
          red.push_back({di, m0, n0, (int32_t)nchunks, slots});
          for (int64_t ch = 0; ch < nchunks; ch++) {
            const int64_t k0 = ch * KCHUNK, k1 = std::min<int64_t>(g.k, k0 + KCHUNK);
            jobs.push_back({di, m0, n0, (int32_t)slots++, k0, k1});
          }
        }
      }
  }
  if (jobs.empty()) return;
  // biggest jobs first (k extent), so long tiles start early
  std::stable_sort(jobs.begin(), jobs.end(),
                   [](const GemmJob& a, const GemmJob& b) { return (a.k1 - a.k0) > (b.k1 - b.k0); });
  DevBuf<GemmJob> dj(jobs.size(), c.stream);
  dj.upload(jobs);
  DevBuf<double> parts((size_t)slots * BM * BN, c.stream);
  k_gemm<WTM, WTN, WM, WN><<<(unsigned)jobs.size(), CF::NT, 0, c.stream>>>(dd, dj.p, parts.p);
  check_launch("k_gemm");
  if (!red.empty()) {
    DevBuf<ReduceJob> dr(red.size(), c.stream);
    dr.upload(red);
    k_gemm_reduce<BM, BN><<<(unsigned)red.size(), 256, 0, c.stream>>>(dd, dr.p, parts.p);
    check_launch("k_gemm_reduce");
  }
}

}  // namespace

void gemm_batched(Ctx& c, const std::vector<GemmDesc>& descs, const char* name) {
  if (descs.empty()) return;
  std::vector<int32_t> s64, s72, s32;
  for (int32_t di = 0; di < (int32_t)descs.size(); di++) {
    const GemmDesc& g = descs[di];
    if (g.m <= 0 || g.n <= 0) continue;
    const int64_t v64 = padded(g, Cfg64::BM, Cfg64::BN), v72 = padded(g, Cfg72::BM, Cfg72::BN),
                  v32 = padded(g, Cfg32::BM, Cfg32::BN);
    if (v32 < std::min(v64, v72)) s32.push_back(di);
    else (v72 < v64 ? s72 : s64).push_back(di);
  }
  if (s64.empty() && s72.empty() && s32.empty()) return;
  DevBuf<GemmDesc> dd(descs.size(), c.stream);
  dd.upload(descs);
  TimedLaunch tl(c, name);
  if (!s72.empty()) run_tiling<Cfg72, 3, 3, 3, 3>(c, dd.p, descs, s72);
  if (!s64.empty()) run_tiling<Cfg64, 4, 4, 2, 2>(c, dd.p, descs, s64);
  if (!s32.empty()) run_tiling<Cfg32, 4, 2, 2, 2>(c, dd.p, descs, s32);
}

}  // namespace mlk
