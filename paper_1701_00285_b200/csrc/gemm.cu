// Batched variable-size FP64 GEMM on DMMA.8x8x4 (row-major NN, optional transposed store).
// Used for the basis transfers Phi_q/W_q = Q^T (Phi_L (+) Phi_R) and for the second
// contraction B = W_a U of the assembly.  Tile 64 x 64 x 16, 4 warps (32 x 32 each),
// cp.async double buffering; k > KCHUNK is split into fixed chunks reduced in order.
#include <algorithm>

#include "api.cuh"
#include "dmma.cuh"

namespace mlk {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int AS = BK + 4;   // A tile row stride (doubles): conflict-free fragment reads
constexpr int BS = BN + 8;   // B tile row stride
constexpr int64_t KCHUNK = 8192;

struct GemmJob {
  int32_t desc;
  int32_t m0, n0;
  int32_t part;  // -1: final store; else partial slot index
  int64_t k0, k1;
};

__device__ __forceinline__ void load_tiles(const GemmDesc& g, int m0, int n0, int64_t kk, int64_t k1,
                                           double* As, double* Bs) {
  int tid = threadIdx.x;
  // A: 64 x 16
#pragma unroll
  for (int r = 0; r < 8; r++) {
    int e = tid + r * 128;
    int row = e / BK, col = e % BK;
    int gm = m0 + row;
    int64_t gk = kk + col;
    bool ok = gm < g.m && gk < k1;
    const double* src = ok ? g.A + (int64_t)gm * g.lda + gk : g.A;
    cp_async8(As + row * AS + col, src, ok);
  }
  // B: 16 x 64
#pragma unroll
  for (int r = 0; r < 8; r++) {
    int e = tid + r * 128;
    int row = e / BN, col = e % BN;
    int64_t gk = kk + row;
    int gn = n0 + col;
    bool ok = gk < k1 && gn < g.n;
    const double* src = ok ? g.B + gk * g.ldb + gn : g.B;
    cp_async8(Bs + row * BS + col, src, ok);
  }
}

__global__ void __launch_bounds__(128) k_gemm(const GemmDesc* __restrict__ descs, const GemmJob* __restrict__ jobs,
                                              double* __restrict__ partials) {
  __shared__ __align__(16) double As[2][BM * AS];
  __shared__ __align__(16) double Bs[2][BK * BS];
  const GemmJob job = jobs[blockIdx.x];
  const GemmDesc g = descs[job.desc];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  int64_t nk = (job.k1 - job.k0 + BK - 1) / BK;
  if (nk > 0) load_tiles(g, job.m0, job.n0, job.k0, job.k1, As[0], Bs[0]);
  cp_async_commit();
  for (int64_t it = 0; it < nk; it++) {
    int cur = it & 1;
    if (it + 1 < nk) load_tiles(g, job.m0, job.n0, job.k0 + (it + 1) * BK, job.k1, As[cur ^ 1], Bs[cur ^ 1]);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* A = As[cur];
    const double* B = Bs[cur];
#pragma unroll
    for (int ks = 0; ks < BK / 4; ks++) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; i++) af[i] = A[(wm + i * 8 + (lane >> 2)) * AS + ks * 4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; j++) bf[j] = B[(ks * 4 + (lane & 3)) * BS + wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
#pragma unroll
      for (int e = 0; e < 2; e++) {
        int r = wm + i * 8 + (lane >> 2);
        int cc = wn + j * 8 + 2 * (lane & 3) + e;
        if (job.part >= 0) {
          partials[(int64_t)job.part * BM * BN + r * BN + cc] = acc[i][j][e];
        } else {
          int gm = job.m0 + r, gn = job.n0 + cc;
          if (gm < g.m && gn < g.n) {
            double v = acc[i][j][e];
            if (g.diag >= 0) v = ((int64_t)gm + g.diag == gn ? 1.0 : 0.0) - v;
            if (g.trans_c) g.C[(int64_t)gn * g.ldc + gm] = v;
            else g.C[(int64_t)gm * g.ldc + gn] = v;
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

__global__ void k_gemm_reduce(const GemmDesc* __restrict__ descs, const ReduceJob* __restrict__ jobs,
                              const double* __restrict__ partials) {
  const ReduceJob job = jobs[blockIdx.x];
  const GemmDesc g = descs[job.desc];
  for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
    int r = e / BN, cc = e % BN;
    int gm = job.m0 + r, gn = job.n0 + cc;
    if (gm >= g.m || gn >= g.n) continue;
    double s = 0.0;
    for (int p = 0; p < job.nparts; p++) s += partials[(job.first + p) * BM * BN + e];
    if (g.diag >= 0) s = ((int64_t)gm + g.diag == gn ? 1.0 : 0.0) - s;
    if (g.trans_c) g.C[(int64_t)gn * g.ldc + gm] = s;
    else g.C[(int64_t)gm * g.ldc + gn] = s;
  }
}

}  // namespace

void gemm_batched(Ctx& c, const std::vector<GemmDesc>& descs, const char* name) {
  if (descs.empty()) return;
  std::vector<GemmJob> jobs;
  std::vector<ReduceJob> red;
  int64_t slots = 0;
  for (int32_t di = 0; di < (int32_t)descs.size(); di++) {
    const GemmDesc& g = descs[di];
    if (g.m <= 0 || g.n <= 0) continue;
    int64_t nchunks = g.k <= KCHUNK ? 1 : ceil_div(g.k, KCHUNK);
    for (int m0 = 0; m0 < g.m; m0 += BM)
      for (int n0 = 0; n0 < g.n; n0 += BN) {
        if (nchunks == 1) {
          jobs.push_back({di, m0, n0, -1, 0, (int64_t)g.k});
        } else {
          red.push_back({di, m0, n0, (int32_t)nchunks, slots});
          for (int64_t ch = 0; ch < nchunks; ch++) {
            int64_t k0 = ch * KCHUNK, k1 = std::min<int64_t>(g.k, k0 + KCHUNK);
            jobs.push_back({di, m0, n0, (int32_t)slots++, k0, k1});
          }
        }
      }
  }
  if (jobs.empty()) return;
  // biggest jobs first (k extent), so long tiles start early
  std::stable_sort(jobs.begin(), jobs.end(),
                   [](const GemmJob& a, const GemmJob& b) { return (a.k1 - a.k0) > (b.k1 - b.k0); });
  DevBuf<GemmDesc> dd(descs.size(), c.stream);
  dd.upload(descs);
  DevBuf<GemmJob> dj(jobs.size(), c.stream);
  dj.upload(jobs);
  DevBuf<double> parts((size_t)slots * BM * BN, c.stream);
  {
    TimedLaunch tl(c, name);
    // grid.x limit 2^31-1; jobs count is far below
    k_gemm<<<(unsigned)jobs.size(), 128, 0, c.stream>>>(dd.p, dj.p, parts.p);
    check_launch("k_gemm");
    if (!red.empty()) {
      DevBuf<ReduceJob> dr(red.size(), c.stream);
      dr.upload(red);
      k_gemm_reduce<<<(unsigned)red.size(), 256, 0, c.stream>>>(dd.p, dr.p, parts.p);
      check_launch("k_gemm_reduce");
    }
  }
}

}  // namespace mlk
