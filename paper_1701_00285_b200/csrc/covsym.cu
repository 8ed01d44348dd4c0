// Symmetric b = C a for several vectors (5..16 per launch group): step (2) of the three-step
// product C_W v = W (C (W^T v)) with each covariance entry C_ij, i <= j, evaluated
// once for both of its uses -- the row part b_i += C_ij a_j (j >= i) and the column part
// b_j += C_ij a_i (j > i) -- and both contractions on FP64 DMMA.
//
// Task I = kSymRows = 32 consecutive rows (4 row groups of 8) against the points j >= 32 I,
// streamed through a TMA ring of stages of BN = 64 points: BN rows of the augmented Pb and the
// 8G vector rows of a for those points.  Unlike the assembly kernel (tile.cu), the four warps of
// a CTA split the POINTS of a stage (two 8-point sub-tiles each) and every warp handles all 32
// rows, so that the column part of a sub-tile is complete over the task's rows inside one warp:
//   1. Gram: z^2 for the 4 row groups x 8 points, the B fragment of each k-step reused across
//      the row groups (4 independent DMMA chains);
//   2. correlations in registers (corr.cuh), the same-site entry 1 + nugget/sigma2 (R18, R19);
//   3. row part: the accumulator entries are the A fragments of the contraction with the
//      vectors (as in tile.cu), acc[row group][vector group] -- a per-warp partial over the
//      warp's points, written per task and summed over the four warps in a fixed order;
//   4. column part: the 8 x 8 tile is transposed through a warp-private shared buffer (one
//      16-byte store, two 8-byte loads per lane; rows rotated by 0/8/4/12 doubles so both
//      access patterns are bank-conflict free) into the B fragments of
//      D[vector][point] += a^T[vector][row] C[row][point], with the a^T fragments of the task's
//      rows held in registers; D covers all the task's rows and is stored once per sub-tile.
// Column partials: nvec x (n - 32 I) per task -- n^2 nvec / 64 doubles in all (4x fewer than
// the 8-row partials of tile.cu's SYM variant); k_sym_chunks / k_sym_final add them in a fixed
// order.  Deterministic.  Task height measured (cfg3, 10 vectors, r02 sym1): 64 rows with 255
// registers at 2 CTAs/SM 49.2 ms, 32 rows at 168 registers / 3 CTAs 44.8 ms (a^T from shared
// memory instead of registers: 45.6 ms).
#include <algorithm>
#include <map>
#include <mutex>

#include "corr.cuh"
#include "dmma.cuh"
#include "fastmath.cuh"
#include "tile.cuh"

namespace mlk {
namespace {

constexpr int kRG = kSymRows / 8;  // row groups per task (all in every warp)
constexpr int kTW = 2;             // 8-point sub-tiles per warp and stage
constexpr int kBN = 32 * kTW;      // points per stage
constexpr int kNST = 4;            // deepest ring
#ifndef MLK_SYM_MINB
#define MLK_SYM_MINB 3  // CTAs per SM the register budget targets (A/B switch; 2 with 64-row tasks: 255
                        // registers, cfg3 C a 49.2 ms against 44.8 with 32-row tasks at 3, r02 sym1)
#endif

struct SymArgs {
  const double* Pa;
  int dpa, dk, sdp;
  const double* a;  // nvec x n (the launch's vector group, row stride lda)
  int64_t lda;
  int nvec;
  int64_t n;
  int64_t t0, t1;  // tasks of this rank
  const CUtensorMap* xmap;  // Pb, boxes of kBN rows x sdp
  const CUtensorMap* amap;  // vectors padded to 8G rows, boxes of 8G x kBN
  double* colpart;          // task I: nvec x (n - kSymRows I) at sym_off(I)
  double* rowpart;          // task I: 4 warps x nvec x kSymRows rows
  int* counter;
  int nring;
};

__host__ __device__ inline int64_t sym_off(int64_t I, int64_t t0, int64_t n, int nvec) {
  // nvec * sum_{I' = t0}^{I - 1} (n - kSymRows I')
  return (int64_t)nvec * ((I - t0) * n - (kSymRows / 2) * (I * (I - 1) - t0 * (t0 - 1)));
}

__host__ __device__ constexpr int sym_stage_doubles(int sdp, int nr) { return (kBN * sdp + nr * kBN + 15) / 16 * 16; }

// transposition buffer: row i of the 8 x 8 tile at 16 i, rotated by 8 (i & 1) + 4 ((i >> 1) & 1)
__device__ __forceinline__ int xpos(int i, int j) { return 16 * i + ((j + 8 * (i & 1) + 4 * ((i >> 1) & 1)) & 15); }

template <int FAM, int G>
__global__ void __launch_bounds__(128, MLK_SYM_MINB) k_cov_sym(SymArgs g, KernelParams kp) {
  constexpr int NR = 8 * G;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[kNST];
  __shared__ int cnt[kNST];
  __shared__ int s_task;
  __shared__ double s_tab[kExpTabN];
  __shared__ __align__(16) double xbuf[4][2][128];
#ifdef MLK_SYM_ACOL_SMEM
  constexpr int kAcS = (kSymRows + 11) / 16 * 16 + 4;
  __shared__ double acs[NR * kAcS];
#endif
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sdp = g.sdp, sd = sym_stage_doubles(sdp, NR);
  double* As = sm;                    // kSymRows x sdp
  double* St = sm + kSymRows * sdp;   // ring
  for (int i = tid; i < kExpTabN; i += blockDim.x) s_tab[i] = kExp2Tab[i];
  if (tid == 0) {
    for (int i = 0; i < g.nring; i++) {
      mbar_init(&full[i], 1);
      cnt[i] = 0;
    }
    fence_mbar_init();
  }
  for (int e = tid; e < g.nring * sd; e += 128) St[e] = 0.0;
  fence_proxy_async_smem();
  const int ks_n = g.dk >> 2;
  const bool nmode = g.dk < g.dpa;
  const int lq = lane & 3, lr = lane >> 2;
  int gs = 0;
  while (true) {
    __syncthreads();
    if (tid == 0) s_task = atomicAdd(g.counter, 1);
    __syncthreads();
    const int64_t I = g.t0 + s_task;
    if (I >= g.t1) break;
    const int64_t r0 = (int64_t)kSymRows * I;
    const int rows = (int)min((int64_t)kSymRows, g.n - r0);
    const int s_b = (int)(g.n - r0);
    {
      const int cpr = g.dpa >> 1;
      for (int e = tid; e < kSymRows * cpr; e += 128) {
        const int r = e / cpr, ch = e - r * cpr;
        const bool ok = r < rows;
        cp_async16(As + r * sdp + 2 * ch, ok ? g.Pa + (r0 + r) * g.dpa + 2 * ch : g.Pa, ok);
      }
      cp_async_commit();
    }
    const int nst = (s_b + kBN - 1) / kBN;
    const int slot0 = gs % g.nring;
    const unsigned par0 = (unsigned)((gs / g.nring) & 1);
    auto issue = [&](int s, int slot) {
      if (lane == 0) {
        double* Xs = St + slot * sd;
        mbar_arrive_expect_tx(&full[slot], 8u * kBN * (sdp + NR));
        tma_2d_g2s(Xs, g.xmap, 0, (int)(r0 + (int64_t)s * kBN), &full[slot]);
        tma_2d_g2s(Xs + kBN * sdp, g.amap, (int)(r0 + (int64_t)s * kBN), 0, &full[slot]);
      }
    };
    if (warp == 0)
      for (int s = 0, sl = slot0; s < min(g.nring, nst); s++, sl = sl + 1 == g.nring ? 0 : sl + 1) issue(s, sl);
    // a^T fragments of the task's rows: A[m = vector][k = row], k-step h covers rows 8 r + 4 h + k
#ifndef MLK_SYM_ACOL_SMEM
    double acol[kRG][2][G];
#pragma unroll
    for (int r = 0; r < kRG; r++)
#pragma unroll
      for (int h = 0; h < 2; h++)
#pragma unroll
        for (int q = 0; q < G; q++) {
          const int row = 8 * r + 4 * h + lq, vec = 8 * q + lr;
          acol[r][h][q] = (row < rows && vec < g.nvec) ? g.a[(int64_t)vec * g.lda + r0 + row] : 0.0;
        }
#define ACOL(r, h, q) acol[r][h][q]
#else
    // (A/B variant) the task's vector rows in shared memory, row stride kAcS = 4 (mod 16)
    for (int e = tid; e < NR * kSymRows; e += 128) {
      const int vec = e / kSymRows, row = e - vec * kSymRows;
      acs[vec * kAcS + row] = (row < rows && vec < g.nvec) ? g.a[(int64_t)vec * g.lda + r0 + row] : 0.0;
    }
#define ACOL(r, h, q) acs[(8 * (q) + lr) * kAcS + 8 * (r) + 4 * (h) + lq]
#endif
    cp_async_wait<0>();
    __syncthreads();
    double na[kRG];
#pragma unroll
    for (int r = 0; r < kRG; r++) na[r] = nmode ? As[(8 * r + lr) * sdp + g.dk] : 0.0;
    double acc[kRG][G][2];
#pragma unroll
    for (int r = 0; r < kRG; r++)
#pragma unroll
      for (int q = 0; q < G; q++) acc[r][q][0] = acc[r][q][1] = 0.0;
    const int64_t coff = sym_off(I, g.t0, g.n, g.nvec);
    int slot = slot0;
    unsigned par = par0;
    for (int s = 0; s < nst; s++) {
      const double* Xs = St + slot * sd;
      const double* Ws = Xs + kBN * sdp;
      const int yb = s * kBN;
      mbar_wait(&full[slot], par);
      const bool diag = yb < rows, tail = yb + kBN > s_b;
#pragma unroll
      for (int tt = 0; tt < kTW; tt++) {
        const int t = warp * kTW + tt;
        const int jb = yb + 8 * t;  // first point of the sub-tile (task-local)
        if (jb >= s_b) continue;    // warp-uniform
        // 1. Gram
        double gr[kRG][2];
        if (nmode) {
          const double nb0 = Xs[(8 * t + 2 * lq) * sdp + g.dk], nb1 = Xs[(8 * t + 2 * lq + 1) * sdp + g.dk];
#pragma unroll
          for (int r = 0; r < kRG; r++) {
            gr[r][0] = na[r] + nb0;
            gr[r][1] = na[r] + nb1;
          }
        } else {
#pragma unroll
          for (int r = 0; r < kRG; r++) gr[r][0] = gr[r][1] = 0.0;
        }
        const double* bp = Xs + (8 * t + lr) * sdp + lq;
        const double* ap = As + lr * sdp + lq;
#pragma unroll 2
        for (int ks = 0; ks < ks_n; ks++) {
          const double b = bp[4 * ks];
#pragma unroll
          for (int r = 0; r < kRG; r++) dmma_8x8x4(gr[r][0], gr[r][1], ap[8 * r * sdp + 4 * ks], b);
        }
        // 2. correlations; masks only in the diagonal stage and the last one
        double cv[kRG][2];
#pragma unroll
        for (int r = 0; r < kRG; r++)
#pragma unroll
          for (int e = 0; e < 2; e++) cv[r][e] = corr<FAM>(gr[r][e], s_tab, kp);
        const int j0 = jb + 2 * lq;  // the lane's two points j0, j0 + 1
        if (diag || tail) {
#pragma unroll
          for (int r = 0; r < kRG; r++) {
            const int i = 8 * r + lr;
#pragma unroll
            for (int e = 0; e < 2; e++) {
              const int j = j0 + e;
              if (j == i) cv[r][e] = kp.same_val;
              if (j < i || j >= s_b) cv[r][e] = 0.0;  // row part: j >= i only
            }
          }
        }
        // 3. row part
        double2 w[G];
#pragma unroll
        for (int q = 0; q < G; q++) w[q] = *reinterpret_cast<const double2*>(Ws + (8 * q + lr) * kBN + 8 * t + 2 * lq);
#pragma unroll
        for (int r = 0; r < kRG; r++)
#pragma unroll
          for (int q = 0; q < G; q++) {
            dmma_8x8x4(acc[r][q][0], acc[r][q][1], cv[r][0], w[q].x);
            dmma_8x8x4(acc[r][q][0], acc[r][q][1], cv[r][1], w[q].y);
          }
        // 4. column part (j > i): transpose through the warp's buffer, contract with a^T
        double D[G][2];
#pragma unroll
        for (int q = 0; q < G; q++) D[q][0] = D[q][1] = 0.0;
#pragma unroll
        for (int r = 0; r < kRG; r++) {
          double c0 = cv[r][0], c1 = cv[r][1];
          if (diag) {
            const int i = 8 * r + lr;
            if (j0 == i) c0 = 0.0;
            if (j0 + 1 == i) c1 = 0.0;
          }
          double* X = xbuf[warp][r & 1];
          *reinterpret_cast<double2*>(X + xpos(lr, 2 * lq)) = make_double2(c0, c1);
          __syncwarp();
          const double bt0 = X[xpos(lq, lr)], bt1 = X[xpos(4 + lq, lr)];
#pragma unroll
          for (int q = 0; q < G; q++) {
            dmma_8x8x4(D[q][0], D[q][1], ACOL(r, 0, q), bt0);
            dmma_8x8x4(D[q][0], D[q][1], ACOL(r, 1, q), bt1);
          }
        }
        // D[vector 8 q + lr][point j0 + e], complete over the task's rows
#pragma unroll
        for (int q = 0; q < G; q++) {
          const int vec = 8 * q + lr;
          if (vec < g.nvec) {
            double* cp = g.colpart + coff + (int64_t)vec * s_b;
            if (j0 < s_b) cp[j0] = D[q][0];
            if (j0 + 1 < s_b) cp[j0 + 1] = D[q][1];
          }
        }
      }
      // release the slot: the last of the four warps refills it with stage s + nring
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(&cnt[slot], 1) == 3;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        if (lane == 0) cnt[slot] = 0;
        if (s + g.nring < nst) issue(s + g.nring, slot);
      }
      if (++slot == g.nring) {
        slot = 0;
        par ^= 1u;
      }
    }
    gs += nst;
#undef ACOL
    // row partials of this warp: acc[r][q][e] = U[row 8 r + lr][vector 8 q + 2 lq + e]
    double* rp = g.rowpart + ((I - g.t0) * 4 + warp) * (int64_t)g.nvec * kSymRows;
#pragma unroll
    for (int r = 0; r < kRG; r++)
#pragma unroll
      for (int q = 0; q < G; q++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int vec = 8 * q + 2 * lq + e;
          if (vec < g.nvec) rp[vec * kSymRows + 8 * r + lr] = acc[r][q][e];
        }
  }
}

// tmp[l][c][j] = sum over the tasks I of chunk c (I <= j / kSymRows) of colpart[I][l][j - kSymRows I]
constexpr int kSymChunk = 64;
__global__ void k_sym_chunks(const double* __restrict__ colpart, int64_t t0, int64_t t1, int64_t n, int nvec,
                             int nchunks, double* __restrict__ tmp) {
  const int64_t j = kSymRows * t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c = blockIdx.y, l = blockIdx.z;
  if (j >= n) return;
  const int64_t i0 = t0 + (int64_t)c * kSymChunk;
  const int64_t i1 = std::min<int64_t>({t1, i0 + kSymChunk, j / kSymRows + 1});
  double s = 0.0;
  for (int64_t I = i0; I < i1; I++) {
    const int64_t w = n - kSymRows * I;
    s += colpart[sym_off(I, t0, n, nvec) + (int64_t)l * w + (j - kSymRows * I)];
  }
  tmp[((int64_t)l * nchunks + c) * n + j] = s;
}

// b[l][j] = sigma2 ((row partials of j's task, warps 0..3) + sum over chunks c of tmp)
__global__ void k_sym_final(const double* __restrict__ tmp, const double* __restrict__ rowpart, int64_t t0,
                            int64_t t1, int64_t n, int nvec, int nchunks, double sigma2, double* __restrict__ b,
                            int64_t ldb, int accumulate) {
  const int64_t j = kSymRows * t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (j >= n) return;
  const int64_t I = j / kSymRows;
  double s = 0.0;
  if (I < t1) {
    const double* rp = rowpart + (I - t0) * 4 * (int64_t)nvec * kSymRows + (int64_t)l * kSymRows + (j - kSymRows * I);
    s = ((rp[0] + rp[(int64_t)nvec * kSymRows]) + rp[2 * (int64_t)nvec * kSymRows]) + rp[3 * (int64_t)nvec * kSymRows];
  }
  double t = 0.0;
  for (int c = 0; c < nchunks; c++) t += tmp[((int64_t)l * nchunks + c) * n + j];
  double* bp = b + (int64_t)l * ldb + j;
  *bp = accumulate ? *bp + sigma2 * (s + t) : sigma2 * (s + t);
}

template <int FAM, int G>
void launch_sym(Ctx& c, const SymArgs& ag, const KernelParams& kp, int64_t ntask) {
  auto fn = k_cov_sym<FAM, G>;
  struct Cfg {
    int nring = 0, occ = 0;
    size_t smem = 0;
  };
  static std::mutex mu;
  static std::map<std::pair<int, int>, Cfg> cache;
  static std::map<int, size_t> attr;
  std::lock_guard<std::mutex> lock(mu);
  Cfg& cf = cache[{c.device, ag.sdp}];
  if (cf.nring == 0) {
    cudaFuncAttributes fa;
    CUDA_CHECK(cudaFuncGetAttributes(&fa, fn));
    for (int ns = kNST; ns >= 2; ns--) {
      const size_t sm_ns = sizeof(double) * (size_t)(kSymRows * ag.sdp + ns * sym_stage_doubles(ag.sdp, 8 * G));
      if (sm_ns + fa.sharedSizeBytes > 227 * 1024) continue;
      CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_ns));
      attr[c.device] = std::max(attr[c.device], sm_ns);
      int o = 0;
      CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 128, sm_ns));
      if (cf.nring == 0 || o > cf.occ) {
        cf.nring = ns;
        cf.occ = o;
        cf.smem = sm_ns;
      }
      if (o >= MLK_SYM_MINB) break;
    }
    if (cf.nring == 0) throw Error(MLK_ERR_UNSUPPORTED, "symmetric C a stages do not fit shared memory");
    cf.occ = std::max(cf.occ, 1);
  }
  if (attr[c.device] < cf.smem) {
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf.smem));
    attr[c.device] = cf.smem;
  }
  SymArgs a = ag;
  a.nring = cf.nring;
  const int grid = (int)std::min<int64_t>(ntask, (int64_t)num_sms(c.device) * cf.occ);
  fn<<<grid, 128, cf.smem, c.stream>>>(a, kp);
  check_launch("k_cov_sym");
}

template <int G>
void launch_sym_fam(Ctx& c, const SymArgs& ag, const KernelParams& kp, int64_t ntask) {
  switch (kp.family) {
    case MLK_MATERN_12: launch_sym<MLK_MATERN_12, G>(c, ag, kp, ntask); break;
    case MLK_MATERN_32: launch_sym<MLK_MATERN_32, G>(c, ag, kp, ntask); break;
    case MLK_MATERN_52: launch_sym<MLK_MATERN_52, G>(c, ag, kp, ntask); break;
    case MLK_MATERN_NU: launch_sym<MLK_MATERN_NU, G>(c, ag, kp, ntask); break;
    default: launch_sym<MLK_GAUSSIAN, G>(c, ag, kp, ntask); break;
  }
}

// the vectors of one group copied to 8G rows of ld = n rounded up to 8 (zero rows / columns
// past nvec / n): a TMA-describable source for every n
__global__ void k_pad_vectors(const double* __restrict__ a, int64_t n, int nvec, double* __restrict__ ap, int64_t ld,
                              int rows) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (j >= ld || l >= rows) return;
  ap[(int64_t)l * ld + j] = (l < nvec && j < n) ? a[(int64_t)l * n + j] : 0.0;
}

}  // namespace

int64_t cov_sym_partials(int64_t n, int nvec, int64_t t0, int64_t t1) {
  return t1 > t0 ? sym_off(t1, t0, n, std::min(nvec, 16)) : 0;
}

// Tasks in batches whose column partials fit an eighth of the device (a function of n, nvec and
// the device's total memory only, so every rank cuts the same batches; cfg3's 10 vectors: one
// batch of 21 GB, cfg4's: four).  Batches of 2 GB measured 34 % slower on cfg3 (59.8 against
// 44.7 ms: eleven launches with their tails).  All buffers are allocated before the timed region
// (an allocation inside it once stalled the stream by 50-150 ms, r02 bn).  Batch k adds its
// part of b in batch order: deterministic.
void cov_matvec_sym(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, const double* a, double* b, int nvec,
                    int64_t t0, int64_t t1) {
  const int64_t n = tree->n;
  if (t1 <= t0) return;
  AugCoords aug;
  tile_aug_layout(tree->d, aug);
  const int64_t ld = (n + 7) / 8 * 8;
  const int64_t batch_doubles = std::max<int64_t>(device_total_bytes(c.device) / 8 / 8, 4 * n);
  for (int v0 = 0; v0 < nvec; v0 += 16) {
    const int nv = std::min(16, nvec - v0);
    const int G = nv <= 8 ? 1 : 2;
    // batches [bt[k], bt[k + 1])
    std::vector<int64_t> bt = {t0};
    int64_t cp_max = 0, rows_max = 0;
    for (int64_t I = t0, acc = 0; I < t1; I++) {
      const int64_t w = (int64_t)nv * (n - kSymRows * I);
      if (acc > 0 && acc + w > batch_doubles) {
        bt.push_back(I);
        acc = 0;
      }
      acc += w;
      cp_max = std::max(cp_max, acc);
    }
    bt.push_back(t1);
    for (size_t k = 0; k + 1 < bt.size(); k++) rows_max = std::max(rows_max, bt[k + 1] - bt[k]);
    DevBuf<double> apad((size_t)8 * G * ld, c.stream);
    double* colpart = c.scratch("sym_colpart", (size_t)cp_max);
    DevBuf<double> rowpart((size_t)rows_max * 4 * nv * kSymRows, c.stream);
    const int nchunks_max = (int)ceil_div(rows_max, (int64_t)kSymChunk);
    double* tmp = c.scratch("sym_tmp", (size_t)nv * nchunks_max * n);
    DevBuf<int> counter(bt.size(), c.stream);
    counter.zero();
    TimedLaunch tl(c, "cov_matvec_sym");
    const double* Pa = tile_aug_get(c, tree, kp, aug);
    k_pad_vectors<<<dim3((unsigned)ceil_div(ld, (int64_t)256), (unsigned)(8 * G)), 256, 0, c.stream>>>(
        a + (int64_t)v0 * n, n, nv, apad.p, ld, 8 * G);
    check_launch("k_pad_vectors");
    std::vector<CUtensorMap> maps = {make_map_2d(Pa + (size_t)n * aug.dpa, n, aug.dpa, aug.dpa, kBN, aug.sdp),
                                     make_map_2d(apad.p, 8 * G, ld, ld, 8 * G, kBN)};
    DevBuf<CUtensorMap> maps_d(2, c.stream);
    maps_d.upload(maps);
    for (size_t k = 0; k + 1 < bt.size(); k++) {
      const int64_t b0 = bt[k], b1 = bt[k + 1];
      SymArgs ag;
      ag.Pa = Pa;
      ag.dpa = aug.dpa;
      ag.dk = aug.dk;
      ag.sdp = aug.sdp;
      ag.a = apad.p;
      ag.lda = ld;
      ag.nvec = nv;
      ag.n = n;
      ag.t0 = b0;
      ag.t1 = b1;
      ag.xmap = maps_d.p;
      ag.amap = maps_d.p + 1;
      ag.colpart = colpart;
      ag.rowpart = rowpart.p;
      ag.counter = counter.p + k;
      ag.nring = 0;
      if (G == 1) launch_sym_fam<1>(c, ag, kp, b1 - b0);
      else launch_sym_fam<2>(c, ag, kp, b1 - b0);
      const int nchunks = (int)ceil_div(b1 - b0, (int64_t)kSymChunk);
      const int64_t jn = n - kSymRows * b0;
      dim3 g1((unsigned)ceil_div(jn, (int64_t)256), (unsigned)nchunks, (unsigned)nv);
      k_sym_chunks<<<g1, 256, 0, c.stream>>>(colpart, b0, b1, n, nv, nchunks, tmp);
      check_launch("k_sym_chunks");
      dim3 g2((unsigned)ceil_div(jn, (int64_t)256), (unsigned)nv);
      k_sym_final<<<g2, 256, 0, c.stream>>>(tmp, rowpart.p, b0, b1, n, nv, nchunks, kp.sigma2,
                                            b + (int64_t)v0 * n, n, k > 0 ? 1 : 0);
      check_launch("k_sym_final");
    }
  }
}

}  // namespace mlk
