// mlk_build_basis: the multi-level basis (steps (a)-(f)) as a tree QR.
//  leaves:   P(X_leaf) (s x M monomials, graded TD order, reading R8) -> complete Householder
//            QR (LAPACK convention, reading R7): Phi = Q_1^T, W = Q_2^T, R.
//  internal: [R_L; R_R] (2M x M) -> complete QR; Phi = Q_1^T (Phi_L (+) Phi_R),
//            W = Q_2^T (Phi_L (+) Phi_R) by four DMMA GEMMs per cell (gemm.cu).
// The QR kernel runs one CTA per matrix (batched over the cells of a level).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>

#include "api.cuh"

namespace mlk {
namespace {

// Q (row-major, 2M x 2M) of each job from Q^T (row-major): dst[c][r] = src[r][c]
__global__ void k_keep_q(const double* __restrict__ qt, const int64_t* __restrict__ dst_off, int m2,
                         double* __restrict__ qm) {
  const double* src = qt + (int64_t)blockIdx.y * m2 * m2;
  double* dst = qm + dst_off[blockIdx.y];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)m2 * m2; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / m2), cc = (int)(e - (int64_t)r * m2);
    dst[(int64_t)cc * m2 + r] = src[e];
  }
}

// Index set Lambda(w) of Table multivariate:table1 as factor lists (coordinate
// indices, nondecreasing; a monomial is the left-to-right product of its factors), in graded
// order (R8): total degree, then the factor lists lexicographically -- combinations with
// replacement for TD.  Depth-first over the nonzero coordinates with the set's (monotone)
// budget; at most kMaxM members.
constexpr int kMaxM = 4096;
int sm_f(int p) {
  if (p <= 1) return p;
  int l = 0;
  while ((1 << l) < p) l++;
  return l;  // ceil(log2 p)
}
std::vector<std::vector<int>> index_set_factors(int kind, int d, int w) {
  std::vector<std::vector<int>> out;
  std::vector<int> alpha(d, 0);
  // budget semantics: TD sum alpha <= w; HC prod (alpha + 1) <= w; SM sum f(alpha) <= w;
  // TP max alpha <= w
  std::function<void(int, int64_t)> rec = [&](int start, int64_t budget) {
    if ((int)out.size() > kMaxM) return;
    std::vector<int> fac;
    for (int k = 0; k < d; k++)
      for (int e = 0; e < alpha[k]; e++) fac.push_back(k);
    out.push_back(fac);
    for (int k = start; k < d; k++) {
      for (int e = 1;; e++) {
        int64_t nb;
        if (kind == MLK_INDEX_TD) nb = budget - e;
        else if (kind == MLK_INDEX_HC) nb = budget / (e + 1) >= 1 && (int64_t)(e + 1) <= budget ? budget / (e + 1) : -1;
        else if (kind == MLK_INDEX_SM) nb = budget - sm_f(e);
        else nb = e <= w ? budget : -1;
        if (nb < 0) break;
        alpha[k] = e;
        rec(k + 1, nb);
        alpha[k] = 0;
        if ((int)out.size() > kMaxM) return;
      }
    }
  };
  if (!(kind == MLK_INDEX_HC && w < 1)) rec(0, w);
  std::stable_sort(out.begin(), out.end(), [](const std::vector<int>& a, const std::vector<int>& b) {
    if (a.size() != b.size()) return a.size() < b.size();
    return a < b;
  });
  return out;
}

struct LeafJob {
  int64_t pt_begin;  // first tree position
  int32_t s;         // points
  int64_t a_off;     // offset of the s x M column-major monomial matrix in scratch
};

// monomial matrix P (s x M, column-major) of each leaf; a monomial is the left-to-right
// product of its factors (factor table fac[m * w + j], -1 padded)
__global__ void k_monomials(const double* __restrict__ Xt, int dp, const LeafJob* __restrict__ jobs,
                            const int32_t* __restrict__ fac, int M, int w, double* __restrict__ A) {
  const LeafJob jb = jobs[blockIdx.y];
  int64_t total = (int64_t)jb.s * M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int m = (int)(e / jb.s);
    int i = (int)(e % jb.s);
    const double* x = Xt + (jb.pt_begin + i) * dp;
    double v = 1.0;
    bool first = true;
    for (int j = 0; j < w; j++) {
      int f = fac[m * w + j];
      if (f < 0) break;
      v = first ? x[f] : v * x[f];
      first = false;
    }
    A[jb.a_off + (int64_t)m * jb.s + i] = v;
  }
}

struct QrJob {
  double* A;      // m x nc column-major (lda = m); factorised in place
  int32_t m, nc;
  double* R;      // nc x nc row-major output
  double* V;      // scratch m x nc row-major: unit lower-trapezoidal Householder vectors
  double* T;      // scratch nc x nc: the upper-triangular factor of Q = I - V T V^T
  double* W1T;    // scratch nc x m row-major: T^T V^T
  double* qlo;    // rows j < nc of Q^T (row j at qlo + j*ldq)
  double* qhi;    // rows j >= nc of Q^T at qhi + (j - nc)*ldq
  int64_t ldq;
  int32_t stacked;  // 1: A = [R_L; R_R] (m = 2 nc, both upper triangular), see k_qr_wy
  // stacked jobs: R_L, R_R (nc x nc row-major); the shared-memory QR reads them directly and
  // A is formed (k_stack_r) only for the global-memory and blocked paths
  const double* RL = nullptr;
  const double* RR = nullptr;
};

constexpr int kQrSmemLimit = 225 * 1024;

// Householder QR of one matrix per CTA in the LAPACK dgeqr2 convention (beta = -sign(alpha)
// ||(alpha, x)||, tau = (beta - alpha)/beta, v = x/(alpha - beta), tau = 0 when x = 0), then
// W1T = T^T V^T for the compact-WY form Q = H_0 ... H_{nc-1} = I - V T V^T, so that
// Q^T = I - V W1T is formed by the DMMA GEMM (gemm.cu).
//  * Column step k takes two barriers: (1) thread j forms x . a_j for its column j >= k
//    (serial, four partial sums); the owner of column k (j = k gives |x|^2) forms beta, tau
//    and the scale once; (2) thread j applies H_k to its column j > k, reading the unscaled
//    x (column k's scaling and beta are stored at the start of the next step).
//  * Stacked merges [R_L; R_R] touch only rows {k} and nc..nc+k in step k (the triangles'
//    structure is preserved), a third of the dense work.
//  * T is never formed: with G = V^T V, T^{-1} = triu(G, 1) + diag(1/tau) (the inverse of the
//    dlarft recursion), so W1T solves T^{-T} W1T = V^T by forward substitution,
//    W1T[l][i] = tau_l (V[i][l] - sum_{q<l} G[q][l] W1T[q][i]), one thread per row i, in place
//    of A's row i (R and V are exported first).  A reflector with tau = 0 is the identity and
//    gets a zero row.
// SMEM: the matrix lives in shared memory (odd column stride); GS: G lives there too.
constexpr int kQrThreads = 256;
// phase timestamps of block 0 of the last k_qr_wy launch (diagnostics, MLK_QR_PROFILE)
__device__ long long g_qr_prof[12];
#define QR_STAMP(i) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_qr_prof[i] = clock64();

template <bool SMEM, bool GS>
__global__ void __launch_bounds__(kQrThreads) k_qr_wy(const QrJob* __restrict__ jobs, int* __restrict__ rank_flag) {
  extern __shared__ __align__(16) double sh[];
  __shared__ double s_piv[6];                       // tau, scal, beta of step k at 3 (k & 1)
  const QrJob jb = jobs[blockIdx.x];
  const int m = jb.m, nc = jb.nc;
  const int lda = SMEM ? (m | 1) : m;
  double* taus = sh;                                // nc
  double* dots = taus + nc;                         // nc: x . a_j of the current step (by column)
  double* A = SMEM ? dots + nc : jb.A;
  double* G = GS ? A + (int64_t)lda * nc : jb.T;    // G[q][l], q < l, row-major nc x nc
  const int tid = threadIdx.x, nt = blockDim.x;
  QR_STAMP(0);
  if (SMEM && jb.RL) {
    // [R_L; R_R] straight from the children's R (row-major nc x nc each): coalesced reads in the
    // source order, transposed into the column-major shared copy
    const int nn = nc * nc;
    for (int f0 = tid; f0 < 2 * nn; f0 += 4 * nt) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int f = f0 + u * nt;
        v[u] = f < nn ? jb.RL[f] : (f < 2 * nn ? jb.RR[f - nn] : 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int f = f0 + u * nt;
        if (f < 2 * nn) {
          const int half = f >= nn, r = f - half * nn, il = r / nc, j = r - il * nc;
          A[(int64_t)j * lda + il + half * nc] = v[u];
        }
      }
    }
    __syncthreads();
  } else if (SMEM) {
    // four independent global loads in flight per thread
    const int64_t tot = (int64_t)m * nc;
    for (int64_t e0 = tid; e0 < tot; e0 += 4 * (int64_t)nt) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t e = e0 + u * nt;
        v[u] = e < tot ? jb.A[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t e = e0 + u * nt;
        if (e < tot) {
          const int j = (int)(e / m), i = (int)(e - (int64_t)j * m);
          A[(int64_t)j * lda + i] = v[u];
        }
      }
    }
    __syncthreads();
  }
  QR_STAMP(1);
  // Rows a reflector touches: dense, x = rows k+1..m-1; stacked [R_L; R_R] (both upper
  // triangular), x has nonzeros only in rows nc..nc+k and the structure is preserved, so
  // rows nc..nc+k (exactly the entries LAPACK's dense sweep would change).
  const bool stk = jb.stacked != 0;
  const int lane = tid & 31, sub = tid & 3, cq = tid >> 2, ncq = nt >> 2;
  const unsigned qmask = 0xFu << (lane & ~3);
  // A quad of threads owns column j (below); the odd column stride keeps the column-strided
  // accesses of different quads in distinct banks.  Two barriers per step.
  for (int k = 0; k < nc; k++) {
    const double* ak = A + (int64_t)k * lda;
    const int lo = stk ? nc : k + 1, hi = stk ? nc + k + 1 : m;
    if (k > 0) {  // finish column k - 1 (not read in this step): x scaled into v, beta on the diagonal
      double* ap = A + (int64_t)(k - 1) * lda;
      const double* pv = s_piv + 3 * ((k - 1) & 1);
      const int plo = stk ? nc : k, phi = stk ? nc + k : m;
      for (int i = plo + tid; i < phi; i += nt) ap[i] *= pv[1];
      if (tid == 0) ap[k - 1] = pv[2];
    }
    // (1) dots for the columns j >= k, a quad of threads per column: lane `sub` of the quad
    // sums the rows lo + sub + 4 m (the tail rows go to sub 0), then two in-quad shuffles add
    // (s0 + s1) + (s2 + s3) -- the same partial sums and order as one thread with four
    // accumulators, so the factors are unchanged, at a quarter of the per-thread row work.
    // The owner quad of column k forms the reflector.
    const int nfull = (hi - lo) & ~3;
    for (int j = k + cq; j < nc; j += ncq) {
      const double* aj = A + (int64_t)j * lda;
      double sp = 0.0;
#pragma unroll 4
      for (int i = lo + sub; i < lo + nfull; i += 4) sp = fma(ak[i], aj[i], sp);
      if (sub == 0)
        for (int i = lo + nfull; i < hi; i++) sp = fma(ak[i], aj[i], sp);
      sp += __shfl_xor_sync(qmask, sp, 1);
      sp += __shfl_xor_sync(qmask, sp, 2);
      if (sub == 0) {
        const double sum = sp;
        if (j == k) {
          const double alpha = ak[k];
          double tau = 0.0, scal = 1.0, beta = alpha;
          if (sum > 0.0) {
            beta = -copysign(sqrt(fma(alpha, alpha, sum)), alpha);
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
          }
          taus[k] = tau;
          double* pv = s_piv + 3 * (k & 1);
          pv[0] = tau;
          pv[1] = scal;
          pv[2] = beta;
        } else {
          dots[j] = sum;
        }
      }
    }
    __syncthreads();
    // (2) a_j -= f (e_k + scal x), f = tau (a_kj + scal d_j), for the columns j > k (a quad per
    // column, rows strided over its four lanes)
    const double tau = s_piv[3 * (k & 1)];
    if (tau != 0.0) {
      const double scal = s_piv[3 * (k & 1) + 1];
      for (int j = k + 1 + cq; j < nc; j += ncq) {
        double* __restrict__ aj = A + (int64_t)j * lda;
        const double* __restrict__ xk = ak;
        const double f = tau * fma(scal, dots[j], aj[k]);
        const double g = f * scal;
        __syncwarp(qmask);  // every lane has read aj[k] before sub 0 changes it
        if (sub == 0) aj[k] -= f;
        int i = lo + sub;
        for (; i + 12 < hi; i += 16) {
          double x[4], y[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            x[u] = xk[i + 4 * u];
            y[u] = aj[i + 4 * u];
          }
#pragma unroll
          for (int u = 0; u < 4; u++) aj[i + 4 * u] = fma(-g, x[u], y[u]);
        }
        for (; i < hi; i += 4) aj[i] = fma(-g, xk[i], aj[i]);
      }
    }
    __syncthreads();
  }
  // finish the last column
  {
    double* ap = A + (int64_t)(nc - 1) * lda;
    const double* pv = s_piv + 3 * ((nc - 1) & 1);
    const int plo = nc, phi = stk ? 2 * nc : m;
    for (int i = plo + tid; i < phi; i += nt) ap[i] *= pv[1];
    if (tid == 0) ap[nc - 1] = pv[2];
  }
  __syncthreads();
  QR_STAMP(2);
  // R, rank test (reading R9), V row-major with the unit diagonal made explicit
  for (int e = tid; e < nc * nc; e += nt) {
    int i = e / nc, j = e - i * nc;
    jb.R[e] = j >= i ? A[(int64_t)j * lda + i] : 0.0;
  }
  for (int e = tid; e < m * nc; e += nt) {
    const int i = e / nc, l = e - i * nc;
    jb.V[e] = i == l ? 1.0 : (i > l ? A[(int64_t)l * lda + i] : 0.0);
  }
  if (tid == 0) {
    double mx = 0.0, mn = INFINITY;
    for (int i = 0; i < nc; i++) {
      double v = fabs(A[(int64_t)i * lda + i]);
      mx = fmax(mx, v);
      mn = fmin(mn, v);
    }
    if (!(mn > 1e-13 * mx)) atomicExch(rank_flag, 1);
  }
  QR_STAMP(3);
  // G[q][l] = (V^T V)[q][l] for q < l: column q of V is (0.., 1 at q, A[q*lda + i] for i > q),
  // so G[q][l] = A[q*lda + l] + sum_{i > l} A[q*lda + i] A[l*lda + i].  One thread per pair.
  for (int e = tid; e < nc * nc; e += nt) {
    const int q = e / nc, l = e - q * nc;
    if (q >= l) continue;
    const double* vq = A + (int64_t)q * lda;
    const double* vl = A + (int64_t)l * lda;
    double s0 = vq[l], s1 = 0.0;
    int i = stk ? nc : l + 1;
    const int iend = stk ? nc + q + 1 : m;   // stacked: column q of V is zero past row nc + q
    for (; i + 1 < iend; i += 2) {
      s0 = fma(vq[i], vl[i], s0);
      s1 = fma(vq[i + 1], vl[i + 1], s1);
    }
    if (i < iend) s0 = fma(vq[i], vl[i], s0);
    G[(int64_t)q * nc + l] = s0 + s1;
  }
  __syncthreads();
  QR_STAMP(4);
  // forward substitution, thread per row i (reads only its own row of A, then overwrites it)
  for (int i = tid; i < m; i += nt) {
    for (int l = 0; l < nc; l++) {
      const double tl = taus[l];
      double w = 0.0;
      if (tl != 0.0) {
        const double vil = i == l ? 1.0 : (i > l ? A[(int64_t)l * lda + i] : 0.0);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int q = 0;
        for (; q + 3 < l; q += 4) {
          s0 = fma(G[(int64_t)q * nc + l], A[(int64_t)q * lda + i], s0);
          s1 = fma(G[(int64_t)(q + 1) * nc + l], A[(int64_t)(q + 1) * lda + i], s1);
          s2 = fma(G[(int64_t)(q + 2) * nc + l], A[(int64_t)(q + 2) * lda + i], s2);
          s3 = fma(G[(int64_t)(q + 3) * nc + l], A[(int64_t)(q + 3) * lda + i], s3);
        }
        for (; q < l; q++) s0 = fma(G[(int64_t)q * nc + l], A[(int64_t)q * lda + i], s0);
        w = tl * (vil - ((s0 + s1) + (s2 + s3)));
      }
      A[(int64_t)l * lda + i] = w;   // row i of W1T, in place (entries q < l already replaced)
      jb.W1T[(int64_t)l * m + i] = w;
    }
  }
  __syncthreads();
  QR_STAMP(5);
}

// dynamic shared memory of k_qr_wy: taus, dots (+ A) (+ G)
inline size_t qr_smem(int m, int nc, bool a_in, bool g_in) {
  size_t d = 2 * (size_t)nc;
  if (a_in) d += (size_t)(m | 1) * nc;
  if (g_in) d += (size_t)nc * nc;
  return d * sizeof(double);
}

// [R_L; R_R] (2M x M, column-major) for every internal cell of a level
struct StackJob {
  const double* RL;
  const double* RR;
  double* A;
};
__global__ void k_stack_r(const StackJob* __restrict__ jobs, int M) {
  const StackJob jb = jobs[blockIdx.x];
  for (int e = threadIdx.x; e < 2 * M * M; e += blockDim.x) {
    int j = e / (2 * M), i = e % (2 * M);
    jb.A[e] = i < M ? jb.RL[i * M + j] : jb.RR[(i - M) * M + j];
  }
}

// ---------------------------------------------------------------------------------------------
// Blocked Householder QR for matrices that do not fit in shared memory (LAPACK dgeqrf: dgeqr2
// panels + dlarft + dlarfb, so the reflectors are those of the unblocked kernel above).  The
// job's matrix is augmented to [A | I] (column-major, lda = m); each 32-column panel is
// factorised by one CTA (k_qr_panel) and its block reflector B_p^T = I - V_p T_p^T V_p^T is
// applied to every trailing column on the DMMA GEMM:
//     Wt = A_tr^T (V_p T_p)            (ntr x 32, k = m - c0)
//     A_tr^T -= Wt V_p^T               (ntr x (m - c0), k = 32)
// The identity columns end up holding Q^T I = Q^T, which k_qr_export copies to qlo / qhi.
constexpr int kPanelKB = 32;
constexpr int kPanelThreads = 512;
constexpr int kPanelWarps = kPanelThreads / 32;

struct PanelJob {
  double* A;    // [A | I], column-major, lda = m
  int32_t m;
  double* VT;   // (m - c0) x 32 row-major: V_p T_p
  double* Vt;   // 32 x (m - c0) row-major (ld m): V_p^T, unit diagonal and zeros made explicit
};

// lane c ends with sum over the warp of v[c] (recursive halving; 31 shuffles, fixed order)
__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; i++) {
      const double send = up ? v[i] : v[i + s];
      const double keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// Panel columns c0 .. c0 + kb - 1 (kb <= 32), rows c0 .. m - 1, in the dgeqr2 convention of
// k_qr_wy.  Thread t owns the rows c0 + t + i * 512; step l does ONE pass over the panel that
// (a) scales x_l into v_l, (b) applies H_l to the columns j > l, (c) accumulates the dots of
// step l + 1 (x_{l+1} . a_j, j > l) and (d) the Gram column G[q][l] = v_q . v_l (q < l) that
// dlarft needs — 32 slots, reduced once per step (warp reduce-scatter, then 16 warp partials
// summed in order by warp 0, which then forms the next reflector).  Two barriers per step.
__global__ void __launch_bounds__(kPanelThreads) k_qr_panel(const PanelJob* __restrict__ jobs, int c0, int kb) {
  __shared__ double red[kPanelWarps][kPanelKB + 1];
  __shared__ double Gp[kPanelKB][kPanelKB + 1];  // Gp[q][l], q < l
  __shared__ double Tp[kPanelKB][kPanelKB + 1];
  __shared__ double dsum[kPanelKB];               // dots of the current step, by column
  __shared__ double gcol[kPanelKB];               // f_j * scal of the current step
  __shared__ double taus[kPanelKB];
  __shared__ double s_scal;
  const PanelJob jb = jobs[blockIdx.x];
  const int m = jb.m;
  const int64_t lda = m;
  double* __restrict__ A = jb.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto col = [&](int j) { return A + (int64_t)(c0 + j) * lda; };

  // warp 0: reflector of step l from dsum, then f_j for the columns j > l (row k updated)
  auto pivot = [&](int l) {
    const int k = c0 + l;
    double tau = 0.0, scal = 1.0, beta = 0.0;
    if (lane == 0) {
      const double alpha = col(l)[k], sum = dsum[l];
      beta = alpha;
      if (sum > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, sum)), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
    }
    tau = __shfl_sync(0xffffffffu, tau, 0);
    scal = __shfl_sync(0xffffffffu, scal, 0);
    if (lane > l && lane < kb) {
      double* aj = col(lane);
      const double a = aj[k];
      const double f = tau * fma(scal, dsum[lane], a);
      aj[k] = a - f;
      gcol[lane] = f * scal;
    }
    if (lane == 0) {
      col(l)[k] = beta;
      taus[l] = tau;
      s_scal = scal;
    }
  };

  double p[kPanelKB];
  // initial dots x_0 . a_j over the rows below c0
#pragma unroll
  for (int j = 0; j < kPanelKB; j++) p[j] = 0.0;
  for (int r = c0 + 1 + tid; r < m; r += kPanelThreads) {
    const double x = col(0)[r];
#pragma unroll
    for (int j = 0; j < kPanelKB; j++)
      if (j < kb) p[j] = fma(x, col(j)[r], p[j]);
  }
  {
    const double s = warp_reduce_scatter32(p, lane);
    red[warp][lane] = s;
  }
  __syncthreads();
  if (warp == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kPanelWarps; w++) s += red[w][lane];
    dsum[lane] = s;
    __syncwarp();
    pivot(0);
  }
  __syncthreads();
  for (int l = 0; l < kb; l++) {
    const int k = c0 + l;
    const double scal = s_scal;
#pragma unroll
    for (int j = 0; j < kPanelKB; j++) p[j] = 0.0;
    const double* ak = col(l);
    for (int r = c0 + tid; r < m; r += kPanelThreads) {
      if (r <= k) continue;
      const double x = ak[r];
      const double v = x * scal;
      col(l)[r] = v;
#pragma unroll
      for (int q = 0; q < kPanelKB; q++)
        if (q < l) p[q] = fma(v, col(q)[r], p[q]);
      double xn = 0.0;
      if (l + 1 < kb && r > k + 1) xn = fma(-gcol[l + 1], x, col(l + 1)[r]);
#pragma unroll
      for (int j = 0; j < kPanelKB; j++) {
        if (j > l && j < kb) {
          double* aj = col(j);
          const double y = fma(-gcol[j], x, aj[r]);
          aj[r] = y;
          p[j] = fma(xn, y, p[j]);
        }
      }
    }
    {
      const double s = warp_reduce_scatter32(p, lane);
      red[warp][lane] = s;
    }
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kPanelWarps; w++) s += red[w][lane];
      if (lane < l) Gp[lane][l] = s + col(lane)[k];   // + v_q[k] * v_l[k] (v_l[k] = 1)
      if (lane > l) dsum[lane] = s;
      __syncwarp();
      if (l + 1 < kb) pivot(l + 1);
    }
    __syncthreads();
  }
  // dlarft (forward, columnwise): T[l][l] = tau_l, T[0:l, l] = -tau_l T[0:l, 0:l] G[0:l, l]
  if (warp == 0) {
    for (int l = 0; l < kPanelKB; l++) {
      double t = 0.0;
      if (l < kb) {
        if (lane < l) {
          double s = 0.0;
          for (int q = lane; q < l; q++) s = fma(Tp[lane][q], Gp[q][l], s);
          t = -taus[l] * s;
        } else if (lane == l) {
          t = taus[l];
        }
      }
      Tp[lane][l] = t;
      __syncwarp();
    }
  }
  __syncthreads();
  // V_p^T (explicit) and V_p T_p, rows c0 .. m - 1
  for (int r = c0 + tid; r < m; r += kPanelThreads) {
    const int rho = r - c0;
    double v[kPanelKB];
#pragma unroll
    for (int l = 0; l < kPanelKB; l++) {
      v[l] = l < kb ? (rho == l ? 1.0 : (rho > l ? col(l)[r] : 0.0)) : 0.0;
      jb.Vt[(int64_t)l * m + rho] = v[l];
    }
    double* vt = jb.VT + (int64_t)rho * kPanelKB;
#pragma unroll
    for (int j = 0; j < kPanelKB; j++) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l <= j; l++) s = fma(v[l], Tp[l][j], s);
      vt[j] = s;
    }
  }
}

// [A | I] from the job's column-major A
__global__ void k_qr_aug_init(const QrJob* __restrict__ jobs, double* const* __restrict__ aug, int nc) {
  const QrJob jb = jobs[blockIdx.y];
  double* X = aug[blockIdx.y];
  const int64_t m = jb.m, tot = m * (nc + m);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;
    X[e] = j < nc ? jb.A[e] : (i == j - nc ? 1.0 : 0.0);
  }
}

// R (row-major) and the rank test of reading R9 from the factorised [A | I]
__global__ void k_qr_export_r(const QrJob* __restrict__ jobs, double* const* __restrict__ aug, int nc,
                              int* __restrict__ rank_flag) {
  const QrJob jb = jobs[blockIdx.x];
  const double* X = aug[blockIdx.x];
  const int64_t m = jb.m;
  for (int e = threadIdx.x; e < nc * nc; e += blockDim.x) {
    const int i = e / nc, j = e - i * nc;
    jb.R[e] = j >= i ? X[(int64_t)j * m + i] : 0.0;
  }
  if (threadIdx.x == 0) {
    double mx = 0.0, mn = INFINITY;
    for (int i = 0; i < nc; i++) {
      const double v = fabs(X[(int64_t)i * m + i]);
      mx = fmax(mx, v);
      mn = fmin(mn, v);
    }
    if (!(mn > 1e-13 * mx)) atomicExch(rank_flag, 1);
  }
}

// Q^T[i][j] = X[(nc + j) * m + i]: rows i < nc to qlo, rows i >= nc to qhi (32 x 32 tiles
// through shared memory, both sides coalesced)
__global__ void k_qr_export_q(const QrJob* __restrict__ jobs, double* const* __restrict__ aug, int nc) {
  __shared__ double t[32][33];
  const QrJob jb = jobs[blockIdx.z];
  const double* X = aug[blockIdx.z];
  const int m = jb.m;
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  if (i0 >= m || j0 >= m) return;
  for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
    const int i = i0 + threadIdx.x, j = j0 + jj;
    if (i < m && j < m) t[jj][threadIdx.x] = X[(int64_t)(nc + j) * m + i];
  }
  __syncthreads();
  for (int ii = threadIdx.y; ii < 32; ii += blockDim.y) {
    const int i = i0 + ii, j = j0 + threadIdx.x;
    if (i < m && j < m) {
      double* row = i < nc ? jb.qlo + (int64_t)i * jb.ldq : jb.qhi + (int64_t)(i - nc) * jb.ldq;
      row[j] = t[threadIdx.x][ii];
    }
  }
}

void run_qr_blocked(Ctx& c, const std::vector<QrJob>& all, int nc, int* flag, const char* name) {
  // group jobs so that the augmented matrices and the panel scratch stay within the budget
  const int64_t budget = c.scratch_budget_bytes();
  size_t first = 0;
  while (first < all.size()) {
    size_t last = first;
    int64_t bytes = 0;
    while (last < all.size()) {
      const int64_t m = all[last].m;
      const int64_t b = (m * (nc + m) + 2 * m * kPanelKB + (int64_t)(nc + m) * kPanelKB) * 8;
      if (last > first && bytes + b > budget) break;
      bytes += b;
      last++;
    }
    std::vector<QrJob> jobs(all.begin() + first, all.begin() + last);
    first = last;
    const size_t nj = jobs.size();
    int m_max = 0;
    int64_t tot = 0;
    for (auto& j : jobs) {
      m_max = std::max(m_max, j.m);
      tot += (int64_t)j.m * (nc + j.m) + 2 * (int64_t)j.m * kPanelKB + (int64_t)(nc + j.m) * kPanelKB;
    }
    DevBuf<double> scratch(tot, c.stream);
    std::vector<double*> augp(nj), wtp(nj);
    std::vector<PanelJob> pj(nj);
    int64_t off = 0;
    for (size_t i = 0; i < nj; i++) {
      const int64_t m = jobs[i].m;
      augp[i] = scratch.p + off;
      off += m * (nc + m);
      pj[i] = {augp[i], (int32_t)m, scratch.p + off, scratch.p + off + m * kPanelKB};
      off += 2 * m * kPanelKB;
      wtp[i] = scratch.p + off;
      off += (int64_t)(nc + m) * kPanelKB;
    }
    DevBuf<QrJob> dj(nj, c.stream);
    dj.upload(jobs);
    DevBuf<double*> daug(nj, c.stream);
    daug.upload(augp);
    DevBuf<PanelJob> dpj(nj, c.stream);
    dpj.upload(pj);
    TimedLaunch tl(c, name);
    {
      dim3 grid((unsigned)std::min<int64_t>(1024, ceil_div((int64_t)m_max * (nc + m_max), 256)), (unsigned)nj);
      k_qr_aug_init<<<grid, 256, 0, c.stream>>>(dj.p, daug.p, nc);
      check_launch("k_qr_aug_init");
    }
    for (int c0 = 0; c0 < nc; c0 += kPanelKB) {
      const int kb = std::min(kPanelKB, nc - c0);
      k_qr_panel<<<(unsigned)nj, kPanelThreads, 0, c.stream>>>(dpj.p, c0, kb);
      check_launch("k_qr_panel");
      std::vector<GemmDesc> g1, g3;
      for (size_t i = 0; i < nj; i++) {
        const int32_t m = jobs[i].m;
        const int32_t ntr = nc + m - c0 - kb, mr = m - c0;
        double* Atr = augp[i] + (int64_t)(c0 + kb) * m + c0;  // row-major view: A_tr^T, ld m
        GemmDesc a{Atr, m, pj[i].VT, kPanelKB, wtp[i], kPanelKB, ntr, kb, mr, 0};
        GemmDesc b{wtp[i], kPanelKB, pj[i].Vt, m, Atr, m, ntr, mr, kb, 0};
        b.sub = 1;
        g1.push_back(a);
        g3.push_back(b);
      }
      gemm_batched(c, g1, "qr_panel_w");
      gemm_batched(c, g3, "qr_panel_update");
    }
    k_qr_export_r<<<(unsigned)nj, 256, 0, c.stream>>>(dj.p, daug.p, nc, flag);
    check_launch("k_qr_export_r");
    {
      const unsigned tq = (unsigned)ceil_div(m_max, 32);
      k_qr_export_q<<<dim3(tq, tq, (unsigned)nj), dim3(32, 8), 0, c.stream>>>(dj.p, daug.p, nc);
      check_launch("k_qr_export_q");
    }
  }
}

// QR of every job (one CTA each), then Q^T = I - V W1T on the DMMA GEMM, rows < nc to qlo and
// rows >= nc to qhi.  Matrices beyond shared memory (or MLK_QR_BLOCKED=1) take the blocked path.
// A = [R_L; R_R] for the stacked jobs, for the paths that factor A in global memory
void stack_jobs(Ctx& c, std::vector<QrJob>& jobs, int nc) {
  std::vector<StackJob> sj;
  for (auto& j : jobs)
    if (j.RL) sj.push_back({j.RL, j.RR, j.A});
  if (sj.empty()) return;
  DevBuf<StackJob> sjd(sj.size(), c.stream);
  sjd.upload(sj);
  TimedLaunch tl(c, "basis_stack");
  k_stack_r<<<(unsigned)sj.size(), 256, 0, c.stream>>>(sjd.p, nc);
  check_launch("k_stack_r");
  for (auto& j : jobs) j.RL = j.RR = nullptr;
}

void run_qr(Ctx& c, std::vector<QrJob>& jobs, int nc, int* flag, const char* name) {
  if (jobs.empty()) return;
  {
    int mm = 0;
    for (auto& j : jobs) mm = std::max(mm, j.m);
    const char* eb = std::getenv("MLK_QR_BLOCKED");
    if (qr_smem(mm, nc, true, false) > (size_t)kQrSmemLimit || (eb && eb[0] == '1')) {
      stack_jobs(c, jobs, nc);
      run_qr_blocked(c, jobs, nc, flag, name);
      return;
    }
  }
  int m_max = 0;
  for (auto& j : jobs) m_max = std::max(m_max, j.m);
  // scratch for V, T, W1T
  int64_t per = 0;
  for (auto& j : jobs) per += 2 * (int64_t)j.m * nc + (int64_t)nc * nc;
  DevBuf<double> scratch(per, c.stream);
  int64_t off = 0;
  for (auto& j : jobs) {
    j.V = scratch.p + off;
    off += (int64_t)j.m * nc;
    j.W1T = scratch.p + off;
    off += (int64_t)j.m * nc;
    j.T = scratch.p + off;
    off += (int64_t)nc * nc;
  }
  DevBuf<QrJob> dj(jobs.size(), c.stream);
  dj.upload(jobs);
  {
    TimedLaunch tl(c, name);
    const size_t s_full = qr_smem(m_max, nc, true, true), s_a = qr_smem(m_max, nc, true, false);
    if (s_full <= (size_t)kQrSmemLimit) {
      CUDA_CHECK(cudaFuncSetAttribute(k_qr_wy<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_full));
      k_qr_wy<true, true><<<(unsigned)jobs.size(), kQrThreads, s_full, c.stream>>>(dj.p, flag);
    } else if (s_a <= (size_t)kQrSmemLimit) {
      CUDA_CHECK(cudaFuncSetAttribute(k_qr_wy<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s_a));
      k_qr_wy<true, false><<<(unsigned)jobs.size(), kQrThreads, s_a, c.stream>>>(dj.p, flag);
    } else {
      stack_jobs(c, jobs, nc);
      dj.upload(jobs);
      const size_t s0 = qr_smem(m_max, nc, false, false);
      CUDA_CHECK(cudaFuncSetAttribute(k_qr_wy<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s0));
      k_qr_wy<false, false><<<(unsigned)jobs.size(), kQrThreads, s0, c.stream>>>(dj.p, flag);
    }
    check_launch("k_qr_wy");
    if (std::getenv("MLK_QR_PROFILE")) {
      long long h[12];
      CUDA_CHECK(cudaStreamSynchronize(c.stream));
      CUDA_CHECK(cudaMemcpyFromSymbol(h, g_qr_prof, sizeof(h)));
      std::fprintf(stderr,
                   "[mlk] qr %s m=%d nc=%d jobs=%zu: copy %lld fact %lld export %lld G %lld fs %lld cycles\n", name,
                   m_max, nc, jobs.size(), h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4]);
    }
  }
  std::vector<GemmDesc> gd;
  for (auto& j : jobs) {
    GemmDesc lo{j.V, nc, j.W1T, j.m, j.qlo, j.ldq, nc, j.m, nc, 0};
    lo.diag = 0;
    gd.push_back(lo);
    if (j.m > nc) {
      GemmDesc hi{j.V + (int64_t)nc * nc, nc, j.W1T, j.m, j.qhi, j.ldq, j.m - nc, j.m, nc, 0};
      hi.diag = nc;
      gd.push_back(hi);
    }
  }
  std::string gname = std::string(name) + "_formq";
  gemm_batched(c, gd, gname.c_str());
}

}  // namespace
}  // namespace mlk

namespace mlk {
void basis_sync(const mlk_basis_s* B) {
  if (!B->ready || B->ready_checked) return;
  CUDA_CHECK(cudaEventSynchronize(B->ready));
  int f = 0;
  CUDA_CHECK(cudaMemcpy(&f, B->merge_flag.p, sizeof(int), cudaMemcpyDeviceToHost));
  B->ready_checked = true;
  if (f && !B->keep_deficient)
    throw Error(MLK_ERR_RANK_DEFICIENT, "merged moment matrix is rank deficient (|R_kk| <= 1e-13 max|R_ii|)");
}

void basis_wait(Ctx& c, const mlk_basis_s* B) {
  basis_sync(B);
  if (B->ready) CUDA_CHECK(cudaStreamWaitEvent(c.stream, B->ready, 0));
}
}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_build_basis(mlk_ctx ctx, mlk_tree tree, int32_t w, mlk_basis* out) {
  return mlk_build_basis_ex(ctx, tree, MLK_INDEX_TD, w, 0, out);
}

mlk_status mlk_build_basis_ex(mlk_ctx ctx, mlk_tree tree, int32_t index_set, int32_t w, int32_t flags,
                              mlk_basis* out) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && tree && out, "NULL argument");
  *out = nullptr;
  // MLK_SLOW_MS=<ms>: report host phases of this call that took longer (diagnostics)
  struct SlowMark {
    double thr;
    std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    SlowMark() : thr(std::getenv("MLK_SLOW_MS") ? std::atof(std::getenv("MLK_SLOW_MS")) : -1.0) {}
    void operator()(const char* what) {
      if (thr < 0) return;
      auto now = std::chrono::steady_clock::now();
      const double ms = std::chrono::duration<double, std::milli>(now - last).count();
      if (ms >= thr) std::fprintf(stderr, "[mlk slow] basis.%s %.1f ms\n", what, ms);
      last = now;
    }
  } slow;
  MLK_REQUIRE(index_set >= MLK_INDEX_TD && index_set <= MLK_INDEX_TP, "unknown index set");
  MLK_REQUIRE(w >= 0 && w <= 64, "need 0 <= w <= 64");
  MLK_REQUIRE((flags & ~(MLK_BASIS_KEEP_DEFICIENT | MLK_BASIS_DROP_PHI)) == 0, "unknown basis flags");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  cudaStream_t st = c.stream;
  const int d = tree->d, dp = tree->d_pad, nn = tree->n_nodes;
  auto fac = index_set_factors(index_set, d, w);
  MLK_REQUIRE((int)fac.size() <= kMaxM, "index set has more than 4096 members");
  MLK_REQUIRE(!fac.empty(), "empty index set");
  const int M = (int)fac.size();
  int wmax = 0;
  for (auto& f : fac) wmax = std::max(wmax, (int)f.size());
  MLK_REQUIRE(M < tree->n, "need n > M = |Lambda(w)|");

  auto B = std::make_unique<mlk_basis_s>();
  B->device = c.device;
  B->M = M;
  B->w = wmax;
  B->tree = tree;
  B->p.assign(nn, 0);
  B->cell_pos.assign(nn, -1);
  B->w_off.assign(nn, -1);
  B->phi_off.assign(nn, -1);
  for (int q = 0; q < nn; q++) {
    if (tree->state[q] < 0) continue;
    int64_t s = tree->end[q] - tree->begin[q];
    if (tree->state[q] == 1) {
      if (s < M) throw Error(MLK_ERR_RANK_DEFICIENT, "leaf with fewer points than monomials");
      B->p[q] = (int32_t)(s - M);
    } else {
      B->p[q] = M;
    }
  }
  // C_W order: levels t..0, heap order within a level (R11)
  std::vector<int> order;
  for (int dep = tree->t; dep >= 0; dep--)
    for (int q = (1 << dep) - 1; q < (2 << dep) - 1 && q < nn; q++)
      if (tree->state[q] >= 0) order.push_back(q);
  int64_t woff = 0, phioff = 0, row = 0;
  B->row_off.push_back(0);
  for (int q : order) {
    int64_t s = tree->end[q] - tree->begin[q];
    B->w_off[q] = woff;
    woff += (int64_t)B->p[q] * s;
    B->phi_off[q] = phioff;
    phioff += (int64_t)M * s;
    if (B->p[q] > 0) {
      B->cell_pos[q] = (int32_t)B->cells.size();
      B->cells.push_back(q);
      row += B->p[q];
      B->row_off.push_back(row);
    }
  }
  B->dim = row;
  slow("setup");
  B->W.alloc(std::max<int64_t>(woff, 1), st);
  slow("W.alloc");
  // Phi blocks of every node cost M x n doubles per level (cfg5: 111 GB next to 106 GB of W).
  // They are kept (for mlk_basis_export) only when W + Phi fit in half of the free memory or
  // MLK_BASIS_DROP_PHI is not set; otherwise the construction keeps the leaves' Phi and two
  // alternating level buffers (node q at M begin[q]) and retains only L = Phi_root.
  bool drop_phi = (flags & MLK_BASIS_DROP_PHI) != 0;
  if (!drop_phi && (woff + phioff) * (int64_t)sizeof(double) > ((int64_t)1 << 30)) {
    // (the context's estimate, not cudaMemGetInfo: a driver query per call stalls under NVML polling)
    drop_phi = phioff * (int64_t)sizeof(double) > std::max<int64_t>(ctx_avail_bytes(c), 0) / 2;
  }
  B->phi_dropped = drop_phi;
  const int64_t mn = (int64_t)M * tree->n;
  DevBuf<double> leafphi, lvlphi[2];
  if (drop_phi) {
    leafphi.alloc((size_t)std::max<int64_t>(mn, 1), st);
    std::fill(B->phi_off.begin(), B->phi_off.end(), -1);
    B->phi_off[0] = 0;
  } else {
    B->Phi.alloc(std::max<int64_t>(phioff, 1), st);
  }
  auto phi_ptr = [&](int q) -> double* {
    if (!drop_phi) return B->Phi.p + B->phi_off[q];
    if (tree->state[q] == 1) return leafphi.p + (int64_t)M * tree->begin[q];
    return lvlphi[tree->depth[q] & 1].p + (int64_t)M * tree->begin[q];
  };
  slow("Phi.alloc");
  DevBuf<double> Rbuf((size_t)nn * M * M, st);
  slow("Rbuf.alloc");
  DevBuf<int> flag(1, st);
  flag.zero();

  // factor table
  int wf = std::max(wmax, 1);
  std::vector<int32_t> fh((size_t)M * wf, -1);
  for (int m = 0; m < M; m++)
    for (size_t j = 0; j < fac[m].size(); j++) fh[(size_t)m * wf + j] = fac[m][j];
  DevBuf<int32_t> facd(fh.size(), st);
  facd.upload(fh);

  slow("facd");
  HostTrace trace("basis");
  // ---- leaves
  {
    std::vector<LeafJob> lj;
    std::vector<QrJob> qj;
    int64_t aoff = 0;
    int32_t smax = 0;
    for (int q : order) {
      if (tree->state[q] != 1) continue;
      int32_t s = (int32_t)(tree->end[q] - tree->begin[q]);
      lj.push_back({tree->begin[q], s, aoff});
      aoff += (int64_t)s * M;
      smax = std::max(smax, s);
    }
    DevBuf<double> A(std::max<int64_t>(aoff, 1), st);
    DevBuf<LeafJob> ljd(lj.size(), st);
    ljd.upload(lj);
    {
      TimedLaunch tl(c, "basis_monomials");
      dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(64, ceil_div((int64_t)smax * M, 256))),
                (unsigned)lj.size());
      k_monomials<<<grid, 256, 0, st>>>(tree->Xt.p, dp, ljd.p, facd.p, M, wf, A.p);
      check_launch("k_monomials");
    }
    size_t k = 0;
    for (int q : order) {
      if (tree->state[q] != 1) continue;
      int32_t s = (int32_t)(tree->end[q] - tree->begin[q]);
      QrJob jb;
      jb.A = A.p + lj[k].a_off;
      jb.m = s;
      jb.nc = M;
      jb.R = Rbuf.p + (int64_t)q * M * M;
      jb.qlo = phi_ptr(q);
      jb.qhi = B->W.p + B->w_off[q];
      jb.ldq = s;
      jb.stacked = 0;
      qj.push_back(jb);
      k++;
    }
    run_qr(c, qj, M, flag.p, "basis_leaf_qr");
  }
  trace.mark("leaves");
  slow("leaves");
  {
    auto fl = flag.download(1);
    if (fl[0] && !(flags & MLK_BASIS_KEEP_DEFICIENT))
      throw Error(MLK_ERR_RANK_DEFICIENT, "moment matrix is rank deficient (|R_kk| <= 1e-13 max|R_ii|)");
  }
  B->keep_deficient = (flags & MLK_BASIS_KEEP_DEFICIENT) != 0;
  trace.mark("leaf_check");
  slow("leaf_check");
  // ---- internal levels, bottom-up, on the auxiliary stream: the call returns while they run
  // ([R_L; R_R] has full column rank whenever R_L does, so the synchronous leaf check above is
  // the one that can fail; merge_flag re-checks numerically when the basis is first used)
  if (!c.aux_stream) CUDA_CHECK(cudaStreamCreateWithFlags(&c.aux_stream, cudaStreamNonBlocking));
  CUDA_CHECK(cudaEventCreateWithFlags(&B->ready, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventRecord(B->ready, st));
  CUDA_CHECK(cudaStreamWaitEvent(c.aux_stream, B->ready, 0));
  const cudaStream_t main_stream = st;
  st = c.aux_stream;
  c.stream = st;  // run_qr / gemm_batched / TimedLaunch use the context stream
  struct RestoreStream {
    Ctx& c;
    cudaStream_t s;
    ~RestoreStream() { c.stream = s; }
  } restore{c, main_stream};
  B->merge_flag.alloc(1, st);
  B->merge_flag.zero();
  Rbuf.s = st;  // freed behind the merges
  leafphi.s = st;
  if (drop_phi)
    for (auto& lb : lvlphi) lb.alloc((size_t)std::max<int64_t>(mn, 1), st);
  DevBuf<double> Qt(0, st);
  DevBuf<double> Ast(0, st);
  // keep the merge Q factors for the nested assembly when they are small (cfg2-4: 7-43 MB)
  {
    int64_t nint = 0;
    for (int q = 0; q < nn; q++)
      if (tree->state[q] == 0) nint++;
    const int64_t qbytes = nint * 4 * (int64_t)M * M * (int64_t)sizeof(double);
    B->q_off.assign(nn, -1);
    if (nint > 0 && qbytes <= ((int64_t)1 << 30)) {
      B->Qm.alloc((size_t)nint * 4 * M * M, st);
      int64_t o = 0;
      for (int q = 0; q < nn; q++)
        if (tree->state[q] == 0) {
          B->q_off[q] = o;
          o += 4 * (int64_t)M * M;
        }
    }
  }
  // cells of a level in groups whose stacked matrices and Q^T (6 M^2 doubles per cell) fit a
  // quarter of the scratch budget (cfg5: 84 MB per cell; a whole level of 256 took 22 GB)
  const int64_t per_cell = 6 * (int64_t)M * M * (int64_t)sizeof(double);
  const size_t group_max = (size_t)std::max<int64_t>(1, c.scratch_budget_bytes() / 4 / per_cell);
  for (int dep = tree->t - 1; dep >= 0; dep--) {
    std::vector<int> level_cells;
    for (int q = (1 << dep) - 1; q < (2 << dep) - 1; q++)
      if (tree->state[q] == 0) level_cells.push_back(q);
    for (size_t g0 = 0; g0 < level_cells.size(); g0 += group_max) {
      std::vector<int> cellsq(level_cells.begin() + g0,
                              level_cells.begin() + std::min(level_cells.size(), g0 + group_max));
      size_t nc = cellsq.size();
      Ast.alloc(nc * 2 * M * M, st);
      Qt.alloc(nc * 4 * (size_t)M * M, st);
      std::vector<StackJob> sj;
      std::vector<QrJob> qj;
      for (size_t i = 0; i < nc; i++) {
        int q = cellsq[i];
        sj.push_back({Rbuf.p + (int64_t)(2 * q + 1) * M * M, Rbuf.p + (int64_t)(2 * q + 2) * M * M,
                      Ast.p + i * 2 * M * M});
        QrJob jb;
        jb.A = Ast.p + i * 2 * M * M;
        jb.m = 2 * M;
        jb.nc = M;
        jb.R = Rbuf.p + (int64_t)q * M * M;
        jb.qlo = Qt.p + i * 4 * (size_t)M * M;       // Q column-major == Q^T row-major
        jb.qhi = jb.qlo + (size_t)M * 2 * M;
        jb.ldq = 2 * M;
        jb.stacked = 1;
        jb.RL = sj.back().RL;
        jb.RR = sj.back().RR;
        qj.push_back(jb);
      }
      trace.mark("lvl_stack");
      run_qr(c, qj, M, B->merge_flag.p, "basis_merge_qr");
      trace.mark("lvl_qr");
      if (B->Qm.p) {
        std::vector<int64_t> qo(nc);
        for (size_t i = 0; i < nc; i++) qo[i] = B->q_off[cellsq[i]];
        DevBuf<int64_t> qo_d(nc, st);
        qo_d.upload(qo);
        k_keep_q<<<dim3(8, (unsigned)nc), 256, 0, st>>>(Qt.p, qo_d.p, 2 * M, B->Qm.p);
        check_launch("k_keep_q");
      }
      // Phi_q / W_q = (Q^T)[rows, cols of child] x Phi_child
      std::vector<GemmDesc> gd;
      for (size_t i = 0; i < nc; i++) {
        int q = cellsq[i];
        int l = 2 * q + 1, r = 2 * q + 2;
        int64_t s = tree->end[q] - tree->begin[q];
        int32_t nl = (int32_t)(tree->end[l] - tree->begin[l]), nr = (int32_t)(tree->end[r] - tree->begin[r]);
        const double* Qrow = Qt.p + i * 4 * (size_t)M * M;  // (Q^T)[i][c] at Qrow[i*2M + c]
        for (int half = 0; half < 2; half++) {
          const double* Pc = phi_ptr(half ? r : l);
          int32_t ncol = half ? nr : nl;
          int64_t coff = half ? nl : 0;
          GemmDesc g1{Qrow + (half ? M : 0), 2 * M, Pc, ncol, phi_ptr(q) + coff, s, M, ncol, M, 0};
          GemmDesc g2{Qrow + (int64_t)M * 2 * M + (half ? M : 0), 2 * M, Pc, ncol, B->W.p + B->w_off[q] + coff, s, M,
                      ncol, M, 0};
          gd.push_back(g1);
          gd.push_back(g2);
        }
      }
      gemm_batched(c, gd, "basis_transfer_gemm");
      trace.mark("lvl_gemm");
    }
  }
  trace.mark("levels");
  slow("levels");
  if (drop_phi) {
    // L = Phi_root: the root's level buffer (or the leaf buffer when the root is a leaf)
    B->Phi = std::move(tree->state[0] == 1 ? leafphi : lvlphi[0]);
    B->Phi.s = st;
  }
  CUDA_CHECK(cudaEventRecord(B->ready, st));
  *out = B.release();
  MLK_API_END
}


void mlk_basis_free(mlk_basis basis) {
  if (!basis) return;
  cudaSetDevice(basis->device);
  // the creating context's stream may already be gone: drain the device, free on stream 0
  cudaDeviceSynchronize();
  basis->W.s = nullptr;
  basis->Phi.s = nullptr;
  basis->Qm.s = nullptr;
  basis->merge_flag.s = nullptr;
  if (basis->ready) cudaEventDestroy(basis->ready);
  delete basis;
}

mlk_status mlk_basis_info(mlk_basis basis, int32_t* M, int64_t* dim, int32_t* n_cells) {
  MLK_API_BEGIN
  MLK_REQUIRE(basis, "basis is NULL");
  if (M) *M = basis->M;
  if (dim) *dim = basis->dim;
  if (n_cells) *n_cells = (int32_t)basis->cells.size();
  MLK_API_END
}

mlk_status mlk_basis_export(mlk_basis basis, int32_t* cells, int64_t* cell_row_off, int32_t node, double* W_block,
                            double* Phi_block, double* L) {
  MLK_API_BEGIN
  MLK_REQUIRE(basis, "basis is NULL");
  CUDA_CHECK(cudaSetDevice(basis->device));
  // cells / row offsets are host-side; only the device blocks wait for the merge levels
  if (node >= 0 || L) basis_sync(basis);
  const mlk_tree_s* tree = basis->tree;
  if (cells) std::copy(basis->cells.begin(), basis->cells.end(), cells);
  if (cell_row_off) std::copy(basis->row_off.begin(), basis->row_off.end(), cell_row_off);
  if (node >= 0) {
    MLK_REQUIRE(node < tree->n_nodes && tree->state[node] >= 0, "node out of range");
    int64_t s = tree->end[node] - tree->begin[node];
    if (W_block && basis->p[node] > 0)
      CUDA_CHECK(cudaMemcpy(W_block, basis->W.p + basis->w_off[node], sizeof(double) * basis->p[node] * s,
                            cudaMemcpyDefault));
    if (Phi_block) {
      if (basis->phi_off[node] < 0)
        throw Error(MLK_ERR_UNSUPPORTED, "Phi blocks of non-root cells were not retained (MLK_BASIS_DROP_PHI "
                                         "or W + Phi beyond half of the free device memory); L is available");
      CUDA_CHECK(cudaMemcpy(Phi_block, basis->Phi.p + basis->phi_off[node], sizeof(double) * basis->M * s,
                            cudaMemcpyDefault));
    }
  }
  if (L)
    CUDA_CHECK(cudaMemcpy(L, basis->Phi.p + basis->phi_off[0], sizeof(double) * basis->M * tree->n, cudaMemcpyDefault));
  MLK_API_END
}

}  // extern "C"
