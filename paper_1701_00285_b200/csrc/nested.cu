// Transfers of the nested assembly (assemble.cu, DESIGN.md section 6 "Nested assembly"):
// for every internal cell c of one tree level and every row i of the current row chunk,
//   [S_c[i] | V_c[i]] = [S_cL[i] S_cR[i]] Q_c        (1 x 2M) (2M x 2M)
// with Q_c the complete orthogonal factor of the QR of [R_cL; R_cR] kept by the basis (steps
// (c)-(e) of P:1427-1515: Phi_c = Q_c[:, :M]^T (Phi_cL (+) Phi_cR), W_c = Q_c[:, M:]^T (...)).
//
// k_transfer: one CTA per (cell, block of 256 rows); Q_c (2M x 2M, row stride 4 (mod 16)
// doubles so the B-fragment loads of a half-warp hit 16 distinct 8-byte banks) stays in shared
// memory for the CTA's rows; 8 warps, each 8 rows x all 2M columns per 64-row pass, on FP64
// DMMA.8x8x4 (k = 2M padded to a multiple of 8); the A fragments ([S_cL S_cR] rows) are read
// straight from global memory into registers at the start of each pass (each element once,
// 32-byte row segments, one round trip per pass).  8 M^2 flops per (row, cell).
#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <map>
#include <mutex>

#include "api.cuh"
#include "dmma.cuh"

namespace mlk {
namespace {

constexpr int kTrRows = 64;       // rows per pass (8 warps x 8)
// passes per CTA: 4 x 64 rows (Q_c loaded once per 256 rows; adaptive pass counts that keep
// only ~2 CTAs per SM busy measured slower: 134 -> 167 ms at cfg4, r02j)
constexpr int kTrMaxM2 = 144;     // 2M limit of the shared-memory kernel (M <= 72)
// (a tiled variant with Q_c and double-buffered 64-row A tiles in shared memory, 8 warps as
// 2 row halves x 4 column quarters, one CTA per SM, measured 1.75x slower on cfg4: 199 against
// 114 ms, r02 tr2 -- the A tile went through shared memory once per column warp); so did a
// variant with 16 warps, one CTA per SM and each warp's next-pass A rows staged by 8-byte
// cp.async into its own shared buffer during the current pass's DMMAs (cfg4 97.1 vs 82.8 ms,
// cfg3 16.5 vs 13.8 ms, bit-identical; r02 trasync): the load latency is not what limits it)

struct TransferJob {
  const double* Sch;     // [S_cL S_cR], rows x 2M, row stride ld
  const double* Q;       // 2M x 2M row-major
  double* Sout;          // rows x M (stride ld), or nullptr (the root: S_0 is not needed)
  double* Vout;          // rows x M (stride ld)
  const uint8_t* vflag;  // per 64-row block: 1 if some row of it needs V_c (nullptr: all)
};

__host__ __device__ constexpr int tr_stride(int m2p) { return (m2p + 11) / 16 * 16 + 4; }  // >= m2p, 4 mod 16

template <int NT, bool PF>  // NT = 2M padded / 8 column tiles; PF: prefetch the next pass's A (NT <= 8)
#ifndef MLK_TR_MINB
#define MLK_TR_MINB 2  // CTAs per SM the register budget targets (128 registers; 1: 212 registers,
                       // one CTA per SM: cfg4 transfers 167 vs 145 ms, r02j)
#endif
__global__ void __launch_bounds__(256, MLK_TR_MINB) k_transfer(const TransferJob* __restrict__ jobs, int M, int64_t rows,
                                                     int64_t ld, int passes) {
  extern __shared__ __align__(16) double sm[];
  constexpr int M2P = NT * 8;            // 2M padded to a multiple of 8 (k and n)
  constexpr int SQ = tr_stride(M2P);
  constexpr int KS = M2P / 4;
  const TransferJob jb = jobs[blockIdx.y];
  const int M2 = 2 * M;
  double* Qs = sm;                       // M2P x SQ, zero padded
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < M2P * M2P; e += blockDim.x) {
    const int r = e / M2P, cc = e - r * M2P;
    Qs[r * SQ + cc] = (r < M2 && cc < M2) ? jb.Q[(int64_t)r * M2 + cc] : 0.0;
  }
  const int64_t r_begin = (int64_t)blockIdx.x * kTrRows * passes;
  const double* bp = Qs + (lane & 3) * SQ + (lane >> 2);
  // the lane's A elements of one pass: one memory round trip per pass, not per k-step
  auto load = [&](int pass, double (&dst)[KS]) {
    const int64_t r = r_begin + (int64_t)pass * kTrRows + warp * 8 + (lane >> 2);
    const bool rok = r < rows;
    const double* ap = jb.Sch + (rok ? r : 0) * ld + (lane & 3);
#pragma unroll
    for (int ks = 0; ks < KS; ks++) {
      const int k = 4 * ks + (lane & 3);
      dst[ks] = (rok && k < M2) ? __ldg(ap + 4 * ks) : 0.0;
    }
  };
  double areg[KS], anext[PF ? KS : 1];
  if (PF && r_begin + warp * 8 < rows) load(0, areg);  // in flight while Q_c is staged
  __syncthreads();
  for (int pass = 0; pass < passes; pass++) {
    const int64_t r = r_begin + (int64_t)pass * kTrRows + warp * 8 + (lane >> 2);  // the lane's A row
    if (r_begin + (int64_t)pass * kTrRows + warp * 8 >= rows) break;              // warp-uniform
    const bool rok = r < rows;
    if constexpr (PF) {
      if (pass + 1 < passes && r_begin + (int64_t)(pass + 1) * kTrRows + warp * 8 < rows) load(pass + 1, anext);
    } else {
      load(pass, areg);
    }
    // V_c only where a block with contracted-first cell c has rows (the S half is needed for
    // every row: the parents' sums); warp-uniform: a pass is one 64-row block
    const int64_t blk = (r_begin >> 6) + pass;
    const int nt_use = (jb.vflag == nullptr || jb.vflag[blk]) ? NT : (NT + 1) / 2;  // (NT + 1) / 2 = ceil(M / 8)
    double acc[NT][2];
#pragma unroll
    for (int t = 0; t < NT; t++) acc[t][0] = acc[t][1] = 0.0;
    // the tile count is a compile-time constant in each branch: a DMMA predicated off by a
    // runtime test still occupies the pipe (the S-only passes, 96 % of the (row, cell) pairs at
    // cfg4, ran 13 DMMA tiles for 7 useful ones: 71 % DMMA-active at 38 % of the FP64 peak, r02)
    auto mm = [&](auto ntc) {
      constexpr int NU = decltype(ntc)::value;
#pragma unroll
      for (int ks = 0; ks < KS; ks++) {
        const double* bk = bp + 4 * ks * SQ;
#pragma unroll
        for (int t = 0; t < NU; t++) dmma_8x8x4(acc[t][0], acc[t][1], areg[ks], bk[8 * t]);
      }
    };
    if (nt_use == NT) mm(std::integral_constant<int, NT>{});
    else mm(std::integral_constant<int, (NT + 1) / 2>{});
    if (rok) {
#pragma unroll
      for (int t = 0; t < NT; t++) {
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int col = 8 * t + 2 * (lane & 3) + e;
          if (col < M) {
            if (jb.Sout) jb.Sout[r * ld + col] = acc[t][e];
          } else if (col < M2 && t < nt_use) {
            jb.Vout[r * ld + col - M] = acc[t][e];
          }
        }
      }
    }
    if constexpr (PF) {
#pragma unroll
      for (int ks = 0; ks < KS; ks++) areg[ks] = anext[ks];
    }
  }
}

template <int NT>
void launch_transfer(Ctx& c, const TransferJob* jobs, int njobs, int M, int64_t rows, int64_t ld) {
  constexpr int M2P = NT * 8;
  const size_t smem = sizeof(double) * (size_t)M2P * tr_stride(M2P);
  // prefetch of the next pass's A fragments where the registers allow it without spilling
  // (2M <= 64: cfg3's transfers 15.9 -> 14.5 ms, r02 pf; at cfg4's NT = 13 the extra 26
  // registers spilled at the 128-register budget and the transfers took 214 against 114 ms,
  // and one CTA per SM without spills 154 ms).  MLK_TR_NOPF: A/B switch.
  static const bool pf_env = std::getenv("MLK_TR_NOPF") == nullptr;
  auto fn = k_transfer<NT, false>;
  if constexpr (NT <= 8) {
    if (pf_env) fn = k_transfer<NT, true>;
  }
  static std::mutex mu;
  static std::map<int, bool> set;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!set[c.device]) {
      CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      set[c.device] = true;
    }
  }
  const int64_t row_blocks = ceil_div(rows, (int64_t)kTrRows);
#ifndef MLK_TR_PASSES
#define MLK_TR_PASSES 4
#endif
  // fewer passes per CTA where a level has few cells (the top levels), so that the level still
  // spreads over ~2 CTAs per SM
  const int64_t want = 2LL * 2 * num_sms(c.device);
  const int passes = (int)std::max<int64_t>(1, std::min<int64_t>({row_blocks, (int64_t)MLK_TR_PASSES,
                                                                   row_blocks * njobs / want}));
  dim3 grid((unsigned)ceil_div(row_blocks, (int64_t)passes), (unsigned)njobs);
  fn<<<grid, 256, smem, c.stream>>>(jobs, M, rows, ld, passes);
  check_launch("k_transfer");
}

}  // namespace

bool transfer_kernel_ok(int M) { return 2 * M <= kTrMaxM2; }

// One tree level of transfers (all cells of the level), rows x (n_nodes M) buffers S, V.
void transfer_level(Ctx& c, const std::vector<std::array<const double*, 4>>& jobs,
                    const std::vector<const uint8_t*>& vflags, int M, int64_t rows, int64_t ld) {
  if (jobs.empty()) return;
  std::vector<TransferJob> hj;
  for (size_t i = 0; i < jobs.size(); i++) {
    const auto& j = jobs[i];
    hj.push_back({j[0], j[1], const_cast<double*>(j[2]), const_cast<double*>(j[3]), vflags[i]});
  }
  DevBuf<TransferJob> dj(hj.size(), c.stream);
  dj.upload(hj);
  TimedLaunch tl(c, "assemble_transfer");
  const int nt = (2 * M + 7) / 8;
  switch (nt) {
#define MLK_TR_CASE(K) \
  case K: launch_transfer<K>(c, dj.p, (int)hj.size(), M, rows, ld); break;
    MLK_TR_CASE(1) MLK_TR_CASE(2) MLK_TR_CASE(3) MLK_TR_CASE(4) MLK_TR_CASE(5) MLK_TR_CASE(6) MLK_TR_CASE(7)
    MLK_TR_CASE(8) MLK_TR_CASE(9) MLK_TR_CASE(10) MLK_TR_CASE(11) MLK_TR_CASE(12) MLK_TR_CASE(13)
    MLK_TR_CASE(14) MLK_TR_CASE(15) MLK_TR_CASE(16) MLK_TR_CASE(17) MLK_TR_CASE(18)
#undef MLK_TR_CASE
    default: throw Error(MLK_ERR_UNSUPPORTED, "transfer kernel: 2M > 144");
  }
}

}  // namespace mlk
