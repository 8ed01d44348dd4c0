// C_W v by the three steps of P:2146-2170 -- (1) a = W^T v, (2) b = C a, (3) y = W b -- and
// the BSR product y = C~_W v.  Step (2) is the fused tile kernel of tile.cu with the vectors
// in place of a wavelet block; steps (1), (3) and the BSR product are HBM-bound passes over
// the stored W blocks / BSR values with a fixed summation order (deterministic).
#include <algorithm>
#include <cstdlib>

#include "api.cuh"
#include "tile.cuh"

namespace mlk {
namespace {

struct CellJob {
  int64_t pt_begin;   // first tree position of the cell
  int32_t s, p;       // points, wavelets
  int64_t row_off;    // C_W row offset
  const double* W;    // p x s
};

// a[v][begin + x] += sum_r W[r][x] v[v][row_off + r] for the cells of one level; the vectors in
// groups of kAwVG, so each W element is read once per group (not once per vector)
constexpr int kAwVG = 8;
template <int VG>
__global__ void k_apply_wt(const CellJob* __restrict__ jobs, const double* __restrict__ v, int64_t dim,
                           double* __restrict__ a, int64_t n, int nvec) {
  const CellJob jb = jobs[blockIdx.x];
  for (int x = blockIdx.y * blockDim.x + threadIdx.x; x < jb.s; x += gridDim.y * blockDim.x) {
    for (int iv0 = 0; iv0 < nvec; iv0 += VG) {
      const int nv = min(VG, nvec - iv0);
      const double* vv = v + (int64_t)iv0 * dim + jb.row_off;
      // four partial sums per vector: four independent W loads in flight per thread (the pass is
      // bound by memory-level parallelism, one accumulator left it latency-bound at ~0.5 TB/s)
      double s0[VG], s1[VG], s2[VG], s3[VG];
#pragma unroll
      for (int q = 0; q < VG; q++) s0[q] = s1[q] = s2[q] = s3[q] = 0.0;
      const double* w = jb.W + x;
      int r = 0;
      for (; r + 3 < jb.p; r += 4) {
        const double w0 = w[(int64_t)r * jb.s], w1 = w[(int64_t)(r + 1) * jb.s], w2 = w[(int64_t)(r + 2) * jb.s],
                     w3 = w[(int64_t)(r + 3) * jb.s];
#pragma unroll
        for (int q = 0; q < VG; q++) {
          if (q < nv) {
            const double* vq = vv + (int64_t)q * dim;
            s0[q] = fma(w0, vq[r], s0[q]);
            s1[q] = fma(w1, vq[r + 1], s1[q]);
            s2[q] = fma(w2, vq[r + 2], s2[q]);
            s3[q] = fma(w3, vq[r + 3], s3[q]);
          }
        }
      }
      for (; r < jb.p; r++) {
        const double w0 = w[(int64_t)r * jb.s];
#pragma unroll
        for (int q = 0; q < VG; q++)
          if (q < nv) s0[q] = fma(w0, vv[(int64_t)q * dim + r], s0[q]);
      }
#pragma unroll
      for (int q = 0; q < VG; q++)
        if (q < nv) a[(int64_t)(iv0 + q) * n + jb.pt_begin + x] += (s0[q] + s1[q]) + (s2[q] + s3[q]);
    }
  }
}

// y[v][row_off + r] = sum_x W[r][x] b[v][begin + x].  A CTA per (cell, chunk of kAwChunk
// points), a warp per row, lanes strided over the chunk's points, vectors in groups of VG (each W
// element read once per group); a cell of one chunk writes y, longer cells write per-chunk
// partials that k_apply_w_reduce adds in chunk order (deterministic).  The root row's p rows
// of n points were one warp each (latency-bound at cfg3: 3.4 ms for 10 vectors).
constexpr int kAwChunk = 4096;
struct WJob {
  int32_t cell;     // index into the level-order job list
  int32_t x0, x1;   // point range of the chunk
  int64_t part;     // partial offset (doubles, nvec x p), or -1: write y
};
template <int VG>
__global__ void k_apply_w(const CellJob* __restrict__ jobs, const WJob* __restrict__ wj, const double* __restrict__ b,
                          int64_t n, double* __restrict__ y, int64_t dim, int nvec, double* __restrict__ part) {
  const WJob w_ = wj[blockIdx.x];
  const CellJob jb = jobs[w_.cell];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < jb.p; r += nw) {
    const double* w = jb.W + (int64_t)r * jb.s;
    for (int iv0 = 0; iv0 < nvec; iv0 += VG) {
      const int nv = min(VG, nvec - iv0);
      const double* bb = b + (int64_t)iv0 * n + jb.pt_begin;
      double s[VG];
#pragma unroll
      for (int q = 0; q < VG; q++) s[q] = 0.0;
      for (int x = w_.x0 + lane; x < w_.x1; x += 32) {
        const double wx = w[x];
#pragma unroll
        for (int q = 0; q < VG; q++)
          if (q < nv) s[q] = fma(wx, bb[(int64_t)q * n + x], s[q]);
      }
#pragma unroll
      for (int q = 0; q < VG; q++) {
        if (q < nv) {  // warp-uniform
          for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
          if (lane == 0) {
            if (w_.part < 0) y[(int64_t)(iv0 + q) * dim + jb.row_off + r] = s[q];
            else part[w_.part + (int64_t)(iv0 + q) * jb.p + r] = s[q];
          }
        }
      }
    }
  }
}

struct WRed {
  int32_t cell, nch;
  int64_t part;  // first chunk's partials; chunk c at part + c nvec p
};
__global__ void k_apply_w_reduce(const CellJob* __restrict__ jobs, const WRed* __restrict__ rj,
                                 const double* __restrict__ part, double* __restrict__ y, int64_t dim, int nvec) {
  const WRed q = rj[blockIdx.x];
  const CellJob jb = jobs[q.cell];
  for (int e = threadIdx.x; e < nvec * jb.p; e += blockDim.x) {
    const int iv = e / jb.p, r = e - iv * jb.p;
    double s = 0.0;
    for (int c = 0; c < q.nch; c++) s += part[q.part + (int64_t)c * nvec * jb.p + e];
    y[(int64_t)iv * dim + jb.row_off + r] = s;
  }
}

// BSR: y_r = sum_{items (r,c)} B v_c + sum_{items (c,r), c != r} B^T v_c over the stored
// items this rank applies -- every block (nranks == 1), the blocks it owns (complete values,
// nranks > 1), or the row-chunk pieces it computed, read straight from its shard (nranks > 1
// before any gather: S§8(e)'s sharded product, the ranks' partial y sum to C~_W v).  Two passes
// read each item once with coalesced loads, then a fixed-order reduction per cell
// (deterministic, no atomics).  HBM-bound: 2 x 8 x (item values) bytes.
//  row pass  (one CTA per item, grid.y = vector group): warp per row i, lanes over the columns,
//            warp reduction -> rp[part_off[k]][iv][i] (p_r values)
//  col pass  (one CTA per item and 256-column panel): thread per column j, loop over the rows
//            -> cp[..][iv][j] (p_c values, off-diagonal items only)
constexpr int kBsrVG = 4;  // vectors per pass

struct BsrItem {
  int32_t r, c;  // cell positions (C_W order)
  int64_t off;   // values at base + off, p_r x p_c row-major
};

__global__ void k_bsr_rows(const BsrItem* __restrict__ items, const int64_t* __restrict__ row_off,
                           const int64_t* __restrict__ part_off, const double* __restrict__ base,
                           const double* __restrict__ v, int64_t dim, int nvec, double* __restrict__ rp) {
  const int k = blockIdx.x, iv0 = blockIdx.y * kBsrVG;
  const BsrItem it = items[k];
  const int64_t r0 = row_off[it.r], c0 = row_off[it.c];
  const int pr = (int)(row_off[it.r + 1] - r0), pc = (int)(row_off[it.c + 1] - c0);
  const int nv = min(kBsrVG, nvec - iv0);
  double* out = rp + part_off[k] * nvec;  // nvec x p_r
  const double* B = base + it.off;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < pr; i += nw) {
    double s[kBsrVG] = {0.0, 0.0, 0.0, 0.0};
    const double* Bi = B + (int64_t)i * pc;
    for (int j = lane; j < pc; j += 32) {
      const double bij = Bi[j];
#pragma unroll
      for (int q = 0; q < kBsrVG; q++)
        if (q < nv) s[q] = fma(bij, v[(int64_t)(iv0 + q) * dim + c0 + j], s[q]);
    }
#pragma unroll
    for (int q = 0; q < kBsrVG; q++) {
      if (q < nv) {  // warp-uniform
        for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
        if (lane == 0) out[(int64_t)(iv0 + q) * pr + i] = s[q];
      }
    }
  }
}

__global__ void k_bsr_cols(const BsrItem* __restrict__ items, const int64_t* __restrict__ row_off,
                           const int64_t* __restrict__ part_off, const double* __restrict__ base,
                           const double* __restrict__ v, int64_t dim, int nvec, double* __restrict__ cp) {
  const int k = blockIdx.x, iv0 = blockIdx.z * kBsrVG;
  const BsrItem it = items[k];
  if (it.r == it.c) return;
  const int64_t r0 = row_off[it.r], c0 = row_off[it.c];
  const int pr = (int)(row_off[it.r + 1] - r0), pc = (int)(row_off[it.c + 1] - c0);
  const int j = blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= pc) return;
  const int nv = min(kBsrVG, nvec - iv0);
  double s[kBsrVG] = {0.0, 0.0, 0.0, 0.0};
  const double* B = base + it.off + j;
#pragma unroll 4
  for (int i = 0; i < pr; i++) {
    const double bij = B[(int64_t)i * pc];
#pragma unroll
    for (int q = 0; q < kBsrVG; q++)
      if (q < nv) s[q] = fma(bij, v[(int64_t)(iv0 + q) * dim + r0 + i], s[q]);
  }
  double* out = cp + part_off[k] * nvec;  // nvec x p_c
#pragma unroll
  for (int q = 0; q < kBsrVG; q++)
    if (q < nv) out[(int64_t)(iv0 + q) * pc + j] = s[q];
}

// y[cell rows] = the row partials of the items in the cell's block row (item order) + the
// column partials of the off-diagonal items in its block column (item order)
__global__ void k_bsr_reduce(const int32_t* __restrict__ rl_ptr, const int64_t* __restrict__ rl,
                             const int32_t* __restrict__ cl_ptr, const int64_t* __restrict__ cl,
                             const int64_t* __restrict__ row_off, const double* __restrict__ rp,
                             const double* __restrict__ cp, int64_t dim, int nvec, double* __restrict__ y) {
  const int r = blockIdx.x;
  const int64_t r0 = row_off[r];
  const int pr = (int)(row_off[r + 1] - r0);
  for (int e = threadIdx.x; e < pr * nvec; e += blockDim.x) {
    const int iv = e / pr, i = e - iv * pr;
    double s = 0.0;
    for (int q = rl_ptr[r]; q < rl_ptr[r + 1]; q++) s += rp[rl[q] * nvec + (int64_t)iv * pr + i];
    for (int q = cl_ptr[r]; q < cl_ptr[r + 1]; q++) s += cp[cl[q] * nvec + (int64_t)iv * pr + i];
    y[(int64_t)iv * dim + r0 + i] = s;
  }
}

}  // namespace

std::vector<std::vector<CellJob>> level_jobs(const mlk_tree_s* tree, const mlk_basis_s* B) {
  std::vector<std::vector<CellJob>> lv(tree->t + 1);
  for (size_t i = 0; i < B->cells.size(); i++) {
    int q = B->cells[i];
    lv[tree->depth[q]].push_back({tree->begin[q], (int32_t)(tree->end[q] - tree->begin[q]), B->p[q],
                                  B->row_off[i], B->W.p + B->w_off[q]});
  }
  return lv;
}

void apply_wt_dev(Ctx& c, const mlk_tree_s* tree, const mlk_basis_s* B, const double* v, double* a, int nvec) {
  CUDA_CHECK(cudaMemsetAsync(a, 0, sizeof(double) * nvec * tree->n, c.stream));
  auto lv = level_jobs(tree, B);
  TimedLaunch tl(c, "apply_wt");
  for (int dep = tree->t; dep >= 0; dep--) {  // fixed level order: t .. 0
    if (lv[dep].empty()) continue;
    DevBuf<CellJob> dj(lv[dep].size(), c.stream);
    dj.upload(lv[dep]);
    int smax = 0;
    for (auto& j : lv[dep]) smax = std::max(smax, j.s);
    dim3 grid((unsigned)lv[dep].size(), (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, ceil_div(smax, 256))));
    if (nvec == 1) k_apply_wt<1><<<grid, 256, 0, c.stream>>>(dj.p, v, B->dim, a, tree->n, nvec);
    else k_apply_wt<kAwVG><<<grid, 256, 0, c.stream>>>(dj.p, v, B->dim, a, tree->n, nvec);
    check_launch("k_apply_wt");
  }
}

void apply_w_dev(Ctx& c, const mlk_tree_s* tree, const mlk_basis_s* B, const double* b, double* y, int nvec) {
  std::vector<CellJob> all;
  for (auto& l : level_jobs(tree, B))
    for (auto& j : l) all.push_back(j);
  if (all.empty()) return;
  std::vector<WJob> wj;
  std::vector<WRed> red;
  int64_t parts = 0;
  for (int32_t i = 0; i < (int32_t)all.size(); i++) {
    const int32_t s = all[i].s, nch = (int32_t)ceil_div((int64_t)s, (int64_t)kAwChunk);
    if (nch == 1) {
      wj.push_back({i, 0, s, -1});
      continue;
    }
    red.push_back({i, nch, parts});
    for (int32_t ch = 0; ch < nch; ch++) {
      wj.push_back({i, ch * kAwChunk, std::min(s, (ch + 1) * kAwChunk), parts});
      parts += (int64_t)nvec * all[i].p;
    }
  }
  DevBuf<CellJob> dj(all.size(), c.stream);
  dj.upload(all);
  DevBuf<WJob> dw(wj.size(), c.stream);
  dw.upload(wj);
  DevBuf<double> part((size_t)std::max<int64_t>(parts, 1), c.stream);
  TimedLaunch tl(c, "apply_w");
  if (nvec == 1) k_apply_w<1><<<(unsigned)wj.size(), 256, 0, c.stream>>>(dj.p, dw.p, b, tree->n, y, B->dim, nvec, part.p);
  else k_apply_w<kAwVG><<<(unsigned)wj.size(), 256, 0, c.stream>>>(dj.p, dw.p, b, tree->n, y, B->dim, nvec, part.p);
  check_launch("k_apply_w");
  if (!red.empty()) {
    DevBuf<WRed> dr(red.size(), c.stream);
    dr.upload(red);
    k_apply_w_reduce<<<(unsigned)red.size(), 256, 0, c.stream>>>(dj.p, dr.p, part.p, y, B->dim, nvec);
    check_launch("k_apply_w_reduce");
  }
}

// Symmetric C a column partials.  This rank's tiles are I_m = r + R m, m = 0 .. T_r - 1 (cyclic
// over the nranks = R ranks: every rank gets the same mix of long and short triangular tasks, so
// its waves fill like the single-rank run's; contiguous tile ranges of equal cost left rank 0
// with ~T/16 full-length tasks -- less than one wave -- and 30 against 21 ms at cfg4 / 8 ranks).
// Tile I_m holds nvec rows of n - 32 I_m columns starting at column 32 I_m (its 4 warps already
// summed in order by the tile kernel), at offset nvec sum_{m' < m} (n - 32 I_m').  Two
// fixed-order levels: tmp[l][c][j] = sum over the tiles of chunk c (kColChunk tiles), then
// b[l][j] += sum over chunks c in order.  Deterministic; R = 1 is the plain tile order.
constexpr int kColChunk = 64;
__device__ __forceinline__ int64_t colpart_off(int64_t m, int64_t r, int64_t R, int64_t n, int nvec) {
  return (int64_t)nvec * (m * n - 32 * (r * m + R * (m * (m - 1) / 2)));
}

__global__ void k_colpart_chunks(const double* __restrict__ colpart, int64_t r, int64_t R, int64_t Tr, int64_t n,
                                 int nvec, int nchunks, double* __restrict__ tmp) {
  const int64_t j = 32 * r + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c = blockIdx.y, l = blockIdx.z;
  if (j >= n) return;
  const int64_t m0 = (int64_t)c * kColChunk;
  // tiles that reach column j: 32 I_m <= j
  const int64_t m1 = std::min<int64_t>({Tr, m0 + kColChunk, (j / 32 - r) / R + 1});
  double s = 0.0;
  for (int64_t m = m0; m < m1; m++) {
    const int64_t I = r + R * m;
    const int64_t w = n - 32 * I;
    s += colpart[colpart_off(m, r, R, n, nvec) + (int64_t)l * w + (j - 32 * I)];
  }
  tmp[((int64_t)l * nchunks + c) * n + j] = s;
}

__global__ void k_colpart_final(const double* __restrict__ tmp, int64_t j0, int64_t n, int nchunks,
                                double* __restrict__ b) {
  const int64_t j = j0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (j >= n) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; c++) s += tmp[((int64_t)l * nchunks + c) * n + j];
  b[(int64_t)l * n + j] += s;
}

// b = C a for this rank's rows (others zero); a, b device, nvec x n.  Symmetric kernels (each
// covariance entry evaluated once for the pair (i, j), i <= j) when their column partials fit:
// up to 4 vectors the lane-local DFMA variant of tile.cu (nvec x n^2 / 64 doubles),
// 5 or more the DMMA kernel of covsym.cu (nvec x n^2 / 128 doubles per group of 16 vectors).
void cov_matvec_dev(Ctx& c, const mlk_tree_s* tree, const mlk_kernel& k, const double* a, double* b, int nvec) {
  const int64_t n = tree->n;
  CUDA_CHECK(cudaMemsetAsync(b, 0, sizeof(double) * nvec * n, c.stream));
  // rows of this rank: 32-row tiles, cyclic over the ranks for the symmetric kernel (tile I belongs
  // to rank I mod nranks), a contiguous range for the row-panel kernel
  const int64_t tiles = ceil_div(n, 32);
  const int64_t R = c.nranks;
  auto sym_count = [&](int64_t r) { return tiles > r ? (tiles - r + R - 1) / R : (int64_t)0; };
  auto sym_partials = [&](int64_t r) {
    int64_t s = 0;
    for (int64_t m = 0; m < sym_count(r); m++) s += (int64_t)nvec * (n - 32 * (r + R * m));
    return s;
  };
  // The symmetric and the row-panel kernels split the rows differently, so every rank must take
  // the same branch: the choice depends only on (n, nvec, nranks) and the device's TOTAL memory
  // (identical across the ranks of one box), never on this rank's free memory.  The symmetric
  // kernel's column partials of the largest rank share must fit a quarter of the device.
  const bool nosym = std::getenv("MLK_NO_SYM_MATVEC") != nullptr;
  // (MLK_SYM_MIN_NVEC: A/B switch for the vector count from which covsym.cu takes over)
  const char* smn = std::getenv("MLK_SYM_MIN_NVEC");
  if (nvec >= (smn ? std::atoi(smn) : 5) && !nosym) {
    // 5 or more vectors: the symmetric kernel with DMMA contractions (covsym.cu), tasks of
    // kSymRows rows split by their triangular costs n - kSymRows I (rank-invariant); it bounds
    // its column partials by processing the tasks in batches
    const int64_t T = ceil_div(n, (int64_t)kSymRows);
    auto cost_before = [&](int64_t I) { return (double)I * n - 0.5 * kSymRows * (double)I * (I - 1); };
    auto range = [&](int r, int64_t& a0, int64_t& a1) {
      const double total = cost_before(T);
      a0 = 0;
      while (a0 < T && cost_before(a0 + 1) <= total * r / c.nranks) a0++;
      a1 = a0;
      while (a1 < T && cost_before(a1 + 1) <= total * (r + 1) / c.nranks) a1++;
      if (r == c.nranks - 1) a1 = T;
    };
    int64_t a0, a1;
    range(c.rank, a0, a1);
    cov_matvec_sym(c, tree, make_kernel_params(k), a, b, nvec, a0, a1);
    return;
  }
  bool sym = nvec <= 4 && !nosym;
  if (sym) {
    int64_t worst = 0;
    for (int r = 0; r < c.nranks; r++) worst = std::max(worst, sym_partials(r));
    sym = worst * (int64_t)sizeof(double) <= device_total_bytes(c.device) / 4;
  }
  const int nv = nvec == 1 ? 1 : nvec == 2 ? 2 : 4;
  std::vector<TileUnit> units;
  if (sym) {
    const int64_t r = c.rank, Tr = sym_count(r);
    if (Tr == 0) return;
    const int64_t cp = sym_partials(r);
    int64_t off = 0;
    for (int64_t m = 0; m < Tr; m++) {
      const int64_t row = 32 * (r + R * m);
      make_tile_units(units, row, (int32_t)std::min<int64_t>(32, n - row), row, (int32_t)(n - row), a, n, nvec,
                      b + row, n, 1, tree->d_pad);
      TileUnit& u = units.back();
      u.rq = -nv;
      u.w_col0 = row;
      u.w_cols = n;
      u.cp_off = off;
      off += (int64_t)nvec * (n - row);
    }
    double* colpart = c.scratch("sym4_colpart", (size_t)cp);
    const int nchunks = (int)ceil_div(Tr, (int64_t)kColChunk);
    double* tmp = c.scratch("sym4_tmp", (size_t)nvec * nchunks * n);
    run_tile_contract(c, tree, make_kernel_params(k), units, "cov_matvec_tile", colpart);
    TimedLaunch tl(c, "cov_matvec_colsum");
    dim3 g1((unsigned)ceil_div(n - 32 * r, 256), (unsigned)nchunks, (unsigned)nvec);
    k_colpart_chunks<<<g1, 256, 0, c.stream>>>(colpart, r, R, Tr, n, nvec, nchunks, tmp);
    check_launch("k_colpart_chunks");
    dim3 g2((unsigned)ceil_div(n - 32 * r, 256), (unsigned)nvec);
    k_colpart_final<<<g2, 256, 0, c.stream>>>(tmp, 32 * r, n, nchunks, b);
    check_launch("k_colpart_final");
    return;
  }
  const int64_t t0 = tiles * c.rank / c.nranks, t1 = tiles * (c.rank + 1) / c.nranks;
  if (t1 <= t0) return;
  const int64_t r0 = t0 * 32, r1 = std::min<int64_t>(n, t1 * 32);
  // rows r0..r1 as an a range; b range = all points; W_b = the vectors a (nvec x n)
  make_tile_units(units, r0, (int32_t)(r1 - r0), 0, (int32_t)n, a, n, nvec, b + r0, n, 1, tree->d_pad);
  // up to 4 vectors: lane-local DFMA contraction instead of 8-column DMMAs (tile.cu, NV)
  if (nvec <= 4)
    for (auto& u : units) u.rq = -nv;
  run_tile_contract(c, tree, make_kernel_params(k), units, "cov_matvec_tile");
}

// y = (this rank's items of) C~_W v, v / y device nvec x dim
void bsr_matvec_dev(Ctx& c, const mlk_basis_s* basis, const mlk_cw_s* cw, const double* v, double* y, int nvec) {
  const int64_t dim = basis->dim;
  const int64_t nb = cw->n_blocks;
  std::vector<BsrItem> items;
  const double* base = cw->vals();
  if (c.nranks == 1) {
    for (int64_t k = 0; k < nb; k++) items.push_back({cw->brow[k], cw->bcol[k], cw->val_off[k]});
  } else if (cw->complete) {
    for (int64_t k = 0; k < nb; k++)
      if (cw->owner[k] == c.rank) items.push_back({cw->brow[k], cw->bcol[k], cw->val_off[k]});
  } else {
    base = cw->shard.p;
    for (int64_t k = 0; k < nb; k++)
      for (int64_t p = cw->piece_ptr[k]; p < cw->piece_ptr[k + 1]; p++)
        if (cw->piece_owner[p] == c.rank) items.push_back({cw->brow[k], cw->bcol[k], cw->piece_off[p]});
  }
  if (items.empty()) {
    CUDA_CHECK(cudaMemsetAsync(y, 0, sizeof(double) * nvec * dim, c.stream));
    return;
  }
  const int64_t ni = (int64_t)items.size();
  const int nc = cw->n_cells;
  // partial offsets (per vector): p_row per item, p_col per off-diagonal item; per cell the
  // lists of row partials (items in its block row) and column partials (its block column)
  std::vector<int64_t> rpo(ni), cpo(ni);
  std::vector<int32_t> rl_ptr(nc + 1, 0), cl_ptr(nc + 1, 0);
  int64_t rtot = 0, ctot = 0;
  int pcmax = 1;
  for (int64_t k = 0; k < ni; k++) {
    const int r = items[k].r, cc = items[k].c;
    const int pr = (int)(basis->row_off[r + 1] - basis->row_off[r]);
    const int pc = (int)(basis->row_off[cc + 1] - basis->row_off[cc]);
    rpo[k] = rtot;
    rtot += pr;
    rl_ptr[r + 1]++;
    cpo[k] = ctot;
    if (r != cc) {
      ctot += pc;
      cl_ptr[cc + 1]++;
    }
    pcmax = std::max(pcmax, pc);
  }
  for (int i = 0; i < nc; i++) {
    rl_ptr[i + 1] += rl_ptr[i];
    cl_ptr[i + 1] += cl_ptr[i];
  }
  std::vector<int64_t> rl(std::max<int32_t>(rl_ptr[nc], 1)), cl(std::max<int32_t>(cl_ptr[nc], 1));
  {
    std::vector<int32_t> rf(rl_ptr.begin(), rl_ptr.end() - 1), cf(cl_ptr.begin(), cl_ptr.end() - 1);
    for (int64_t k = 0; k < ni; k++) {
      rl[rf[items[k].r]++] = rpo[k];
      if (items[k].r != items[k].c) cl[cf[items[k].c]++] = cpo[k];
    }
  }
  DevBuf<BsrItem> it_d(ni, c.stream);
  it_d.upload(items);
  DevBuf<int64_t> ro(basis->row_off.size(), c.stream), rpo_d(ni, c.stream), cpo_d(ni, c.stream);
  ro.upload(basis->row_off);
  rpo_d.upload(rpo);
  cpo_d.upload(cpo);
  DevBuf<int32_t> rlp_d(nc + 1, c.stream), clp_d(nc + 1, c.stream);
  rlp_d.upload(rl_ptr);
  clp_d.upload(cl_ptr);
  DevBuf<int64_t> rl_d(rl.size(), c.stream), cl_d(cl.size(), c.stream);
  rl_d.upload(rl);
  cl_d.upload(cl);
  DevBuf<double> rp((size_t)std::max<int64_t>(rtot * nvec, 1), c.stream);
  DevBuf<double> cp((size_t)std::max<int64_t>(ctot * nvec, 1), c.stream);
  TimedLaunch tl(c, "bsr_matvec");
  const unsigned vg = (unsigned)ceil_div(nvec, kBsrVG);
  k_bsr_rows<<<dim3((unsigned)ni, vg), 256, 0, c.stream>>>(it_d.p, ro.p, rpo_d.p, base, v, dim, nvec, rp.p);
  check_launch("k_bsr_rows");
  k_bsr_cols<<<dim3((unsigned)ni, (unsigned)ceil_div(pcmax, 256), vg), 256, 0, c.stream>>>(it_d.p, ro.p, cpo_d.p,
                                                                                            base, v, dim, nvec, cp.p);
  check_launch("k_bsr_cols");
  k_bsr_reduce<<<(unsigned)nc, 256, 0, c.stream>>>(rlp_d.p, rl_d.p, clp_d.p, cl_d.p, ro.p, rp.p, cp.p, dim, nvec, y);
  check_launch("k_bsr_reduce");
}

void check_kernel(const mlk_kernel* k) {
  MLK_REQUIRE(k != nullptr, "kernel is NULL");
  MLK_REQUIRE(k->family >= MLK_MATERN_12 && k->family <= MLK_MATERN_NU, "unknown covariance family");
  MLK_REQUIRE(k->rho > 0 && k->sigma2 > 0 && k->nugget >= 0, "need rho > 0, sigma2 > 0, nugget >= 0");
  MLK_REQUIRE(k->family != MLK_MATERN_NU || (k->nu > 0 && k->nu <= 50), "MLK_MATERN_NU needs 0 < nu <= 50");
}

}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_apply_wt(mlk_ctx ctx, mlk_basis basis, const double* v, double* a, int32_t nvec) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && basis && v && a, "NULL argument");
  MLK_REQUIRE(nvec >= 1, "need nvec >= 1");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  const mlk_tree_s* tree = basis->tree;
  DevIn<double> vin(v, (size_t)nvec * basis->dim, c.stream);
  DevOut<double> aout(a, (size_t)nvec * tree->n, c.stream);
  basis_wait(c, basis);
  apply_wt_dev(c, tree, basis, vin.p, aout.p, nvec);
  aout.finish();
  MLK_API_END
}

mlk_status mlk_apply_w(mlk_ctx ctx, mlk_basis basis, const double* b, double* y, int32_t nvec) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && basis && b && y, "NULL argument");
  MLK_REQUIRE(nvec >= 1, "need nvec >= 1");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  const mlk_tree_s* tree = basis->tree;
  DevIn<double> bin(b, (size_t)nvec * tree->n, c.stream);
  DevOut<double> yout(y, (size_t)nvec * basis->dim, c.stream);
  basis_wait(c, basis);
  apply_w_dev(c, tree, basis, bin.p, yout.p, nvec);
  yout.finish();
  MLK_API_END
}

mlk_status mlk_cov_matvec(mlk_ctx ctx, mlk_tree tree, const mlk_kernel* kernel, const double* a, double* b,
                          int32_t nvec) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && tree && a && b, "NULL argument");
  check_kernel(kernel);
  MLK_REQUIRE(nvec >= 1 && nvec <= 64, "need 1 <= nvec <= 64");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  DevIn<double> ain(a, (size_t)nvec * tree->n, c.stream);
  DevOut<double> bout(b, (size_t)nvec * tree->n, c.stream);
  cov_matvec_dev(c, tree, *kernel, ain.p, bout.p, nvec);
  bout.finish();
  MLK_API_END
}

mlk_status mlk_cw_matvec(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel, mlk_cw cw,
                         int32_t mode, const double* v, double* y, int32_t nvec) {
  MLK_API_BEGIN
  MLK_REQUIRE(ctx && tree && basis && v && y, "NULL argument");
  MLK_REQUIRE(basis->tree == tree, "basis was built for another tree");
  MLK_REQUIRE(mode == MLK_MATVEC_EXACT || mode == MLK_MATVEC_BSR, "unknown matvec mode");
  MLK_REQUIRE(nvec >= 1 && nvec <= 64, "need 1 <= nvec <= 64");
  Ctx& c = ctx->c;
  CUDA_CHECK(cudaSetDevice(c.device));
  const int64_t dim = basis->dim;
  DevIn<double> vin(v, (size_t)nvec * dim, c.stream);
  DevOut<double> yout(y, (size_t)nvec * dim, c.stream);
  if (mode == MLK_MATVEC_EXACT) {
    check_kernel(kernel);
    DevBuf<double> a((size_t)nvec * tree->n, c.stream), b((size_t)nvec * tree->n, c.stream);
    basis_wait(c, basis);
    apply_wt_dev(c, tree, basis, vin.p, a.p, nvec);
    cov_matvec_dev(c, tree, *kernel, a.p, b.p, nvec);
    apply_w_dev(c, tree, basis, b.p, yout.p, nvec);
    comm_allreduce_sum(c, yout.p, (int64_t)nvec * dim);  // no-op without a communicator
    yout.finish();
  } else {
    MLK_REQUIRE(cw != nullptr, "BSR mode needs the assembled matrix");
    MLK_REQUIRE(cw->n_cells == (int32_t)basis->cells.size(), "cw does not match the basis");
    MLK_REQUIRE(cw->nranks == c.nranks && cw->rank == c.rank, "cw was assembled for another rank layout");
    bsr_matvec_dev(c, basis, cw, vin.p, yout.p, nvec);
    comm_allreduce_sum(c, yout.p, (int64_t)nvec * dim);  // no-op without a communicator
    yout.finish();
  }
  MLK_API_END
}

}  // extern "C"
