// The fused tile-and-contract kernel (K5a): for a cell pair (a, b) it computes
//     U[r, l] = sum_y C(x_{a,r}, x_{b,y}) W_b[l, y]
// with the covariance tile generated in registers -- Gram product x.y on FP64 DMMA, the
// Gram identity r^2 = |x|^2 + |y|^2 - 2 x.y, the Matern/Gaussian closed form -- and
// contracted immediately on FP64 DMMA; C never reaches memory.  It serves the assembly
// (W_b = wavelet block of the contracted-first cell) and the exact product b = C a
// (W_b = the vectors a).
#pragma once
#include <cuda.h>

#include "api.cuh"

namespace mlk {

struct TileUnit {
  int64_t a_begin, b_begin;  // first tree position of the a / b point ranges
  int32_t s_a, s_b;          // points in the ranges
  int32_t row0;              // first a row of the range (tasks cover row0 + 32 i)
  int32_t n_tasks;           // 32-row CTA tasks of the range: ceil((s_a - row0) / 32)
  int32_t c0, qc;            // first column of W_b rows handled, and how many (<= 8 RQ)
  int32_t p_b;               // rows of W_b
  int32_t trans;             // 0: U[r * ldu + c0 + l]; 1: U[(c0 + l) * ldu + r]
  int32_t rq;                // instantiation class (columns padded to 8 rq); -NV: DFMA contraction of NV <= 4 columns
  const double* Wb;          // W_b[l][y] at Wb + l * ldw + y
  int64_t ldw;
  double* U;                 // base of this pair's U
  int64_t ldu;
  double cost;               // for scheduling
  int32_t bulk;              // stages filled by 2-D TMA (else 8-byte cp.async): W_b 16-byte aligned, ldw even
  int32_t xmap, wmap;        // tensor maps of the b rows and of W_b (run_tile_contract)
  int32_t nr;                // columns 8 rq .. 8 rq + nr - 1 of the chunk are done with DFMAs
  int32_t wrows;             // W_b rows staged per stage (8 rq + nr)
  int64_t w_col0;            // W_b column of point b_begin (0, except the symmetric C a tasks)
  int64_t w_cols;            // columns of W_b addressable by the tensor map (s_b by default)
  int64_t cp_off;            // symmetric C a: offset of this task's column partials (NV x s_b)
  int32_t seg;               // > 0: the b range is a run of segments of seg points (the nested
                             // assembly's leaves), each with its own output: U + k seg_off for
                             // segment k (the accumulators are written and cleared at every
                             // segment boundary; seg is a multiple of 8)
  int64_t seg_off;
};

struct KernelParams {
  int32_t family;
  double c1;        // sqrt(2 nu) / rho (Matern) or 1 / rho^2 (Gaussian)
  double sigma2;
  double nugget;
  double same_val;  // 1 + nugget / sigma2: the correlation of a site with itself (R18)
  double scale;     // coordinate pre-scale of the augmented Gram product (c1, or 1 / rho)
  // MLK_MATERN_NU (tile.cu matern_nu): nu, norm = 2^(1 - nu) / Gamma(nu), the trapezoid step
  // scale h0, and for the small-z series g1m = Gamma(1 - nu), rg1p = 1 / Gamma(1 + nu) (used
  // only when nu is at least 0.01 away from an integer: series != 0)
  double nu, norm, h0, g1m, rg1p;
  int32_t series;
};

KernelParams make_kernel_params(const mlk_kernel& k);
// column-class instantiations available to the planner
int tile_rq_class(int qc);  // smallest available rq with 8 rq >= qc
constexpr int kTileMaxRQ = 24;
// remainder columns that go to lane-local DFMA instead of padding to the next 8-column group.
// A DFMA column costs 2 x 2.25 pipe cycles per 64 entries against 4 per column of a padded DMMA
// group, which suggests up to 7; measured on cfg3 (p = 21), 16 + 5 DFMA ran 4 % slower than
// 24 padded (286 vs 274 ms, r01g vs r01f: register pressure and the broadcast W loads), so 3
constexpr int kTileMaxNR = 3;
constexpr int kTileMaxNRWide = 3;
// (5 DFMA columns for the two-group class -- cfg3's p = 21 as 16 + 5 instead of 24 padded --
// measured 3 % slower than the padding on cfg3's K5a, r02c)
__host__ __device__ constexpr int tile_max_nr(int rq) { return rq <= 4 ? kTileMaxNR : kTileMaxNRWide; }
// Run all units (any mix of rq classes) on the context stream.  colpart != nullptr selects the
// symmetric C a kernel (units with rq = -NV; see tile.cu).
void run_tile_contract(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, std::vector<TileUnit>& units,
                       const char* name, double* colpart = nullptr);
// Split a (pair, output) into units: rows in blocks of 32, W_b rows in balanced chunks.
void make_tile_units(std::vector<TileUnit>& out, int64_t a_begin, int32_t s_a, int64_t b_begin, int32_t s_b,
                     const double* Wb, int64_t ldw, int32_t p_b, double* U, int64_t ldu, int32_t trans, int dp);

// Layout of the augmented, pre-scaled coordinates Pa, Pb (n x dpa each, one buffer) of the Gram
// product (tile.cu k_tile_aug): dk Gram columns, dpa doubles per row, sdp = shared-memory row
// stride.  tile_aug_get returns Pa (Pb = Pa + n dpa), formed on the context stream unless the
// tree's cache already holds them for this scale.
struct AugCoords {
  int dpa = 0, dk = 0, sdp = 0;
};
void tile_aug_layout(int d, AugCoords& a);
const double* tile_aug_get(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, const AugCoords& a);
// row-major FP64 matrix (rows x cols, row stride ld elements) read by TMA in boxes of
// box_rows x box_cols (out-of-range elements zero-filled)
CUtensorMap make_map_2d(const double* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows,
                        uint32_t box_cols);
// Symmetric b = C a for 5 or more vectors (covsym.cu): tasks [t0, t1) of kSymRows rows; a and b
// device, nvec x n; b holds this rank's contributions (the caller sums the ranks).
#ifndef MLK_SYM_RG
#define MLK_SYM_RG 4  // row groups of 8 per task (A/B switch, tools/build_variant.py)
#endif
constexpr int kSymRows = 8 * MLK_SYM_RG;
int64_t cov_sym_partials(int64_t n, int nvec, int64_t t0, int64_t t1);  // doubles of column partials
void cov_matvec_sym(Ctx& c, const mlk_tree_s* tree, const KernelParams& kp, const double* a, double* b, int nvec,
                    int64_t t0, int64_t t1);

}  // namespace mlk
