// Handle types shared by the translation units of libmlk, and the ABI try/catch wrapper.
#pragma once
#include <array>
#include <map>
#include <mutex>
#include <new>

#include "common.cuh"

#define MLK_API_BEGIN try {
#define MLK_API_END                                                        \
  }                                                                        \
  catch (const ::mlk::Error& e) {                                          \
    ::mlk::set_last_error(e.what());                                       \
    return e.status;                                                       \
  }                                                                        \
  catch (const std::bad_alloc&) {                                          \
    ::mlk::set_last_error("host allocation failed");                       \
    return MLK_ERR_OUT_OF_MEMORY;                                          \
  }                                                                        \
  catch (const std::exception& e) {                                        \
    ::mlk::set_last_error(e.what());                                       \
    return MLK_ERR_CUDA;                                                   \
  }                                                                        \
  return MLK_OK;
// the status of a nested ABI call, after the caller's own checks
#define MLK_API_END_CALL(expr)                                             \
  }                                                                        \
  catch (const ::mlk::Error& e) {                                          \
    ::mlk::set_last_error(e.what());                                       \
    return e.status;                                                       \
  }                                                                        \
  return (expr);

struct mlk_basis_s;
struct mlk_tree_s;
namespace mlk {
void partition_lpt(const double* cost, int64_t n, int nranks, int32_t* owner);
void shard_plan(const int64_t* val_off, const int32_t* owner, int64_t n, int nranks, int64_t* shard_off,
                int64_t* shard_len);

// make the context stream wait until the basis's asynchronous merge levels have completed;
// the first call also synchronises and reports a rank-deficient merge (MLK_ERR_RANK_DEFICIENT)
void basis_wait(Ctx& c, const mlk_basis_s* B);
void basis_sync(const mlk_basis_s* B);

// The three steps of C_W v (matvec.cu), device vectors, nvec x n (point space, tree order) or
// nvec x dim (C_W space): a = W^T v, b = C a (this rank's rows), y = W b.
void apply_wt_dev(Ctx& c, const mlk_tree_s* tree, const mlk_basis_s* B, const double* v, double* a, int nvec);
void cov_matvec_dev(Ctx& c, const mlk_tree_s* tree, const mlk_kernel& k, const double* a, double* b, int nvec);
void apply_w_dev(Ctx& c, const mlk_tree_s* tree, const mlk_basis_s* B, const double* b, double* y, int nvec);
void check_kernel(const mlk_kernel* k);

// NCCL collectives on the context's communicator (comm.cu)
void* comm_create(int nranks, int rank, const void* unique_id);
void comm_destroy(void* comm);
void comm_allreduce_sum(Ctx& c, double* x, int64_t count);

// padded coordinate count for the DMMA k = 4 Gram steps
inline int pad4(int d) { return (d + 3) / 4 * 4; }
}  // namespace mlk

// Tree (heap-numbered nodes).  Shape arrays are host-side (they depend only on n and the
// leaf size); the permutation, thresholds and tree-ordered points live on the device.
struct mlk_tree_s {
  int device = 0;
  int64_t n = 0;
  int d = 0, d_pad = 0, leaf = 0, kind = 0, t = 0, n_nodes = 0;
  std::vector<int8_t> state;      // -1 empty, 0 internal, 1 leaf
  std::vector<int64_t> begin, end;
  std::vector<int32_t> depth;
  std::vector<double> thr;        // NaN unless internal
  std::vector<double> dir;        // n_nodes x d
  std::vector<int64_t> perm;      // host copy
  mlk::DevBuf<int32_t> perm_d;    // tree position -> original index
  mlk::DevBuf<double> X;          // n x d, original order
  mlk::DevBuf<double> Xt;         // n x d_pad, tree order, zero padded
  mlk::DevBuf<double> norm2;      // |x|^2 in tree order
  mlk::DevBuf<double> thr_d;      // n_nodes
  mlk::DevBuf<double> dir_d;      // n_nodes x d
  // the fused tile kernels' augmented, pre-scaled coordinates Pa, Pb (tile.cu tile_aug_get),
  // cached for the last coordinate scale: formed once per assembly / product, not per launch
  mutable mlk::DevBuf<double> aug;
  mutable double aug_scale = 0.0;
  mutable int aug_dpa = 0;
};

// Basis blocks per heap node; cells (nodes with >= 1 wavelet) listed in C_W order.
struct mlk_basis_s {
  int device = 0;
  int M = 0, w = 0;
  int64_t dim = 0;
  const mlk_tree_s* tree = nullptr;
  std::vector<int32_t> cells;      // C_W order
  std::vector<int64_t> row_off;    // n_cells + 1
  std::vector<int32_t> p;          // wavelets per node (n_nodes)
  std::vector<int32_t> cell_pos;   // node -> position in cells, or -1
  std::vector<int64_t> w_off;      // node -> offset of W block (doubles) in W
  std::vector<int64_t> phi_off;    // node -> offset of Phi block in Phi
  mlk::DevBuf<double> W;           // all W blocks, C_W order, each p x |node| row-major
  mlk::DevBuf<double> Phi;         // all Phi blocks, M x |node| row-major
  // merge factors: for every internal node q the complete Q (2M x 2M, row-major) of the QR of
  // [R_L; R_R] at Qm + q_off[q] (Phi_q = Q[:, :M]^T (Phi_L (+) Phi_R), W_q = Q[:, M:]^T (...));
  // kept when they total <= 1 GB (not cfg5: 29 GB) -- the nested assembly transfers with them
  mlk::DevBuf<double> Qm;
  std::vector<int64_t> q_off;      // node -> offset in Qm, or -1
  // the merge levels run asynchronously on the context's auxiliary stream; `ready` marks
  // their completion and consumers wait on it (mlk::basis_wait), checking merge_flag once
  cudaEvent_t ready = nullptr;
  mlk::DevBuf<int> merge_flag;
  mutable bool ready_checked = false;
  bool keep_deficient = false;     // MLK_BASIS_KEEP_DEFICIENT
  bool phi_dropped = false;        // only L = Phi_root retained (phi_off[0] = 0, others -1)
};

struct mlk_cw_s {
  int device = 0, nranks = 1, rank = 0;
  int32_t n_cells = 0;
  int64_t n_blocks = 0, nnz = 0;
  std::vector<int32_t> brow_ptr, bcol, brow, owner;
  std::vector<int64_t> val_off;
  // pieces: block k = sum of pieces piece_ptr[k]..piece_ptr[k+1] (one per row chunk), piece p
  // stored in rank piece_owner[p]'s shard at piece_off[p]
  std::vector<int64_t> piece_ptr, piece_off;
  std::vector<int32_t> piece_owner, reduce_blocks;
  int64_t shard_len = 0, max_shard_len = 0;
  bool complete = false;           // values hold every block (nranks == 1 or unpacked)
  double entries = 0, flops = 0, own_entries = 0, own_flops = 0;
  double f_gram = 0, f_c1 = 0, f_c2 = 0, f_tr = 0;  // f_tr: nested-assembly transfers
  double f_nested_k5a = 0;         // Gram + first contraction of the nested leaf pass (in f_gram, f_c1)
  bool nested = false;             // internal cells' V_b by the nested evaluation
  mlk::DevBuf<double> values;      // nnz on the device (nranks == 1: at assembly; else at unpack)
  double* hvals = nullptr;         // MLK_VALUES_HOST: nnz in mapped pinned host memory instead
  double* vals() const { return hvals ? hvals : values.p; }
  mlk::DevBuf<double> shard;       // this rank's packed values (nranks > 1)
  // device structure for the BSR matvec
  mlk::DevBuf<int32_t> brow_d, bcol_d, owner_d;
  mlk::DevBuf<int64_t> val_off_d, piece_ptr_d, piece_off_d;
  mlk::DevBuf<int32_t> piece_owner_d, reduce_d;
  mlk::DevBuf<int32_t> csc_ptr_d, csc_blk_d;   // blocks (r, c), r != c, grouped by column c
};

namespace mlk {
// free device memory at the context's first query less the live handles since (ctx.cu): no
// driver call after the first -- cudaMemGetInfo stalls under NVML polling
int64_t ctx_avail_bytes(Ctx& c);
// nested-assembly transfers of one tree level (nested.cu): jobs {[S_cL S_cR], Q_c, S_c (or
// nullptr), V_c}, rows x (n_nodes M) buffers with row stride ld, and per job a device flag per
// 64-row block (V_c needed there; nullptr: everywhere); transfer_kernel_ok(M): 2M <= 144
bool transfer_kernel_ok(int M);
void transfer_level(Ctx& c, const std::vector<std::array<const double*, 4>>& jobs,
                    const std::vector<const uint8_t*>& vflags, int M, int64_t rows, int64_t ld);
// all-gather of the piece shards into the values (nranks > 1, library communicator; comm.cu)
void gather_values(Ctx& c, mlk_cw_s* cw, const double* full);
void gather_plan(int64_t nb, const int64_t* piece_ptr, const int64_t* piece_off, const int32_t* piece_owner,
                 const int64_t* block_len, int nranks, int64_t budget, std::vector<int64_t>& group_ptr,
                 std::vector<int64_t>& group_lo, std::vector<int64_t>& group_count);
// Row-major NN product C = A B (m x k times k x n); if trans_c, C^T is stored (C[j][i]).
// If accumulate, the product is added to C (fixed order: exactly one job per C tile).
struct GemmDesc {
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int32_t m, n, k;
  int32_t trans_c;
  int64_t diag = -1;  // >= 0: store [i + diag == j] - (A B)[i][j] instead of (A B)[i][j]
  int32_t sub = 0;    // 1: C -= A B (read-modify-write; not with diag)
  int32_t trans_a = 0;  // 1: A is stored k x m (row-major, lda >= m) and read transposed
};
// Launch all products on the context stream with FP64 DMMA tiles (64 x 64, 72 x 72 or
// 64 x 32, by padded volume; k steps of 16); large k
// is split into fixed chunks whose partial tiles are reduced in chunk order (deterministic).
void gemm_batched(Ctx& c, const std::vector<GemmDesc>& descs, const char* name);
}  // namespace mlk
