/*
 * mlk.h -- C ABI of the B200-native multi-level covariance library (libmlk.so).
 *
 * The library computes the hot path of multi-level kriging (J. E. Castrillon-Candas,
 * "High Dimensional Multi-Level Covariance Estimation and Kriging", arXiv:1701.00285):
 * the multi-level covariance matrix C_W = W C(theta) W^T and
 * the products C_W v.  "P:n" cites line n of the paper's LaTeX source
 * (PAPER.md); readings of ambiguous passages are numbered R1.. in DESIGN.md.
 *
 * Conventions common to every call
 *  - Every call returns mlk_status; no C++ exception crosses the ABI.  On a non-OK status
 *    mlk_last_error() returns a thread-local description.  Handles passed to a failing call
 *    stay valid; output handles are left NULL.
 *  - Arguments are validated before any launch (MLK_ERR_INVALID_ARG).
 *  - Pointer arguments documented "host or device" are classified with
 *    cudaPointerGetAttributes: device (or managed) memory of the context's device is read
 *    in place, anything else is treated as host memory and staged through the context's
 *    stream.  Output pointers follow the same rule.
 *  - Handles own all device memory they allocate (stream-ordered on the context stream).
 *    Export calls copy into caller memory; passing NULL for an output skips it.
 *  - A context is single-threaded; calls are stream-ordered on the context's stream and
 *    return after the work they enqueue has completed unless stated otherwise.
 *  - Multi-GPU (nranks > 1, S§8(e)): one process per GPU.  Points and basis are replicated
 *    (every rank builds them identically); the assembly's work units and the C_W v rows are
 *    split across ranks.  The only collectives are an all-gather of the BSR pieces after the
 *    assembly and a sum-allreduce of C_W v.  A context created WITH an NCCL unique id
 *    (mlk_ctx_create) issues them itself on its own communicator, over NVLink/NVSwitch:
 *    mlk_assemble_cw(gather = MLK_GATHER_DEVICE / _HOST) returns the complete matrix on every
 *    rank and mlk_cw_matvec returns the summed y.  A context created WITHOUT one leaves them
 *    to the caller: mlk_cw_pack / caller all-gather / mlk_cw_unpack, and a caller allreduce of
 *    mlk_cw_matvec's partial y.  Every rank must make the same calls with the same arguments
 *    (the collective calls are then collective).
 *  - Point-space vectors are in TREE ORDER: entry k belongs to original observation perm[k]
 *    (mlk_tree_export).  C_W-space vectors are in C_W row order (levels t..0, heap order
 *    within a level, reading R11).
 *  - All floating point is IEEE binary64.
 */
#ifndef MLK_H_
#define MLK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MLK_OK = 0,
  MLK_ERR_INVALID_ARG = 1,      /* a size, enum or pointer argument is out of range          */
  MLK_ERR_DUPLICATE_POINTS = 2, /* two observation sites coincide (P:167-169 needs x_i != x_j) */
  MLK_ERR_RANK_DEFICIENT = 3,   /* a moment matrix has rank < M (reading R9)                  */
  MLK_ERR_OUT_OF_MEMORY = 4,    /* a device allocation failed                                 */
  MLK_ERR_CUDA = 5,             /* any other CUDA runtime error                               */
  MLK_ERR_UNSUPPORTED = 6,      /* valid request this build does not implement                */
  MLK_ERR_NCCL = 7              /* libnccl.so.2 missing or an NCCL call failed                */
} mlk_status;

/* Text for the last non-OK status returned on this thread ("" if none). */
const char* mlk_last_error(void);
/* Library version string. */
const char* mlk_version(void);
/* Number of CUDA kernels this process has launched through the library so far. */
int64_t mlk_launch_count(void);

typedef struct mlk_ctx_s* mlk_ctx;
typedef struct mlk_tree_s* mlk_tree;
typedef struct mlk_basis_s* mlk_basis;
typedef struct mlk_cw_s* mlk_cw;

/* ------------------------------------------------------------------------------------------
 * Context.  device: CUDA ordinal.  nranks >= 1, 0 <= rank < nranks.
 *  nccl_unique_id  NULL, or the 128-byte ncclUniqueId (mlk_nccl_unique_id on one rank,
 *                  distributed by the caller, e.g. a torch.distributed broadcast): the context
 *                  then creates and owns an NCCL communicator of nranks ranks
 *                  (ncclCommInitRank -- collective over the ranks) and issues the path's
 *                  collectives itself.  NCCL is loaded at run time (libnccl.so.2);
 *                  MLK_ERR_NCCL if it is missing or the initialisation fails.
 *  cuda_stream     a cudaStream_t the library launches on (NULL: the library creates and owns
 *                  one).  Collectives run on the same stream.
 */
mlk_status mlk_ctx_create(int device, int nranks, int rank, const void* nccl_unique_id, void* cuda_stream,
                          mlk_ctx* out);
/* A fresh ncclUniqueId (128 bytes into id) for mlk_ctx_create; host only, call on one rank. */
mlk_status mlk_nccl_unique_id(void* id);
void mlk_ctx_destroy(mlk_ctx ctx); /* NULL-safe */
/* The cudaStream_t the context launches on. */
void* mlk_ctx_stream(mlk_ctx ctx);
/* Per-kernel timing with CUDA events recorded on the context stream around every launch
 * (enable != 0).  Stats accumulate until mlk_ctx_reset_stats. */
mlk_status mlk_ctx_set_timing(mlk_ctx ctx, int enable);
mlk_status mlk_ctx_reset_stats(mlk_ctx ctx);
/* Kernel stats: idx in [0, *count).  Call with name == NULL to get *count only.
 * name receives the kernel name (NUL-terminated, truncated to name_len), launches the
 * number of launches, ms the summed event-measured duration. */
mlk_status mlk_ctx_kernel_stats(mlk_ctx ctx, int idx, int* count, char* name, int name_len,
                                int64_t* launches, double* ms);

/* ------------------------------------------------------------------------------------------
 * mlk_build_tree -- binary median-split tree, Algorithm 1 with ChooseRule RP (Alg 2) or kD
 * (Alg 2-kd).
 *  X           n x d row-major observation sites, host or device.  Sites must be distinct
 *              (MLK_ERR_DUPLICATE_POINTS otherwise).
 *  leaf_size   a cell is a leaf iff it holds <= leaf_size points (R1).
 *  kind        MLK_TREE_KD: direction e_(depth mod d) (R4); MLK_TREE_RP: `directions`.
 *  directions  RP only: n_dir_rows x d row-major unit vectors, host or device, row q used
 *              as given for heap node q (R3); needs n_dir_rows >= 2^t - 1 where t is the
 *              tree depth (smallest delta with ceil(n / 2^delta) <= leaf_size).
 * Split rule (R2): sort the cell by (x.v, original index); the first ceil(s/2) go left;
 * threshold = median (midpoint of the two middle projections for even s).  Projections are
 * summed left to right with separately rounded products and sums (R6).
 * Nodes are numbered in heap order (children of q are 2q+1, 2q+2; R5).
 * Cost: O(n d t) projections + one segmented sort per level, all on the device.
 */
typedef enum { MLK_TREE_KD = 0, MLK_TREE_RP = 1 } mlk_tree_kind;
mlk_status mlk_build_tree(mlk_ctx ctx, const double* X, int64_t n, int32_t d, int32_t leaf_size,
                          int32_t kind, const double* directions, int64_t n_dir_rows,
                          mlk_tree* out);
void mlk_tree_free(mlk_tree tree); /* NULL-safe */
/* t: depth; n_nodes = 2^(t+1) - 1 heap slots. */
mlk_status mlk_tree_info(mlk_tree tree, int32_t* t, int32_t* n_nodes, int64_t* n, int32_t* d);
/* Host copies (any may be NULL).  perm[n]: tree position -> original index.  Per heap slot
 * (n_nodes): begin/end range in perm (0,0 if the slot is empty), depth, state (-1 empty,
 * 0 internal, 1 leaf), thr (NaN unless internal), dir (n_nodes x d, zero unless internal). */
mlk_status mlk_tree_export(mlk_tree tree, int64_t* perm, int64_t* begin, int64_t* end,
                           int32_t* depth, int32_t* state, double* thr, double* dir);

/* ------------------------------------------------------------------------------------------
 * mlk_build_basis -- multi-level basis, steps (a)-(f) P:1427-1515, with the orthonormal
 * split of step (b) taken from a complete Householder QR in the LAPACK convention (R7):
 * leaf: P(X_leaf) = Q R (s x M, total-degree-w monomials of the raw coordinates, R8),
 *       Phi = Q_1^T, W = Q_2^T;
 * internal: [R_L; R_R] = Q R (2M x M), Phi = Q_1^T (Phi_L (+) Phi_R), W = Q_2^T (...).
 * M = C(d + w, w).  L = Phi_root (R10).  MLK_ERR_RANK_DEFICIENT if a leaf has fewer than M
 * points or |R_kk| <= 1e-13 max_i |R_ii| in any cell (R9).
 * Asynchrony: the leaf level is factored before the call returns (its rank test is the one
 * that can fail: [R_L; R_R] has full column rank whenever R_L does); the merge levels -- a
 * latency-bound chain of small QRs -- are left running on the context's auxiliary stream so
 * they overlap the caller's next host work (e.g. the admission search and planning of
 * mlk_assemble_cw).  Every call that reads the blocks (mlk_basis_export of W / Phi / L,
 * mlk_apply_wt, mlk_apply_w, mlk_assemble_cw, mlk_cw_matvec EXACT) waits for them first and
 * reports a numerically rank-deficient merge there (MLK_ERR_RANK_DEFICIENT).
 */
mlk_status mlk_build_basis(mlk_ctx ctx, mlk_tree tree, int32_t w, mlk_basis* out);
/* The same with the index set of Table multivariate:table1 (NEXT-3): total degree
 * (TD, sum p_i <= w, M = C(d + w, w)), hyperbolic cross (HC, prod (p_i + 1) <= w), Smolyak
 * (SM, sum f(p_i) <= w, f(0) = 0, f(1) = 1, f(p) = ceil(log2 p)) or tensor product (TP,
 * max p_i <= w), in the graded order of reading R8.  M <= 4096. */
typedef enum { MLK_INDEX_TD = 0, MLK_INDEX_HC = 1, MLK_INDEX_SM = 2, MLK_INDEX_TP = 3 } mlk_index_set;
/* flags: MLK_BASIS_KEEP_DEFICIENT keeps p = M wavelet-free directions in a numerically rank-
 * deficient cell instead of failing (reading R24: the paper's Table 1 sphere workload, where
 * sum x_i^2 = 1 makes the HC moment matrix rank M - 1, is built with p = M -- its Size column
 * 20592 = 8 (4000 - 1426)).  W stays orthonormal and annihilates the polynomials; only the
 * direction of the deficient column inside the cell is then set by rounding. */
#define MLK_BASIS_KEEP_DEFICIENT 1
/* MLK_BASIS_DROP_PHI retains only L = Phi_root after the construction instead of the Phi block
 * of every node (M x n doubles per tree level: 111 GB at BASELINE cfg5).  It is also applied
 * automatically when the Phi blocks exceed half of the free device memory.  mlk_basis_export
 * of a non-root Phi_block then fails with MLK_ERR_UNSUPPORTED; W, L and every other call are
 * unaffected. */
#define MLK_BASIS_DROP_PHI 2
mlk_status mlk_build_basis_ex(mlk_ctx ctx, mlk_tree tree, int32_t index_set, int32_t w, int32_t flags,
                              mlk_basis* out);
void mlk_basis_free(mlk_basis basis); /* NULL-safe */
/* M; dim = N - M rows of W; n_cells = cells with at least one wavelet. */
mlk_status mlk_basis_info(mlk_basis basis, int32_t* M, int64_t* dim, int32_t* n_cells);
/* Host copies.  cells[n_cells]: heap node of each cell in C_W order; cell_row_off[n_cells+1]
 * prefix sums of the wavelet counts.  If node >= 0: W_block (p_node x |node| row-major,
 * columns = the node's points in tree order) and Phi_block (M x |node|).  L: M x n. */
mlk_status mlk_basis_export(mlk_basis basis, int32_t* cells, int64_t* cell_row_off, int32_t node,
                            double* W_block, double* Phi_block, double* L);
/* a = W^T v (step (1) of P:2146-2170).  v: nvec x dim, a: nvec x n (host or device). */
mlk_status mlk_apply_wt(mlk_ctx ctx, mlk_basis basis, const double* v, double* a, int32_t nvec);
/* y = W b (step (3)).  b: nvec x n, y: nvec x dim. */
mlk_status mlk_apply_w(mlk_ctx ctx, mlk_basis basis, const double* b, double* y, int32_t nvec);

/* ------------------------------------------------------------------------------------------
 * Covariance C(x, y) = sigma2 phi(|x - y|) + nugget [same observation] (R18), phi one of
 * the Matern closed forms nu = 1/2, 3/2, 5/2 with z = sqrt(2 nu) r / rho (R16)
 * or the Gaussian exp(-r^2 / rho^2) (R17).  rho > 0, sigma2 > 0, nugget >= 0.
 */
/* MLK_MATERN_NU (NEXT-3): the definition of P:970 for any nu > 0 (the paper's workloads use
 * nu = 1.25, 3/4), with K_nu evaluated in the kernel from its integral representation
 * int_0^inf exp(-z cosh t) cosh(nu t) dt (trapezoidal rule) or, for z < 2 and non-integer nu,
 * the I_-nu - I_nu power series; 0 < nu <= 50; nu is read only for this family. */
typedef enum { MLK_MATERN_12 = 0, MLK_MATERN_32 = 1, MLK_MATERN_52 = 2, MLK_GAUSSIAN = 3, MLK_MATERN_NU = 4 } mlk_family;
typedef struct {
  int32_t family;
  double rho, sigma2, nugget;
  double nu;
} mlk_kernel;

/* Sparsity: MLK_PAIRS_ALL admits every cell pair (dense C_W); MLK_PAIRS_PAPER_TAU admits the
 * pairs of Algorithm 6 with tau_{i,j} = tau 2^(t-(i+j)/2) (R15),
 * the symmetric projection rule (R12), the root row dense (R21) and self pairs. tau >= 0. */
typedef enum { MLK_PAIRS_ALL = 0, MLK_PAIRS_PAPER_TAU = 1 } mlk_pairs;
typedef struct {
  int32_t mode;
  double tau;
} mlk_sparsity;

/* Precision of the block computation.  FP64: FP64 DMMA tiles (Gram identity + fused kernel
 * evaluation + two contractions).  DD: double-double tile generation and contractions for
 * workloads at the FP64 floor (e.g. BASELINE cfg1). */
typedef enum { MLK_PREC_FP64 = 0, MLK_PREC_DD = 1 } mlk_precision;

/* Gather of the per-rank pieces after the assembly (nranks > 1; nothing to do for nranks == 1):
 *  MLK_GATHER_NONE    each rank keeps its shard of pieces (mlk_cw_pack / mlk_cw_unpack, or the
 *                     sharded mlk_cw_matvec BSR, which needs no gather at all).  This is the
 *                     mode for matrices no single GPU or host holds (BASELINE cfg5: 184 GB of
 *                     values).
 *  MLK_GATHER_DEVICE  the library all-gathers the pieces over its NCCL communicator, in block
 *                     groups sized to a staging buffer (no rank ever holds the nranks x shard
 *                     receive buffer), and reduces them in chunk order into device values: every
 *                     rank returns the complete C~_W, bit-identical to nranks == 1.
 *  MLK_GATHER_HOST    the same into mapped pinned host memory (MLK_VALUES_HOST placement).
 * The GATHER modes need a context created with an NCCL unique id. */
typedef enum { MLK_GATHER_NONE = 0, MLK_GATHER_DEVICE = 1, MLK_GATHER_HOST = 2 } mlk_gather;

/* ------------------------------------------------------------------------------------------
 * mlk_assemble_cw -- the sparse multi-level covariance matrix C~_W (Algorithm 6; blocks
 * W_i C W_j^T of P:1636-1653) in variable-block BSR form:
 *  block rows/cols = cells in C_W order; each admitted unordered pair is stored once as
 *  (row, col) with row <= col in C_W order, row-major p_row x p_col, blocks sorted by
 *  (row, col).  Every block is computed exactly (no approximation inside a block).
 * Work decomposition ("Nested assembly"): for each block one
 * cell b is contracted first; V_b = C(X_R, X_b) W_b^T is formed once for the union R of the
 * row points of all blocks sharing b (for ancestor pairs R = X_b itself), in work units of
 * <= 4096 rows, either directly on the fused tile kernel or -- the nested plan, for every
 * internal b at once -- from the leaves' scaling sums C(X_R, X_l) Phi_l^T and the merge factors
 * of the basis; a block is W_a V_b[X_a], summed over the 4096-row chunks ("pieces") of X_a in
 * chunk order (mlk_cw_plan reports the plan; MLK_ASSEMBLY=direct|nested overrides it).
 * With nranks > 1 the units are LPT-partitioned over ranks, each rank writes the pieces of
 * its units into its shard, and `gather` (mlk_gather) decides how the shards are combined.
 * Results are bit-identical for every nranks.
 */
mlk_status mlk_assemble_cw(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel,
                           const mlk_sparsity* sparsity, int32_t precision, int32_t gather, mlk_cw* out);
/* mlk_assemble_cw_ex -- as mlk_assemble_cw, with the placement of the nnz BSR values:
 *  MLK_VALUES_DEVICE: device memory (what mlk_assemble_cw does);
 *  MLK_VALUES_HOST:   mapped pinned host memory allocated by the library (cudaHostAlloc), for
 *                     matrices beyond HBM (BASELINE cfg5: 184 GB of values next to 106 GB of
 *                     W).  The kernels store the finished blocks straight over the host link;
 *                     the piece shards and all scratch stay on the device (nranks > 1: the gather
 *                     reduces into it).  mlk_cw_values_device then returns the host pointer;
 *                     mlk_cw_matvec BSR reads the values over the host link.
 *  gather: MLK_GATHER_NONE or MLK_GATHER_DEVICE (= "gather into the placement"). */
typedef enum { MLK_VALUES_DEVICE = 0, MLK_VALUES_HOST = 1 } mlk_values_placement;
mlk_status mlk_assemble_cw_ex(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel,
                              const mlk_sparsity* sparsity, int32_t precision, int32_t placement, int32_t gather,
                              mlk_cw* out);
void mlk_cw_free(mlk_cw cw); /* NULL-safe */
/* n_cells; n_blocks; nnz values; entries = sum over blocks |row cell| |col cell| (the
 * covariance pairs C~_W is made of); flops = FP64 flops the kernels execute (Gram 2d per
 * evaluated entry + both contractions, see mlk_cw_flops); own_entries = covariance entries
 * this rank evaluates, own_flops = its share of flops. */
mlk_status mlk_cw_info(mlk_cw cw, int32_t* n_cells, int64_t* n_blocks, int64_t* nnz,
                       double* entries, double* flops, double* own_entries, double* own_flops);
/* Host copies of the structure (brow_ptr[n_cells+1], bcol[n_blocks], val_off[n_blocks+1])
 * and, if values != NULL, of all nnz values (host or device pointer).  With nranks > 1 the
 * values are complete only after mlk_cw_unpack. */
mlk_status mlk_cw_export(mlk_cw cw, int32_t* brow_ptr, int32_t* bcol, int64_t* val_off,
                         double* values);
/* Asynchronous export of all nnz BSR values into `values` (host or device memory): the copy is
 * enqueued on the context's copy stream behind the work already enqueued on the context stream,
 * and the call returns without waiting, so the transfer overlaps later calls (e.g. the C_W v
 * product).  Pinned host memory gives a true DMA overlap.  mlk_ctx_wait_copies blocks until
 * every copy enqueued this way has landed; `values` and `cw` must stay valid until then.  With
 * nranks > 1 call it after mlk_cw_unpack. */
mlk_status mlk_cw_export_async(mlk_ctx ctx, mlk_cw cw, double* values);
mlk_status mlk_ctx_wait_copies(mlk_ctx ctx);
/* Executed FP64 flops by stage (all ranks): gram = 2 d per evaluated covariance entry,
 * contract1 = the fused tile products V_b = C W_b^T (2 p_b per entry), contract2 = the
 * products W_a V_b[X_a] (2 p_a |X_a| p_b per block). */
mlk_status mlk_cw_flops(mlk_cw cw, double* gram, double* contract1, double* contract2);
/* The assembly plan: *nested = 1 if the internal cells' V_b came from the nested evaluation
 * (leaves' scaling sums + merge-factor transfers; MLK_ASSEMBLY=direct|nested
 * overrides the cost model), transfer_flops = the FP64 flops of those transfers (all ranks; not
 * part of mlk_cw_flops' three stages), nested_tile_flops = the part of mlk_cw_flops' gram +
 * contract1 done by the nested leaf pass (kernel timing name "assemble_tile_nested"; the rest is
 * the direct units, "assemble_tile_contract").  Any output may be NULL. */
mlk_status mlk_cw_plan(mlk_cw cw, int32_t* nested, double* transfer_flops, double* nested_tile_flops);
/* Owner rank of every block (n_blocks): the rank of its first piece; mlk_cw_matvec BSR with
 * nranks > 1 applies the blocks a rank owns. */
mlk_status mlk_cw_owner(mlk_cw cw, int32_t* owner);
/* Gather support (nranks > 1).  shard_len: doubles of pieces this rank produced;
 * max_shard_len: the maximum over ranks.  mlk_cw_pack writes this rank's pieces, in
 * (block, chunk) order, to `dst` (device, >= max_shard_len doubles, tail zero-filled).  After
 * the caller's all-gather of the packed shards into `gathered` (device, nranks x
 * max_shard_len, rank-major), mlk_cw_unpack sums every block's pieces in chunk order into
 * the BSR values (no-op for nranks == 1), group by group exactly as MLK_GATHER_DEVICE does. */
mlk_status mlk_cw_shard_len(mlk_cw cw, int64_t* shard_len, int64_t* max_shard_len);
mlk_status mlk_cw_pack(mlk_ctx ctx, mlk_cw cw, double* dst);
mlk_status mlk_cw_unpack(mlk_ctx ctx, mlk_cw cw, const double* gathered);
/* The piece layout behind the gather (for checking one rank's share without the all-gather):
 * piece_ptr[n_blocks+1] (block k = sum of pieces piece_ptr[k] .. piece_ptr[k+1]-1 in order),
 * piece_off[n_pieces] (offset in its owner's shard; meaningful for pieces not written straight
 * into the values, i.e. all pieces when nranks > 1), piece_owner[n_pieces], and a copy of this
 * rank's shard (shard_len doubles, host or device).  Any output may be NULL; n_pieces =
 * piece_ptr[n_blocks]. */
mlk_status mlk_cw_export_pieces(mlk_cw cw, int64_t* piece_ptr, int64_t* piece_off, int32_t* piece_owner,
                                double* shard);
/* Pointer to the BSR values (device memory, or mapped host memory under MLK_VALUES_HOST;
 * valid while cw lives; with nranks > 1 NULL until mlk_cw_unpack allocated them). */
mlk_status mlk_cw_values_device(mlk_cw cw, double** values);

/* ------------------------------------------------------------------------------------------
 * mlk_cov_matvec -- b = C a, exact direct summation with on-the-fly covariance tiles (step
 * (2) of P:2146-2170).  a, b: nvec x n in tree order (host or device), 1 <= nvec <= 64.
 * With nranks > 1, b is this rank's partial sum and the caller sums b over the ranks: the
 * rank owns a set of 32-row tiles I and adds C(I, J) a_J to b_I and, for the symmetric
 * product (nvec <= 4, each pair (i, j) evaluated once), C(I, J)^T a_I to b_J (J > I).
 */
mlk_status mlk_cov_matvec(mlk_ctx ctx, mlk_tree tree, const mlk_kernel* kernel, const double* a,
                          double* b, int32_t nvec);

/* mlk_cw_matvec -- y = C_W v.  EXACT: y = W (C (W^T v)) by the three steps of
 * P:2146-2170 (cw may be NULL).  BSR: y = C~_W v on the assembled blocks (mirrored lower
 * triangle).  v, y: nvec x dim (host or device).
 * nranks > 1: each rank applies its share -- EXACT its row panel of C; BSR the blocks it owns
 * when cw is complete (gathered / unpacked), otherwise the pieces of its own shard (S§8(e): "each
 * rank applies its own blocks and their mirrors", no gather needed).  With a library
 * communicator (mlk_ctx_create with an NCCL id) y is then sum-allreduced and every rank returns
 * C_W v; without one y is this rank's partial sum and the caller allreduces it.  The EXACT
 * row split is a function of (n, nvec, nranks) and the device's total memory only, identical on
 * every rank. */
typedef enum { MLK_MATVEC_EXACT = 0, MLK_MATVEC_BSR = 1 } mlk_matvec_mode;
mlk_status mlk_cw_matvec(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel,
                         mlk_cw cw, int32_t mode, const double* v, double* y, int32_t nvec);

/* ------------------------------------------------------------------------------------------
 * mlk_pcg_solve -- gamma_W = C_W^-1 z_W by preconditioned conjugate gradient (the
 * survey's NEXT-1).  Products C_W p by the EXACT three-step product.
 *  precond 1: P_W = diag of the self blocks W_k C W_k^T of every cell, taken from
 *             the assembled `cw` (which must contain every self block -- always the case for
 *             mlk_assemble_cw -- and be complete), Cholesky-factored once; MLK_ERR_RANK_DEFICIENT
 *             if a block is not positive definite.  precond 0: P_W = I (cw may be NULL).
 *  z_w, gamma_w: dim doubles (host or device).  Iterates from gamma = 0 until the recursive
 *  residual satisfies ||r|| <= tol ||z_W|| or max_iter iterations; *iters receives the count and
 *  *rel_residual the TRUE unpreconditioned residual ||z_W - C_W gamma|| / ||z_W||,
 *  recomputed with one extra product.  Deterministic (fixed-order reductions).  nranks == 1 only
 *  (MLK_ERR_UNSUPPORTED otherwise).
 */
mlk_status mlk_pcg_solve(mlk_ctx ctx, mlk_tree tree, mlk_basis basis, const mlk_kernel* kernel, mlk_cw cw,
                         int32_t precond, const double* z_w, double* gamma_w, double tol, int32_t max_iter,
                         int32_t* iters, double* rel_residual);

/* ------------------------------------------------------------------------------------------
 * mlk_loglik -- the level-truncated multi-level log-likelihood of P:1954-1971 (the survey's
 * NEXT-4):
 *   l~^n_W = -N~/2 log(2 pi) - 1/2 log det C~^n_W - 1/2 (Z^n_W)^T (C~^n_W)^-1 Z^n_W,
 * with C~^n_W the upper-left N~ x N~ block of the assembled C~_W = the rows of the cells of
 * levels t .. `level` (0 <= level <= t; level 0 is the whole C~_W), and Z^n_W the first N~
 * entries of z_w = W Z (dim doubles, host or device; e.g. from mlk_apply_w).  Computed from a
 * block-sparse Cholesky factor of C~^n_W (log det = 2 sum log G_ii, the quadratic
 * form by the same factor), right-looking over the BSR cells in C_W order with the fill of
 * the block pattern; deterministic.  Outputs (any may be NULL): loglik, logdet, quad =
 * (Z^n_W)^T (C~^n_W)^-1 Z^n_W, n_tilde = N~.  cw must be complete; nranks == 1.
 * MLK_ERR_RANK_DEFICIENT if a pivot is not positive (C~^n_W not positive definite).
 */
mlk_status mlk_loglik(mlk_ctx ctx, mlk_basis basis, mlk_cw cw, int32_t level, const double* z_w,
                      double* loglik, double* logdet, double* quad, int64_t* n_tilde);

/* ------------------------------------------------------------------------------------------
 * Host-only helpers (no device needed).
 * mlk_partition_lpt: longest-processing-time assignment of n units with the given costs to
 * nranks ranks (largest first to the least-loaded rank; ties to the lower rank), the
 * partition mlk_assemble_cw uses.  owner[n] receives ranks.
 */
mlk_status mlk_partition_lpt(const double* cost, int64_t n, int32_t nranks, int32_t* owner);
/* mlk_shard_plan: the gather layout mlk_assemble_cw uses.  Given piece offsets val_off[n+1]
 * (prefix sums of piece lengths) and owner[n], shard_off[k] = offset of piece k inside its
 * owner's packed shard (pieces in order), shard_len[nranks] = doubles per rank.  The gathered
 * buffer holds rank r's shard at r * max(shard_len). */
mlk_status mlk_shard_plan(const int64_t* val_off, const int32_t* owner, int64_t n, int32_t nranks,
                          int64_t* shard_off, int64_t* shard_len);

/* mlk_gather_plan: the block groups of the chunked all-gather (MLK_GATHER_DEVICE / _HOST and
 * mlk_cw_unpack).  Inputs: n_blocks, piece_ptr[n_blocks+1], piece_off[n_pieces] (offset in the
 * owner's shard), piece_owner[n_pieces], block_len[n_blocks] (doubles per block), nranks, and the
 * receive budget (doubles).  Group g covers blocks group_ptr[g] .. group_ptr[g+1]-1; rank r
 * contributes its shard slice [group_lo[g*nranks + r], + group_count[g]) (pieces of the group are
 * contiguous in every shard), so a group is one equal-count all-gather of nranks x
 * group_count[g] <= budget doubles (a single larger block is a group of its own).  Call with
 * the three group arrays NULL to get *n_groups; group_ptr needs n_groups + 1 entries. */
mlk_status mlk_gather_plan(int64_t n_blocks, const int64_t* piece_ptr, const int64_t* piece_off,
                           const int32_t* piece_owner, const int64_t* block_len, int32_t nranks, int64_t budget,
                           int64_t* n_groups, int64_t* group_ptr, int64_t* group_lo, int64_t* group_count);

#ifdef __cplusplus
}
#endif
#endif /* MLK_H_ */
