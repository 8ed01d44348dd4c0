"""Blocks of C_W = W C W^T (oracle; test infrastructure only).

P:1636-1653  C_W^{i,j} = W_i C W_j^T; each entry is (psi^i_k)^T C psi^j_l.
P:1777-1800  Algorithm 6: compute (psi^i_k)^T C psi^j_l for every admitted pair of cells.
Every block is formed exactly as written: the dense covariance tile C(X_row, X_col) by
direct differences (oracle/covariance.py), then W_row @ C @ W_col^T.

BSR layout: block rows are cells in C_W order; each admitted
unordered pair is stored once as (row, col) with row first in C_W order, row-major
p_row x p_col, blocks sorted by (row, col).
"""
from dataclasses import dataclass

import numpy as np

from .basis import dense_W
from .covariance import cov


@dataclass
class BSR:
    cells: list          # C_W order
    row_off: np.ndarray  # int64[n_cells + 1]
    brow_ptr: np.ndarray  # int32[n_cells + 1]
    bcol: np.ndarray     # int32[n_blocks]  (cell position in C_W order)
    val_off: np.ndarray  # int64[n_blocks + 1]
    values: np.ndarray   # float64[nnz]


def cell_points(tree, q):
    return tree.perm[tree.begin[q]:tree.end[q]], np.arange(tree.begin[q], tree.end[q])


def block(X, tree, basis, kern, a, b, dtype=np.float64):
    """B_ab = W_a C(X_a, X_b) W_b^T.  dtype=np.longdouble for the cfg1 reference."""
    ia, _ = cell_points(tree, a)
    ib, _ = cell_points(tree, b)
    Xa = np.asarray(X[ia], dtype=dtype)
    Xb = np.asarray(X[ib], dtype=dtype)
    C = cov(Xa, Xb, ia, ib, kern["family"], dtype(kern["rho"]), dtype(kern.get("sigma2", 1.0)),
            dtype(kern.get("nugget", 0.0)), nu=kern.get("nu"))
    Wa = np.asarray(basis.W[a], dtype=dtype)
    Wb = np.asarray(basis.W[b], dtype=dtype)
    return Wa @ C @ Wb.T


def bsr_structure(basis, pairs):
    cells = basis.cells
    pos = {q: k for k, q in enumerate(cells)}
    nc = len(cells)
    row_off = np.zeros(nc + 1, np.int64)
    for k, q in enumerate(cells):
        row_off[k + 1] = row_off[k] + basis.p(q)
    brow_ptr = np.zeros(nc + 1, np.int32)
    bcol = np.zeros(len(pairs), np.int32)
    val_off = np.zeros(len(pairs) + 1, np.int64)
    for k, (a, b) in enumerate(pairs):
        brow_ptr[pos[a] + 1] += 1
        bcol[k] = pos[b]
        val_off[k + 1] = val_off[k] + basis.p(a) * basis.p(b)
    brow_ptr = np.cumsum(brow_ptr).astype(np.int32)
    return cells, row_off, brow_ptr, bcol, val_off


def assemble(X, tree, basis, kern, pairs, dtype=np.float64):
    """Sparse C~_W in BSR form: one block per admitted pair (Alg 6)."""
    cells, row_off, brow_ptr, bcol, val_off = bsr_structure(basis, pairs)
    values = np.zeros(int(val_off[-1]), dtype=dtype)
    for k, (a, b) in enumerate(pairs):
        values[val_off[k]:val_off[k + 1]] = block(X, tree, basis, kern, a, b, dtype).ravel()
    return BSR(cells, row_off, brow_ptr, bcol, val_off, values)


def dense_cw(X, tree, basis, kern):
    """C_W = W C W^T formed densely; small n only."""
    W = dense_W(tree, basis)
    ids = tree.perm
    Xt = np.asarray(X)[ids]
    C = cov(Xt, Xt, ids, ids, kern["family"], kern["rho"], kern.get("sigma2", 1.0),
            kern.get("nugget", 0.0), nu=kern.get("nu"))
    return W @ C @ W.T, C, W


def bsr_to_dense(bsr):
    """Symmetric dense matrix from the upper-triangle BSR (mirrors off-diagonal blocks)."""
    n = int(bsr.row_off[-1])
    A = np.zeros((n, n), dtype=bsr.values.dtype)
    nc = len(bsr.cells)
    for r in range(nc):
        for k in range(bsr.brow_ptr[r], bsr.brow_ptr[r + 1]):
            c = bsr.bcol[k]
            r0, r1 = bsr.row_off[r], bsr.row_off[r + 1]
            c0, c1 = bsr.row_off[c], bsr.row_off[c + 1]
            blk = bsr.values[bsr.val_off[k]:bsr.val_off[k + 1]].reshape(r1 - r0, c1 - c0)
            A[r0:r1, c0:c1] = blk
            if r != c:
                A[c0:c1, r0:r1] = blk.T
    return A
