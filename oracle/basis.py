"""Multi-level basis W and L (oracle; test infrastructure only).

P:1427-1515  steps (a)-(f): at each leaf cell form the moment matrix
             calM = (M~)^T V of the cell's vectors, split R^s into the orthonormal
             complement of its null space (scaling vectors phi) and the null space
             (multi-level / wavelet vectors psi, which satisfy eq. hbconstruction:eqn1);
             go up one level, replacing the leaf unit vectors by the children's scaling
             vectors; stop at the root.
P:1541-1566  W = [W_t; ...; W_0; W_-1], L = scaling vectors of the root, P = [W; L]
             orthonormal.

Readings:
  R7  the orthonormal split of step (b)(ii)-(iii) is taken from a COMPLETE Householder QR
      in the LAPACK convention (numpy.linalg.qr, mode='complete') instead of an SVD: the
      SVD basis of the null space is not unique, the QR split spans the same two
      subspaces and is canonical.  For a leaf, calM^T = P(X_leaf) (s x M) = Q R, so
      phi = Q_1^T, psi = Q_2^T.  For an internal cell V = [Phi_L ; Phi_R] (block
      diagonal), calM^T = V M~ = [R_L ; R_R] (2M x M) = Q R, phi = Q_1^T V, psi = Q_2^T V.
  R8  raw monomials (no centring) of the TD set in graded order.
  R9  rank a = M at every cell, else RankDeficient (|R_kk| <= 1e-13 max_i |R_ii|, or a
      leaf with fewer than M points).
  R10 a = 0, p~ = p = M: W_-1 is empty and L = Phi_root.
  R11 row order of W: levels t, t-1, ..., 0; heap order within a level; QR complement
      column order within a cell.  Cells with no wavelets take no rows.
Columns of every block are the cell's points in tree order (perm).
"""
from dataclasses import dataclass, field

import numpy as np

from .index_set import monomials, td_exponents


class RankDeficient(ValueError):
    pass


RANK_TOL = 1e-13


@dataclass
class Basis:
    M: int
    exps: list
    W: dict = field(default_factory=dict)      # node -> (p_node x |node|)
    Phi: dict = field(default_factory=dict)    # node -> (M x |node|)
    R: dict = field(default_factory=dict)      # node -> (M x M)
    cells: list = field(default_factory=list)  # C_W order (R11), cells with p > 0
    row_off: dict = field(default_factory=dict)
    dim: int = 0
    L: np.ndarray = None                       # M x n, tree order

    def p(self, q):
        return self.W[q].shape[0]


def _check_rank(R, M):
    dg = np.abs(np.diag(R[:M, :M]))
    if dg.size and dg.min() <= RANK_TOL * dg.max():
        raise RankDeficient("moment matrix is rank deficient")


def _node_step(X, tree, exps, B, q):
    """Phi_q, W_q, R_q of one node from its points (leaf, steps (a)-(b)) or from its
    children's R and Phi (internal, steps (c)-(e)), readings R7-R9."""
    M = len(exps)
    b, e = tree.begin[q], tree.end[q]
    if tree.is_leaf[q]:
        s = e - b
        if s < M:
            raise RankDeficient("leaf with fewer points than monomials")
        P = monomials(X[tree.perm[b:e]], exps)   # calM^T for the leaf unit vectors
        Q, R = np.linalg.qr(P, mode="complete")
        _check_rank(R, M)
        B.Phi[q] = Q[:, :M].T.copy()
        B.W[q] = Q[:, M:].T.copy()
        B.R[q] = R[:M, :].copy()
    else:
        lq, rq = 2 * q + 1, 2 * q + 2
        A = np.vstack([B.R[lq], B.R[rq]])          # calM^T = [R_L; R_R]
        Q, R = np.linalg.qr(A, mode="complete")
        _check_rank(R, M)
        nl = tree.end[lq] - tree.begin[lq]
        V = np.zeros((2 * M, e - b))
        V[:M, :nl] = B.Phi[lq]
        V[M:, nl:] = B.Phi[rq]
        B.Phi[q] = Q[:, :M].T @ V
        B.W[q] = Q[:, M:].T @ V
        B.R[q] = R[:M, :].copy()


def build_subtree_basis(X, tree, w, root, exps=None):
    """W, Phi, R of the nodes of the subtree rooted at `root` only.  The construction is
    bottom-up and a node's blocks depend only on its own points, so these equal the
    corresponding blocks of build_basis (same steps, same order); used to check sampled
    cells of workloads whose full basis does not fit the host (BASELINE cfg5).  `cells`,
    `row_off` and `L` are left empty."""
    X = np.asarray(X, dtype=np.float64)
    exps = td_exponents(tree.d, w) if exps is None else list(exps)
    B = Basis(M=len(exps), exps=exps)
    sub, stack = [], [root]
    while stack:
        q = stack.pop()
        if q < tree.n_nodes and tree.exists[q]:
            sub.append(q)
            if not tree.is_leaf[q]:
                stack += [2 * q + 1, 2 * q + 2]
    for q in sorted(sub, reverse=True):              # children before parents
        _node_step(X, tree, exps, B, q)
    return B


def build_basis(X, tree, w, exps=None):
    """Steps (a)-(f) of P:1427-1515 with readings R7-R11 (TD set unless `exps` is given)."""
    X = np.asarray(X, dtype=np.float64)
    exps = td_exponents(tree.d, w) if exps is None else list(exps)
    M = len(exps)
    if M >= tree.n:
        raise RankDeficient("need n > M")
    B = Basis(M=M, exps=exps)
    for q in range(tree.n_nodes - 1, -1, -1):       # children before parents, finest first
        if tree.exists[q]:
            _node_step(X, tree, exps, B, q)
    # C_W order (R11)
    order = sorted((q for q in range(tree.n_nodes) if tree.exists[q]),
                   key=lambda q: (-int(tree.depth[q]), q))
    off = 0
    for q in order:
        p = B.W[q].shape[0]
        if p == 0:
            continue
        B.cells.append(q)
        B.row_off[q] = off
        off += p
    B.dim = off
    B.L = B.Phi[0]
    return B


def dense_W(tree, B):
    """W as a dense (N - M) x N matrix, columns in tree order (small n only)."""
    W = np.zeros((B.dim, tree.n))
    for q in B.cells:
        o = B.row_off[q]
        W[o:o + B.p(q), tree.begin[q]:tree.end[q]] = B.W[q]
    return W


def level_rows(tree, B):
    """Number of rows of W_q for each level q = t..0 (Lemma 1)."""
    out = {}
    for q in B.cells:
        out[int(tree.depth[q])] = out.get(int(tree.depth[q]), 0) + B.p(q)
    return out
