"""Level-truncated multi-level log-likelihood (oracle; test infrastructure only).

P:1954-1971   l~^n_W(theta) = -N~/2 log(2 pi) - 1/2 log det C~^n_W(theta)
                               - 1/2 (Z^n_W)^T C~^n_W(theta)^-1 Z^n_W,
              Z^n_W = [W_t^T, ..., W_n^T]^T Z (the first N~ entries of W Z in C_W order, levels
              t .. n), C~^n_W the N~ x N~ upper-left sub-matrix of the sparse C~_W.
P:2104-2116   log det C~^n_W = 2 sum_i log G_ii for the Cholesky factor G G^T = C~^n_W.
P:2118-2136   the quadratic form from the same factor: with y = G^-1 Z^n_W it is y^T y.

The oracle forms C~^n_W densely from the oracle's BSR (oracle.assemble.bsr_to_dense), factors it
with numpy.linalg.cholesky and solves with numpy.linalg.solve (small sizes only).  It shares no
code with the CUDA path.
"""
import numpy as np

from . import assemble as OAs


def truncation(tree, basis, level):
    """(number of leading cells, N~): the cells of depth >= level, a prefix of the C_W order."""
    K = 0
    while K < len(basis.cells) and tree.depth[basis.cells[K]] >= level:
        K += 1
    n_tilde = int(sum(basis.p(q) for q in basis.cells[:K]))
    return K, n_tilde


def loglik_dense(Ct, z):
    """(l, log det, quad) of a zero-mean Gaussian with covariance Ct at z (P:1954-1971,
    P:2104-2136) through the Cholesky factor G G^T = Ct."""
    Ct = np.asarray(Ct, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    n = Ct.shape[0]
    G = np.linalg.cholesky(Ct)
    logdet = 2.0 * np.sum(np.log(np.diag(G)))
    y = np.linalg.solve(G, z)
    quad = float(y @ y)
    return -0.5 * n * np.log(2.0 * np.pi) - 0.5 * logdet - 0.5 * quad, float(logdet), quad


def loglik(bsr, tree, basis, z_w, level):
    """l~^n_W for the assembled BSR C~_W (oracle.assemble.assemble) and z_w = W Z (dim)."""
    _, n_tilde = truncation(tree, basis, level)
    A = OAs.bsr_to_dense(bsr)[:n_tilde, :n_tilde]
    return loglik_dense(A, np.asarray(z_w)[:n_tilde]) + (n_tilde,)
