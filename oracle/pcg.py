"""Preconditioned conjugate gradient for C_W gamma_W = Z_W (oracle; test infrastructure only).

P:2058-2064   Z_W = W Z and C_W(theta) gamma_W = Z_W (W M = 0 removes the mean term).
P:2065-2083   the preconditioner P_W = diag(P^{i,k}) over every cell B^i_k, where P^{i,k} is the
              block of C_W between the cell's own basis vectors, i.e. W_k C W_k^T (the self
              block of Algorithm 6's assembly).  P_W = I ("no preconditioner") is allowed.
P:2084-2097   Theorem (multi-levelkriging:lemma2): P_W is symmetric positive definite.
P:2146-2170   the products C_W gamma^n in the iteration are computed in three steps
              a = W^T gamma, b = C a, y = W b (oracle.matvec.cw_matvec_exact).
P:2186-2194   the accuracy is set on the *unpreconditioned* system: stop when
              ||Z_W - C_W gamma|| <= eps ||Z_W||.

The iteration is the textbook PCG (Hestenes-Stiefel with a left preconditioner M = P_W):
    x = 0, r = z, s = M^-1 r, p = s, rs = r.s
    repeat: q = C_W p; alpha = rs / (p.q); x += alpha p; r -= alpha q;
            stop if ||r|| <= eps ||z||; s = M^-1 r; rs' = r.s; p = s + (rs'/rs) p; rs = rs'
M^-1 is applied block by block with the Cholesky factors of the P^{i,k} (numpy.linalg).
"""
import numpy as np

from . import assemble as OAs
from . import matvec as OM


def preconditioner_blocks(X, tree, basis, kern):
    """The self blocks P^{i,k} = W_k C(X_k, X_k) W_k^T of every cell, in C_W order."""
    return [OAs.block(X, tree, basis, kern, q, q) for q in basis.cells]


def apply_block_inverse(blocks, row_off, r):
    """s = P_W^-1 r with P_W = diag(blocks): two triangular solves per block (Cholesky)."""
    s = np.empty_like(r)
    for k, P in enumerate(blocks):
        a, b = row_off[k], row_off[k + 1]
        L = np.linalg.cholesky(P)
        y = np.linalg.solve(L, r[a:b])
        s[a:b] = np.linalg.solve(L.T, y)
    return s


def pcg(matvec, z, tol, max_iter, precond=None):
    """Returns (x, iterations, ||z - A x|| / ||z|| of the recursive residual).  precond(r) -> M^-1 r
    or None for M = I."""
    z = np.asarray(z, dtype=np.float64)
    x = np.zeros_like(z)
    r = z.copy()
    nz = np.linalg.norm(z)
    if nz == 0.0:
        return x, 0, 0.0
    s = precond(r) if precond else r.copy()
    p = s.copy()
    rs = float(r @ s)
    it = 0
    while it < max_iter:
        q = matvec(p)
        alpha = rs / float(p @ q)
        x += alpha * p
        r -= alpha * q
        it += 1
        if np.linalg.norm(r) <= tol * nz:
            break
        s = precond(r) if precond else r.copy()
        rs_new = float(r @ s)
        p = s + (rs_new / rs) * p
        rs = rs_new
    return x, it, float(np.linalg.norm(r) / nz)


def solve_cw(X, tree, basis, kern, z_w, tol=1e-10, max_iter=1000, use_precond=True):
    """gamma_W = C_W^-1 z_W with the EXACT three-step product."""
    blocks = preconditioner_blocks(X, tree, basis, kern) if use_precond else None
    row_off = np.array([basis.row_off[q] for q in basis.cells] + [basis.dim], dtype=np.int64)
    matvec = lambda v: OM.cw_matvec_exact(X, tree, basis, kern, v)[0]
    pre = (lambda r: apply_block_inverse(blocks, row_off, r)) if use_precond else None
    return pcg(matvec, z_w, tol, max_iter, pre)
