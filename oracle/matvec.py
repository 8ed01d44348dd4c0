"""C_W v (oracle; test infrastructure only).

P:2146-2170  the PCG matrix-vector product C_W gamma is computed in three steps:
             (1) a = W^T gamma, (2) b = C a, (3) y = W b.   (EXACT mode, reading R20)
The BSR mode applies the assembled sparse C~_W (Alg 6 output) instead.
Point-space vectors are in tree order (entry k <-> original observation perm[k]).
"""
import numpy as np

from .covariance import cov


def apply_wt(tree, basis, v):
    """a = W^T v, v in C_W order (step (1)); v may be (dim,) or (nvec, dim)."""
    v = np.atleast_2d(v)
    a = np.zeros((v.shape[0], tree.n))
    for q in basis.cells:
        o = basis.row_off[q]
        a[:, tree.begin[q]:tree.end[q]] += v[:, o:o + basis.p(q)] @ basis.W[q]
    return a


def apply_w(tree, basis, b):
    """y = W b, b in tree order (step (3))."""
    b = np.atleast_2d(b)
    y = np.zeros((b.shape[0], basis.dim))
    for q in basis.cells:
        o = basis.row_off[q]
        y[:, o:o + basis.p(q)] = b[:, tree.begin[q]:tree.end[q]] @ basis.W[q].T
    return y


def cov_matvec(X, tree, kern, a, panel=2048, rows=None):
    """b = C a (step (2)), exact direct summation in row panels; optionally only `rows`."""
    a = np.atleast_2d(a)
    ids = tree.perm
    Xt = np.asarray(X)[ids]
    rows = np.arange(tree.n) if rows is None else np.asarray(rows)
    b = np.zeros((a.shape[0], rows.size))
    for s in range(0, rows.size, panel):
        rr = rows[s:s + panel]
        C = cov(Xt[rr], Xt, ids[rr], ids, kern["family"], kern["rho"], kern.get("sigma2", 1.0),
                kern.get("nugget", 0.0), nu=kern.get("nu"))
        b[:, s:s + rr.size] = (C @ a.T).T
    return b


def cw_matvec_exact(X, tree, basis, kern, v):
    """y = W (C (W^T v))."""
    return apply_w(tree, basis, cov_matvec(X, tree, kern, apply_wt(tree, basis, v)))


def cw_matvec_bsr(bsr, v):
    """y = C~_W v on the symmetric upper-triangle BSR."""
    v = np.atleast_2d(v)
    y = np.zeros_like(v, dtype=np.float64)
    nc = len(bsr.cells)
    for r in range(nc):
        r0, r1 = bsr.row_off[r], bsr.row_off[r + 1]
        for k in range(bsr.brow_ptr[r], bsr.brow_ptr[r + 1]):
            c = bsr.bcol[k]
            c0, c1 = bsr.row_off[c], bsr.row_off[c + 1]
            blk = bsr.values[bsr.val_off[k]:bsr.val_off[k + 1]].reshape(r1 - r0, c1 - c0)
            y[:, r0:r1] += v[:, c0:c1] @ blk.T
            if r != c:
                y[:, c0:c1] += v[:, r0:r1] @ blk
    return y
