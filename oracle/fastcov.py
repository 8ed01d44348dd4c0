"""Full-size oracle references through the plain-C covariance tile (oracle/csrc/cov_tile.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The C routine is `oracle.covariance.cov`
written out in C (direct differences, the same closed forms, one entry at a time); the
contractions stay NumPy matmuls (library primitives), exactly as in oracle/assemble.py.

  cov_c(Xa, Xb, ia, ib, kern)        C(X_a, X_b)                    (R16-R18)
  block_streamed(X, tree, basis, kern, a, b)
                                      B_ab = W_a C(X_a, X_b) W_b^T, formed as
                                      sum over row panels P of X_a of W_a[:, P] (C(X_P, X_b) W_b^T)
                                      -- the definition, with the sum over the rows of C split
                                      into panels so C never exists whole
  cov_rows(X, tree, kern, a, rows)   (C a)[rows] (step (2) of P:2146-2170) on selected rows

Pinned in tests/test_oracle.py against oracle.covariance.cov / oracle.assemble.block (which
are pinned to the paper independently) and against a scalar double sum.
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "cov_tile.c")
_LIB = os.path.join(_HERE, "_cov_tile.so")
# no -ffast-math, no FP contraction: every entry is the plain expression of the source
_CFLAGS = ["-O3", "-mavx2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]
_lib = None


def build(force=False):
    """Compile oracle/_cov_tile.so with gcc (called by __graft_entry__.build() and on demand)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".%d.tmp" % os.getpid()
        subprocess.run(["gcc"] + _CFLAGS + [_SRC, "-o", tmp, "-lm"], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        P = C.c_void_p
        lib.oracle_cov_tile.restype = C.c_int
        lib.oracle_cov_tile.argtypes = [P, P, C.c_int64, P, P, C.c_int64, C.c_int32, C.c_int32,
                                        C.c_double, C.c_double, C.c_double, P]
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def cov_c(Xa, Xb, ia, ib, kern):
    """C(X_a, X_b) (na x nb) for the closed-form families (MATERN_NU: use oracle.covariance)."""
    lib = _load()
    Xa = np.ascontiguousarray(Xa, dtype=np.float64)
    Xb = np.ascontiguousarray(Xb, dtype=np.float64)
    ia = np.ascontiguousarray(ia, dtype=np.int64)
    ib = np.ascontiguousarray(ib, dtype=np.int64)
    na, d = Xa.shape
    nb = Xb.shape[0]
    out = np.empty((na, nb), np.float64)
    st = lib.oracle_cov_tile(_p(Xa), _p(ia), na, _p(Xb), _p(ib), nb, d, int(kern["family"]),
                             float(kern["rho"]), float(kern.get("sigma2", 1.0)),
                             float(kern.get("nugget", 0.0) or 0.0), _p(out))
    if st != 0:
        raise ValueError("oracle_cov_tile: unsupported family %r" % kern["family"])
    return out


def _panel_rows(nb, budget=1 << 27):
    """Rows per panel so one C panel holds about `budget` entries (1 GiB)."""
    return int(max(1, min(1 << 16, budget // max(nb, 1))))


def block_streamed(X, tree, basis, kern, a, b, Wa=None, Wb=None):
    """B_ab = W_a C(X_a, X_b) W_b^T = sum_P W_a[:, P] (C(X_P, X_b) W_b^T)."""
    ia = tree.perm[tree.begin[a]:tree.end[a]]
    ib = tree.perm[tree.begin[b]:tree.end[b]]
    Wa = basis.W[a] if Wa is None else Wa
    Wb = basis.W[b] if Wb is None else Wb
    Xb = np.asarray(X)[ib]
    out = np.zeros((Wa.shape[0], Wb.shape[0]))
    step = _panel_rows(ib.size)
    for s in range(0, ia.size, step):
        P = slice(s, min(s + step, ia.size))
        Cp = cov_c(np.asarray(X)[ia[P]], Xb, ia[P], ib, kern)
        out += Wa[:, P] @ (Cp @ Wb.T)
    return out


def cov_rows(X, tree, kern, a, rows):
    """(C a)[:, rows] in tree order: a is (nvec, n) in tree order, rows tree-order indices."""
    a = np.atleast_2d(a)
    ids = tree.perm
    Xt = np.asarray(X)[ids]
    rows = np.asarray(rows, dtype=np.int64)
    out = np.zeros((a.shape[0], rows.size))
    step = _panel_rows(tree.n)
    for s in range(0, rows.size, step):
        rr = rows[s:s + step]
        Cp = cov_c(Xt[rr], Xt, ids[rr], ids, kern)
        out[:, s:s + rr.size] = (Cp @ a.T).T
    return out
