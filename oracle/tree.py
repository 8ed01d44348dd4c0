"""Binary median-split tree: MakeTree + ChooseRule (oracle; test infrastructure only).

P:1005-1031  root B^0_0 holds all observations; split a cell by projecting onto a unit
             vector v and splitting at the median of the projections; repeat until a cell
             holds at most the leaf size.
P:1037-1069  Algorithm 1 MakeTree (node number, currentdepth, threshold, v per cell).
P:1071-1084  Algorithm 2 ChooseRule (RP): random unit v, Rule(x) := x.v <= median.
P:1086-1097  Algorithm 2-kd ChooseRule (kD): a coordinate direction.

Readings:
  R1  leaf iff |cell| <= leaf_size.
  R2  threshold = median of the projections (midpoint of the two middle values when the
      cell size s is even).  Membership by rank: sort the cell by (projection, original
      id); the first ceil(s/2) go left, the rest right, each keeping that sorted order.
  R3  RP directions are inputs (one unit row per heap index of an internal node).
  R4  kD axis = depth mod d.
  R5  nodes are numbered in heap (BFS) order: children of q are 2q+1, 2q+2.
  R6  projections are x_0 v_0 (+) x_1 v_1 (+) ... summed left to right, every product and
      sum rounded separately (no fused multiply-add).
Distinct sites are required: duplicate rows raise DuplicatePoints.
"""
from dataclasses import dataclass

import numpy as np

KD, RP = 0, 1


class DuplicatePoints(ValueError):
    pass


def tree_depth(n, leaf_size):
    """Depth t of the tree: the smallest delta with ceil(n / 2^delta) <= leaf_size (R1, R2)."""
    t = 0
    s = n
    while s > leaf_size:
        s = (s + 1) // 2
        t += 1
    return t


def project(Xs, v):
    """p_i = sum_k Xs[i,k] v[k], summed left to right without FMA (reading R6)."""
    acc = Xs[:, 0] * v[0]
    for k in range(1, Xs.shape[1]):
        acc = acc + Xs[:, k] * v[k]
    return acc


@dataclass
class Tree:
    n: int
    d: int
    t: int                 # maximal depth
    n_nodes: int           # heap slots 2^(t+1) - 1
    exists: np.ndarray     # bool[n_nodes]
    is_leaf: np.ndarray    # bool[n_nodes]
    begin: np.ndarray      # int64[n_nodes], range in perm
    end: np.ndarray        # int64[n_nodes]
    depth: np.ndarray      # int32[n_nodes]
    thr: np.ndarray        # float64[n_nodes] (NaN for leaves / missing)
    dirs: np.ndarray       # float64[n_nodes, d] (0 rows for leaves / missing)
    perm: np.ndarray       # int64[n]: tree position -> original index

    def children(self, q):
        return 2 * q + 1, 2 * q + 2


def check_distinct(X):
    """Distinct observation sites."""
    if np.unique(X, axis=0).shape[0] != X.shape[0]:
        raise DuplicatePoints("duplicate observation locations")


def build_tree(X, leaf_size, kind, directions=None):
    """Algorithm 1 with ChooseRule RP (Alg 2) or kD (Alg 2-kd), nodes in heap order (R5)."""
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    if n < 1 or d < 1 or leaf_size < 1:
        raise ValueError("invalid arguments")
    check_distinct(X)
    t = tree_depth(n, leaf_size)
    n_nodes = 2 ** (t + 1) - 1
    exists = np.zeros(n_nodes, bool)
    is_leaf = np.zeros(n_nodes, bool)
    begin = np.zeros(n_nodes, np.int64)
    end = np.zeros(n_nodes, np.int64)
    depth = np.zeros(n_nodes, np.int32)
    thr = np.full(n_nodes, np.nan)
    dirs = np.zeros((n_nodes, d))
    perm = np.arange(n, dtype=np.int64)
    if kind == RP:
        directions = np.asarray(directions, dtype=np.float64)
        if directions.shape[0] < 2 ** t - 1 or directions.shape[1] != d:
            raise ValueError("RP tree needs one direction per internal heap node")
    exists[0] = True
    begin[0], end[0] = 0, n
    for q in range(n_nodes):                      # heap order == BFS order
        if not exists[q]:
            continue
        depth[q] = (q + 1).bit_length() - 1
        b, e = begin[q], end[q]
        s = e - b
        if s <= leaf_size:                        # R1
            is_leaf[q] = True
            continue
        if kind == KD:                            # Alg 2-kd, R4
            v = np.zeros(d)
            v[depth[q] % d] = 1.0
        else:                                     # Alg 2, R3
            v = directions[q]
        ids = perm[b:e]
        p = project(X[ids], v)                    # R6
        order = np.lexsort((ids, p))              # sort by (projection, original id)
        ids, p = ids[order], p[order]
        perm[b:e] = ids
        h = (s + 1) // 2
        thr[q] = p[h - 1] if s % 2 == 1 else (p[h - 1] + p[h]) / 2   # R2 median
        dirs[q] = v
        lq, rq = 2 * q + 1, 2 * q + 2
        exists[lq] = exists[rq] = True
        begin[lq], end[lq] = b, b + h
        begin[rq], end[rq] = b + h, e
    return Tree(n, d, t, n_nodes, exists, is_leaf, begin, end, depth, thr, dirs, perm)
