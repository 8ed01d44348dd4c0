"""Admission of cell pairs (oracle; test infrastructure only).

P:1655-1668  for a cell K = B^l_k, the Targetdepth is the desired tree level.
P:1669-1683  find the cells at Targetdepth that overlap a ball of radius tau around the
             projections of the points of K onto Tree.v, searching from the root.
P:1685-1737  Algorithms 3 (SearchTree), 4 (LocalSearchTree), 5 (ChooseSecondRule).
P:1771-1775  symmetry: only blocks with j >= i are computed.
P:1777-1800  Algorithm 6: for every cell B^i_m at level i, the cells B^j_q returned by
             LocalSearchTree(Tree, K = B^i_m, Targetdepth, tau_{i,j}) are admitted.
P:3130-3134  levels -1 and 0 are never truncated (E^{i,j} = 0 for i or j in {-1, 0}).
P:3140-3143  Assumption: tau_{i,j} = tau 2^{t - (i+j)/2}; P:3541-3546 the same radius.

Readings:
  R12 symmetric projection rule: at node (v, thr) with projections of K onto v,
      descend left iff min - tau <= thr and right iff max + tau > thr.
  R13 Alg 6's "Targetdepth(i)" is read as Targetdepth(j).
  R14 i < j: the level-i cell searches; i = j: the union of both directions.
      Self pairs are always admitted.
  R15 tau_{i,j} computed exactly as ldexp(tau, floor(e/2)) * (sqrt(2) if e odd), e = 2t-i-j.
  R21 pairs involving the root (level 0) are always admitted.
Output: unordered pairs {a, b} stored as (row, col) with row the cell that comes first in
C_W order, sorted by (row position, col position).
"""
import math

import numpy as np

from .tree import project

PAIRS_ALL, PAIRS_PAPER_TAU = 0, 1


def tau_ij(tau, t, i, j):
    """tau_{i,j} = tau 2^{t-(i+j)/2}, reading R15."""
    e = 2 * t - i - j
    return math.ldexp(tau, e // 2) * (math.sqrt(2.0) if e % 2 else 1.0)


def local_search(X, tree, K_ids, target_depth, tau, node, out):
    """Algorithm 4 LocalSearchTree with the ChooseSecondRule of Algorithm 5 (reading R12)."""
    if tree.depth[node] == target_depth:
        out.append(node)
        return
    if tree.is_leaf[node]:
        return
    p = project(X[K_ids], tree.dirs[node])
    if p.min() - tau <= tree.thr[node]:
        local_search(X, tree, K_ids, target_depth, tau, 2 * node + 1, out)
    if p.max() + tau > tree.thr[node]:
        local_search(X, tree, K_ids, target_depth, tau, 2 * node + 2, out)


def search_tree(X, tree, K_ids, target_depth, tau):
    """Algorithm 3 SearchTree."""
    out = []
    local_search(X, tree, K_ids, target_depth, tau, 0, out)
    return out


def admitted_pairs(X, tree, basis, mode, tau=0.0):
    """Algorithm 6 admission over all level pairs j >= i, readings R12-R15, R21."""
    X = np.asarray(X, dtype=np.float64)
    cells = basis.cells
    pos = {q: k for k, q in enumerate(cells)}
    has = set(cells)
    pairs = set()

    def add(a, b):
        if a in has and b in has:
            pairs.add((a, b) if pos[a] <= pos[b] else (b, a))

    if mode == PAIRS_ALL:
        for x in range(len(cells)):
            for y in range(x, len(cells)):
                pairs.add((cells[x], cells[y]))
    elif mode == PAIRS_PAPER_TAU:
        t = tree.t
        for a in cells:
            add(a, a)                                   # R14 self pairs
            if tree.depth[a] == 0:                      # R21 root row/column dense
                for b in cells:
                    add(a, b)
                continue
            i = int(tree.depth[a])
            K = tree.perm[tree.begin[a]:tree.end[a]]
            for j in range(i, t + 1):
                for b in search_tree(X, tree, K, j, tau_ij(tau, t, i, j)):
                    add(a, b)
    else:
        raise ValueError("unknown mode")
    return sorted(pairs, key=lambda ab: (pos[ab[0]], pos[ab[1]]))


def ancestor_pattern_count(tree, basis):
    """Number of unordered ancestor/descendant-or-self pairs among cells with wavelets."""
    cells = set(basis.cells)
    cnt = 0
    for a in cells:
        q = a
        while True:
            if q in cells:
                cnt += 1
            if q == 0:
                break
            q = (q - 1) // 2
    return cnt
