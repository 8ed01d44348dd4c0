"""Monomial index sets Lambda(w) and design matrices (oracle; test infrastructure only).

P:223-231  Q^d_h = {x^alpha : |alpha| <= h}, cardinality C(d+h, h) (total degree).
P:303-327  Table multivariate:table1: TP (max p_i <= w), TD (sum p_i <= w),
           SM (sum f(p_i) <= w), HC (prod (p_i + 1) <= w).

Ordering (paper-silent; reading R8): graded -- degree 0, then degree 1
(x_1..x_d), then each higher degree in combinations-with-replacement order
(x_1^2, x_1 x_2, ..., x_1 x_d, x_2^2, ...).  A monomial is evaluated as the
left-to-right product of its factors in that order.
"""
import itertools
import math

import numpy as np


def td_exponents(d, w):
    """Total-degree set {alpha in N^d : |alpha| <= w} in graded order (Table 1 TD)."""
    out = []
    for deg in range(w + 1):
        for combo in itertools.combinations_with_replacement(range(d), deg):
            a = [0] * d
            for k in combo:
                a[k] += 1
            out.append(tuple(a))
    return out


def td_cardinality(d, w):
    """|TD(d, w)| = C(d + w, w)."""
    return math.comb(d + w, w)


def _graded_key(a):
    """Sort key: total degree, then the factor tuple (k1 <= k2 <= ...) lexicographically.

    For TD this reproduces combinations_with_replacement order (reading R8)."""
    factors = []
    for k, e in enumerate(a):
        factors.extend([k] * e)
    return (sum(a), tuple(factors))


def hc_exponents(d, w):
    """Hyperbolic cross {alpha : prod_i (alpha_i + 1) <= w} (Table multivariate:table1).

    Enumerated by depth-first choice of the nonzero coordinates, graded order."""
    out = []

    def rec(start, budget, cur):
        out.append(tuple(cur))
        for k in range(start, d):
            e = 1
            while budget // (e + 1) >= 1 and (e + 1) <= budget:
                cur[k] = e
                rec(k + 1, budget // (e + 1), cur)
                cur[k] = 0
                e += 1

    if w >= 1:
        rec(0, w, [0] * d)
    return sorted(out, key=_graded_key)


def hc_count(d, w):
    """|HC(d, w)| = #{alpha : prod_i (alpha_i + 1) <= w} (Table multivariate:table1).

    Counted exactly by recursion over the number of nonzero coordinates: choose the
    multiset of factors (alpha_i + 1) >= 2 whose product is <= w, then the positions.
    """
    # count ordered assignments: f(k, budget) = number of alpha in N^k with prod(alpha+1) <= budget
    memo = {}

    def f(k, budget):
        if budget < 1:
            return 0
        if k == 0:
            return 1
        key = (k, budget)
        if key in memo:
            return memo[key]
        total = 0
        a = 0
        while a + 1 <= budget:
            total += f(k - 1, budget // (a + 1))
            a += 1
        memo[key] = total
        return total

    return f(d, w)


def sm_f(p):
    """Smolyak level function f(p) of Table multivariate:table1."""
    if p == 0:
        return 0
    if p == 1:
        return 1
    return math.ceil(math.log2(p))


def sm_exponents(d, w):
    """Smolyak set {alpha : sum_i f(alpha_i) <= w} (Table multivariate:table1), graded order."""
    out = []

    def rec(start, budget, cur):
        out.append(tuple(cur))
        for k in range(start, d):
            e = 1
            while sm_f(e) <= budget:
                cur[k] = e
                rec(k + 1, budget - sm_f(e), cur)
                cur[k] = 0
                e += 1

    rec(0, w, [0] * d)
    return sorted(out, key=_graded_key)


def tp_exponents(d, w):
    """Tensor-product set {alpha : max_i alpha_i <= w} (Table multivariate:table1), graded order."""
    return sorted(itertools.product(range(w + 1), repeat=d), key=_graded_key)


TD, HC, SM, TP = 0, 1, 2, 3


def exponents(kind, d, w):
    """The index set Lambda(w) of Table multivariate:table1 in graded order (R8)."""
    return {TD: td_exponents, HC: hc_exponents, SM: sm_exponents, TP: tp_exponents}[kind](d, w)


def monomials(X, exps):
    """Design matrix P(X)[i, m] = prod_k X[i, k]^alpha_m[k] (the matrix M of P:172-173).

    Each monomial is the left-to-right product of its factors in coordinate order.
    """
    X = np.asarray(X)
    n = X.shape[0]
    P = np.empty((n, len(exps)), dtype=X.dtype)
    for m, a in enumerate(exps):
        col = None
        for k, e in enumerate(a):
            for _ in range(e):
                col = X[:, k].copy() if col is None else col * X[:, k]
        P[:, m] = np.ones(n, dtype=X.dtype) if col is None else col
    return P
