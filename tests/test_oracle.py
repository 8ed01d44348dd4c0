"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Every test here checks the oracle against something other than itself: values printed in
PAPER.md (tests/golden/*.json, each with its citation), closed forms, textbook special
cases (sorting, the Haar basis, the Bessel-function Matern definition), invariants
(P P^T = I, W M = 0, Theorem 1 / interlacing, symmetry) and brute force on tiny inputs.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import workloads as wl
from oracle import admission as A
from oracle import assemble as As
from oracle import basis as Bm
from oracle import covariance as cv
from oracle import index_set as I
from oracle import matvec as Mv
from oracle import tree as T

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def small_setup(n=256, d=2, w=2, leaf=16, kind=T.KD, points="uniform", seed=0, tau=0.0,
                mode=A.PAIRS_ALL):
    X = wl.points(points, n, d, seed)
    t = T.tree_depth(n, leaf)
    dirs = wl.directions(2 ** t - 1, d, seed) if kind == T.RP else None
    tr = T.build_tree(X, leaf, kind, dirs)
    B = Bm.build_basis(X, tr, w)
    pairs = A.admitted_pairs(X, tr, B, mode, tau)
    return X, tr, B, pairs


# ----------------------------------------------------------------------------- index sets
def test_td_cardinality_formula_and_brute_force():
    for d in range(1, 6):
        for w in range(0, 5):
            bf = [a for a in itertools.product(range(w + 1), repeat=d) if sum(a) <= w]
            ex = I.td_exponents(d, w)
            assert len(ex) == len(set(ex)) == len(bf) == I.td_cardinality(d, w)
            assert sorted(ex) == sorted(bf)
    # BASELINE configs: M = 6, 66, 21, 51, 1326
    assert [I.td_cardinality(d, w) for d, w in [(2, 2), (10, 2), (20, 1), (50, 1), (50, 2)]] == \
        [6, 66, 21, 51, 1326]


def test_index_set_cardinalities_printed_in_paper():
    g = json.load(open(os.path.join(GOLD, "index_set_cardinalities.json")))
    for e in g["td"]:
        assert len(I.td_exponents(e["d"], e["w"])) == e["p"], e["cite"]
    for e in g["hc"]:
        assert len(I.hc_exponents(e["d"], e["w"])) == e["p"], e["cite"]
        assert I.hc_count(e["d"], e["w"]) == e["p"], e["cite"]


def test_hc_brute_force_small():
    for d, w in [(3, 6), (4, 8), (2, 12)]:
        bf = [a for a in itertools.product(range(w + 1), repeat=d)
              if math.prod(x + 1 for x in a) <= w]
        assert sorted(bf) == sorted(I.hc_exponents(d, w))


def test_graded_order_and_monomials():
    assert I.td_exponents(2, 2) == [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)]
    X = np.array([[2.0, 3.0], [-1.0, 0.5]])
    P = I.monomials(X, I.td_exponents(2, 2))
    assert np.array_equal(P, np.array([[1, 2, 3, 4, 6, 9], [1, -1, 0.5, 1, -0.5, 0.25]]))


# ----------------------------------------------------------------------------- covariance
@pytest.mark.parametrize("family,nu", [(cv.MATERN_12, 0.5), (cv.MATERN_32, 1.5), (cv.MATERN_52, 2.5)])
def test_matern_closed_forms_match_bessel_definition(family, nu):
    r = np.linspace(1e-4, 12.0, 2001)
    for rho in (0.5, 1.0, 3.0):
        a = cv.phi(r, family, rho)
        b = cv.matern_bessel(r, nu, rho)
        assert np.max(np.abs(a - b) / np.abs(b)) < 1e-13
    assert cv.phi(np.array([0.0]), family, 1.0)[0] == 1.0
    assert np.all(np.diff(cv.phi(r, family, 1.0)) < 0)


def test_gaussian_is_the_large_nu_limit():
    # nu -> inf gives exp(-r^2/(2 rho'^2)); BASELINE's exp(-r^2/rho^2) is rho' = rho/sqrt 2
    r = np.linspace(0.01, 3.0, 300)
    rho = 1.3
    g = cv.phi(r, cv.GAUSSIAN, rho)
    e10 = np.max(np.abs(g - cv.matern_bessel(r, 10.0, rho / math.sqrt(2.0))))
    e60 = np.max(np.abs(g - cv.matern_bessel(r, 60.0, rho / math.sqrt(2.0))))
    assert e60 < 1e-2 and e60 < e10 / 4


def test_cov_nugget_only_on_same_index():
    X = wl.points("uniform", 5, 3)
    C = cv.cov(X, X, np.arange(5), np.arange(5), cv.GAUSSIAN, 1.0, 2.0, 0.25)
    assert np.allclose(np.diag(C), 2.25)
    D = cv.cov(X, X, np.arange(5), np.arange(5) + 5, cv.GAUSSIAN, 1.0, 2.0, 0.25)
    assert np.allclose(np.diag(D), 2.0)


# ----------------------------------------------------------------------------- tree
def test_kd_tree_in_one_dimension_is_a_sort():
    rng = np.random.default_rng(5)
    for n, leaf in [(64, 4), (1000, 7), (38, 37), (38, 1)]:
        X = rng.uniform(-1, 1, (n, 1))
        tr = T.build_tree(X, leaf, T.KD)
        assert np.array_equal(tr.perm, np.argsort(X[:, 0], kind="stable"))
        xs = np.sort(X[:, 0])
        for q in range(tr.n_nodes):
            if tr.exists[q] and not tr.is_leaf[q]:
                b, e = tr.begin[q], tr.end[q]
                s = e - b
                h = (s + 1) // 2
                med = np.median(xs[b:e])
                assert tr.thr[q] == med and tr.end[2 * q + 1] - b == h


def test_tree_shape_partition_and_median():
    for name in ("cfg1",):
        inp = wl.make(name)
        c = inp["cfg"]
        tr = T.build_tree(inp["X"], c["leaf"], c["tree"], inp["dirs"])
        assert tr.t == 5 and sorted(tr.perm) == list(range(c["n"]))
        leaves = [q for q in range(tr.n_nodes) if tr.exists[q] and tr.is_leaf[q]]
        assert len(leaves) == 32 and all(tr.end[q] - tr.begin[q] == 32 for q in leaves)
    X = wl.points("normal", 3000, 7, seed=3)
    t = T.tree_depth(3000, 50)
    tr = T.build_tree(X, 50, T.RP, wl.directions(2 ** t - 1, 7, seed=3))
    for q in range(tr.n_nodes):
        if tr.exists[q] and not tr.is_leaf[q]:
            v = tr.dirs[q]
            assert abs(np.dot(v, v) - 1) < 1e-14
            pl = X[tr.perm[tr.begin[2 * q + 1]:tr.end[2 * q + 1]]] @ v
            pr = X[tr.perm[tr.begin[2 * q + 2]:tr.end[2 * q + 2]]] @ v
            assert pl.max() <= tr.thr[q] + 1e-12 and pr.min() >= tr.thr[q] - 1e-12
            allp = np.concatenate([pl, pr])
            assert abs(tr.thr[q] - np.median(allp)) < 1e-12
            sl, sr = pl.size, pr.size
            assert sl - sr in (0, 1)


def test_ragged_tree_sizes():
    X = wl.points("uniform", 1000, 3)
    tr = T.build_tree(X, 32, T.KD)
    assert tr.t == T.tree_depth(1000, 32) == 5
    for dep in range(tr.t + 1):
        sizes = [tr.end[q] - tr.begin[q] for q in range(2 ** dep - 1, 2 ** (dep + 1) - 1)
                 if tr.exists[q]]
        assert max(sizes) - min(sizes) <= 1 and sum(sizes) == 1000


def test_tree_root_leaf_and_duplicates():
    X = wl.points("uniform", 10, 2)
    tr = T.build_tree(X, 10, T.KD)
    assert tr.t == 0 and tr.is_leaf[0]
    Xd = np.vstack([X, X[3:4]])
    with pytest.raises(T.DuplicatePoints):
        T.build_tree(Xd, 4, T.KD)


# ----------------------------------------------------------------------------- basis
def test_basis_orthonormal_and_vanishing_moments_cfg1():
    inp = wl.make("cfg1")
    c = inp["cfg"]
    X = inp["X"]
    tr = T.build_tree(X, c["leaf"], c["tree"], inp["dirs"])
    B = Bm.build_basis(X, tr, c["w"])
    W = Bm.dense_W(tr, B)
    P = np.vstack([W, B.L])
    assert P.shape == (1024, 1024) and B.dim == 1018
    assert np.max(np.abs(P @ P.T - np.eye(1024))) < 1e-13
    Mx = I.monomials(X[tr.perm], B.exps)
    assert np.max(np.abs(W @ Mx)) / np.max(np.abs(Mx)) < 1e-13      # eq hbconstruction:eqn1
    assert Bm.level_rows(tr, B) == {5: 832, 4: 96, 3: 48, 2: 24, 1: 12, 0: 6}   # Lemma 1 counts


def test_subtree_basis_equals_full_basis_blocks():
    """build_subtree_basis (used for sampled cfg5 cells) reproduces build_basis exactly on every
    node of the subtree, and its W blocks are orthonormal and annihilate the monomials."""
    inp = wl.make("cfg2", n=4096)
    c = inp["cfg"]
    X = inp["X"]
    tr = T.build_tree(X, c["leaf"], c["tree"], inp["dirs"])
    B = Bm.build_basis(X, tr, c["w"])
    for root in (1, 4, 2 ** tr.t - 1):
        S = Bm.build_subtree_basis(X, tr, c["w"], root)
        assert root in S.W
        for q in S.W:
            assert np.array_equal(S.W[q], B.W[q]) and np.array_equal(S.Phi[q], B.Phi[q])
        ids = tr.perm[tr.begin[root]:tr.end[root]]
        Wr = S.W[root]
        assert np.max(np.abs(Wr @ Wr.T - np.eye(Wr.shape[0]))) < 1e-13
        Mx = I.monomials(X[ids], B.exps)
        assert np.max(np.abs(Wr @ Mx)) / np.max(np.abs(Mx)) < 1e-12


def test_table1_size_column_reproduced():
    """Size of C~^i_W = sum of rows(W_q) for q >= i, Table numericalresults:table1."""
    g = json.load(open(os.path.join(GOLD, "table1_structure.json")))
    X = wl.points("uniform", 32000, 50)
    tr = T.build_tree(X, 4000, T.RP, wl.directions(7, 50))
    B = Bm.build_basis(X, tr, 5, exps=I.hc_exponents(50, 5))
    assert B.M == g["p"]
    rows = Bm.level_rows(tr, B)
    for r in g["rows"]:
        if r["N"] == 32000:
            assert sum(rows[q] for q in rows if q >= r["i"]) == r["size"]


def test_haar_special_case():
    """w = 0, one point per leaf, d = 1: W is the orthonormal Haar basis up to signs."""
    n = 16
    X = np.sort(np.random.default_rng(1).uniform(-1, 1, (n, 1)), axis=0)
    tr = T.build_tree(X, 1, T.KD)
    B = Bm.build_basis(X, tr, 0)
    W = Bm.dense_W(tr, B)
    H = []
    for dep in range(tr.t, -1, -1):
        for q in range(2 ** dep - 1, 2 ** (dep + 1) - 1):
            s = tr.end[q] - tr.begin[q]
            if s < 2:
                continue
            h = np.zeros(n)
            h[tr.begin[q]:tr.begin[q] + s // 2] = 1.0
            h[tr.begin[q] + s // 2:tr.end[q]] = -1.0
            H.append(h / math.sqrt(s))
    H = np.array(H)
    assert W.shape == H.shape == (15, 16)
    assert np.max(np.abs(np.abs(W) - np.abs(H))) < 1e-15


def test_rank_deficient_points_raise():
    x = np.linspace(-1, 1, 64)
    X = np.stack([x, 0.5 * x], axis=1) + 0.0
    tr = T.build_tree(X, 16, T.KD)
    with pytest.raises(Bm.RankDeficient):
        Bm.build_basis(X, tr, 1)


# ----------------------------------------------------------------------------- admission
def test_tau_schedule():
    for t in range(1, 10):
        for i in range(1, t + 1):
            for j in range(i, t + 1):
                a = A.tau_ij(1e-7, t, i, j)
                assert a == A.tau_ij(1e-7, t, j, i)
                assert abs(a - 1e-7 * 2.0 ** (t - (i + j) / 2)) <= 2e-16 * a


def test_tau_zero_gives_ancestor_pattern_and_infinite_tau_all_pairs():
    X, tr, B, pairs = small_setup(n=256, d=3, w=1, leaf=16, kind=T.RP, points="normal",
                                  mode=A.PAIRS_PAPER_TAU, tau=0.0)
    assert tr.t == 4
    assert len(pairs) == tr.t * 2 ** (tr.t + 1) + 1 == A.ancestor_pattern_count(tr, B) == 129
    for a, b in pairs:
        x, y = sorted((a, b))
        while y > x:
            y = (y - 1) // 2
        assert x == y                         # one is an ancestor-or-self of the other
    allp = A.admitted_pairs(X, tr, B, A.PAIRS_PAPER_TAU, 1e9)
    nc = len(B.cells)
    assert len(allp) == nc * (nc + 1) // 2 == len(A.admitted_pairs(X, tr, B, A.PAIRS_ALL))


def _seq_dot(x, v):
    acc = x[0] * v[0]
    for k in range(1, len(x)):
        acc = acc + x[k] * v[k]
    return acc


def _path_rule_admits(X, tr, a, b, tau):
    """Independent statement of the rule: every proper ancestor q of b must let a's
    projection interval [min - tau, max + tau] reach the side of q that holds b."""
    K = X[tr.perm[tr.begin[a]:tr.end[a]]]
    node = b
    while node != 0:
        par = (node - 1) // 2
        v = tr.dirs[par]
        proj = np.array([math.fsum([0.0]) + _seq_dot(x, v) for x in K])
        if node == 2 * par + 1 and not (proj.min() - tau <= tr.thr[par]):
            return False
        if node == 2 * par + 2 and not (proj.max() + tau > tr.thr[par]):
            return False
        node = par
    return True


def test_search_matches_path_rule_brute_force():
    X, tr, B, _ = small_setup(n=192, d=3, w=1, leaf=12, kind=T.RP, points="uniform", seed=2)
    tau = 0.05
    pairs = set(A.admitted_pairs(X, tr, B, A.PAIRS_PAPER_TAU, tau))
    pos = {q: k for k, q in enumerate(B.cells)}
    expect = set()
    for a in B.cells:
        expect.add((a, a))
        i = int(tr.depth[a])
        for b in B.cells:
            j = int(tr.depth[b])
            if i == 0:
                ok = True
            elif j > i:
                ok = _path_rule_admits(X, tr, a, b, A.tau_ij(tau, tr.t, i, j))
            elif j == i:
                tij = A.tau_ij(tau, tr.t, i, j)
                ok = _path_rule_admits(X, tr, a, b, tij) or _path_rule_admits(X, tr, b, a, tij)
            else:
                continue
            if ok:
                expect.add((a, b) if pos[a] <= pos[b] else (b, a))
    assert pairs == expect
    assert len(A.ancestor_pattern_count(tr, B) * [0]) < len(pairs) < len(B.cells) ** 2


def test_admission_contains_every_geometric_neighbour():
    """Cells at levels i <= j with points closer than tau_ij are always admitted."""
    X, tr, B, _ = small_setup(n=256, d=2, w=1, leaf=16, kind=T.RP, points="uniform", seed=4)
    tau = 0.02
    pairs = set(A.admitted_pairs(X, tr, B, A.PAIRS_PAPER_TAU, tau))
    pos = {q: k for k, q in enumerate(B.cells)}
    hits = 0
    for a in B.cells:
        for b in B.cells:
            i, j = int(tr.depth[a]), int(tr.depth[b])
            if j < i:
                continue
            Xa = X[tr.perm[tr.begin[a]:tr.end[a]]]
            Xb = X[tr.perm[tr.begin[b]:tr.end[b]]]
            dmin = np.sqrt(((Xa[:, None, :] - Xb[None, :, :]) ** 2).sum(-1)).min()
            if dmin < A.tau_ij(tau, tr.t, max(i, 1), max(j, 1)) * (1 - 1e-9):
                hits += 1
                assert ((a, b) if pos[a] <= pos[b] else (b, a)) in pairs
    assert hits > 50


def _nz_pct(p_leaf, p_int, t, i):
    """Lower-triangle nonzero fraction of C~^i_W for the ancestor pattern of a balanced tree."""
    cnt = 0
    size = 0
    for dep in range(i, t + 1):
        p = p_leaf if dep == t else p_int
        size += 2 ** dep * p
        cnt += 2 ** dep * p * (p + 1) // 2                      # self blocks, lower triangle
        for anc in range(i, dep):                               # ancestor blocks (full)
            pa = p_int
            cnt += 2 ** dep * p * pa
    return 100.0 * cnt / size ** 2


def test_table1_nz_matches_ancestor_pattern_at_tiny_tau():
    """At tau = 1e-7 the printed nz% is the ancestor/descendant pattern, which
    is what the symmetric rule admits at tau -> 0 (reading R12)."""
    g = json.load(open(os.path.join(GOLD, "table1_structure.json")))
    # the pattern the oracle admits at tau = 0 on a real tree is the ancestor pattern
    X, tr, B, pairs = small_setup(n=512, d=3, w=1, leaf=32, kind=T.RP, mode=A.PAIRS_PAPER_TAU,
                                  tau=0.0)
    assert len(pairs) == A.ancestor_pattern_count(tr, B)
    for r in g["rows"]:
        if r["tau"] == 1e-7:
            leaf = r["N"] // 2 ** r["t"]
            assert round(_nz_pct(leaf - g["p"], g["p"], r["t"], r["i"]), 1) == r["nz_pct"]


# ----------------------------------------------------------------------------- assembly
def test_all_pairs_bsr_is_dense_cw_and_spectrum_interlaces():
    X, tr, B, pairs = small_setup(n=256, d=2, w=2, leaf=16)
    kern = dict(family=cv.MATERN_12, rho=0.5, sigma2=1.0, nugget=0.0)
    bsr = As.assemble(X, tr, B, kern, pairs)
    D = As.bsr_to_dense(bsr)
    CW, C, W = As.dense_cw(X, tr, B, kern)
    assert np.max(np.abs(D - CW)) < 1e-13
    assert np.max(np.abs(CW - CW.T)) < 1e-14
    lc = np.linalg.eigvalsh(C)
    lw = np.linalg.eigvalsh(CW)
    M = B.M
    assert np.all(lc[:-M] <= lw * (1 + 1e-10)) and np.all(lw <= lc[M:] * (1 + 1e-10))   # Cauchy
    assert lw[-1] / lw[0] <= lc[-1] / lc[0]                                     # Theorem 1


def test_identity_pin_gaussian_tiny_rho():
    inp = wl.make("cfg1")
    c = inp["cfg"]
    X = inp["X"]
    tr = T.build_tree(X, c["leaf"], c["tree"], inp["dirs"])
    B = Bm.build_basis(X, tr, c["w"])
    kern = dict(family=cv.GAUSSIAN, rho=1e-5, sigma2=1.0, nugget=0.0)
    CW, C, _ = As.dense_cw(X, tr, B, kern)
    assert np.array_equal(C, np.eye(1024))
    assert np.max(np.abs(CW - np.eye(B.dim))) < 1e-13


def test_polynomial_kernel_is_annihilated():
    X, tr, B, _ = small_setup(n=200, d=3, w=2, leaf=20, kind=T.RP, points="normal")
    W = Bm.dense_W(tr, B)
    Xt = X[tr.perm]
    Pm = I.monomials(Xt, B.exps)
    G = np.random.default_rng(0).standard_normal((B.M, B.M))
    kern = dict(family=cv.MATERN_32, rho=1.0)
    C = cv.cov(Xt, Xt, tr.perm, tr.perm, cv.MATERN_32, 1.0)
    a = W @ C @ W.T
    b = W @ (C + Pm @ G @ Pm.T) @ W.T
    assert np.max(np.abs(a - b)) < 1e-9 * np.max(np.abs(Pm @ G @ Pm.T))


def test_block_entries_brute_force_scalar():
    """A few entries psi_k^T C psi_l by explicit scalar double sums with math.exp/math.sqrt."""
    X, tr, B, pairs = small_setup(n=64, d=2, w=1, leaf=8, kind=T.KD)
    kern = dict(family=cv.MATERN_52, rho=0.7)
    rng = np.random.default_rng(3)
    for idx in rng.choice(len(pairs), 6, replace=False):
        a, b = pairs[idx]
        blk = As.block(X, tr, B, kern, a, b)
        ia = tr.perm[tr.begin[a]:tr.end[a]]
        ib = tr.perm[tr.begin[b]:tr.end[b]]
        k = rng.integers(B.p(a))
        l = rng.integers(B.p(b))
        s = 0.0
        for x in range(len(ia)):
            for y in range(len(ib)):
                r = math.sqrt(sum((X[ia[x], m] - X[ib[y], m]) ** 2 for m in range(2)))
                z = math.sqrt(5.0) * r / 0.7
                s += B.W[a][k, x] * (1 + z + z * z / 3) * math.exp(-z) * B.W[b][l, y]
        assert abs(s - blk[k, l]) <= 1e-12 * max(1.0, abs(s))


def test_theorem2_nested_condition_numbers():
    X, tr, B, pairs = small_setup(n=256, d=2, w=2, leaf=16)
    CW, _, _ = As.dense_cw(X, tr, B, dict(family=cv.MATERN_52, rho=0.2))
    kap = []
    for lev in range(tr.t, -1, -1):
        rows = [k for q in B.cells if tr.depth[q] >= lev
                for k in range(B.row_off[q], B.row_off[q] + B.p(q))]
        ev = np.linalg.eigvalsh(CW[np.ix_(rows, rows)])
        kap.append(ev[-1] / ev[0])
    assert all(kap[k] <= kap[k + 1] * (1 + 1e-12) for k in range(len(kap) - 1))


def test_longdouble_block_agrees_with_fp64():
    X, tr, B, pairs = small_setup(n=128, d=2, w=2, leaf=16)
    kern = dict(family=cv.MATERN_12, rho=0.5)
    for a, b in pairs[:: max(1, len(pairs) // 20)]:
        x = As.block(X, tr, B, kern, a, b)
        y = As.block(X, tr, B, kern, a, b, dtype=np.longdouble).astype(np.float64)
        assert np.linalg.norm(x - y) <= 1e-9 * np.linalg.norm(y)


# ----------------------------------------------------------------------------- matvec
def test_matvec_exact_bsr_and_round_trip():
    X, tr, B, pairs = small_setup(n=256, d=2, w=2, leaf=16)
    kern = dict(family=cv.MATERN_32, rho=0.8)
    v = np.random.default_rng(0).standard_normal((3, B.dim))
    CW, C, W = As.dense_cw(X, tr, B, kern)
    y = Mv.cw_matvec_exact(X, tr, B, kern, v)
    assert np.max(np.abs(y - v @ CW.T)) < 1e-12 * np.max(np.abs(y))
    bsr = As.assemble(X, tr, B, kern, pairs)
    yb = Mv.cw_matvec_bsr(bsr, v)
    assert np.max(np.abs(yb - y)) < 1e-12 * np.max(np.abs(y))
    x = np.random.default_rng(1).standard_normal((2, 256))
    back = Mv.apply_wt(tr, B, Mv.apply_w(tr, B, x)) + (x @ B.L.T) @ B.L
    assert np.max(np.abs(back - x)) < 1e-13
    rows = np.array([0, 17, 255])
    a = Mv.apply_wt(tr, B, v)
    assert np.allclose(Mv.cov_matvec(X, tr, kern, a, rows=rows), Mv.cov_matvec(X, tr, kern, a)[:, rows])


# ----------------------------------------------------------------------------- PCG (NEXT-1)
from oracle import pcg as Pc  # noqa: E402


def test_pcg_finite_termination_and_dense_solve():
    """CG on an SPD matrix with 3 distinct eigenvalues stops in 3 iterations (Krylov space of
    the minimal polynomial); the result equals numpy.linalg.solve."""
    rng = np.random.default_rng(7)
    Q, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    A = Q @ np.diag(np.repeat([1.0, 2.5, 7.0], [14, 13, 13])) @ Q.T
    z = rng.standard_normal(40)
    x, it, res = Pc.pcg(lambda v: A @ v, z, 1e-12, 100)
    assert it == 3 and res <= 1e-12
    assert np.linalg.norm(x - np.linalg.solve(A, z)) <= 1e-11 * np.linalg.norm(x)
    # an exact preconditioner (M = A) converges in one step
    x1, it1, _ = Pc.pcg(lambda v: A @ v, z, 1e-12, 100, precond=lambda r: np.linalg.solve(A, r))
    assert it1 == 1 and np.linalg.norm(x1 - x) <= 1e-11 * np.linalg.norm(x)


def test_pcg_cw_against_dense_system():
    """gamma_W of the PCG (with and without P_W) solves the dense C_W = W C W^T system: the true
    residual, not the recursive one, is below the tolerance, and both agree with a dense solve.
    P_W's blocks are the diagonal blocks of the dense C_W and are SPD (Theorem)."""
    X, tr, B, pairs = small_setup(n=512, d=2, w=2, leaf=32)
    kern = dict(family=cv.MATERN_12, rho=0.2)   # cond(C_W) ~ 7e2
    CW, _, _ = As.dense_cw(X, tr, B, kern)
    z = np.random.default_rng(3).standard_normal(B.dim)
    blocks = Pc.preconditioner_blocks(X, tr, B, kern)
    row_off = np.array([B.row_off[q] for q in B.cells] + [B.dim])
    for k, P in enumerate(blocks):
        a, b = row_off[k], row_off[k + 1]
        assert np.allclose(P, CW[a:b, a:b], rtol=0, atol=1e-12 * np.abs(CW).max())
        assert np.linalg.eigvalsh(P).min() > 0
    xd = np.linalg.solve(CW, z)
    its = []
    for use in (True, False):
        x, it, res = Pc.solve_cw(X, tr, B, kern, z, tol=1e-10, max_iter=2000, use_precond=use)
        its.append(it)
        assert res <= 1e-10
        assert np.linalg.norm(z - CW @ x) <= 2e-10 * np.linalg.norm(z)
        assert np.linalg.norm(x - xd) <= 1e-7 * np.linalg.norm(xd)
    assert its[0] < its[1]   # P_W pays off on this instance (63 vs 198 iterations)


def test_sm_and_tp_sets_brute_force():
    """SM and TP sets equal brute-force filters of a box with the Table 1 predicates; |TP| =
    (w + 1)^d; all four sets start with the constant and are in graded order."""
    for d, w in [(2, 3), (3, 3), (4, 2)]:
        box = list(itertools.product(range(2 ** w + 1), repeat=d))
        sm = [a for a in box if sum(I.sm_f(p) for p in a) <= w]
        assert sorted(sm) == sorted(I.sm_exponents(d, w))
        assert len(I.tp_exponents(d, w)) == (w + 1) ** d
        for kind in (I.TD, I.HC, I.SM, I.TP):
            e = I.exponents(kind, d, w)
            assert e[0] == (0,) * d and [sum(a) for a in e] == sorted(sum(a) for a in e)


@pytest.mark.parametrize("name,count", [("cfg3", 20819), ("cfg4", 13668), ("cfg5", 16803)])
def test_golden_pair_lists(name, count):
    """tests/golden/pairs_<cfg>.npz (tools/make_golden_pairs.py, oracle only) at full BASELINE
    size: unique unordered pairs in C_W order, a superset of the ancestor/descendant-or-self
    pattern (the tau = 0 structure, sum_j 2^j (j + 1) = 9217 pairs at t = 9), the root row dense
    (R21), and the count the survey measured independently on the same recipe (S§8 [M13])."""
    g = np.load(os.path.join(GOLD, "pairs_%s.npz" % name))
    P = g["pairs"]
    assert len(P) == count
    t = 9
    depth = lambda q: int(np.floor(np.log2(q + 1)))
    key = lambda q: (-depth(q), q)                        # C_W order (R11)
    assert all(key(a) <= key(b) for a, b in P)
    assert len({(int(a), int(b)) for a, b in P}) == len(P)
    S = {(int(a), int(b)) for a, b in P}
    anc = 0
    for q in range(2 ** (t + 1) - 1):
        a = q
        while True:
            pr = (q, a) if key(q) <= key(a) else (a, q)
            assert pr in S
            anc += 1
            if a == 0:
                break
            a = (a - 1) // 2
    assert anc == sum(2 ** j * (j + 1) for j in range(t + 1)) == 9217
    assert all(((0, q) in S or (q, 0) in S) for q in range(2 ** (t + 1) - 1))


from oracle import likelihood as Ll  # noqa: E402


def test_loglik_dense_matches_scipy_gaussian_logpdf():
    """The oracle's Cholesky log-likelihood equals the Gaussian
    log-density of scipy.stats on a random SPD matrix and on a small C~_W."""
    from scipy.stats import multivariate_normal
    rng = np.random.default_rng([0, 11])
    R = rng.standard_normal((40, 40))
    S = R @ R.T + 40 * np.eye(40)
    z = rng.standard_normal(40)
    l, ld, q = Ll.loglik_dense(S, z)
    assert abs(l - multivariate_normal(mean=np.zeros(40), cov=S).logpdf(z)) <= 1e-10 * abs(l)
    assert abs(ld - np.linalg.slogdet(S)[1]) <= 1e-12 * abs(ld)
    assert abs(q - z @ np.linalg.solve(S, z)) <= 1e-12 * q
    inp = wl.make("cfg1", n=256)
    c = inp["cfg"]
    X = inp["X"]
    tr = T.build_tree(X, 16, c["tree"], inp["dirs"])
    B = Bm.build_basis(X, tr, c["w"])
    kern = dict(family=cv.MATERN_12, rho=0.5)
    pairs = A.admitted_pairs(X, tr, B, A.PAIRS_PAPER_TAU, 0.05)
    bsr = As.assemble(X, tr, B, kern, pairs)
    zw = rng.standard_normal(B.dim)
    for level in (0, 2, tr.t):
        l, ld, q, nt = Ll.loglik(bsr, tr, B, zw, level)
        Ct = As.bsr_to_dense(bsr)[:nt, :nt]
        ref = multivariate_normal(mean=np.zeros(nt), cov=Ct).logpdf(zw[:nt])
        assert abs(l - ref) <= 1e-10 * abs(ref)


def test_loglik_truncation_sizes_and_identity_pin():
    """N~ per level is the Lemma 1 row count of levels t .. n (cfg1: 832, 96, 48, 24, 12, 6),
    and the identity pin (Gaussian rho = 1e-5 => C = I => C~_W = I) gives log det = 0 and
    quad = |Z^n_W|^2."""
    inp = wl.make("cfg1")
    c = inp["cfg"]
    X = inp["X"]
    tr = T.build_tree(X, c["leaf"], c["tree"], inp["dirs"])
    B = Bm.build_basis(X, tr, c["w"])
    rows = [832, 96, 48, 24, 12, 6]            # levels 5 .. 0
    for level in range(6):
        assert Ll.truncation(tr, B, level)[1] == sum(rows[:6 - level])
    kern = dict(family=cv.GAUSSIAN, rho=1e-5)
    pairs = A.admitted_pairs(X, tr, B, A.PAIRS_PAPER_TAU, 1e-7)
    bsr = As.assemble(X, tr, B, kern, pairs)
    zw = np.random.default_rng([0, 12]).standard_normal(B.dim)
    for level in (0, 3, 5):
        l, ld, q, nt = Ll.loglik(bsr, tr, B, zw, level)
        assert abs(ld) <= 1e-12 * nt and abs(q - zw[:nt] @ zw[:nt]) <= 1e-12 * q
        assert abs(l - (-0.5 * nt * np.log(2 * np.pi) - 0.5 * zw[:nt] @ zw[:nt])) <= 1e-12 * abs(l)


# ----------------------------------------------------------------------------- sm_f (NEXT-3)
def test_smolyak_level_function_pinned_to_table1():
    """f of Table multivariate:table1: f(0) = 0, f(1) = 1, f(p) = ceil(log2 p) for
    p >= 2 -- values written out by hand, so a floor/ceil or off-by-one slip fails; and
    |SM(d = 2, w = 2)| = 13 counted by hand (f-classes {0}, {1, 2}, {3, 4}: 1 + 4 + 4 + 4)."""
    expect = {0: 0, 1: 1, 2: 1, 3: 2, 4: 2, 5: 3, 6: 3, 7: 3, 8: 3, 9: 4, 15: 4, 16: 4, 17: 5, 32: 5, 33: 6}
    for p, f in expect.items():
        assert I.sm_f(p) == f, (p, I.sm_f(p), f)
    assert len(I.sm_exponents(2, 2)) == 13
    assert sorted(I.sm_exponents(2, 1)) == sorted([(0, 0), (1, 0), (0, 1), (2, 0), (0, 2)])


# ----------------------------------------------------------------------------- plain-C tiles
from oracle import fastcov as Fc  # noqa: E402


@pytest.mark.parametrize("family", [cv.MATERN_12, cv.MATERN_32, cv.MATERN_52, cv.GAUSSIAN])
def test_fastcov_tile_equals_numpy_cov(family):
    """The C tile (oracle/csrc/cov_tile.c) is oracle.covariance.cov written out: same entries
    (to the last bits of the k-sum order), nugget only where the global indices agree, ragged
    shapes that are not multiples of its 16 x 512 loop blocking."""
    rng = np.random.default_rng([1, 7])
    Xa = rng.standard_normal((37, 11))
    Xb = np.vstack([rng.standard_normal((1000, 11)), Xa[:5]])
    ia = np.arange(37) + 1000
    ib = np.concatenate([np.arange(1000), ia[:5]])
    kern = dict(family=family, rho=1.7, sigma2=1.3, nugget=1e-3)
    got = Fc.cov_c(Xa, Xb, ia, ib, kern)
    ref = cv.cov(Xa, Xb, ia, ib, family, 1.7, 1.3, 1e-3)
    assert np.max(np.abs(got - ref)) <= 4e-16 * 1.3
    assert np.all(np.abs(got[np.arange(5), 1000 + np.arange(5)] - (1.3 + 1e-3)) <= 1e-15)


def test_fastcov_block_streamed_brute_force_and_panels(monkeypatch):
    """block_streamed = W_a C W_b^T: against oracle.assemble.block on every admitted block
    (with one-row panels forced, so the panel sum is exercised), against explicit scalar
    double sums with math.exp, and the identity pin (Gaussian rho = 1e-5: C = I, so the self
    block is W_a W_a^T = I)."""
    X, tr, B, pairs = small_setup(n=96, d=3, w=1, leaf=12, kind=T.RP, points="normal")
    kern = dict(family=cv.MATERN_12, rho=0.9, sigma2=1.1)
    monkeypatch.setattr(Fc, "_panel_rows", lambda nb, budget=0: 7)
    for a, b in pairs:
        ref = As.block(X, tr, B, kern, a, b)
        got = Fc.block_streamed(X, tr, B, kern, a, b)
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    a, b = pairs[len(pairs) // 2]
    blk = Fc.block_streamed(X, tr, B, kern, a, b)
    ia = tr.perm[tr.begin[a]:tr.end[a]]
    ib = tr.perm[tr.begin[b]:tr.end[b]]
    s = 0.0
    for x in range(len(ia)):
        for y in range(len(ib)):
            r = math.sqrt(sum((X[ia[x], m] - X[ib[y], m]) ** 2 for m in range(3)))
            s += B.W[a][0, x] * 1.1 * math.exp(-r / 0.9) * B.W[b][0, y]
    assert abs(s - blk[0, 0]) <= 1e-12 * max(1.0, abs(s))
    eye = Fc.block_streamed(X, tr, B, dict(family=cv.GAUSSIAN, rho=1e-5), a, a)
    assert np.max(np.abs(eye - np.eye(B.p(a)))) < 1e-14


def test_fastcov_rows_equal_panel_matvec():
    X, tr, B, pairs = small_setup(n=300, d=4, w=1, leaf=20, kind=T.RP, points="uniform")
    kern = dict(family=cv.MATERN_52, rho=0.6, nugget=1e-4)
    a = np.random.default_rng(2).standard_normal((2, 300))
    rows = np.array([0, 5, 150, 299])
    ref = Mv.cov_matvec(X, tr, kern, a, rows=rows)
    got = Fc.cov_rows(X, tr, kern, a, rows)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_full_size_goldens_match_the_sample(name):
    """tests/golden/blocks_<cfg>.npz holds exactly the expensive blocks of tests/sampling.py's
    fixed sample (so the GPU test checks what the golden script computed), each with the block
    shape p_a x p_b of the oracle's cell sizes; matvec_<cfg>.npz holds a y of length n - M."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import sampling
    inp = wl.make(name)
    c = inp["cfg"]
    tr = T.build_tree(inp["X"], c["leaf"], c["tree"], inp["dirs"])
    gp = os.path.join(GOLD, "pairs_%s.npz" % name)
    if os.path.exists(gp):
        pairs = [tuple(int(v) for v in p) for p in np.load(gp)["pairs"]]
    else:
        B = Bm.build_basis(inp["X"], tr, c["w"])
        pairs = A.admitted_pairs(inp["X"], tr, B, c["pairs"], c["tau"])
    g = np.load(os.path.join(GOLD, "blocks_%s.npz" % name))
    idx = sampling.select_blocks(name, pairs, tr)
    need = sampling.golden_needed(pairs, tr, idx)
    assert list(g["index"]) == need and len(need) >= 1
    M = math.comb(c["d"] + c["w"], c["w"])
    p = lambda q: (tr.end[q] - tr.begin[q]) - M if tr.is_leaf[q] else M
    for k in need:
        a, b = pairs[k]
        assert g["k%d" % k].shape == (p(a), p(b))
    root = [k for k, (a, b) in enumerate(pairs) if a == 0 and b == 0]
    assert root[0] in need
    mv = np.load(os.path.join(GOLD, "matvec_%s.npz" % name))
    assert mv["y_exact"].shape == (c["n"] - M,)


def test_cfg5_entries_golden_structure():
    """tests/golden/entries_cfg5.npz (tools/make_golden_cfg5.py, oracle only): 4 x 4 seeded
    entries psi_k^T C psi_l of the level-1 blocks B_11 and B_12 at full cfg5 size, with row and
    column indices inside the cells' wavelet counts (M = 1326 for internal cells) and finite,
    non-trivial values (checked against the GPU by tools/cfg5_all_ranks.py,
    profiles/cfg5_level1_entries_r02.json)."""
    g = np.load(os.path.join(GOLD, "entries_cfg5.npz"))
    assert sorted(tuple(int(v) for v in b) for b in g["blocks"]) == [(1, 1), (1, 2)]
    for p, q in ((1, 1), (1, 2)):
        e = g["entries_%d_%d" % (p, q)]
        assert e.shape == (4, 4) and np.all(np.isfinite(e)) and np.max(np.abs(e)) > 0
        assert np.all(g["rows_%d_%d" % (p, q)] < 1326) and np.all(g["cols_%d_%d" % (p, q)] < 1326)
    # the diagonal block's entries with equal row and column index are psi_k^T C psi_k > 0
    r, c = g["rows_1_1"], g["cols_1_1"]
    e = g["entries_1_1"]
    for i in range(4):
        for j in range(4):
            if r[i] == c[j]:
                assert e[i, j] > 0
