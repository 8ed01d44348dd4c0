"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module is shared by the tests, the oracle side and the GPU side.  It holds only the
random input recipes (points, RP tree directions, matvec vectors) and plain configuration
parameters -- none of the method's arithmetic.  The paper's own data sets are synthetic
recipes too (random hypercube and n-sphere points); none is a file.

Random streams are NumPy PCG64 (`np.random.default_rng`).  Random unit directions of the
RP tree (Alg 2 "choose a random unit vector") are drawn here and passed to both
implementations, which use them as given.
"""
import math

import numpy as np

KD, RP = 0, 1
MATERN_12, MATERN_32, MATERN_52, GAUSSIAN, MATERN_NU = 0, 1, 2, 3, 4
PAIRS_ALL, PAIRS_PAPER_TAU = 0, 1

CONFIGS = {
    "cfg1": dict(n=1024, d=2, w=2, leaf=32, tree=KD, family=MATERN_12, rho=0.5, sigma2=1.0,
                 nugget=0.0, pairs=PAIRS_ALL, tau=0.0, points="uniform"),
    "cfg2": dict(n=32768, d=10, w=2, leaf=256, tree=RP, family=MATERN_32, rho=1.0, sigma2=1.0,
                 nugget=0.0, pairs=PAIRS_PAPER_TAU, tau=1e-6, points="uniform"),
    "cfg2_dense": dict(n=32768, d=10, w=2, leaf=256, tree=RP, family=MATERN_32, rho=1.0,
                       sigma2=1.0, nugget=0.0, pairs=PAIRS_ALL, tau=0.0, points="uniform"),
    "cfg3": dict(n=131072, d=20, w=1, leaf=256, tree=RP, family=MATERN_52, rho=2.0, sigma2=1.0,
                 nugget=0.0, pairs=PAIRS_PAPER_TAU, tau=1e-7, points="normal", nvec=10),
    "cfg4": dict(n=262144, d=50, w=1, leaf=512, tree=RP, family=MATERN_12, rho=3.0, sigma2=1.0,
                 nugget=0.0, pairs=PAIRS_PAPER_TAU, tau=1e-7, points="mixture"),
    "cfg5": dict(n=1048576, d=50, w=2, leaf=2048, tree=RP, family=GAUSSIAN, rho=4.0, sigma2=1.0,
                 nugget=1e-6, pairs=PAIRS_PAPER_TAU, tau=1e-7, points="uniform"),
    # NEXT-3: the paper's own Table 1 workload: N = 32 000 points on
    # the sphere S^49 (d = 50), hyperbolic cross w = 5 (p = 1426), Matern nu = 1.25, rho = 10,
    # RP tree with t = 3 (leaf 4000), tau = 1e-6
    "paper_t1": dict(n=32000, d=50, w=5, leaf=4000, tree=RP, family=MATERN_NU, rho=10.0, sigma2=1.0,
                     nugget=0.0, pairs=PAIRS_PAPER_TAU, tau=1e-6, points="sphere", index_set=1, nu=1.25),
}


def tree_levels(n, leaf):
    """Number of split levels t (pure integer shape arithmetic: sizes ceil(s/2), floor(s/2))."""
    t, s = 0, n
    while s > leaf:
        s = (s + 1) // 2
        t += 1
    return t


def points(kind, n, d, seed=0):
    """Observation locations X (n x d, float64)."""
    r = np.random.default_rng([seed, 0])
    if kind == "uniform":                     # random hypercube [-1,1]^d
        return r.uniform(-1.0, 1.0, (n, d))
    if kind == "normal":                      # N(0, I_d) (BASELINE cfg3)
        return r.standard_normal((n, d))
    if kind == "mixture":                     # 8-component isotropic mixture (BASELINE cfg4)
        means = r.uniform(-3.0, 3.0, (8, d))
        labels = r.integers(0, 8, n)
        return means[labels] + 0.5 * r.standard_normal((n, d))
    if kind == "sphere":                      # random n-sphere S^{d-1}
        g = r.standard_normal((n, d))
        return g / np.sqrt(np.sum(g * g, axis=1, keepdims=True))
    raise ValueError(kind)


def directions(n_rows, d, seed=0):
    """Unit directions for the RP tree, one row per heap index of an internal node."""
    G = np.random.default_rng([seed, 1]).standard_normal((max(n_rows, 1), d))
    out = np.empty_like(G)
    for k in range(G.shape[0]):
        out[k] = G[k] / np.sqrt(np.sum(G[k] * G[k]))
    return out


def vectors(nvec, dim, seed=0):
    """Random N(0,1) vectors for C_W v (BASELINE cfg3: 10 vectors)."""
    return np.random.default_rng([seed, 2]).standard_normal((nvec, dim))


def make(name_or_cfg, n=None, seed=0):
    """Inputs for a config (optionally with a smaller n): dict(X, dirs, cfg)."""
    cfg = dict(CONFIGS[name_or_cfg]) if isinstance(name_or_cfg, str) else dict(name_or_cfg)
    if n is not None:
        cfg["n"] = n
    X = points(cfg["points"], cfg["n"], cfg["d"], seed)
    t = tree_levels(cfg["n"], cfg["leaf"])
    dirs = directions(2 ** t - 1, cfg["d"], seed) if cfg["tree"] == RP else None
    return dict(X=X, dirs=dirs, cfg=cfg, t=t)


def kernel_dict(cfg):
    return dict(family=cfg["family"], rho=cfg["rho"], sigma2=cfg["sigma2"], nugget=cfg["nugget"],
                nu=cfg.get("nu"))


def mtd(d, w):
    return math.comb(d + w, w)
