"""cfg5 (n = 2^20, d = 50, w = 2 -> M = 1326, leaf 2048, Gaussian rho = 4 + nugget 1e-6) oracle
entries psi_k^T C psi_l of the level-1 blocks B_11 and B_12 (S§8(c) "large configs": "8 single
entries psi_a^T C psi_b with a, b at levels 0-1") -> tests/golden/entries_cfg5.npz.

The full oracle basis at cfg5 (W 106 GB + Phi 11 GB per level) does not fit this host, so the
basis is built level by level with the oracle's own node step (oracle.basis._node_step, steps
(a)-(e) of P:1427-1515): a node's Phi / R are dropped once its parent exists, W is kept only for
the cells 1 and 2.  Then for each block (a, b) in ((1, 1), (1, 2)) one pass over C(X_a, X_b) in
row panels (oracle.fastcov: direct differences, plain C) gives U = C(X_a, X_b) psi_l^T for NCOL
rows l of W_b, and B_ab[k, l] = psi_k U[:, l] for NROW rows k of W_a: NROW x NCOL entries of
each block.  Rows k, l are seeded (default_rng([0, 3, 5])).  Calls only oracle/ and workloads/.
Each C pass is 2.7e11 covariance entries (~1 h on 8 host cores).

    OMP_NUM_THREADS=6 python tools/make_golden_cfg5.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402
from oracle import basis as OB  # noqa: E402
from oracle import fastcov as F  # noqa: E402
from oracle import tree as OT  # noqa: E402
from oracle.index_set import td_exponents  # noqa: E402

NROW, NCOL = 4, 4
BLOCKS = ((1, 1), (1, 2))
OUT = os.path.join(ROOT, "tests", "golden", "entries_cfg5.npz")


def streamed_basis(X, tr, w, keep, top=1):
    """W of the cells in `keep`, by the oracle's node step, finest level first up to depth
    `top`, dropping every node's Phi / R as soon as its parent has been formed (the root level,
    which the level-1 blocks do not need, would take ~50 GB of dense NumPy temporaries)."""
    exps = td_exponents(tr.d, w)
    B = OB.Basis(M=len(exps), exps=exps)
    for dep in range(tr.t, top - 1, -1):
        t0 = time.time()
        nodes = [q for q in range(2 ** dep - 1, 2 ** (dep + 1) - 1) if q < tr.n_nodes and tr.exists[q]]
        for q in nodes:
            OB._node_step(X, tr, exps, B, q)
            if q not in keep:
                del B.W[q]
            if not tr.is_leaf[q]:
                for ch in (2 * q + 1, 2 * q + 2):
                    B.Phi.pop(ch, None)
                    B.R.pop(ch, None)
        print("  level %d: %d nodes in %.0f s" % (dep, len(nodes), time.time() - t0), flush=True)
    return B


def main():
    t0 = time.time()
    inp = wl.make("cfg5")
    c = inp["cfg"]
    X = inp["X"]
    tr = OT.build_tree(X, c["leaf"], c["tree"], inp["dirs"])
    print("tree %.0f s" % (time.time() - t0), flush=True)
    B = streamed_basis(X, tr, c["w"], keep={1, 2})
    kern = wl.kernel_dict(c)
    rng = np.random.default_rng([0, 3, 5])
    out = {}
    for a, b in BLOCKS:
        rows = np.sort(rng.choice(B.W[a].shape[0], NROW, replace=False))
        cols = np.sort(rng.choice(B.W[b].shape[0], NCOL, replace=False))
        t1 = time.time()
        ent = F.block_streamed(X, tr, B, kern, a, b, Wa=B.W[a][rows], Wb=B.W[b][cols])
        print("  block (%d, %d): %d x %d entries in %.0f s" % (a, b, NROW, NCOL, time.time() - t1), flush=True)
        out["rows_%d_%d" % (a, b)] = rows
        out["cols_%d_%d" % (a, b)] = cols
        out["entries_%d_%d" % (a, b)] = ent
        np.savez_compressed(OUT, blocks=np.array([p for p in BLOCKS if "entries_%d_%d" % p in out], np.int32),
                            source="oracle (tree, basis node steps, fastcov C tiles) on workloads.make('cfg5'), "
                                   "tools/make_golden_cfg5.py", **out)
    print("done in %.0f s -> %s" % (time.time() - t0, OUT), flush=True)


if __name__ == "__main__":
    main()
