"""Write the expensive full-size oracle references used by tests/test_gpu_parity.py:

  tests/golden/blocks_<cfg>.npz   B_ab = W_a C(X_a, X_b) W_b^T for the sampled blocks of
                                  tests/sampling.py whose evaluation exceeds 2^26 covariance
                                  entries (the root-root block, level <= 2 blocks, ...)
  tests/golden/matvec_<cfg>.npz   y = C_W v, EXACT three-step product for
                                  v = workloads.vectors(1, dim, seed=0); for cfg2 also the BSR
                                  product C~_W v on all admitted blocks

Calls only oracle/ (tree, basis, admission, the plain-C direct-difference tile of
oracle/fastcov.py) and workloads/ (the seeded input recipe): no value comes from the GPU path.

    python tools/make_golden_blocks.py cfg2 cfg3 cfg4
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import sampling  # noqa: E402
import workloads as wl  # noqa: E402
from oracle import admission as OA  # noqa: E402
from oracle import assemble as OAs  # noqa: E402
from oracle import basis as OB  # noqa: E402
from oracle import fastcov as F  # noqa: E402
from oracle import matvec as OM  # noqa: E402
from oracle import tree as OT  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def oracle_setup(name):
    inp = wl.make(name)
    c = inp["cfg"]
    X = inp["X"]
    tr = OT.build_tree(X, c["leaf"], c["tree"], inp["dirs"])
    B = OB.build_basis(X, tr, c["w"])
    gp = os.path.join(GOLD, "pairs_%s.npz" % name)
    if os.path.exists(gp):
        pairs = [tuple(int(v) for v in p) for p in np.load(gp)["pairs"]]
    else:
        pairs = OA.admitted_pairs(X, tr, B, c["pairs"], c["tau"])
    return inp, c, X, tr, B, pairs


def main(names):
    for name in names:
        t0 = time.time()
        inp, c, X, tr, B, pairs = oracle_setup(name)
        kern = wl.kernel_dict(c)
        print("%s: oracle tree/basis/pairs %.0f s (%d pairs)" % (name, time.time() - t0, len(pairs)), flush=True)
        idx = sampling.select_blocks(name, pairs, tr)
        need = sampling.golden_needed(pairs, tr, idx)
        out = {}
        # reuse blocks an earlier run of this script already wrote (same pair index and cells)
        old_path = os.path.join(GOLD, "blocks_%s.npz" % name)
        old = {}
        if os.path.exists(old_path):
            g = np.load(old_path)
            old = {int(k): (tuple(int(v) for v in p), g["k%d" % k]) for k, p in zip(g["index"], g["pairs"])}
        for k in need:
            a, b = pairs[k]
            if k in old and old[k][0] == (a, b):
                out["k%d" % k] = old[k][1]
                continue
            t1 = time.time()
            out["k%d" % k] = F.block_streamed(X, tr, B, kern, a, b)
            print("  block %d (%d, %d) |a||b| = %.2e: %.0f s" % (k, a, b, sampling.size(tr, a) * sampling.size(tr, b),
                                                               time.time() - t1), flush=True)
        np.savez_compressed(os.path.join(GOLD, "blocks_%s.npz" % name), index=np.array(need, np.int64),
                            pairs=np.array([pairs[k] for k in need], np.int32),
                            source="oracle.fastcov.block_streamed on workloads.make('%s') (seed 0), "
                                   "tools/make_golden_blocks.py" % name, **out)
        if os.environ.get("GOLDEN_BLOCKS_ONLY"):
            continue
        # C_W v, EXACT: y = W (C (W^T v)) with C a by row panels of the C tile
        v = wl.vectors(1, B.dim, seed=0)
        t1 = time.time()
        a = OM.apply_wt(tr, B, v)
        b = F.cov_rows(X, tr, kern, a, np.arange(tr.n))
        y = OM.apply_w(tr, B, b)
        mv = dict(v_seed=0, y_exact=y[0])
        print("  EXACT C_W v: %.0f s" % (time.time() - t1), flush=True)
        if name == "cfg2":
            t1 = time.time()
            cells, row_off, brow_ptr, bcol, val_off = OAs.bsr_structure(B, pairs)
            values = np.zeros(int(val_off[-1]))
            for k, (pa, pb) in enumerate(pairs):
                values[val_off[k]:val_off[k + 1]] = F.block_streamed(X, tr, B, kern, pa, pb).ravel()
            bsr = OAs.BSR(cells, row_off, brow_ptr, bcol, val_off, values)
            mv["y_bsr"] = OM.cw_matvec_bsr(bsr, v)[0]
            print("  BSR C~_W v (all %d blocks): %.0f s" % (len(pairs), time.time() - t1), flush=True)
        np.savez_compressed(os.path.join(GOLD, "matvec_%s.npz" % name),
                            source="oracle (apply_wt, fastcov.cov_rows, apply_w%s) on workloads.make('%s'), "
                                   "tools/make_golden_blocks.py" % (", BSR of fastcov blocks" if name == "cfg2" else "",
                                                                    name), **mv)
        print("%s done in %.0f s" % (name, time.time() - t0), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg3", "cfg4"])
