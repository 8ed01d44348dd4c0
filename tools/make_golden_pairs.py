"""Write tests/golden/pairs_<cfg>.npz: the oracle's admitted pair list (Algorithm 6 with the
symmetric rule R12, tau_ij of R15) for a BASELINE configuration at full size.

Calls only oracle/ and workloads/ (the seeded input recipe); the GPU path never writes a
golden value.  The oracle search takes ~1 min (cfg3) / ~5 min (cfg4) on 16 host cores, which
is why the full-size parity tests read the list instead of recomputing it.

    python tools/make_golden_pairs.py cfg3 cfg4 cfg5
"""
import os
import sys
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402
from oracle import admission as OA  # noqa: E402
from oracle import basis as OB  # noqa: E402
from oracle import tree as OT  # noqa: E402


def main(names):
    for name in names:
        t0 = time.time()
        inp = wl.make(name)
        c = inp["cfg"]
        X = inp["X"]
        tr = OT.build_tree(X, c["leaf"], c["tree"], inp["dirs"])
        if name == "cfg5":
            # the oracle basis at n = 2^20, M = 1326 (~110 GB of Phi blocks) does not fit this
            # host; the search only needs the C_W cell order (R11), and every cfg5 cell has
            # p > 0 (leaves 2048 - 1326 = 722, internal cells M), so the order is all nodes by
            # (deepest level first, heap index) -- the rule oracle.basis.build_basis applies
            order = sorted((q for q in range(tr.n_nodes) if tr.exists[q]), key=lambda q: (-int(tr.depth[q]), q))
            B = types.SimpleNamespace(cells=order)
        else:
            B = OB.build_basis(X, tr, c["w"])
        pairs = np.array(OA.admitted_pairs(X, tr, B, c["pairs"], c["tau"]), dtype=np.int32)
        out = os.path.join(ROOT, "tests", "golden", "pairs_%s.npz" % name)
        np.savez_compressed(out, pairs=pairs, n=c["n"], d=c["d"], leaf=c["leaf"], w=c["w"], tau=c["tau"],
                            source="oracle.admission.admitted_pairs on workloads.make('%s') (seed 0), "
                                   "tools/make_golden_pairs.py" % name)
        print("%s: %d pairs in %.0f s -> %s" % (name, len(pairs), time.time() - t0, out))


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg3", "cfg4"])
