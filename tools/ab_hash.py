"""Hash of the basis (L, all W blocks) and the assembled values of a config for the library
selected by MLK_LIB_VARIANT (A/B bit-identity checks of refactorings)."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1701_00285_b200 import mlk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
inp = wl.make(name)
c = inp["cfg"]
ctx = mlk.Ctx(0)
tr = mlk.build_tree(ctx, inp["X"], c["leaf"], c["tree"], inp["dirs"])
B = mlk.build_basis(ctx, tr, c["w"])
h = hashlib.sha256()
h.update(B.L().tobytes())
e = tr.export()
for q in B.cells:
    h.update(B.block(int(q), int(e["end"][q] - e["begin"][q]), phi=False)[0].tobytes())
cw = mlk.assemble_cw(ctx, tr, B, wl.kernel_dict(c), dict(mode=c["pairs"], tau=c["tau"]))
h.update(cw.export()["values"].tobytes())
print(name, os.environ.get("MLK_LIB_VARIANT", "default"), h.hexdigest())
