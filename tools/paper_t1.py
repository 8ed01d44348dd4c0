"""The paper's Table 1 workload on the GPU (NEXT-3): timings and the C~^i_W structure (Size,
lower-triangle nz%) printed at P:3665-3668 for N = 32 000, t = 3, tau = 1e-6."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as wl
from paper_1701_00285_b200 import mlk

inp = wl.make("paper_t1"); c = inp["cfg"]
ctx = mlk.Ctx(0)
t0 = time.time()
g = mlk.build_tree(ctx, inp["X"], c["leaf"], c["tree"], inp["dirs"]); t1 = time.time()
B = mlk.build_basis(ctx, g, c["w"], index_set=c["index_set"], flags=mlk.BASIS_KEEP_DEFICIENT); B.L(); t2 = time.time()
kern = wl.kernel_dict(c)
cw = mlk.assemble_cw(ctx, g, B, kern, dict(mode=c["pairs"], tau=c["tau"])); t3 = time.time()
print("M %d dim %d; tree %.2f s basis %.2f s assemble %.2f s (%.3g pairs, %.3g flops)" % (B.M, B.dim, t1 - t0, t2 - t1, t3 - t2, cw.entries, cw.flops))
te = g.export(); brow_ptr, bcol, val_off = cw.structure()
depth = te["depth"][B.cells]
rows = np.diff(B.row_off)
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "table1_structure.json")))
for i in range(g.t, -1, -1):
    keep = depth >= i
    size = int(rows[keep].sum())
    # lower-triangle nonzeros of C~^i_W: blocks with both cells at level >= i, counted once
    nnz = 0
    for r in range(len(B.cells)):
        for k in range(brow_ptr[r], brow_ptr[r + 1]):
            cc = bcol[k]
            if keep[r] and keep[cc]:
                nnz += rows[r] * rows[cc] if r != cc else rows[r] * (rows[r] + 1) // 2
    nz = 100.0 * nnz / (size * size)
    ref = [e for e in gold["rows"] if e["N"] == 32000 and e["i"] == i]
    print("i=%d size %d nz %.2f%%  paper: %s" % (i, size, nz, ref[0] if ref else "-"))
