"""cfg5-shaped mini run (d = 50, w = 2 -> M = 1326, leaf 2048, Gaussian rho = 4 + nugget 1e-6,
tau = 1e-7) at reduced n: GPU assembly + C_W v against the oracle, with timings."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as wl
from oracle import admission as OA, assemble as OAs, basis as OB, matvec as OM, tree as OT
from paper_1701_00285_b200 import mlk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cfg = dict(wl.CONFIGS["cfg5"])
inp = wl.make(cfg, n=n)
c = inp["cfg"]; X = inp["X"]
ctx = mlk.Ctx(0)
t0 = time.time()
g = mlk.build_tree(ctx, X, c["leaf"], c["tree"], inp["dirs"]); t1 = time.time()
gb = mlk.build_basis(ctx, g, c["w"]); _ = gb.L(); t2 = time.time()
kern = wl.kernel_dict(c)
cw = mlk.assemble_cw(ctx, g, gb, kern, dict(mode=c["pairs"], tau=c["tau"])); t3 = time.time()
got = cw.export()
v = wl.vectors(1, gb.dim)
y = mlk.cw_matvec(ctx, g, gb, kern, None, mlk.MATVEC_EXACT, v); t4 = time.time()
print("gpu: tree %.2f basis %.2f assemble %.2f matvec %.2f s; M %d dim %d blocks %d" % (t1-t0, t2-t1, t3-t2, t4-t3, gb.M, gb.dim, cw.n_blocks))
o = OT.build_tree(X, c["leaf"], c["tree"], inp["dirs"])
ob = OB.build_basis(X, o, c["w"])
assert np.array_equal(g.export()["perm"], o.perm)
pairs = OA.admitted_pairs(X, o, ob, c["pairs"], c["tau"])
_, _, rp, bc, vo = OAs.bsr_structure(ob, pairs)
assert np.array_equal(got["val_off"], vo) and np.array_equal(got["bcol"], bc)
worst = 0.0
wW = 0.0
for q in ob.cells:
    Wg, _ = gb.block(q, int(o.end[q] - o.begin[q]))
    wW = max(wW, np.linalg.norm(Wg - ob.W[q]) / np.linalg.norm(ob.W[q]))
for k, (a, b) in enumerate(pairs):
    ref = OAs.block(X, o, ob, kern, a, b).ravel()
    e = np.linalg.norm(got["values"][vo[k]:vo[k+1]] - ref) / np.linalg.norm(ref)
    worst = max(worst, e)
yr = OM.cw_matvec_exact(X, o, ob, kern, v)
print("parity: W %.2e, blocks %.2e over %d, matvec %.2e" % (wW, worst, len(pairs), np.linalg.norm(y - yr) / np.linalg.norm(yr)))
