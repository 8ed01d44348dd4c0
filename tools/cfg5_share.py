"""BASELINE cfg5 at full size (n = 2^20, d = 50, M = 1326, leaf 2048, Gaussian rho = 4 + nugget
1e-6, tau = 1e-7) on ONE B200: the share of rank `--rank` of an `--nranks`-rank job.

cfg5 is an 8-GPU workload (S§8e): W (106 GB) is replicated on every rank and the
block pairs are LPT-partitioned; this run executes exactly what one rank of that job executes
(tree, basis, its LPT share of the assembly into its piece shard, its row panel of the EXACT
C_W v), timed with CUDA events on the library stream.  No rank waits on another: the all-gather
of the shards is the only step left out, and nothing here stands in for it.

    python tools/cfg5_share.py [--nranks 8] [--rank 0] [--check] [--out gpurun_out/cfg5.json]

--check (test infrastructure; calls oracle/):
  * tree permutation / thresholds bit-exact against the oracle tree;
  * the admitted pair list (BSR structure) bit-exact against tests/golden/pairs_cfg5.npz
    (written by tools/make_golden_pairs.py from oracle/ only);
  * sampled blocks this rank owns completely (every piece in its shard), both cells at depth
    >= t - 1 (|tau| |kappa| <= 2^23): the sum of the block's pieces against the oracle's
    W_a C(X_a, X_b) W_b^T with W from oracle.basis.build_subtree_basis, <= 1e-11 relative;
  * sampled rows of the full b = C a (a single-rank context) against direct sums, <= 1e-11;
  * W W^T v = v (orthonormal rows) through mlk_apply_wt / mlk_apply_w.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nranks", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--n", type=int, default=None, help="reduced n (dry runs)")
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--rows", type=int, default=64)
    ap.add_argument("--stop-after-basis", action="store_true", help="diagnostics")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cfg5_share.json"))
    a = ap.parse_args()

    import torch

    from paper_1701_00285_b200 import mlk

    t_start = time.time()
    inp = wl.make("cfg5", n=a.n)
    c = inp["cfg"]
    X, dirs = inp["X"], inp["dirs"]
    kern = wl.kernel_dict(c)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    ctx = mlk.Ctx(0, a.nranks, a.rank, stream.cuda_stream)
    X_d = torch.from_numpy(X).to(dev)
    D_d = torch.from_numpy(dirs).to(dev)
    torch.cuda.synchronize()
    ctx.reset_stats()
    ctx.set_timing(True)
    ev = {}

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        ev[name] = e

    wall = {}
    mark("start")
    t0 = time.perf_counter()
    tr = mlk.build_tree(ctx, X_d, c["leaf"], c["tree"], D_d)
    mark("tree")
    print("tree built", flush=True)
    B = mlk.build_basis(ctx, tr, c["w"], flags=mlk.BASIS_DROP_PHI)
    print("basis leaf level done", flush=True)
    if a.stop_after_basis:
        L = B.L()
        print("basis complete, |L| = %.6e" % float(np.linalg.norm(L)), flush=True)
        return
    wall["tree+basis(leaf level)"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    cw = mlk.assemble_cw(ctx, tr, B, kern, dict(mode=c["pairs"], tau=c["tau"]))
    mark("assemble")
    wall["assemble"] = time.perf_counter() - t0
    print("assembled", flush=True)
    v = torch.from_numpy(wl.vectors(1, B.dim, seed=0)).to(dev)
    y = torch.empty_like(v)
    t0 = time.perf_counter()
    mlk.cw_matvec(ctx, tr, B, kern, None, mlk.MATVEC_EXACT, v, out=y, allreduce=False)
    mark("matvec")
    stream.synchronize()
    wall["matvec"] = time.perf_counter() - t0
    stats = ctx.kernel_stats()
    ctx.set_timing(False)
    ms = {k: ev["start"].elapsed_time(e) for k, e in ev.items() if k != "start"}
    sf = cw.stage_flops()
    sl, msl = cw.shard_len()
    own_k5a = sum(v["ms"] for k, v in stats.items() if k == "assemble_tile_contract")
    own_k5b = sum(v["ms"] for k, v in stats.items() if k == "assemble_wa_gemm")
    peak = 37.062
    res = {
        "what": "BASELINE cfg5, share of rank %d of %d, on one B200 (CUDA events, library stream)" % (a.rank, a.nranks),
        "n": c["n"], "d": c["d"], "M": B.M, "dim": B.dim, "leaf": c["leaf"], "tau": c["tau"],
        "n_blocks": cw.n_blocks, "nnz_values_total": cw.nnz, "shard_doubles": sl, "max_shard_doubles": msl,
        "entries_total": cw.entries, "own_entries": cw.own_entries,
        "flops_total": cw.flops, "own_flops": cw.own_flops, "stage_flops_total": sf,
        "ms_cumulative": ms, "host_wall_s": wall,
        "assembly_ms": ms["assemble"] - ms["tree"], "matvec_ms": ms["matvec"] - ms["assemble"],
        "own_assembly_tflops": cw.own_flops / ((ms["assemble"] - ms["tree"]) * 1e-3) / 1e12,
        "kernels_ms": {k: v["ms"] for k, v in sorted(stats.items())},
        "k5a_ms": own_k5a, "k5b_ms": own_k5b, "peak_tflops": peak,
    }
    res["own_assembly_pct_of_fp64_peak"] = 100.0 * res["own_assembly_tflops"] / peak
    print(json.dumps(res, indent=1), flush=True)

    if a.check:
        chk = check(a, mlk, ctx, tr, B, cw, X, dirs, c, kern)
        res["check"] = chk
        print(json.dumps(chk, indent=1), flush=True)
    res["total_wall_s"] = time.time() - t_start
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


def check(a, mlk, ctx, tr, B, cw, X, dirs, c, kern):
    from oracle import assemble as OAs
    from oracle import basis as OB
    from oracle import covariance as OC
    from oracle import tree as OT

    out = {}
    t0 = time.time()
    o = OT.build_tree(X, c["leaf"], c["tree"], dirs)
    e = tr.export()
    out["tree_bit_exact"] = bool(np.array_equal(e["perm"], o.perm) and
                                 np.array_equal(e["thr"][o.exists & ~o.is_leaf], o.thr[o.exists & ~o.is_leaf]))
    out["oracle_tree_s"] = time.time() - t0
    # pair list: GPU BSR structure -> (node, node) pairs in C_W order vs the golden list
    brow_ptr, bcol, val_off = cw.structure()
    cells = np.asarray(B.cells)
    rows = np.repeat(np.arange(len(brow_ptr) - 1), np.diff(brow_ptr))
    gpairs = np.stack([cells[rows], cells[bcol]], axis=1).astype(np.int32)
    gold = os.path.join(ROOT, "tests", "golden", "pairs_cfg5.npz")
    if a.n is None and os.path.exists(gold):
        ref = np.load(gold)["pairs"]
        out["pairs_bit_exact"] = bool(gpairs.shape == ref.shape and np.array_equal(gpairs, ref))
        out["pairs"] = int(len(ref))
    pairs = [tuple(p) for p in gpairs]
    # sampled blocks owned entirely by this rank, both cells at depth >= t - 1
    pp, po, pw, shard = cw.pieces()
    t = tr.t
    depth = e["depth"]
    cand = [k for k, (p, q) in enumerate(pairs)
            if depth[p] >= t - 1 and depth[q] >= t - 1 and pp[k + 1] > pp[k] and np.all(pw[pp[k]:pp[k + 1]] == a.rank)]
    rng = np.random.default_rng([0, 3])
    selfs = [k for k in cand if pairs[k][0] == pairs[k][1]]
    others = [k for k in cand if pairs[k][0] != pairs[k][1]]
    pick = list(rng.choice(selfs, min(len(selfs), a.blocks // 2), replace=False)) if selfs else []
    pick += list(rng.choice(others, min(len(others), a.blocks - len(pick)), replace=False)) if others else []
    errs = []
    t0 = time.time()
    for k in pick:
        p, q = pairs[int(k)]
        ln = int(val_off[k + 1] - val_off[k])
        got = np.zeros(ln)
        for i in range(pp[k], pp[k + 1]):
            got = got + shard[po[i]:po[i] + ln]
        sb = OB.build_subtree_basis(X, o, c["w"], int(p))
        if q != p:
            sb.W.update(OB.build_subtree_basis(X, o, c["w"], int(q)).W)
        ref = OAs.block(X, o, sb, kern, int(p), int(q)).ravel()
        errs.append({"pair": [int(p), int(q)], "rel_frob": float(np.linalg.norm(got - ref) / np.linalg.norm(ref))})
        print("block", errs[-1], flush=True)
    out["blocks"] = errs
    out["blocks_max_rel"] = max((x["rel_frob"] for x in errs), default=None)
    out["blocks_s"] = time.time() - t0
    # b = C a in full (a nranks = 1 context: a rank's b is only a partial sum, see mlk.h) on
    # seeded sampled rows (tree order) against direct sums
    n = X.shape[0]
    av = np.random.default_rng([0, 4]).standard_normal((1, n))
    ctx1 = mlk.Ctx(0)
    tr1 = mlk.build_tree(ctx1, X, c["leaf"], c["tree"], dirs)
    t0 = time.time()
    b = mlk.cov_matvec(ctx1, tr1, kern, av)
    out["cov_matvec_full_s"] = time.time() - t0
    rows = rng.choice(n, a.rows, replace=False)
    Xt = X[o.perm]
    rel, got_s, ref_s = [], [], []
    for i in rows:
        ci = OC.cov(Xt[i:i + 1], Xt, o.perm[i:i + 1], o.perm, kern["family"], kern["rho"], kern.get("sigma2", 1.0),
                    kern.get("nugget", 0.0))[0]
        ref = float(ci @ av[0])
        rel.append(abs(b[0, i] - ref) / (np.abs(ci) @ np.abs(av[0])))
        got_s.append(b[0, i])
        ref_s.append(ref)
    out["cov_matvec_rows"] = int(len(rows))
    out["cov_matvec_rel_sampled"] = float(np.linalg.norm(np.array(got_s) - np.array(ref_s)) / np.linalg.norm(ref_s))
    out["cov_matvec_max_rel_componentwise"] = float(max(rel)) if rel else None
    # W W^T v = v
    v = wl.vectors(1, B.dim, seed=7)
    aw = mlk.apply_wt(ctx, B, v)
    vv = mlk.apply_w(ctx, B, aw)
    out["WWt_roundtrip_rel"] = float(np.linalg.norm(vv - v) / np.linalg.norm(v))
    return out


if __name__ == "__main__":
    main()
