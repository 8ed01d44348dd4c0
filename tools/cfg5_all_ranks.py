"""BASELINE cfg5 at full size on ONE B200: the shares of ALL ranks of an `--nranks`-rank job, one
after another (no rank waits on another; the all-gather is replaced by summing each block's
pieces on the host in the library's chunk order).  This completes the blocks no single rank
holds -- the level-0/1 blocks, whose row chunks are spread over the ranks by the LPT partition --
and checks them against the oracle's entries of tests/golden/entries_cfg5.npz
(tools/make_golden_cfg5.py: psi_k^T C psi_l of B_11 and B_12, oracle only).

Also reports each rank's assembly time (CUDA events on the library stream): the max over ranks
is what the 8-GPU job's assembly would take with this partition, a per-rank measurement on one
GPU -- NOT a multi-GPU measurement.

    python tools/cfg5_all_ranks.py [--nranks 8] [--out gpurun_out/cfg5_all.json]
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
    ap.add_argument("--n", type=int, default=None, help="reduced n (dry runs)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cfg5_all_ranks.json"))
    a = ap.parse_args()

    import torch

    from paper_1701_00285_b200 import mlk

    t_start = time.time()
    inp = wl.make("cfg5", n=a.n)
    c = inp["cfg"]
    kern = wl.kernel_dict(c)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    ctx0 = mlk.Ctx(0, a.nranks, 0, stream.cuda_stream)
    X_d = torch.from_numpy(inp["X"]).to(dev)
    D_d = torch.from_numpy(inp["dirs"]).to(dev)
    tr = mlk.build_tree(ctx0, X_d, c["leaf"], c["tree"], D_d)
    B = mlk.build_basis(ctx0, tr, c["w"], flags=mlk.BASIS_DROP_PHI)
    L = B.L()   # waits for the merge levels
    print("tree + basis %.0f s" % (time.time() - t_start), flush=True)
    cells = np.asarray(B.cells)
    # target blocks: every admitted block whose two cells sit at levels <= 1
    gold_path = os.path.join(ROOT, "tests", "golden", "entries_cfg5.npz")
    gold = np.load(gold_path) if os.path.exists(gold_path) and a.n is None else None
    sums, struct, ranks = {}, None, []
    for r in range(a.nranks):
        ctx = mlk.Ctx(0, a.nranks, r, stream.cuda_stream)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cw = mlk.assemble_cw(ctx, tr, B, kern, dict(mode=c["pairs"], tau=c["tau"]), gather=mlk.GATHER_NONE)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        if struct is None:
            brow_ptr, bcol, val_off = cw.structure()
            rows = np.repeat(np.arange(len(brow_ptr) - 1), np.diff(brow_ptr))
            pairs = [(int(cells[i]), int(cells[j])) for i, j in zip(rows, bcol)]
            e = tr.export()
            depth = e["depth"]
            targets = [k for k, (p, q) in enumerate(pairs) if depth[p] <= 1 and depth[q] <= 1]
            struct = (pairs, val_off, targets)
        pairs, val_off, targets = struct
        pp, po, pw, shard = cw.pieces()
        # the library's reduction order: block k = ((0 + piece_0) + piece_1) + ... over ALL its
        # pieces in chunk order; pieces of other ranks arrive in later passes, so keep them apart
        for k in targets:
            ln = int(val_off[k + 1] - val_off[k])
            for i in range(pp[k], pp[k + 1]):
                if pw[i] == r:
                    sums.setdefault(k, {})[i] = shard[po[i]:po[i] + ln].copy()
        ranks.append({"rank": r, "assembly_ms": ms, "own_flops": cw.own_flops,
                      "own_tflops": cw.own_flops / (ms * 1e-3) / 1e12, "shard_doubles": int(cw.shard_len()[0])})
        print("rank %d: %.1f s, %.2f TFLOP/s" % (r, ms / 1e3, ranks[-1]["own_tflops"]), flush=True)
        del cw, ctx, shard
    pairs, val_off, targets = struct
    res = {"what": "cfg5, all %d rank shares on one B200, one after another" % a.nranks, "n": c["n"],
           "ranks": ranks, "max_rank_assembly_ms": max(x["assembly_ms"] for x in ranks),
           "sum_rank_assembly_ms": sum(x["assembly_ms"] for x in ranks), "targets": []}
    blocks = {}
    for k in targets:
        ln = int(val_off[k + 1] - val_off[k])
        s = np.zeros(ln)
        for i in sorted(sums[k]):
            s = s + sums[k][i]
        blocks[pairs[k]] = s
        res["targets"].append({"pair": list(pairs[k]), "pieces": len(sums[k])})
    pos = {q: i for i, q in enumerate(cells)}
    # the completed level-1 blocks B_11, B_12 (the oracle's entries_cfg5 blocks), for a host-side
    # comparison with the oracle entries when those are computed after this run (28 MB)
    keep = {k: v for k, v in blocks.items() if k in ((1, 1), (1, 2), (2, 1))}
    np.savez_compressed(os.path.join(os.path.dirname(a.out), "cfg5_level1_blocks.npz"),
                        pairs=np.array(list(keep.keys()), np.int32),
                        shapes=np.array([[int(B.row_off[pos[p] + 1] - B.row_off[pos[p]]),
                                          int(B.row_off[pos[q] + 1] - B.row_off[pos[q]])] for p, q in keep], np.int64),
                        **{"b_%d_%d" % k: v for k, v in keep.items()})
    if gold is not None:
        chk = []
        for (p, q) in [tuple(int(v) for v in b) for b in gold["blocks"]]:
            key = (p, q) if (p, q) in blocks else (q, p)
            pr = int(B.row_off[pos[key[0]] + 1] - B.row_off[pos[key[0]]])
            pc = int(B.row_off[pos[key[1]] + 1] - B.row_off[pos[key[1]]])
            blk = blocks[key].reshape(pr, pc)
            if key != (p, q):
                blk = blk.T
            rr, cc = gold["rows_%d_%d" % (p, q)], gold["cols_%d_%d" % (p, q)]
            got = blk[np.ix_(rr, cc)]
            ref = gold["entries_%d_%d" % (p, q)]
            chk.append({"block": [p, q], "entries": int(ref.size),
                        "rel_frob": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
                        "max_abs": float(np.max(np.abs(got - ref))), "ref_max": float(np.max(np.abs(ref)))})
            print("oracle entries", chk[-1], flush=True)
        res["oracle_entries"] = chk
    res["total_wall_s"] = time.time() - t_start
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "targets"}, indent=1))


if __name__ == "__main__":
    main()
