"""Per-rank step time of an R-rank job, measured on ONE B200: every rank's share of the bench step
(tree + basis + its LPT share of the assembly into its piece shard + its share of the EXACT
C_W v), run one after another through contexts (device 0, nranks = R, rank = r).  No rank waits
on another; the collectives (the all-gather of the shards, the allreduce of y) are left out and
their volume is reported instead.  The max over ranks is what the R-GPU step would take with this
partition apart from the collectives -- a load-balance measurement, NOT a multi-GPU measurement.

    python tools/rank_shares.py [--config cfg4] [--ranks 1,2,4,8] [--out gpurun_out/rank_shares_cfg4.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out_path = a.out or os.path.join(ROOT, "gpurun_out", "rank_shares_%s.json" % a.config)

    import torch

    from paper_1701_00285_b200 import mlk

    inp = wl.make(a.config)
    c = inp["cfg"]
    kern = wl.kernel_dict(c)
    spars = dict(mode=c["pairs"], tau=c["tau"])
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    X_d = torch.from_numpy(inp["X"]).to(dev)
    D_d = torch.from_numpy(inp["dirs"]).to(dev) if inp["dirs"] is not None else None
    nvec = c.get("nvec", 1)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    res = {"config": a.config, "what": __doc__.split("\n\n")[0], "runs": []}
    t1 = None
    for R in [int(x) for x in a.ranks.split(",")]:
        per_rank = []
        for r in range(R):
            ctx = mlk.Ctx(0, R, r, stream.cuda_stream)
            v = y = None
            best = None
            info = {}
            for rep in range(a.reps + 1):   # first pass untimed (warm-up, scratch buffers)
                flush.fill_(1.0)
                torch.cuda.synchronize()
                ctx.reset_stats()
                ctx.set_timing(True)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                tr = mlk.build_tree(ctx, X_d, c["leaf"], c["tree"], D_d)
                B = mlk.build_basis(ctx, tr, c["w"])
                cw = mlk.assemble_cw(ctx, tr, B, kern, spars, gather=mlk.GATHER_NONE)
                if v is None:
                    v = torch.from_numpy(wl.vectors(nvec, B.dim, seed=0)).to(dev)
                    y = torch.empty_like(v)
                mlk.cw_matvec(ctx, tr, B, kern, None, mlk.MATVEC_EXACT, v, out=y, allreduce=False)
                e1.record(stream)
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                st = ctx.kernel_stats()
                ctx.set_timing(False)
                if rep > 0 and (best is None or ms < best):
                    best = ms
                    info = {"own_flops": cw.own_flops, "flops": cw.flops, "shard_doubles": int(cw.shard_len()[0]),
                            "nested": bool(cw.plan()["nested"]),
                            "kernels_ms": {k: round(s["ms"], 3) for k, s in st.items() if s["ms"] >= 0.5}}
                del tr, B, cw
            per_rank.append(dict(rank=r, ms=best, **info))
            print("R=%d rank %d: %.1f ms (own flops %.3e)" % (R, r, best, info["own_flops"]), flush=True)
            del ctx
        mx = max(p["ms"] for p in per_rank)
        if R == 1:
            t1 = mx
        run = {"nranks": R, "max_ms": mx, "mean_ms": float(np.mean([p["ms"] for p in per_rank])),
               "allgather_bytes_total": 8 * int(sum(p["shard_doubles"] for p in per_rank)) if R > 1 else 0,
               "allreduce_bytes": 8 * int(nvec) * int(v.shape[1]) if R > 1 else 0,
               "ranks": per_rank}
        if t1:
            run["speedup_without_collectives"] = t1 / mx
            run["efficiency_without_collectives"] = t1 / mx / R
        res["runs"].append(run)
        print("R=%d: max %.1f ms, mean %.1f ms%s" % (R, mx, run["mean_ms"], (", speedup %.2f" % (t1 / mx)) if t1 else ""),
              flush=True)
        os.makedirs(os.path.dirname(out_path), exist_ok=True)
        json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
