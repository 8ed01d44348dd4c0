"""The N > 1 protocol on CPU: world_size 2 over gloo.  Each rank computes (with the oracle)
exactly the blocks the library's LPT partition gives it, packs them with the library's shard
plan, all-gathers with torch.distributed and unpacks; the result must equal the full BSR
bit for bit.  The distributed C_W v (row panels of C per rank + allreduce) must match the
single-process product."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import workloads as wl
    from oracle import admission as OA, assemble as OAs, basis as OB, tree as OT, matvec as OM
    from paper_1701_00285_b200 import mlk

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = wl.points("uniform", 512, 3, seed=5)
        t = wl.tree_levels(512, 32)
        dirs = wl.directions(2 ** t - 1, 3, seed=5)
        tr = OT.build_tree(X, 32, OT.RP, dirs)
        B = OB.build_basis(X, tr, 1)
        pairs = OA.admitted_pairs(X, tr, B, OA.PAIRS_PAPER_TAU, 0.05)
        kern = dict(family=1, rho=0.6)
        full = OAs.assemble(X, tr, B, kern, pairs)
        cost = np.array([(tr.end[a] - tr.begin[a]) * (tr.end[b] - tr.begin[b]) for a, b in pairs], float)
        owner = mlk.partition_lpt(cost, world)
        so, sl = mlk.shard_plan(full.val_off, owner, world)
        mx = int(sl.max())
        shard = np.zeros(mx)
        for k in np.nonzero(owner == rank)[0]:
            blk = OAs.block(X, tr, B, kern, *pairs[k]).ravel()
            shard[so[k]:so[k] + blk.size] = blk
        recv = torch.zeros(world * mx, dtype=torch.float64)
        dist.all_gather_into_tensor(recv, torch.from_numpy(shard))
        g = recv.numpy()
        vals = np.zeros_like(full.values)
        for k in range(len(pairs)):
            a, b = full.val_off[k], full.val_off[k + 1]
            vals[a:b] = g[owner[k] * mx + so[k]: owner[k] * mx + so[k] + (b - a)]
        ok_gather = np.array_equal(vals, full.values)
        # distributed exact matvec: rank owns a contiguous range of 32-row tiles of C
        v = wl.vectors(2, B.dim, seed=5)
        a_vec = OM.apply_wt(tr, B, v)
        tiles = -(-tr.n // 32)
        r0, r1 = 32 * (tiles * rank // world), min(tr.n, 32 * (tiles * (rank + 1) // world))
        b_part = np.zeros_like(a_vec)
        b_part[:, r0:r1] = OM.cov_matvec(X, tr, kern, a_vec, rows=np.arange(r0, r1))
        y_part = torch.from_numpy(OM.apply_w(tr, B, b_part))
        dist.all_reduce(y_part)
        y_ref = OM.cw_matvec_exact(X, tr, B, kern, v)
        ok_mv = np.max(np.abs(y_part.numpy() - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
        q.put((rank, ok_gather, ok_mv))
    finally:
        dist.destroy_process_group()


def test_gather_and_allreduce_world2():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in ps)
    assert all(r[1] and r[2] for r in res), res
