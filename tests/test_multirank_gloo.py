"""The N > 1 protocol on CPU: world_size 2 over gloo.  Blocks are split into row-chunk pieces
(the libmlk decomposition); each rank computes (with the oracle) exactly the pieces the
library's LPT partition gives it, packs them with the library's shard plan, all-gathers with
torch.distributed and sums each block's pieces in chunk order; the result must equal the
single-process piece sum bit for bit and the oracle blocks to rounding.  The distributed C_W v (row panels of C per rank + allreduce) must match the
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
    from oracle import covariance as OAs_cov
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
        # pieces: block (a, b) split into row chunks of X_a (chunk = 64 rows here; 4096 in
        # libmlk), piece = W_a[:, chunk] C(X_a[chunk], X_b) W_b^T; block = sum in chunk order
        CH = 64
        pieces = []
        for k, (r, cc) in enumerate(pairs):
            for c0 in range(tr.begin[r] // CH, (tr.end[r] - 1) // CH + 1):
                pieces.append((k, c0))
        cost = np.array([1.0 + (tr.end[pairs[k][1]] - tr.begin[pairs[k][1]]) for k, _ in pieces])
        owner = mlk.partition_lpt(cost, world)
        plen = np.array([full.val_off[k + 1] - full.val_off[k] for k, _ in pieces])
        poff = np.concatenate([[0], np.cumsum(plen)])
        so, sl = mlk.shard_plan(poff, owner, world)
        mx = int(sl.max())

        def piece_val(k, c0):
            r, cc = pairs[k]
            ia = tr.perm[tr.begin[r]:tr.end[r]]
            ib = tr.perm[tr.begin[cc]:tr.end[cc]]
            lo = max(tr.begin[r], c0 * CH) - tr.begin[r]
            hi = min(tr.end[r], (c0 + 1) * CH) - tr.begin[r]
            C = OAs_cov.cov(X[ia[lo:hi]], X[ib], ia[lo:hi], ib, kern["family"], kern["rho"])
            return (B.W[r][:, lo:hi] @ (C @ B.W[cc].T)).ravel()

        shard = np.zeros(mx)
        for i, (k, c0) in enumerate(pieces):
            if owner[i] == rank:
                shard[so[i]:so[i] + plen[i]] = piece_val(k, c0)
        recv = torch.zeros(world * mx, dtype=torch.float64)
        dist.all_gather_into_tensor(recv, torch.from_numpy(shard))
        g = recv.numpy()
        vals = np.zeros_like(full.values)
        single = np.zeros_like(full.values)
        for i, (k, c0) in enumerate(pieces):
            a = full.val_off[k]
            vals[a:a + plen[i]] += g[owner[i] * mx + so[i]: owner[i] * mx + so[i] + plen[i]]
            single[a:a + plen[i]] += piece_val(k, c0)
        multi = sum(1 for k in range(len(pairs)) if sum(1 for kk, _ in pieces if kk == k) > 1)
        ok_gather = (np.array_equal(vals, single) and multi > 0 and
                     np.max(np.abs(vals - full.values)) <= 1e-12 * np.max(np.abs(full.values)))
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
