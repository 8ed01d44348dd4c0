"""The N > 1 protocol on CPU: world_size 2 over gloo.  Blocks are split into row-chunk pieces
(the libmlk decomposition); each rank computes (with the oracle) exactly the pieces the
library's LPT partition gives it, packs them with the library's shard plan, all-gathers with
torch.distributed and sums each block's pieces in chunk order; the result must equal the
single-process piece sum bit for bit and the oracle blocks to rounding.  The distributed C_W v (row panels of C per rank + allreduce) must match the
single-process product.  The library's chunked all-gather plan (mlk_gather_plan) and the sharded
BSR product (each rank applies its own pieces and their mirrors, then one allreduce) are run
the same way."""
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
        # the library's CHUNKED all-gather plan (mlk_gather_plan, what MLK_GATHER_DEVICE runs over
        # NCCL): per group one equal-count all-gather of every rank's contiguous shard slice,
        # then the fixed-order piece sums -- bit-identical to the one-shot gather
        piece_ptr = np.zeros(len(pairs) + 1, np.int64)
        for k, _ in pieces:
            piece_ptr[k + 1] += 1
        piece_ptr = np.cumsum(piece_ptr)
        blen = np.diff(full.val_off).astype(np.int64)
        gptr, glo, gcnt = mlk.gather_plan(piece_ptr, so, owner, blen, world, budget=4 * int(blen.max()))
        chunked = np.zeros_like(full.values)
        for gi in range(len(gcnt)):
            cnt = int(gcnt[gi])
            send = np.zeros(max(cnt, 1))
            mylen = max(0, min(cnt, mx - int(glo[gi, rank])))
            send[:mylen] = shard[glo[gi, rank]:glo[gi, rank] + mylen]
            rv = torch.zeros(world * max(cnt, 1), dtype=torch.float64)
            dist.all_gather_into_tensor(rv, torch.from_numpy(send))
            rv = rv.numpy()
            for k in range(gptr[gi], gptr[gi + 1]):
                a = full.val_off[k]
                for i in range(piece_ptr[k], piece_ptr[k + 1]):
                    o = owner[i] * max(cnt, 1) + so[i] - glo[gi, owner[i]]
                    chunked[a:a + plen[i]] += rv[o:o + plen[i]]
        ok_chunked = np.array_equal(chunked, single) and len(gcnt) > 3
        # the sharded BSR product (S§8(e)): each rank applies its own pieces and their mirrors
        # straight from its shard, then one allreduce -- equals the single-rank C~_W v
        vb = wl.vectors(2, B.dim, seed=6)
        yb = np.zeros_like(vb)
        ro = full.row_off
        pos = {q: i for i, q in enumerate(full.cells)}
        for i, (k, c0) in enumerate(pieces):
            if owner[i] != rank:
                continue
            r, cc = pos[pairs[k][0]], pos[pairs[k][1]]
            P = shard[so[i]:so[i] + plen[i]].reshape(ro[r + 1] - ro[r], ro[cc + 1] - ro[cc])
            yb[:, ro[r]:ro[r + 1]] += vb[:, ro[cc]:ro[cc + 1]] @ P.T
            if r != cc:
                yb[:, ro[cc]:ro[cc + 1]] += vb[:, ro[r]:ro[r + 1]] @ P
        ybt = torch.from_numpy(yb)
        dist.all_reduce(ybt)
        yref = OM.cw_matvec_bsr(full, vb)
        ok_bsr = np.max(np.abs(ybt.numpy() - yref)) <= 1e-12 * np.max(np.abs(yref))
        multi = sum(1 for k in range(len(pairs)) if sum(1 for kk, _ in pieces if kk == k) > 1)
        ok_gather = (ok_chunked and ok_bsr and np.array_equal(vals, single) and multi > 0 and
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
