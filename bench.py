"""Benchmark: C_W assembly covariance pairs/s and FP64 TFLOP/s (BASELINE.json metric).

A step is one pass of the whole hot path on one synthetic input of the workload (SURVEY.md
section 8(a) rows a1-a7): mlk_build_tree -> mlk_build_basis -> mlk_assemble_cw (admission,
fused tiles, W_a contraction, NCCL all-gather of the BSR shards when N > 1) -> mlk_cw_matvec
EXACT (allreduce when N > 1).  value = covariance pairs (sum over admitted blocks |a||b|)
processed per second of step time (max over ranks), device-resident inputs.  e2e = the same
metric through the same public API with host (pinned) inputs and the BSR values + C_W v read
back to host inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl reference]
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402

PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "k5a_traffic_%s.json")  # per config, from ncu --set full


K5A_SOURCES = ["tile.cu", "tile.cuh", "dmma.cuh", "fastmath.cuh", "common.cuh"]


def k5a_source_sha():
    """sha256 over K5a's sources: a committed ncu traffic figure is reported only for the code
    it was measured on (tools/traffic_from_ncu.py stamps the same hash)."""
    import hashlib
    h = hashlib.sha256()
    for f in K5A_SOURCES:
        h.update(open(os.path.join(ROOT, "paper_1701_00285_b200", "csrc", f), "rb").read())
    return h.hexdigest()[:16]


def fp64_peak():
    d = json.load(open(PEAK_FILE))
    return float(max(d["fp64_peak_tflops_dmma"], d["fp64_peak_tflops_dfma"]))


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every 100 ms during the timed region
    (in-process, so the sampling does not stall the host thread that drives the GPU)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            try:
                import pynvml
                pynvml.nvmlInit()
                h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            except Exception:
                return
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, mx, rs))
                except Exception:
                    pass
                self._stop.wait(0.1)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4}
        reasons = sorted({k for _, _, rs in self.samples for k, b in bits.items() if rs & b})
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": float(max(s[1] for s in self.samples)), "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args, argv):
    """--gpus N > 1 without a torchrun environment: re-launch this script as N ranks (one per
    GPU) with torch.distributed.run on 127.0.0.1 and return its exit code.  Rank 0 prints the
    JSON line.  --dry-run needs no GPU (used by tests/test_bench_launch.py)."""
    import subprocess
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": "--gpus %d but only %d CUDA devices are visible" % (args.gpus, have)}))
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % args.gpus,
           "--master-addr=127.0.0.1", "--master-port=%d" % _free_port(), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def dry_run(args):
    """Launch check without GPU work: every rank reports its environment over gloo."""
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
        got = [None] * ws
        dist.all_gather_object(got, {"rank": rank, "world_size": ws, "local_rank": local})
        dist.destroy_process_group()
    else:
        got = [{"rank": rank, "world_size": ws, "local_rank": local}]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "gpus_flag": args.gpus, "ranks": got}))
    return 0


# --------------------------------------------------------------------------- reference arm
METRIC = "C_W assembly covariance pairs/s (FP64 TFLOP/s and % of FP64 peak in 'fp64')"


def config_dict(name, ws):
    c = wl.CONFIGS[name]
    return {"workload": name, "n": c["n"], "d": c["d"], "w": c["w"], "leaf": c["leaf"], "family": c["family"],
            "rho": c["rho"], "tau": c["tau"], "pairs_mode": c["pairs"], "parallelism": "pairs%d" % ws,
            "l2": "flushed (512 MB write) between timed steps",
            "nvec": c.get("nvec", 1),
            "step": "build_tree + build_basis + assemble_cw(+all-gather) + cw_matvec EXACT nvec=%d" % c.get("nvec", 1)}


class OracleSampler:
    """The oracle (as it stands) on bounded, seeded, STRATIFIED samples of a workload's admitted
    blocks.  Tree, basis and the admitted pair list are built once, untimed (the pair list of
    cfg3-5 is the oracle's own, read from tests/golden/pairs_<cfg>.npz, written by
    tools/make_golden_pairs.py from oracle/ only).  A sample walks the level pairs (depth a,
    depth b) round-robin -- every level pair gets a block before any gets a second -- taking
    seeded random blocks of at most CAP covariance entries, each computed as W_a C(X_a, X_b) W_b^T
    by the oracle (oracle.fastcov: direct-difference C tile in plain C, NumPy contractions), until
    the time budget is spent and at least MIN_BLOCKS blocks were done."""

    CAP = 1 << 26
    MIN_BLOCKS = 64

    def __init__(self, cfg_name):
        from oracle import admission as OA
        from oracle import basis as OB
        from oracle import tree as OT

        inp = wl.make(cfg_name)
        c = inp["cfg"]
        self.name = cfg_name
        self.X = inp["X"]
        self.tr = OT.build_tree(self.X, c["leaf"], c["tree"], inp["dirs"])
        self.B = OB.build_basis(self.X, self.tr, c["w"])
        gp = os.path.join(ROOT, "tests", "golden", "pairs_%s.npz" % cfg_name)
        if os.path.exists(gp):
            self.pairs = [tuple(int(v) for v in p) for p in np.load(gp)["pairs"]]
        else:
            self.pairs = OA.admitted_pairs(self.X, self.tr, self.B, c["pairs"], c["tau"])
        self.kern = wl.kernel_dict(c)
        tr = self.tr
        self.strata = {}
        for k, (a, b) in enumerate(self.pairs):
            key = (int(tr.depth[a]), int(tr.depth[b]))
            self.strata.setdefault(key, []).append(k)

    def _order(self, seed_tag):
        """Round-robin over the level pairs of seeded permutations of their blocks."""
        rng = np.random.default_rng([0, 3, seed_tag])
        queues = [list(rng.permutation(ks)) for key, ks in sorted(self.strata.items()) if ks]
        out = []
        while any(queues):
            for q in queues:
                if q:
                    out.append(int(q.pop(0)))
        return out

    def sample(self, budget_s, seed_tag=0, min_blocks=None):
        """Oracle pairs/s on a stratified sample.  Blocks above CAP entries (level pairs near the
        root) are timed on a seeded contiguous panel of the row cell's points holding CAP
        entries: W_a[:, P] C(X_P, X_b) W_b^T, the oracle's own block arithmetic restricted to
        rows P (its pairs count is |P| |b|)."""
        from oracle import fastcov as F

        min_blocks = self.MIN_BLOCKS if min_blocks is None else min_blocks
        tr = self.tr
        rng = np.random.default_rng([0, 3, 7, seed_tag])
        ent = 0.0
        nb = npanel = 0
        seen = set()
        t0 = time.perf_counter()
        for k in self._order(seed_tag):
            a, b = self.pairs[k]
            sa, sb = int(tr.end[a] - tr.begin[a]), int(tr.end[b] - tr.begin[b])
            if sa * sb <= self.CAP:
                F.block_streamed(self.X, tr, self.B, self.kern, a, b)
                ent += float(sa) * float(sb)
            else:
                rows = max(1, self.CAP // sb)
                p0 = int(rng.integers(0, sa - rows + 1))
                ia = tr.perm[tr.begin[a] + p0:tr.begin[a] + p0 + rows]
                ib = tr.perm[tr.begin[b]:tr.end[b]]
                Cp = F.cov_c(self.X[ia], self.X[ib], ia, ib, self.kern)
                self.B.W[a][:, p0:p0 + rows] @ (Cp @ self.B.W[b].T)
                ent += float(rows) * float(sb)
                npanel += 1
            nb += 1
            seen.add((int(tr.depth[a]), int(tr.depth[b])))
            if time.perf_counter() - t0 >= budget_s and nb >= min_blocks:
                break
        dt = time.perf_counter() - t0
        cores = omp_threads()
        try:
            from threadpoolctl import threadpool_info
            blas = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
        except Exception:
            blas = None
        desc = ("sampled: %d of %d admitted %s blocks, stratified over %d of %d level pairs (depth a, depth b) "
                "round-robin, seeded; %d blocks above 2^26 covariance entries timed on a seeded 2^26-entry row "
                "panel; oracle W_a C W_b^T = oracle.fastcov (plain-C direct-difference tile, OpenMP %d threads) + "
                "NumPy contractions (BLAS threads %s); %.1f s budget; tree/basis/pair list built once, untimed"
                % (nb, len(self.pairs), self.name, len(seen), len(self.strata), npanel, cores, blas, budget_s))
        return ent / dt, desc, cores

    def matvec_sample(self, rows=256):
        """Oracle C_W v pieces: a = W^T v and y = W b in full, b = C a on `rows` seeded rows."""
        from oracle import fastcov as F
        from oracle import matvec as OM

        tr, B = self.tr, self.B
        v = wl.vectors(1, B.dim, seed=0)
        t0 = time.perf_counter()
        a = OM.apply_wt(tr, B, v)
        t1 = time.perf_counter()
        rr = np.sort(np.random.default_rng([0, 3]).choice(tr.n, rows, replace=False))
        F.cov_rows(self.X, tr, self.kern, a, rr)
        t2 = time.perf_counter()
        OM.apply_w(tr, B, a)
        t3 = time.perf_counter()
        return {"kind": "oracle", "sample": "C a on %d seeded rows of %d (oracle.fastcov.cov_rows); W^T v and W b "
                                            "in full (oracle.matvec)" % (rows, tr.n),
                "apply_wt_s": t1 - t0, "apply_w_s": t3 - t2, "cov_rows_s": t2 - t1,
                "cov_entries_per_s": rows * float(tr.n) / (t2 - t1)}


def omp_threads():
    """Threads the oracle's OpenMP tile uses (OMP_NUM_THREADS if set, else the affinity mask)."""
    n = len(os.sched_getaffinity(0))
    try:
        return max(1, min(n, int(os.environ["OMP_NUM_THREADS"])))
    except (KeyError, ValueError):
        return n


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    if ws > 1:
        # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 runs alone here, so give the oracle the
        # host's cores (read when the oracle's C tile library is first loaded)
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
        try:
            from threadpoolctl import threadpool_limits
            threadpool_limits(len(os.sched_getaffinity(0)))
        except Exception:
            pass
    sampler = OracleSampler(args.config)
    for w in range(args.warmup):
        sampler.sample(min(3.0, args.ref_budget), seed_tag=100 + w, min_blocks=1)
    vals = []
    desc = cores = None
    step_s = []
    for s in range(args.steps):
        t0 = time.perf_counter()
        v, desc, cores = sampler.sample(args.ref_budget, seed_tag=s + 1)
        step_s.append(time.perf_counter() - t0)
        vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "covariance pairs/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        # one step = one bounded sample of the workload (host wall clock; no GPU work in this arm)
        "ms_per_step": 1e3 * float(np.mean(step_s)), "scaling": "weak", "gpu_launches": 0,
        "higher_is_better": True, "dtype": "f64", "data": "synthetic", "config": config_dict(args.config, ws),
        "cpu_baseline": {"value": value, "unit": "covariance pairs/s", "cores": cores, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": "covariance pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4",
                    help="BASELINE workload; cfg4 (n = 262144, d = 50) is the largest that fits one B200")
    ap.add_argument("--impl", default="ours")
    ap.add_argument("--ref-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--pcg-tol", type=float, default=None,
                    help="PCG solve reported after the bench (0: skip; default 1e-8 up to cfg3 size, skipped above)")
    ap.add_argument("--dry-run", action="store_true", help="launch check only (no GPU work)")
    ap.add_argument("--no-matvec-report", dest="matvec_report", action="store_false",
                    help="skip the C_W v timings reported after the bench")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args, sys.argv[1:])
    ws_env = dist_env()[0]
    if ws_env != args.gpus and not (args.gpus == 1 and ws_env > 1):
        print(json.dumps({"error": "--gpus %d but WORLD_SIZE=%d" % (args.gpus, ws_env)}))
        return 2
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.pcg_tol is None:
        args.pcg_tol = 1e-8 if wl.CONFIGS[args.config]["n"] <= 131072 else 0.0

    import torch
    import torch.distributed as dist

    from paper_1701_00285_b200 import mlk

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_id = None
    if ws > 1:
        # torch.distributed (gloo, host side) carries only the plumbing: the NCCL unique id, the
        # barriers and the max-over-ranks timings.  The data-path collectives (the all-gather of
        # the BSR pieces, the allreduce of C_W v) run inside libmlk on its own NCCL communicator.
        dist.init_process_group("gloo")
        idl = [mlk.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(idl, src=0)
        nccl_id = idl[0]
    stream = torch.cuda.Stream(dev)
    ctx = mlk.Ctx(local, ws, rank, stream.cuda_stream, nccl_id=nccl_id)
    inp = wl.make(args.config)
    c = inp["cfg"]
    kern = wl.kernel_dict(c)
    spars = dict(mode=c["pairs"], tau=c["tau"])
    X_d = torch.from_numpy(inp["X"]).to(dev)
    dirs = inp["dirs"]
    dirs_d = torch.from_numpy(dirs).to(dev) if dirs is not None else None
    nvec = c.get("nvec", 1)   # BASELINE cfg3: 10 C_W v products with N(0,1) vectors
    torch.cuda.synchronize()

    api_ms = {}
    vec_cache = {}

    def timed(name, fn, *a, **kw):
        t0 = time.perf_counter()
        r = fn(*a, **kw)
        api_ms[name] = api_ms.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
        return r

    def step(X, D, v_host=None, out_vals=None, out_y=None):
        tr = timed("build_tree", mlk.build_tree, ctx, X, c["leaf"], c["tree"], D)
        B = timed("build_basis", mlk.build_basis, ctx, tr, c["w"], c.get("index_set", 0),
                  mlk.BASIS_KEEP_DEFICIENT if c.get("index_set", 0) else 0)
        # nranks > 1: the library all-gathers the pieces (MLK_GATHER_DEVICE over NCCL)
        cw = timed("assemble_cw", mlk.assemble_cw, ctx, tr, B, kern, spars)
        if v_host is None:
            if "v" not in vec_cache:
                vec_cache["v"] = torch.from_numpy(wl.vectors(nvec, B.dim, seed=0)).to(dev)
                vec_cache["y"] = torch.empty_like(vec_cache["v"])
            v, y = vec_cache["v"], vec_cache["y"]
        else:
            v, y = v_host, out_y
        if out_vals is not None:
            # the BSR read-back (pinned host memory) overlaps the C_W v product
            timed("export_async", cw.export_async, ctx, out_vals)
        timed("cw_matvec", mlk.cw_matvec, ctx, tr, B, kern, None, mlk.MATVEC_EXACT, v, out=y)
        if out_vals is not None:
            timed("wait_copies", ctx.wait_copies)
        return tr, B, cw

    # L2 flush buffer (> 126 MB L2) written between timed steps, outside the timed events
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)

    for _ in range(args.warmup):
        step(X_d, dirs_d)
    torch.cuda.synchronize()
    # one untimed pass for the structure numbers
    tr, B, cw = step(X_d, dirs_d)
    entries, flops, own_flops = cw.entries, cw.flops, cw.own_flops
    plan = cw.plan()
    sf = cw.stage_flops()
    nnz, dim = cw.nnz, B.dim
    del tr, B, cw

    sampler = ClockSampler(local) if rank == 0 and not os.environ.get("MLK_BENCH_NO_SAMPLER") else None
    ctx.reset_stats()
    ctx.set_timing(True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
    launches0 = mlk.launch_count()
    api_ms.clear()
    step_ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(X_d, dirs_d)   # the library's collectives run on `stream` too
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = mlk.launch_count() - launches0
    api_timed = {k: v / args.steps for k, v in api_ms.items()}
    clocks = sampler.stop() if sampler else None
    stats = ctx.kernel_stats()
    ctx.set_timing(False)
    total_ms = float(np.sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = entries * args.steps / (total_ms * 1e-3)

    # ---- e2e: host (pinned) inputs, BSR values + C_W v read back, through the same API
    Xh = torch.from_numpy(inp["X"]).pin_memory()
    Dh = torch.from_numpy(dirs).pin_memory() if dirs is not None else None
    vh = torch.from_numpy(wl.vectors(nvec, dim, seed=0)).pin_memory()
    yh = torch.empty((nvec, dim), dtype=torch.float64).pin_memory()
    valsh = torch.empty(max(nnz, 1), dtype=torch.float64).pin_memory()
    e2e_ms = []
    if args.e2e_steps > 0:  # one untimed e2e step first (copy stream, host staging buffers)
        step(Xh.numpy(), Dh.numpy() if Dh is not None else None, vh.numpy(), valsh.numpy()[:nnz], yh.numpy())
        torch.cuda.synchronize()
    for _ in range(args.e2e_steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        step(Xh.numpy(), Dh.numpy() if Dh is not None else None, vh.numpy(), valsh.numpy()[:nnz], yh.numpy())
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_total = float(np.sum(e2e_ms)) if e2e_ms else float("nan")
    if ws > 1 and e2e_ms:
        t = torch.tensor([e2e_total], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_val = entries * args.e2e_steps / (e2e_total * 1e-3) if e2e_ms else None
    h2d = inp["X"].nbytes + (dirs.nbytes if dirs is not None else 0) + vh.numel() * 8
    d2h = nnz * 8 + yh.numel() * 8

    # ---- C_W v timings (outside the timed step, S§8d): EXACT per call with nvec = 1 (x10
    # sequential) and batched nvec = 10, BSR nvec = 1; CUDA events on the library stream
    mv = None
    if args.matvec_report and ws == 1:
        trm = mlk.build_tree(ctx, X_d, c["leaf"], c["tree"], dirs_d)
        Bm = mlk.build_basis(ctx, trm, c["w"], c.get("index_set", 0),
                             mlk.BASIS_KEEP_DEFICIENT if c.get("index_set", 0) else 0)
        cwm = mlk.assemble_cw(ctx, trm, Bm, kern, spars)
        v10 = torch.from_numpy(wl.vectors(10, Bm.dim, seed=1)).to(dev)
        y10 = torch.empty_like(v10)

        def ev_ms(fn):
            fn()  # warm
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            fn()
            a1.record(stream)
            a1.synchronize()
            return a0.elapsed_time(a1)

        def seq10():
            for i in range(10):
                mlk.cw_matvec(ctx, trm, Bm, kern, None, mlk.MATVEC_EXACT, v10[i:i + 1], out=y10[i:i + 1])

        mv = {"exact_nvec1_x10_sequential_ms": ev_ms(seq10),
              "exact_nvec10_batched_ms": ev_ms(lambda: mlk.cw_matvec(ctx, trm, Bm, kern, None, mlk.MATVEC_EXACT,
                                                                     v10, out=y10)),
              "bsr_nvec1_ms": ev_ms(lambda: mlk.cw_matvec(ctx, trm, Bm, kern, cwm, mlk.MATVEC_BSR, v10[0:1],
                                                          out=y10[0:1]))}
        del trm, Bm, cwm

    # ---- NEXT-1 (outside the timed step): one PCG solve C_W gamma = z with P_W, N(0,1) z
    pcg = None
    if args.pcg_tol > 0 and ws == 1:
        trp = mlk.build_tree(ctx, X_d, c["leaf"], c["tree"], dirs_d)
        Bp = mlk.build_basis(ctx, trp, c["w"], c.get("index_set", 0),
                             mlk.BASIS_KEEP_DEFICIENT if c.get("index_set", 0) else 0)
        cwp = mlk.assemble_cw(ctx, trp, Bp, kern, spars)
        zp = torch.from_numpy(wl.vectors(1, Bp.dim, seed=9)[0]).to(dev)
        gp = torch.empty_like(zp)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, it, rr = mlk.pcg_solve(ctx, trp, Bp, kern, cwp, zp, tol=args.pcg_tol, max_iter=5000, out=gp)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        pcg = {"tol": args.pcg_tol, "precond": "block-diagonal P_W (self blocks)", "iterations": it,
               "true_rel_residual": rr, "seconds": dt, "ms_per_iteration": 1e3 * dt / max(it, 1)}
        # NEXT-4: the level-truncated log-likelihood l~^n_W of the same data, full (n = 0) and
        # the finest level only (n = t)
        ll = {}
        for lev in (0, trp.t):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            try:
                r = mlk.loglik(ctx, Bp, cwp, zp, lev)
            except mlk.RankDeficient:   # the tau-sparsified C~^n_W need not be positive definite
                r = {"not_positive_definite": True}
            torch.cuda.synchronize()
            ll["level%d" % lev] = dict(r, seconds=time.perf_counter() - t0)
        pcg["loglik"] = ll
        del trp, Bp, cwp

    if rank == 0:
        peak = fp64_peak()
        # K5a = the fused tile kernel, both its assembly uses: the nested plan's leaf pass
        # ("assemble_tile_nested") and the direct units ("assemble_tile_contract")
        own = own_flops / flops if flops > 0 else 1.0
        kd = stats.get("assemble_tile_contract", {"ms": 0.0, "launches": 0})
        kn = stats.get("assemble_tile_nested", {"ms": 0.0, "launches": 0})
        k5 = {"ms": kd["ms"] + kn["ms"], "launches": kd["launches"] + kn["launches"]}
        k5_ms_per_step = k5["ms"] / args.steps
        # this rank's share of the K5a flops (its LPT units; the whole job when ws == 1)
        k5_flops = (sf["gram"] + sf["contract1"]) * own
        achieved = k5_flops / (k5_ms_per_step * 1e-3) / 1e12
        nf = plan["nested_tile_flops"] * own
        k5_split = {"nested_leaf_pass": {"ms_per_step": kn["ms"] / args.steps, "flops": nf,
                                         "frac": (nf / (kn["ms"] / args.steps * 1e-3) / 1e12 / fp64_peak())
                                         if kn["ms"] > 0 else None},
                    "direct_units": {"ms_per_step": kd["ms"] / args.steps, "flops": k5_flops - nf,
                                     "frac": ((k5_flops - nf) / (kd["ms"] / args.steps * 1e-3) / 1e12 / fp64_peak())
                                     if kd["ms"] > 0 else None}}
        traffic, traffic_src = None, "no ncu capture for this config"
        if os.path.exists(TRAFFIC_FILE % args.config):
            tj = json.load(open(TRAFFIC_FILE % args.config))
            if tj.get("k5a_source_sha") == k5a_source_sha():
                # dram bytes of the launch(es) of one step, per launch like `achieved`
                traffic = tj.get("bytes_per_launch")
                traffic_src = "ncu --set full, %s (K5a sources sha %s)" % (tj.get("source"), tj["k5a_source_sha"])
            else:
                traffic_src = "stale: %s was captured on other K5a sources" % os.path.basename(TRAFFIC_FILE % args.config)
        asm_ms = sum(stats.get(k, {"ms": 0.0})["ms"] for k in
                     ("search", "assemble_tile_contract", "assemble_tile_nested", "assemble_transfer",
                      "assemble_transfer_gemm", "assemble_wa_gemm")) / args.steps
        cpu = None
        if not args.no_cpu_baseline and ws == 1:
            if wl.CONFIGS[args.config].get("index_set", 0):
                # the oracle builds total-degree bases only, and the paper's sphere workload is
                # rank-deficient by design (reading R24), so it has no oracle baseline
                cpu = {"unavailable": "oracle basis covers total-degree sets without reading R24"}
            else:
                osamp = OracleSampler(args.config)
                v, desc, cores = osamp.sample(args.ref_budget)
                cpu = {"value": v, "unit": "covariance pairs/s", "cores": cores, "kind": "oracle", "sample": desc,
                       "matvec": osamp.matvec_sample()}
        line = {
            "metric": METRIC,
            "value": value, "unit": "covariance pairs/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "steps_ms": [round(x, 2) for x in step_ms],
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(args.config, ws),
            "fp64": {"assembly_flops_per_step": flops, "tflops_step": flops / (ms_per_step * 1e-3) / 1e12,
                     "tflops_assembly": flops / (asm_ms * 1e-3) / 1e12 if asm_ms > 0 else None,
                     "pct_of_peak_step": 100.0 * flops / (ms_per_step * 1e-3) / 1e12 / peak,
                     "peak_tflops": peak, "peak_source": "measured, profiles/fp64_peak_r01.json (DMMA loop)"},
            "roofline": {"kernel": "k_tile_contract (K5a: assemble_tile_nested + assemble_tile_contract)", "bound": "tensor",
                         "peak_source": "of measured: FP64 DMMA loop on this pool's B200 (tools/fp64_peak.cu, "
                                        "profiles/fp64_peak_r01.json; MEASURED_PEAKS.json holds bf16/HBM only)",
                         "pipe": "FP64 DMMA.8x8x4 (shares the FP64 pipe with DFMA, DESIGN.md section 6)", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "launches_per_step": k5["launches"] / args.steps, "split": k5_split,
                         "algorithmic_flops_per_step": k5_flops, "ms_per_step": k5_ms_per_step},
            "kernels_ms_per_step": {k: v["ms"] / args.steps for k, v in sorted(stats.items())},
            "api_wall_ms_per_step": api_timed,
            "entries_per_step": entries, "blocks_nnz": nnz,
            "assembly_plan": {"nested": plan["nested"], "transfer_flops": plan["transfer_flops"],
                              "nested_tile_flops": plan["nested_tile_flops"],
                              "k5a_flops": sf["gram"] + sf["contract1"], "k5b_flops": sf["contract2"]},
            "clocks": clocks, "gpu_launches": launches,
            "e2e": {"value": e2e_val, "unit": "covariance pairs/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": e2e_total / args.e2e_steps if e2e_ms else None,
                    "steps_ms": [round(x, 3) for x in e2e_ms]},
            "cpu_baseline": cpu,
            "matvec": mv,
            "pcg": pcg,
        }
        print(json.dumps(line))
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
