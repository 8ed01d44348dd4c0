"""Thin ctypes binding of libmlk.so (include/mlk.h).  Argument marshalling only: every step of
the path runs in the library's CUDA kernels.  There is no CPU fallback -- importing this module
fails loudly when the in-tree libmlk.so is missing.

Arrays: host inputs may be NumPy arrays (float64, C-contiguous); device inputs/outputs may be
torch CUDA tensors (float64, contiguous).  Results are returned as NumPy arrays unless a torch
`out=` tensor is supplied.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MLK_LIB_VARIANT=name loads the in-tree libmlk_<name>.so (A/B experiments, tools/build_variant.py)
LIB_PATH = os.path.join(_HERE, "libmlk%s.so" % ("_" + os.environ["MLK_LIB_VARIANT"]
                                               if os.environ.get("MLK_LIB_VARIANT") else ""))
if not os.path.exists(LIB_PATH):
    raise ImportError("libmlk.so is not built (run `python -m paper_1701_00285_b200.build` or "
                      "__graft_entry__.build()); there is no CPU fallback")
_lib = C.CDLL(LIB_PATH)

# enums (include/mlk.h)
OK, ERR_INVALID_ARG, ERR_DUPLICATE_POINTS, ERR_RANK_DEFICIENT, ERR_OUT_OF_MEMORY, ERR_CUDA, \
    ERR_UNSUPPORTED, ERR_NCCL = range(8)
TREE_KD, TREE_RP = 0, 1
MATERN_12, MATERN_32, MATERN_52, GAUSSIAN, MATERN_NU = 0, 1, 2, 3, 4
PAIRS_ALL, PAIRS_PAPER_TAU = 0, 1
PREC_FP64, PREC_DD = 0, 1
VALUES_DEVICE, VALUES_HOST = 0, 1
MATVEC_EXACT, MATVEC_BSR = 0, 1
GATHER_NONE, GATHER_DEVICE, GATHER_HOST = 0, 1, 2
INDEX_TD, INDEX_HC, INDEX_SM, INDEX_TP = 0, 1, 2, 3

SYMBOLS = [
    "mlk_last_error", "mlk_version", "mlk_ctx_create", "mlk_ctx_destroy", "mlk_ctx_stream",
    "mlk_ctx_set_timing", "mlk_ctx_reset_stats", "mlk_ctx_kernel_stats", "mlk_build_tree",
    "mlk_tree_free", "mlk_tree_info", "mlk_tree_export", "mlk_build_basis", "mlk_basis_free",
    "mlk_basis_info", "mlk_basis_export", "mlk_apply_wt", "mlk_apply_w", "mlk_assemble_cw",
    "mlk_cw_free", "mlk_cw_info", "mlk_cw_export", "mlk_cw_owner", "mlk_cw_shard_len", "mlk_cw_pack",
    "mlk_cw_unpack", "mlk_cw_values_device", "mlk_cov_matvec", "mlk_cw_matvec", "mlk_partition_lpt",
    "mlk_shard_plan", "mlk_launch_count", "mlk_cw_flops", "mlk_cw_export_async", "mlk_ctx_wait_copies",
    "mlk_pcg_solve", "mlk_build_basis_ex", "mlk_assemble_cw_ex", "mlk_cw_export_pieces", "mlk_loglik",
    "mlk_nccl_unique_id", "mlk_gather_plan", "mlk_cw_plan",
]


class MlkError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("mlk status %d: %s" % (status, msg))
        self.status = status


class DuplicatePoints(MlkError):
    pass


class RankDeficient(MlkError):
    pass


class KernelSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("rho", C.c_double), ("sigma2", C.c_double), ("nugget", C.c_double),
                ("nu", C.c_double)]


class SparsitySpec(C.Structure):
    _fields_ = [("mode", C.c_int32), ("tau", C.c_double)]


P = C.c_void_p
_sig = {
    "mlk_last_error": (C.c_char_p, []),
    "mlk_version": (C.c_char_p, []),
    "mlk_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, P, P, C.POINTER(P)]),
    "mlk_nccl_unique_id": (C.c_int, [P]),
    "mlk_gather_plan": (C.c_int, [C.c_int64, P, P, P, P, C.c_int32, C.c_int64, P, P, P, P]),
    "mlk_ctx_destroy": (None, [P]),
    "mlk_ctx_stream": (P, [P]),
    "mlk_ctx_set_timing": (C.c_int, [P, C.c_int]),
    "mlk_ctx_reset_stats": (C.c_int, [P]),
    "mlk_ctx_kernel_stats": (C.c_int, [P, C.c_int, C.POINTER(C.c_int), C.c_char_p, C.c_int,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_double)]),
    "mlk_build_tree": (C.c_int, [P, P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, P, C.c_int64,
                                 C.POINTER(P)]),
    "mlk_tree_free": (None, [P]),
    "mlk_tree_info": (C.c_int, [P, P, P, P, P]),
    "mlk_tree_export": (C.c_int, [P, P, P, P, P, P, P, P]),
    "mlk_build_basis": (C.c_int, [P, P, C.c_int32, C.POINTER(P)]),
    "mlk_build_basis_ex": (C.c_int, [P, P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]),
    "mlk_basis_free": (None, [P]),
    "mlk_basis_info": (C.c_int, [P, P, P, P]),
    "mlk_basis_export": (C.c_int, [P, P, P, C.c_int32, P, P, P]),
    "mlk_apply_wt": (C.c_int, [P, P, P, P, C.c_int32]),
    "mlk_apply_w": (C.c_int, [P, P, P, P, C.c_int32]),
    "mlk_assemble_cw": (C.c_int, [P, P, P, C.POINTER(KernelSpec), C.POINTER(SparsitySpec), C.c_int32,
                                  C.c_int32, C.POINTER(P)]),
    "mlk_assemble_cw_ex": (C.c_int, [P, P, P, C.POINTER(KernelSpec), C.POINTER(SparsitySpec), C.c_int32,
                                     C.c_int32, C.c_int32, C.POINTER(P)]),
    "mlk_cw_export_pieces": (C.c_int, [P, P, P, P, P]),
    "mlk_loglik": (C.c_int, [P, P, P, C.c_int32, P, P, P, P, P]),
    "mlk_cw_free": (None, [P]),
    "mlk_cw_info": (C.c_int, [P, P, P, P, P, P, P, P]),
    "mlk_cw_export": (C.c_int, [P, P, P, P, P]),
    "mlk_cw_owner": (C.c_int, [P, P]),
    "mlk_cw_shard_len": (C.c_int, [P, P, P]),
    "mlk_cw_pack": (C.c_int, [P, P, P]),
    "mlk_cw_unpack": (C.c_int, [P, P, P]),
    "mlk_cw_values_device": (C.c_int, [P, C.POINTER(P)]),
    "mlk_cov_matvec": (C.c_int, [P, P, C.POINTER(KernelSpec), P, P, C.c_int32]),
    "mlk_cw_matvec": (C.c_int, [P, P, P, C.POINTER(KernelSpec), P, C.c_int32, P, P, C.c_int32]),
    "mlk_partition_lpt": (C.c_int, [P, C.c_int64, C.c_int32, P]),
    "mlk_shard_plan": (C.c_int, [P, P, C.c_int64, C.c_int32, P, P]),
    "mlk_launch_count": (C.c_int64, []),
    "mlk_cw_flops": (C.c_int, [P, P, P, P]),
    "mlk_cw_plan": (C.c_int, [P, P, P, P]),
    "mlk_cw_export_async": (C.c_int, [P, P, P]),
    "mlk_ctx_wait_copies": (C.c_int, [P]),
    "mlk_pcg_solve": (C.c_int, [P, P, P, C.POINTER(KernelSpec), P, C.c_int32, P, P, C.c_double, C.c_int32,
                                C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
}
for _n, (_r, _a) in _sig.items():
    _f = getattr(_lib, _n)
    _f.restype = _r
    _f.argtypes = _a


def _check(st):
    if st != OK:
        msg = _lib.mlk_last_error().decode()
        if st == ERR_DUPLICATE_POINTS:
            raise DuplicatePoints(st, msg)
        if st == ERR_RANK_DEFICIENT:
            raise RankDeficient(st, msg)
        raise MlkError(st, msg)


def version():
    return _lib.mlk_version().decode()


def launch_count():
    """Kernels launched through libmlk in this process so far."""
    return int(_lib.mlk_launch_count())


_TORCH_DTYPE = {np.float64: "torch.float64", np.int64: "torch.int64", np.int32: "torch.int32"}


def _ptr(x, dtype=np.float64, device=None, out=False):
    """(pointer, keepalive) for a NumPy array or torch tensor (no copy for contiguous inputs).

    Torch tensors are passed by address, so their dtype must be exactly `dtype` and a CUDA
    tensor must live on the context's `device` (the library writes / reads nvec x dim x 8 bytes
    there).  NumPy inputs are converted; a NumPy output (out=True) must already be a C-contiguous
    array of `dtype`, since a converted copy would silently swallow the result."""
    if x is None:
        return None, None
    if hasattr(x, "data_ptr") and hasattr(x, "is_cuda"):
        if str(x.dtype) != _TORCH_DTYPE[dtype]:
            raise TypeError("tensor dtype %s, expected %s" % (x.dtype, _TORCH_DTYPE[dtype]))
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if x.is_cuda and device is not None and x.device.index != device:
            raise ValueError("CUDA tensor on cuda:%d, the context is on cuda:%d" % (x.device.index, device))
        return C.c_void_p(x.data_ptr()), x
    if out:
        if not (isinstance(x, np.ndarray) and x.dtype == dtype and x.flags["C_CONTIGUOUS"] and x.flags["WRITEABLE"]):
            raise TypeError("output must be a writeable C-contiguous %s array" % np.dtype(dtype).name)
        return x.ctypes.data_as(C.c_void_p), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data_as(C.c_void_p), a


def _np(ptr_holder):
    return ptr_holder.ctypes.data_as(C.c_void_p)


def kernel_spec(family, rho, sigma2=1.0, nugget=0.0, nu=0.0):
    return KernelSpec(int(family), float(rho), float(sigma2), float(nugget), float(nu or 0.0))


def _kspec(k):
    if isinstance(k, KernelSpec):
        return k
    return kernel_spec(k["family"], k["rho"], k.get("sigma2", 1.0), k.get("nugget", 0.0), k.get("nu") or 0.0)


def nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (bytes) for Ctx(..., nccl_id=...); call on one rank."""
    buf = C.create_string_buffer(128)
    _check(_lib.mlk_nccl_unique_id(buf))
    return buf.raw


class Ctx:
    """mlk_ctx_create.  nccl_id (128 bytes from nccl_unique_id(), the same on every rank): the
    library creates its own NCCL communicator and issues the all-gather / allreduce itself."""

    def __init__(self, device=0, nranks=1, rank=0, stream=None, nccl_id=None):
        h = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes")
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        _check(_lib.mlk_ctx_create(int(device), int(nranks), int(rank), idbuf,
                                   C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h
        self.device, self.nranks, self.rank = device, nranks, rank
        self.has_comm = nccl_id is not None

    @property
    def stream(self):
        return _lib.mlk_ctx_stream(self.h)

    def set_timing(self, on=True):
        _check(_lib.mlk_ctx_set_timing(self.h, 1 if on else 0))

    def reset_stats(self):
        _check(_lib.mlk_ctx_reset_stats(self.h))

    def kernel_stats(self):
        cnt = C.c_int()
        _check(_lib.mlk_ctx_kernel_stats(self.h, 0, C.byref(cnt), None, 0, None, None))
        out = {}
        buf = C.create_string_buffer(128)
        for i in range(cnt.value):
            l = C.c_int64()
            ms = C.c_double()
            _check(_lib.mlk_ctx_kernel_stats(self.h, i, None, buf, 128, C.byref(l), C.byref(ms)))
            out[buf.value.decode()] = dict(launches=l.value, ms=ms.value)
        return out

    def wait_copies(self):
        """Block until every mlk_cw_export_async copy of this context has landed."""
        _check(_lib.mlk_ctx_wait_copies(self.h))

    def close(self):
        if getattr(self, "h", None):
            _lib.mlk_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Tree:
    def __init__(self, h, ctx=None):
        self.h = h
        self.ctx = ctx  # keeps the context (and its stream) alive while the tree lives
        t, nn, n, d = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int32()
        _check(_lib.mlk_tree_info(h, C.byref(t), C.byref(nn), C.byref(n), C.byref(d)))
        self.t, self.n_nodes, self.n, self.d = t.value, nn.value, n.value, d.value

    def export(self):
        nn, n, d = self.n_nodes, self.n, self.d
        perm = np.empty(n, np.int64)
        begin = np.empty(nn, np.int64)
        end = np.empty(nn, np.int64)
        depth = np.empty(nn, np.int32)
        state = np.empty(nn, np.int32)
        thr = np.empty(nn, np.float64)
        dirs = np.empty((nn, d), np.float64)
        _check(_lib.mlk_tree_export(self.h, _np(perm), _np(begin), _np(end), _np(depth), _np(state),
                                    _np(thr), _np(dirs)))
        return dict(perm=perm, begin=begin, end=end, depth=depth, state=state, thr=thr, dirs=dirs)

    def __del__(self):
        if getattr(self, "h", None):
            _lib.mlk_tree_free(self.h)
            self.h = None


def build_tree(ctx, X, leaf_size, kind, directions=None):
    Xp, keep = _ptr(X, device=ctx.device)
    n, d = X.shape
    Dp, keep2 = _ptr(directions, device=ctx.device)
    nrows = 0 if directions is None else directions.shape[0]
    h = C.c_void_p()
    _check(_lib.mlk_build_tree(ctx.h, Xp, n, d, int(leaf_size), int(kind), Dp, nrows, C.byref(h)))
    return Tree(h, ctx)


class Basis:
    def __init__(self, h, tree, ctx=None):
        self.h = h
        self.tree = tree
        self.ctx = ctx
        M, dim, nc = C.c_int32(), C.c_int64(), C.c_int32()
        _check(_lib.mlk_basis_info(h, C.byref(M), C.byref(dim), C.byref(nc)))
        self.M, self.dim, self.n_cells = M.value, dim.value, nc.value
        self.cells = np.empty(self.n_cells, np.int32)
        self.row_off = np.empty(self.n_cells + 1, np.int64)
        _check(_lib.mlk_basis_export(h, _np(self.cells), _np(self.row_off), -1, None, None, None))

    def block(self, node, size, phi=True):
        """(W_node, Phi_node) host copies; size = number of points of the node.  phi=False
        skips Phi (returns None for it), as needed when the basis kept only L (BASIS_DROP_PHI)."""
        pos = np.nonzero(self.cells == node)[0]
        p = int(self.row_off[pos[0] + 1] - self.row_off[pos[0]]) if pos.size else 0
        W = np.empty((p, size), np.float64)
        Phi = np.empty((self.M, size), np.float64) if phi else None
        _check(_lib.mlk_basis_export(self.h, None, None, int(node), _np(W), _np(Phi) if phi else None, None))
        return W, Phi

    def L(self):
        L = np.empty((self.M, self.tree.n), np.float64)
        _check(_lib.mlk_basis_export(self.h, None, None, -1, None, None, _np(L)))
        return L

    def __del__(self):
        if getattr(self, "h", None):
            _lib.mlk_basis_free(self.h)
            self.h = None


BASIS_KEEP_DEFICIENT = 1
BASIS_DROP_PHI = 2


def build_basis(ctx, tree, w, index_set=INDEX_TD, flags=0):
    h = C.c_void_p()
    if index_set == INDEX_TD and flags == 0:
        _check(_lib.mlk_build_basis(ctx.h, tree.h, int(w), C.byref(h)))
    else:
        _check(_lib.mlk_build_basis_ex(ctx.h, tree.h, int(index_set), int(w), int(flags), C.byref(h)))
    return Basis(h, tree, ctx)


def _numel(x):
    return int(x.numel()) if hasattr(x, "numel") and callable(x.numel) else int(np.size(x))


def _vec_io(x, in_cols, out, out_cols, device=None):
    """Marshal an (nvec, in_cols) input and an (nvec, out_cols) output (checked sizes / dtypes)."""
    xp, keep = _ptr(x, device=device)
    nvec = 1 if x.ndim == 1 else x.shape[0]
    if _numel(x) != nvec * in_cols:
        raise ValueError("input has %d entries, expected %d x %d" % (_numel(x), nvec, in_cols))
    if out is None:
        res = np.empty((nvec, out_cols), np.float64)
        op = _np(res)
    else:
        if _numel(out) != nvec * out_cols:
            raise ValueError("output has %d entries, expected %d x %d" % (_numel(out), nvec, out_cols))
        res = out
        op, _ = _ptr(out, device=device, out=True)
    return xp, keep, nvec, res, op


def apply_wt(ctx, basis, v, out=None):
    vp, keep, nvec, res, op = _vec_io(v, basis.dim, out, basis.tree.n, ctx.device)
    _check(_lib.mlk_apply_wt(ctx.h, basis.h, vp, op, nvec))
    return res


def apply_w(ctx, basis, b, out=None):
    bp, keep, nvec, res, op = _vec_io(b, basis.tree.n, out, basis.dim, ctx.device)
    _check(_lib.mlk_apply_w(ctx.h, basis.h, bp, op, nvec))
    return res


class CW:
    def __init__(self, h, owners=()):
        self.h = h
        self._owners = owners  # ctx, tree, basis outlive the matrix
        nc, nb, nnz = C.c_int32(), C.c_int64(), C.c_int64()
        ent, fl, oent, ofl = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        _check(_lib.mlk_cw_info(h, C.byref(nc), C.byref(nb), C.byref(nnz), C.byref(ent), C.byref(fl),
                                C.byref(oent), C.byref(ofl)))
        self.n_cells, self.n_blocks, self.nnz = nc.value, nb.value, nnz.value
        self.entries, self.flops = ent.value, fl.value
        self.own_entries, self.own_flops = oent.value, ofl.value

    def structure(self):
        brow_ptr = np.empty(self.n_cells + 1, np.int32)
        bcol = np.empty(self.n_blocks, np.int32)
        val_off = np.empty(self.n_blocks + 1, np.int64)
        _check(_lib.mlk_cw_export(self.h, _np(brow_ptr), _np(bcol), _np(val_off), None))
        return brow_ptr, bcol, val_off

    def export(self, out=None):
        brow_ptr, bcol, val_off = self.structure()
        vals = np.empty(self.nnz, np.float64) if out is None else out
        if _numel(vals) < self.nnz:
            raise ValueError("output holds %d values, need %d" % (_numel(vals), self.nnz))
        vp, _ = _ptr(vals, out=True)
        _check(_lib.mlk_cw_export(self.h, None, None, None, vp))
        return dict(brow_ptr=brow_ptr, bcol=bcol, val_off=val_off, values=vals)

    def export_async(self, ctx, out):
        """Enqueue the copy of all BSR values into `out` (NumPy array or torch tensor, ideally
        pinned) behind the work already on the context stream; ctx.wait_copies() completes it."""
        if _numel(out) < self.nnz:
            raise ValueError("output holds %d values, need %d" % (_numel(out), self.nnz))
        vp, _ = _ptr(out, device=ctx.device, out=True)
        _check(_lib.mlk_cw_export_async(ctx.h, self.h, vp))
        self._async_keep = out
        return out

    def stage_flops(self):
        g, a, b = C.c_double(), C.c_double(), C.c_double()
        _check(_lib.mlk_cw_flops(self.h, C.byref(g), C.byref(a), C.byref(b)))
        return dict(gram=g.value, contract1=a.value, contract2=b.value)

    def plan(self):
        """dict(nested, transfer_flops, nested_tile_flops) of mlk_cw_plan."""
        nst, tf, nf = C.c_int32(), C.c_double(), C.c_double()
        _check(_lib.mlk_cw_plan(self.h, C.byref(nst), C.byref(tf), C.byref(nf)))
        return dict(nested=bool(nst.value), transfer_flops=tf.value, nested_tile_flops=nf.value)

    def owner(self):
        o = np.empty(self.n_blocks, np.int32)
        _check(_lib.mlk_cw_owner(self.h, _np(o)))
        return o

    def shard_len(self):
        a, b = C.c_int64(), C.c_int64()
        _check(_lib.mlk_cw_shard_len(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def values_ptr(self):
        p = C.c_void_p()
        _check(_lib.mlk_cw_values_device(self.h, C.byref(p)))
        return p.value

    def pieces(self, with_shard=True):
        """(piece_ptr, piece_off, piece_owner, shard): the piece layout and this rank's shard."""
        pp = np.empty(self.n_blocks + 1, np.int64)
        _check(_lib.mlk_cw_export_pieces(self.h, _np(pp), None, None, None))
        npc = int(pp[-1])
        po = np.empty(max(npc, 1), np.int64)
        pw = np.empty(max(npc, 1), np.int32)
        sl, _ = self.shard_len()
        sh = np.empty(max(sl, 1), np.float64) if with_shard else None
        _check(_lib.mlk_cw_export_pieces(self.h, None, _np(po), _np(pw), _np(sh) if with_shard else None))
        return pp, po[:npc], pw[:npc], (sh[:sl] if with_shard else None)

    def host_values(self):
        """Zero-copy NumPy view of the values of a VALUES_HOST matrix (valid while cw lives)."""
        if getattr(self, "placement", VALUES_DEVICE) != VALUES_HOST:
            raise MlkError(1, "host_values() needs placement VALUES_HOST")
        arr = np.ctypeslib.as_array(C.cast(self.values_ptr(), C.POINTER(C.c_double)), shape=(max(self.nnz, 1),))
        return arr[:self.nnz]

    def __del__(self):
        if getattr(self, "h", None):
            _lib.mlk_cw_free(self.h)
            self.h = None


def assemble_cw(ctx, tree, basis, kernel, sparsity, precision=PREC_FP64, placement=VALUES_DEVICE, gather=None):
    """mlk_assemble_cw_ex: values in device memory (VALUES_DEVICE) or mapped pinned host memory
    (VALUES_HOST, for matrices beyond HBM).  gather (nranks > 1): GATHER_NONE keeps this rank's
    shard, GATHER_DEVICE all-gathers over the context's NCCL communicator; default: gather iff the
    context has a communicator."""
    h = C.c_void_p()
    ks = _kspec(kernel)
    sp = sparsity if isinstance(sparsity, SparsitySpec) else SparsitySpec(int(sparsity["mode"]),
                                                                           float(sparsity.get("tau", 0.0)))
    if gather is None:
        gather = GATHER_DEVICE if getattr(ctx, "has_comm", False) else GATHER_NONE
    _check(_lib.mlk_assemble_cw_ex(ctx.h, tree.h, basis.h, C.byref(ks), C.byref(sp), int(precision),
                                   int(placement), 1 if gather else 0, C.byref(h)))
    cw = CW(h, (ctx, tree, basis))
    cw.placement = placement
    return cw


def gather_cw(ctx, cw, group=None):
    """Caller-side all-gather of the BSR shards over a torch.distributed group (for contexts
    without a library communicator): pack this rank's pieces, all_gather_into_tensor, unpack
    into BSR order.  Contexts with a communicator gather inside assemble_cw."""
    import torch
    import torch.distributed as dist

    if ctx.nranks == 1 or getattr(ctx, "has_comm", False):
        return
    _, mx = cw.shard_len()
    dev = torch.device("cuda", ctx.device)
    send = torch.empty(max(mx, 1), dtype=torch.float64, device=dev)
    _check(_lib.mlk_cw_pack(ctx.h, cw.h, C.c_void_p(send.data_ptr())))
    recv = torch.empty(ctx.nranks * max(mx, 1), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    torch.cuda.current_stream(dev).synchronize()
    _check(_lib.mlk_cw_unpack(ctx.h, cw.h, C.c_void_p(recv.data_ptr())))


def pack_cw(ctx, cw, dst):
    _check(_lib.mlk_cw_pack(ctx.h, cw.h, C.c_void_p(dst.data_ptr())))


def unpack_cw(ctx, cw, gathered):
    _check(_lib.mlk_cw_unpack(ctx.h, cw.h, C.c_void_p(gathered.data_ptr())))


def cov_matvec(ctx, tree, kernel, a, out=None):
    ap, keep, nvec, res, op = _vec_io(a, tree.n, out, tree.n, ctx.device)
    ks = _kspec(kernel)
    _check(_lib.mlk_cov_matvec(ctx.h, tree.h, C.byref(ks), ap, op, nvec))
    return res


def cw_matvec(ctx, tree, basis, kernel, cw, mode, v, out=None, allreduce=True, group=None):
    """y = C_W v.  nranks > 1: a context with a library communicator returns the allreduced y;
    otherwise the partial results are sum-allreduced here over `group` (torch.distributed)
    unless allreduce=False."""
    vp, keep, nvec, res, op = _vec_io(v, basis.dim, out, basis.dim, ctx.device)
    ks = _kspec(kernel) if kernel is not None else kernel_spec(0, 1.0)
    _check(_lib.mlk_cw_matvec(ctx.h, tree.h, basis.h, C.byref(ks), cw.h if cw is not None else None,
                              int(mode), vp, op, nvec))
    if ctx.nranks > 1 and allreduce and not getattr(ctx, "has_comm", False):
        import torch
        import torch.distributed as dist

        if isinstance(res, np.ndarray):
            t = torch.from_numpy(res).to(torch.device("cuda", ctx.device))
            dist.all_reduce(t, group=group)
            res[...] = t.cpu().numpy()
        else:
            dist.all_reduce(res, group=group)
    return res


def pcg_solve(ctx, tree, basis, kernel, cw, z_w, tol=1e-10, max_iter=1000, precond=True, out=None):
    """gamma_W = C_W^-1 z_W by PCG with the block-diagonal preconditioner (cw's self blocks) or
    none.  Returns (gamma_W, iterations, true relative residual)."""
    zp, keep = _ptr(z_w, device=ctx.device)
    if _numel(z_w) != basis.dim:
        raise ValueError("z_w has %d entries, expected %d" % (_numel(z_w), basis.dim))
    if out is None:
        res = np.empty(basis.dim, np.float64)
        op = _np(res)
    else:
        if _numel(out) != basis.dim:
            raise ValueError("out has %d entries, expected %d" % (_numel(out), basis.dim))
        res = out
        op, _ = _ptr(out, device=ctx.device, out=True)
    it = C.c_int32()
    rr = C.c_double()
    _check(_lib.mlk_pcg_solve(ctx.h, tree.h, basis.h, C.byref(_kspec(kernel)), cw.h if cw is not None else None,
                              1 if precond else 0, zp, op, float(tol), int(max_iter), C.byref(it), C.byref(rr)))
    return res, it.value, rr.value


def loglik(ctx, basis, cw, z_w, level=0):
    """Level-truncated multi-level log-likelihood (mlk_loglik): returns dict(loglik, logdet,
    quad, n_tilde) for the cells of levels t .. level."""
    zp, keep = _ptr(z_w, device=ctx.device)
    if _numel(z_w) != basis.dim:
        raise ValueError("z_w has %d entries, expected %d" % (_numel(z_w), basis.dim))
    ll, ld, q, nt = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
    _check(_lib.mlk_loglik(ctx.h, basis.h, cw.h, int(level), zp, C.byref(ll), C.byref(ld), C.byref(q), C.byref(nt)))
    return dict(loglik=ll.value, logdet=ld.value, quad=q.value, n_tilde=nt.value)


def partition_lpt(cost, nranks):
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    owner = np.empty(cost.size, np.int32)
    _check(_lib.mlk_partition_lpt(_np(cost), cost.size, int(nranks), _np(owner)))
    return owner


def gather_plan(piece_ptr, piece_off, piece_owner, block_len, nranks, budget):
    """(group_ptr, group_lo[n_groups, nranks], group_count) of the chunked all-gather (host only)."""
    pp = np.ascontiguousarray(piece_ptr, dtype=np.int64)
    po = np.ascontiguousarray(piece_off, dtype=np.int64)
    pw = np.ascontiguousarray(piece_owner, dtype=np.int32)
    bl = np.ascontiguousarray(block_len, dtype=np.int64)
    nb = bl.size
    ng = C.c_int64()
    _check(_lib.mlk_gather_plan(nb, _np(pp), _np(po), _np(pw), _np(bl), int(nranks), int(budget), C.byref(ng),
                                None, None, None))
    g = ng.value
    gp = np.empty(g + 1, np.int64)
    gl = np.empty(max(g * nranks, 1), np.int64)
    gc = np.empty(max(g, 1), np.int64)
    _check(_lib.mlk_gather_plan(nb, _np(pp), _np(po), _np(pw), _np(bl), int(nranks), int(budget), C.byref(ng),
                                _np(gp), _np(gl), _np(gc)))
    return gp, gl[:g * nranks].reshape(g, nranks), gc[:g]


def shard_plan(val_off, owner, nranks):
    """(shard_off[n], shard_len[nranks]) -- the gather layout of mlk_assemble_cw (host only)."""
    val_off = np.ascontiguousarray(val_off, dtype=np.int64)
    owner = np.ascontiguousarray(owner, dtype=np.int32)
    n = owner.size
    so = np.empty(n, np.int64)
    sl = np.empty(int(nranks), np.int64)
    _check(_lib.mlk_shard_plan(_np(val_off), _np(owner), n, int(nranks), _np(so), _np(sl)))
    return so, sl
