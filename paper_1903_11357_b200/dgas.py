"""Thin ctypes binding of libdgas.so (include/dgas.h). Argument marshalling only: every step of the
method runs in the library's CUDA kernels. There is no CPU fallback: if the shared library is
missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdgas.so")
_lib = None
_P = ctypes.c_void_p

OK, NOT_CONVERGED = 0, 1
E_INVALID_ARG, E_MESH, E_NOT_SPD, E_BREAKDOWN, E_CUDA, E_NOMEM = -1, -2, -3, -4, -5, -6

EXPORTS = ["dgas_setup", "dgas_rhs", "dgas_spmv", "dgas_apply", "dgas_pcg", "dgas_pcg_host", "dgas_info",
           "dgas_history", "dgas_debug_block", "dgas_debug_basis", "dgas_debug_A0", "dgas_bench_kernels",
           "dgas_destroy", "dgas_strerror", "dgas_error_detail", "dgas_set_precond", "dgas_shard",
           "dgas_shard_begin", "dgas_shard_precond", "dgas_shard_direction", "dgas_shard_spmv", "dgas_shard_update",
           "dgas_shard_finish"]
PRECOND = {"two_level": 0, "one_level": 1, "coarse": 2, "none": 3}   # DGAS_PRECOND_* (include/dgas.h)


class Mesh(ctypes.Structure):
    _fields_ = [("n_vertices", ctypes.c_int32), ("xy", _P), ("n_cells", ctypes.c_int32), ("cell_ptr", _P),
                ("cell_vtx", _P)]


class Coarse(ctypes.Structure):
    _fields_ = [("n_coarse", ctypes.c_int32), ("parent", _P), ("n_overlaps", ctypes.c_int32), ("ov_fine", _P),
                ("ov_coarse", _P), ("ov_ptr", _P), ("ov_xy", _P)]


class Info(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("N0", ctypes.c_int64),
                ("n_cells", ctypes.c_int32), ("n_p", ctypes.c_int32), ("n_q", ctypes.c_int32),
                ("n_subdomains", ctypes.c_int32), ("n_coarse", ctypes.c_int32), ("n_faces", ctypes.c_int32),
                ("n_overlaps", ctypes.c_int32), ("coarse_dense", ctypes.c_int32), ("coarse_band", ctypes.c_int32),
                ("nnz_blocks", ctypes.c_int64), ("bytes_A", ctypes.c_int64), ("bytes_U", ctypes.c_int64),
                ("bytes_Dinv", ctypes.c_int64), ("bytes_G", ctypes.c_int64), ("bytes_coarse", ctypes.c_int64),
                ("alg_bytes_spmv", ctypes.c_int64), ("alg_bytes_apply", ctypes.c_int64),
                ("alg_bytes_iter", ctypes.c_int64), ("last_iters", ctypes.c_int32), ("last_status", ctypes.c_int32),
                ("last_cond", ctypes.c_double), ("last_lmin", ctypes.c_double), ("last_lmax", ctypes.c_double),
                ("last_relres", ctypes.c_double), ("coarse_mode", ctypes.c_int32), ("launches_per_iter", ctypes.c_int32),
                ("launches_per_solve", ctypes.c_int32), ("coarse_refine", ctypes.c_int32),
                ("coarse_solve_relerr", ctypes.c_double), ("unroll", ctypes.c_int32),
                ("local_kernel", ctypes.c_int32), ("local_ctas_per_sm", ctypes.c_int32),
                ("bytes_local", ctypes.c_int64), ("local_inv_err", ctypes.c_double),
                ("dedup_A_bytes", ctypes.c_int64), ("dedup_local_bytes", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def load():
    """Load the in-tree library; raise if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libdgas.so not built at {LIB_PATH}: run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    L.dgas_setup.argtypes = [ctypes.POINTER(_P), ctypes.POINTER(Mesh), ctypes.c_int, _P, ctypes.c_int32,
                             ctypes.POINTER(Coarse), ctypes.c_int, _P, ctypes.c_double, _P]
    L.dgas_rhs.argtypes = [_P, ctypes.c_int, _P, _P]
    L.dgas_spmv.argtypes = [_P, _P, _P, _P]
    L.dgas_apply.argtypes = [_P, _P, _P, _P]
    L.dgas_pcg.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                           ctypes.POINTER(ctypes.c_double), _P]
    L.dgas_pcg_host.argtypes = L.dgas_pcg.argtypes
    L.dgas_info.argtypes = [_P, ctypes.POINTER(Info)]
    L.dgas_history.argtypes = [_P, _P, _P, ctypes.c_int]
    L.dgas_debug_block.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, _P]
    L.dgas_debug_basis.argtypes = [_P, ctypes.c_int32, _P]
    L.dgas_debug_A0.argtypes = [_P, _P]
    L.dgas_bench_kernels.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P]
    L.dgas_set_precond.argtypes = [_P, ctypes.c_int]
    L.dgas_destroy.argtypes = [_P]
    L.dgas_shard.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, _P]
    L.dgas_shard_begin.argtypes = [_P, _P, _P, _P]
    L.dgas_shard_precond.argtypes = [_P, _P, _P, _P]
    L.dgas_shard_direction.argtypes = [_P, _P, _P, ctypes.c_int32, _P]
    L.dgas_shard_spmv.argtypes = [_P, _P, _P, _P]
    L.dgas_shard_update.argtypes = [_P, _P, _P, _P]
    L.dgas_shard_finish.argtypes = [_P, ctypes.c_int32, _P, _P, _P]
    L.dgas_strerror.restype = ctypes.c_char_p
    L.dgas_strerror.argtypes = [ctypes.c_int]
    L.dgas_error_detail.restype = ctypes.c_char_p
    L.dgas_error_detail.argtypes = [_P]
    _lib = L
    return L


class DgasError(RuntimeError):
    def __init__(self, code, detail=""):
        msg = load().dgas_strerror(code).decode()
        super().__init__(f"dgas status {code} ({msg}){': ' + detail if detail else ''}")
        self.code = code


def _stream(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dptr(t):
    import torch
    assert isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
    return ctypes.c_void_p(t.data_ptr())


class Solver:
    """One dgas context built from a generated problem (dgas_gen.Problem) or raw arrays."""

    def __init__(self, problem, p=None, q=None, penalty=None, stream=None):
        L = load()
        P = problem
        self.p = P.p if p is None else p
        self.q = P.q if q is None else q
        self._keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a.ctypes.data

        mesh = Mesh(P.xy.shape[0], arr(P.xy, np.float64), P.n_cells, arr(P.cell_ptr, np.int32),
                    arr(P.cell_vtx, np.int32))
        if P.nested:
            coarse = Coarse(P.n_coarse, arr(P.parent, np.int32), 0, None, None, None, None)
        else:
            coarse = Coarse(P.n_coarse, None, len(P.ov_fine), arr(P.ov_fine, np.int32), arr(P.ov_coarse, np.int32),
                            arr(P.ov_ptr, np.int32), arr(P.ov_xy, np.float64))
        ctx = _P()
        st = L.dgas_setup(ctypes.byref(ctx), ctypes.byref(mesh), self.p, arr(P.part, np.int32), P.n_sub,
                          ctypes.byref(coarse), self.q, arr(P.kappa, np.float64),
                          P.penalty if penalty is None else penalty, _stream(stream))
        self.ctx = ctx
        if st != 0:
            detail = L.dgas_error_detail(ctx).decode() if ctx.value else ""
            if ctx.value:
                L.dgas_destroy(ctx)
                self.ctx = None
            raise DgasError(st, detail)
        self._keep = []
        self.info = self.get_info()
        self.N = self.info["N"]
        self.N0 = self.info["N0"]

    def close(self):
        if getattr(self, "ctx", None):
            load().dgas_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st < 0:
            raise DgasError(st, load().dgas_error_detail(self.ctx).decode())
        return st

    def get_info(self):
        inf = Info()
        self._check(load().dgas_info(self.ctx, ctypes.byref(inf)))
        return inf.as_dict()

    # -------------------------------------------------------------- device-vector API (torch tensors)
    def rhs(self, f_kind, out=None, stream=None):
        import torch
        b = torch.empty(self.N, dtype=torch.float64, device="cuda") if out is None else out
        self._check(load().dgas_rhs(self.ctx, f_kind, _dptr(b), _stream(stream)))
        return b

    def spmv(self, x, out=None, stream=None):
        import torch
        y = torch.empty_like(x) if out is None else out
        self._check(load().dgas_spmv(self.ctx, _dptr(x), _dptr(y), _stream(stream)))
        return y

    def apply(self, r, out=None, stream=None):
        import torch
        z = torch.empty_like(r) if out is None else out
        self._check(load().dgas_apply(self.ctx, _dptr(r), _dptr(z), _stream(stream)))
        return z

    def set_precond(self, mode):
        """mode: "two_level" (default), "one_level", "coarse" or "none" (plain CG)."""
        self._check(load().dgas_set_precond(self.ctx, PRECOND[mode] if isinstance(mode, str) else int(mode)))

    def pcg(self, b, x=None, rtol=1e-8, maxit=5000, stream=None):
        """Solve A x = b (device tensors). Returns (x, iters, cond, status)."""
        import torch
        x = torch.zeros_like(b) if x is None else x
        it = ctypes.c_int(0)
        cond = ctypes.c_double(0)
        st = self._check(load().dgas_pcg(self.ctx, _dptr(b), _dptr(x), rtol, maxit, ctypes.byref(it),
                                         ctypes.byref(cond), _stream(stream)))
        return x, it.value, cond.value, st

    def pcg_host(self, b_host, x_host, rtol=1e-8, maxit=5000, stream=None):
        """Same with host (ideally pinned) float64 tensors or numpy arrays."""
        it = ctypes.c_int(0)
        cond = ctypes.c_double(0)
        bp = b_host.data_ptr() if hasattr(b_host, "data_ptr") else b_host.ctypes.data
        xp = x_host.data_ptr() if hasattr(x_host, "data_ptr") else x_host.ctypes.data
        st = self._check(load().dgas_pcg_host(self.ctx, ctypes.c_void_p(bp), ctypes.c_void_p(xp), rtol, maxit,
                                              ctypes.byref(it), ctypes.byref(cond), _stream(stream)))
        return it.value, cond.value, st

    def history(self):
        n = self.get_info()["last_iters"]
        a = np.zeros(max(n, 1)); b = np.zeros(max(n, 1))
        load().dgas_history(self.ctx, a.ctypes.data, b.ctypes.data, n)
        return a[:n], b[:n]

    def bench_kernels(self, which, reps, stream=None):
        self._check(load().dgas_bench_kernels(self.ctx, which, reps, _stream(stream)))

    # -------------------------------------------------------------- diagnostics (host)
    def block(self, i, j):
        np_ = self.info["n_p"]
        out = np.zeros((np_, np_))
        ok = self._check(load().dgas_debug_block(self.ctx, i, j, out.ctypes.data))
        return out, bool(ok)

    def basis(self, i):
        np_ = self.info["n_p"]
        out = np.zeros((np_, np_))
        self._check(load().dgas_debug_basis(self.ctx, i, out.ctypes.data))
        return out

    def A0(self):
        out = np.zeros((self.N0, self.N0))
        self._check(load().dgas_debug_A0(self.ctx, out.ctypes.data))
        return out


class ShardBackend:
    """Marshalling of the dgas_shard_* entry points (include/dgas.h) for one rank of a Solver."""

    def __init__(self, solver, rank, nranks):
        import torch
        self.S = solver
        info = np.zeros(6, np.int64)
        solver._check(load().dgas_shard(solver.ctx, rank, nranks, info.ctypes.data))
        self.dof_begin, self.dof_end, self.cap, self.N, self.N0, self.n_sub_own = (int(v) for v in info)
        self.device = torch.device("cuda", torch.cuda.current_device())

    def zeros(self, n):
        import torch
        return torch.zeros(n, dtype=torch.float64, device=self.device)

    def begin(self, b, red0):
        self.S._check(load().dgas_shard_begin(self.S.ctx, _dptr(b), _dptr(red0), _stream()))

    def precond(self, red0, red1):
        self.S._check(load().dgas_shard_precond(self.S.ctx, _dptr(red0), _dptr(red1), _stream()))

    def direction(self, red1, hsend, first):
        self.S._check(load().dgas_shard_direction(self.S.ctx, _dptr(red1), _dptr(hsend), int(first), _stream()))

    def spmv(self, hall, red2):
        self.S._check(load().dgas_shard_spmv(self.S.ctx, _dptr(hall), _dptr(red2), _stream()))

    def update(self, red2, red0):
        self.S._check(load().dgas_shard_update(self.S.ctx, _dptr(red2), _dptr(red0), _stream()))

    def finish(self, iters, x, lanczos):
        return self.S._check(load().dgas_shard_finish(self.S.ctx, int(iters), _dptr(x), _dptr(lanczos), _stream()))


class ShardedSolver:
    """Subdomain-sharded ASPCG over torch.distributed ranks (include/dgas.h "Sharded").

    Every rank owns a contiguous range of subdomains of its (replicated) Solver; the arithmetic runs in the
    dgas_shard_* kernels, the collectives are torch.distributed calls between them (NCCL on GPUs, gloo in
    the tests). `backend` defaults to the rank's ShardBackend; the tests substitute a CPU mock with the same
    buffer semantics to check this driver's collective schedule."""

    def __init__(self, solver=None, group=None, backend=None):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        self.B = backend if backend is not None else ShardBackend(solver, self.rank, self.nranks)

    def _sum(self, t):
        import torch.distributed as dist
        if self.nranks > 1:
            dist.all_reduce(t, group=self.group)

    def _gather(self, hall, hsend):
        import torch.distributed as dist
        if self.nranks > 1:
            dist.all_gather(list(hall.view(self.nranks, -1).unbind(0)), hsend, group=self.group)
        else:
            hall.copy_(hsend)

    def pcg(self, b, rtol=1e-8, maxit=5000):
        """Solve A x = b (b: the full right-hand side, caller order, on every rank). Returns
        (x, iters, cond, status) with x the full solution on every rank (PAPER.md:741 protocol, R11/R12)."""
        B, N0 = self.B, self.B.N0
        red0, red1, red2 = B.zeros(N0 + 2), B.zeros(1), B.zeros(1)
        hsend, hall = B.zeros(B.cap), B.zeros(self.nranks * B.cap)
        B.begin(b, red0)
        self._sum(red0)
        bb = float(red0[N0 + 1])
        stop2 = rtol * rtol * bb
        it, status = 0, 1  # DGAS_NOT_CONVERGED until the stop test holds
        if bb > 0:
            B.precond(red0, red1)
            self._sum(red1)
            B.direction(red1, hsend, True)
            self._gather(hall, hsend)
            while it < maxit:
                B.spmv(hall, red2)
                self._sum(red2)
                B.update(red2, red0)
                self._sum(red0)
                it += 1
                if float(red0[N0]) <= stop2:  # ||r||^2 <= rtol^2 ||b||^2 after the update (R11)
                    status = 0
                    break
                B.precond(red0, red1)
                self._sum(red1)
                B.direction(red1, hsend, False)
                self._gather(hall, hsend)
        else:
            status = 0
        x, lz = B.zeros(B.N), B.zeros(3)
        st = B.finish(it, x, lz)
        self._sum(x)
        cond = float(lz[2]) if it > 0 else 1.0
        return x, it, cond, st if st < 0 else status
