"""CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle.cpp header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this package. The product path (paper_1903_11357_b200) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None
_P = ctypes.c_void_p


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.or_create.restype = _P
        L.or_create.argtypes = [ctypes.c_int, _P, ctypes.c_int, _P, _P, _P, ctypes.c_int, _P, ctypes.c_int,
                                ctypes.c_double]
        L.or_message.restype = ctypes.c_char_p
        L.or_message.argtypes = [_P]
        L.or_status.argtypes = [_P]
        L.or_free.argtypes = [_P]
        L.or_sizes.argtypes = [_P, _P]
        L.or_basis.argtypes = [_P, ctypes.c_int, _P, _P]
        L.or_eval_basis.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P]
        L.or_block.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P]
        L.or_dense_A.argtypes = [_P, _P]
        L.or_spmv.argtypes = [_P, _P, _P]
        L.or_rhs.argtypes = [_P, ctypes.c_int, _P]
        L.or_spmv_abs.argtypes = [_P, _P, _P]
        L.or_project.argtypes = [_P, ctypes.c_int, _P]
        L.or_errors.argtypes = [_P, _P, _P]
        L.or_setup_schwarz.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, _P, ctypes.c_int, ctypes.c_int]
        L.or_apply.argtypes = [_P, _P, _P]
        L.or_apply_ld.argtypes = [_P, _P, _P]
        L.or_apply_sampled.argtypes = [_P, ctypes.c_int, _P, _P, _P]
        L.or_apply_sampled_ld.argtypes = [_P, ctypes.c_int, _P, _P, _P]
        L.or_set_refine.argtypes = [_P, ctypes.c_int]
        L.or_set_perturb.argtypes = [_P, ctypes.c_double, ctypes.c_uint64]
        L.or_perturb_A.argtypes = [_P, ctypes.c_double, ctypes.c_uint64]
        L.or_get_G.argtypes = [_P, _P]
        L.or_get_A0.argtypes = [_P, _P]
        L.or_coarse_basis.argtypes = [_P, ctypes.c_int, _P, _P]
        L.or_pcg.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P]
        L.or_pcg_ext.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P,
                                 ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P]
        L.or_set_threads.argtypes = [ctypes.c_int]
        L.or_get_threads.restype = ctypes.c_int
        L.or_lanczos.argtypes = [ctypes.c_int, _P, _P, _P]
        L.or_triangle_rule.argtypes = [ctypes.c_int, _P]
        L.or_gauss_legendre.argtypes = [ctypes.c_int, _P, _P]
        L.or_poly_monomial.restype = ctypes.c_double
        L.or_poly_monomial.argtypes = [ctypes.c_int, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class Oracle:
    """Oracle for one generated Problem (caller's cell order; dof (cell c, mode a) = c*n_p + a)."""

    def __init__(self, P, p=None, q=None, penalty=None, part=None, n_sub=None):
        L = lib()
        self.P = P
        self.p = P.p if p is None else p
        self.q = P.q if q is None else q
        self.np_ = (self.p + 1) * (self.p + 2) // 2
        self.nq_ = (self.q + 1) * (self.q + 2) // 2
        self.part = np.ascontiguousarray(P.part if part is None else part, dtype=np.int32)
        self.n_sub = P.n_sub if n_sub is None else n_sub
        self._keep = [np.ascontiguousarray(P.xy, dtype=np.float64), np.ascontiguousarray(P.cell_ptr, np.int32),
                      np.ascontiguousarray(P.cell_vtx, np.int32), self.part, np.ascontiguousarray(P.kappa, np.float64)]
        xy, cp, cv, pt, ka = self._keep
        self.h = L.or_create(xy.shape[0], _ptr(xy), P.n_cells, _ptr(cp), _ptr(cv), _ptr(pt), self.n_sub, _ptr(ka),
                             self.p, P.penalty if penalty is None else penalty)
        self._check()
        self.N = P.n_cells * self.np_
        self.N0 = None

    def _check(self, code=None):
        L = lib()
        st = L.or_status(self.h) if code is None else code
        if st != 0:
            raise OracleError(st, L.or_message(self.h).decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_free(self.h)
            self.h = None

    # ------------------------------------------------------------------ assembly
    def basis(self, cell):
        C = np.zeros((self.np_, self.np_)); bb = np.zeros(4)
        lib().or_basis(self.h, cell, _ptr(C), _ptr(bb))
        return C, bb

    def eval_basis(self, cell, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        n = pts.shape[0]
        phi = np.zeros((n, self.np_)); px = np.zeros_like(phi); py = np.zeros_like(phi)
        lib().or_eval_basis(self.h, cell, n, _ptr(pts), _ptr(phi), _ptr(px), _ptr(py))
        return phi, px, py

    def block(self, i, j):
        out = np.zeros((self.np_, self.np_))
        ok = lib().or_block(self.h, i, j, _ptr(out))
        return out, bool(ok)

    def dense_A(self):
        A = np.zeros((self.N, self.N))
        lib().or_dense_A(self.h, _ptr(A))
        return A

    def spmv(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.N)
        lib().or_spmv(self.h, _ptr(x), _ptr(y))
        return y

    def spmv_abs(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.N)
        lib().or_spmv_abs(self.h, _ptr(x), _ptr(y))
        return y

    def rhs(self, f_kind=None):
        b = np.zeros(self.N)
        lib().or_rhs(self.h, self.P.f_kind if f_kind is None else f_kind, _ptr(b))
        return b

    def project(self, u_kind=0):
        out = np.zeros(self.N)
        lib().or_project(self.h, u_kind, _ptr(out))
        return out

    def errors(self, x):
        out = np.zeros(2)
        x = np.ascontiguousarray(x, dtype=np.float64)
        lib().or_errors(self.h, _ptr(x), _ptr(out))
        return out

    # ------------------------------------------------------------------ Schwarz
    def setup_schwarz(self, use_coarse=True, use_local=True, sample=None, long_double=False, dense_max=8192,
                      coarse=None):
        """coarse: optional (n_coarse, ov_fine, ov_coarse, ov_ptr, ov_xy) overriding the problem's."""
        if coarse is None:
            ncoarse = self.P.n_coarse
            f, c, ptr, xy = self.P.overlaps()
        else:
            ncoarse, f, c, ptr, xy = coarse
        self._ov = [np.ascontiguousarray(f, np.int32), np.ascontiguousarray(c, np.int32),
                    np.ascontiguousarray(ptr, np.int32), np.ascontiguousarray(xy, np.float64)]
        f, c, ptr, xy = self._ov
        smp = None if sample is None else np.ascontiguousarray(sample, np.int32)
        self._smp = smp
        st = lib().or_setup_schwarz(self.h, ncoarse, self.q, f.shape[0], _ptr(f), _ptr(c), _ptr(ptr), _ptr(xy),
                                    int(use_coarse), int(use_local), -1 if smp is None else smp.shape[0], _ptr(smp),
                                    int(long_double), dense_max)
        self._check(st)
        self.n_ov = f.shape[0]
        self.n_coarse = ncoarse
        self.N0 = ncoarse * self.nq_
        return self

    def apply(self, r, long_double=False):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.N)
        st = (lib().or_apply_ld if long_double else lib().or_apply)(self.h, _ptr(r), _ptr(z))
        if st:
            raise OracleError(st, "apply failed (missing factors?)")
        return z

    def set_refine(self, steps):
        """Iterative-refinement steps of the banded coarse solve (R30)."""
        lib().or_set_refine(self.h, steps)

    def set_perturb(self, eps, seed=1):
        """Relative perturbation of G before A0 is formed (sensitivity probe, R30)."""
        lib().or_set_perturb(self.h, eps, seed)

    def perturb_A(self, eps, seed=1):
        """A <- A (1 + eps u), symmetric (sensitivity probe, R22/R30); before setup_schwarz."""
        lib().or_perturb_A(self.h, eps, seed)

    def apply_sampled(self, r, sample, long_double=False):
        r = np.ascontiguousarray(r, dtype=np.float64)
        s = np.ascontiguousarray(sample, np.int32)
        z = np.zeros(self.N)
        f = lib().or_apply_sampled_ld if long_double else lib().or_apply_sampled
        st = f(self.h, s.shape[0], _ptr(s), _ptr(r), _ptr(z))
        if st:
            raise OracleError(st, "sampled apply failed")
        return z

    def G(self):
        out = np.zeros((self.n_ov, self.np_, self.nq_))
        lib().or_get_G(self.h, _ptr(out))
        return out

    def A0(self):
        out = np.zeros((self.N0, self.N0))
        if lib().or_get_A0(self.h, _ptr(out)) != 0:
            raise OracleError(-1, "A0 not stored densely")
        return out

    def coarse_basis(self, J):
        C = np.zeros((self.nq_, self.nq_)); bb = np.zeros(4)
        lib().or_coarse_basis(self.h, J, _ptr(C), _ptr(bb))
        return C, bb

    def dense_precond(self):
        """P^{-1} as a dense matrix (tiny problems only)."""
        M = np.zeros((self.N, self.N))
        e = np.zeros(self.N)
        for i in range(self.N):
            e[:] = 0; e[i] = 1
            M[:, i] = self.apply(e)
        return M

    # ------------------------------------------------------------------ PCG
    def pcg(self, b, rtol=1e-8, maxit=5000, precond=True, x0=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.N) if x0 is None else np.array(x0, dtype=np.float64)
        it = ctypes.c_int(0)
        al = np.zeros(maxit); be = np.zeros(maxit); res = np.zeros(maxit)
        st = lib().or_pcg(self.h, _ptr(b), _ptr(x), rtol, maxit, int(precond), ctypes.byref(it), _ptr(al), _ptr(be),
                          _ptr(res))
        k = it.value
        lz = lanczos(al[:k], be[:max(k - 1, 0)]) if k >= 1 else (np.nan, np.nan, np.nan)
        return dict(status=st, x=x, iters=k, alphas=al[:k], betas=be[:max(k - 1, 0)], resid=res[:k],
                    lmin=lz[0], lmax=lz[1], cond=lz[2])


    def pcg_history(self, b, idx, rtol=1e-8, maxit=5000, extra=2, n_hist=5):
        """PCG as pcg(), also keeping x[idx] after each of the last n_hist iterations and running `extra`
        iterations past the stop test (reference outputs for full-size parity, tools/make_golden.py).
        Returns pcg()'s dict (iters = stopping iteration; alphas/betas of the stopping run) plus
        hist = {j: x_j[idx]} for the iterations j kept and iters_run."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        x = np.zeros(self.N)
        it = ctypes.c_int(0); run = ctypes.c_int(0)
        al = np.zeros(maxit + extra); be = np.zeros(maxit + extra); res = np.zeros(maxit + extra)
        hist = np.zeros((n_hist, idx.shape[0]))
        st = lib().or_pcg_ext(self.h, _ptr(b), _ptr(x), rtol, maxit, 1, ctypes.byref(it), _ptr(al), _ptr(be),
                              _ptr(res), idx.shape[0], _ptr(idx), n_hist, _ptr(hist), extra, ctypes.byref(run))
        k, kr = it.value, run.value
        lz = lanczos(al[:k], be[:max(k - 1, 0)]) if k >= 1 else (np.nan, np.nan, np.nan)
        kept = {j: hist[j % n_hist].copy() for j in range(max(1, kr - n_hist + 1), kr + 1)}
        return dict(status=st, iters=k, iters_run=kr, alphas=al[:k], betas=be[:max(k - 1, 0)], resid=res[:kr],
                    lmin=lz[0], lmax=lz[1], cond=lz[2], hist=kept, x=x)


def set_threads(n):
    """OpenMP threads for the independent-subdomain loops (bitwise-identical results for any n)."""
    lib().or_set_threads(int(n))


def get_threads():
    return lib().or_get_threads()


def lanczos(alphas, betas):
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    b = np.ascontiguousarray(betas if len(betas) else np.zeros(1), dtype=np.float64)
    out = np.zeros(3)
    lib().or_lanczos(a.shape[0], _ptr(a), _ptr(b), _ptr(out))
    return out


def triangle_rule(m):
    out = np.zeros((m * m, 3))
    n = lib().or_triangle_rule(m, _ptr(out))
    return out[:n]


def gauss_legendre(m):
    x = np.zeros(m); w = np.zeros(m)
    lib().or_gauss_legendre(m, _ptr(x), _ptr(w))
    return x, w


def poly_monomial(poly_xy, a, b, m, fan=0):
    xy = np.ascontiguousarray(poly_xy, dtype=np.float64)
    return lib().or_poly_monomial(xy.shape[0], _ptr(xy), a, b, m, fan)
