"""Seeded synthetic input generator (shared by the oracle and the CUDA path; input generation only).

Holds none of the method's arithmetic: it makes meshes, partitions, coarse agglomerates, overlap
pieces (pure geometry) and the rho field, plus counter-based N(0,1) test vectors. See gen.cpp and
DESIGN.md "Input recipe". The five BASELINE.json configs are `config(k)`.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.cpp")
_LIB = os.path.join(_HERE, "libdgas_gen.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.dgas_gen_problem.restype = ctypes.c_void_p
        _lib.dgas_gen_problem.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int]
        _lib.dgas_gen_error.restype = ctypes.c_char_p
        _lib.dgas_gen_error.argtypes = [ctypes.c_void_p]
        _lib.dgas_gen_sizes.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        _lib.dgas_gen_copy.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 12
        _lib.dgas_gen_free.argtypes = [ctypes.c_void_p]
        _lib.dgas_gen_normal.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
    return _lib


F_SINSIN, F_ONE, F_POLY = 0, 1, 2   # f = 2 pi^2 sin(pi x) sin(pi y) | 1 | 2[x(1-x)+y(1-y)]


@dataclass
class Problem:
    """One generated input instance (caller's cell order)."""
    name: str
    xy: np.ndarray          # [n_vertices, 2] float64
    cell_ptr: np.ndarray    # [n_cells+1] int32
    cell_vtx: np.ndarray    # CCW vertex loops, int32
    part: np.ndarray        # [n_cells] subdomain id (T_HH), int32
    n_sub: int
    n_coarse: int
    nested: bool
    parent: np.ndarray | None       # [n_cells] coarse id if nested
    ov_fine: np.ndarray | None      # non-nested: overlap pieces kappa ∩ D_J
    ov_coarse: np.ndarray | None
    ov_ptr: np.ndarray | None       # [n_ov+1] offsets into ov_xy (points)
    ov_xy: np.ndarray | None        # [n_pts, 2]
    cpoly_ptr: np.ndarray | None    # coarse polygons (non-nested only; informational)
    cpoly_xy: np.ndarray | None
    kappa: np.ndarray               # [n_cells] rho per cell (> 0)
    p: int = 1
    q: int = 1
    f_kind: int = F_SINSIN
    penalty: float = 10.0
    meta: dict = field(default_factory=dict)

    @property
    def n_cells(self) -> int:
        return int(self.cell_ptr.shape[0] - 1)

    @property
    def n_p(self) -> int:
        return (self.p + 1) * (self.p + 2) // 2

    @property
    def n_q(self) -> int:
        return (self.q + 1) * (self.q + 2) // 2

    @property
    def N(self) -> int:
        return self.n_cells * self.n_p

    @property
    def N0(self) -> int:
        return self.n_coarse * self.n_q

    def overlaps(self):
        """Overlap pieces (fine, coarse, ptr, xy); for nested problems the pieces are the fine cells."""
        if not self.nested:
            return self.ov_fine, self.ov_coarse, self.ov_ptr, self.ov_xy
        nc = self.n_cells
        fine = np.arange(nc, dtype=np.int32)
        return fine, self.parent.astype(np.int32), self.cell_ptr.copy(), self.xy[self.cell_vtx]


def generate(kind: int, n: int, seed: int = 0, lloyd: int = 5, sub_mode: int = 0, sub_tile: int = 8,
             n_sub: int = 1, coarse_mode: int = 0, coarse_tile: int = 1, n_coarse: int = 1, kappa_mode: int = 0,
             name: str = "custom", **kw) -> Problem:
    lib = _load()
    h = lib.dgas_gen_problem(kind, n, seed, lloyd, sub_mode, sub_tile, n_sub, coarse_mode, coarse_tile, n_coarse,
                             kappa_mode)
    try:
        err = lib.dgas_gen_error(h)
        if err:
            raise RuntimeError("generator: " + err.decode())
        s = np.zeros(9, np.int64)
        lib.dgas_gen_sizes(h, s.ctypes.data)
        nv, nc, ncv, nsub, ncoarse, nested, nov, novp, ncp = [int(v) for v in s]
        xy = np.zeros((nv, 2)); cptr = np.zeros(nc + 1, np.int32); cvtx = np.zeros(ncv, np.int32)
        part = np.zeros(nc, np.int32); parent = np.zeros(nc, np.int32); kappa = np.zeros(nc)
        ovf = np.zeros(nov, np.int32); ovc = np.zeros(nov, np.int32); ovp = np.zeros(nov + 1, np.int32)
        ovxy = np.zeros((novp, 2)); cpp = np.zeros(ncoarse + 1, np.int32); cpxy = np.zeros((ncp, 2))
        lib.dgas_gen_copy(h, xy.ctypes.data, cptr.ctypes.data, cvtx.ctypes.data, part.ctypes.data,
                          parent.ctypes.data, kappa.ctypes.data, ovf.ctypes.data, ovc.ctypes.data, ovp.ctypes.data,
                          ovxy.ctypes.data, cpp.ctypes.data, cpxy.ctypes.data)
    finally:
        lib.dgas_gen_free(h)
    nested = bool(nested)
    return Problem(name=name, xy=xy, cell_ptr=cptr, cell_vtx=cvtx, part=part, n_sub=nsub, n_coarse=ncoarse,
                   nested=nested, parent=parent if nested else None,
                   ov_fine=None if nested else ovf, ov_coarse=None if nested else ovc,
                   ov_ptr=None if nested else ovp, ov_xy=None if nested else ovxy,
                   cpoly_ptr=None if nested else cpp, cpoly_xy=None if nested else cpxy,
                   kappa=kappa, **kw)


def normal(seed: int, n: int) -> np.ndarray:
    """Counter-based N(0,1) vector (same bits on every machine)."""
    out = np.zeros(n)
    _load().dgas_gen_normal(seed, n, out.ctypes.data)
    return out


# ---------------------------------------------------------------- BASELINE.json configs (B:7-11)
CONFIG5_PQ = [(1, 1)] + [pq for p in range(2, 7) for pq in ((p, 1), (p, p))]


def config(k: int, p: int | None = None, q: int | None = None, scale: str = "full") -> Problem:
    """BASELINE.json configs[k-1]. `scale="small"` gives a structurally identical reduced instance
    (same generator modes, p, q, rho and f; fewer cells) that the oracle can solve end to end."""
    small = scale == "small"
    if k == 1:
        return generate(0, 16, sub_mode=0, sub_tile=8, coarse_mode=0, name="cfg1", p=1, q=1, f_kind=F_SINSIN)
    if k == 2:
        return generate(1, 1024 if not small else 256, seed=2, lloyd=5, sub_mode=1, n_sub=16 if not small else 4,
                        coarse_mode=1, n_coarse=64 if not small else 16, name="cfg2" + ("s" if small else ""),
                        p=2, q=1, f_kind=F_SINSIN)
    if k == 3:
        n = 512 if not small else 32
        return generate(0, n, sub_mode=0, sub_tile=8, coarse_mode=2, coarse_tile=4, name="cfg3" + ("s" if small else ""),
                        p=3, q=1, f_kind=F_SINSIN)
    if k == 4:
        nc = 65536 if not small else 1024
        ns = 1024 if not small else 16
        return generate(1, nc, seed=4, lloyd=5, sub_mode=1, n_sub=ns, coarse_mode=3, n_coarse=ns, kappa_mode=1,
                        name="cfg4" + ("s" if small else ""), p=4, q=2, f_kind=F_ONE)
    if k == 5:
        p = 1 if p is None else p
        q = p if q is None else q
        nc = 16384 if not small else 1024
        ns = 256 if not small else 16
        return generate(1, nc, seed=5, lloyd=5, sub_mode=1, n_sub=ns, coarse_mode=0,
                        name=f"cfg5{'s' if small else ''}_p{p}q{q}", p=p, q=q, f_kind=F_SINSIN)
    raise ValueError(k)


# ---------------------------------------------------------------- paper regime
PAPER_EX2 = {  # Table tab:ASPCG_P1_poly / _P3_poly: K (iters), rows H, cols N_h
    1: {16: {64: (20.70, 45), 256: (72.31, 86), 1024: (269.70, 163), 4096: (818.09, 289)},
        8: {256: (21.89, 46), 1024: (73.42, 86), 4096: (261.36, 163)},
        4: {1024: (20.91, 46), 4096: (83.77, 91)},
        2: {4096: (23.08, 48)}},
    3: {16: {64: (88.63, 80), 256: (291.77, 145), 1024: (1137.55, 276), 4096: (3241.64, 513)},
        8: {256: (102.96, 82), 1024: (278.15, 140), 4096: (949.21, 271)},
        4: {1024: (90.30, 79), 4096: (343.19, 148)},
        2: {4096: (104.24, 82)}},
}
PAPER_EX4 = {  # Table tab:ASPCG_Cond_Nest0_hHfine_HHcoarse_P1 / _P3: rows N_H, cols N_h
    1: {16: {64: (23.29, 38), 256: (92.13, 77), 1024: (387.61, 159), 4096: (1624.26, 324), 16384: (6370.86, 657)},
        64: {256: (25.91, 39), 1024: (106.42, 84), 4096: (411.02, 167), 16384: (1774.19, 342)},
        256: {1024: (26.73, 41), 4096: (100.89, 82), 16384: (425.97, 169)},
        1024: {4096: (31.81, 44), 16384: (118.61, 86)},
        4096: {16384: (30.56, 43)}},
    3: {16: {64: (148.36, 83), 256: (429.84, 143), 1024: (1602.53, 275), 4096: (5405.40, 529), 16384: (21263.66, 1058)},
        64: {256: (142.42, 76), 1024: (405.44, 135), 4096: (1525.94, 263), 16384: (5170.13, 498)},
        256: {1024: (157.47, 80), 4096: (452.41, 137), 16384: (1469.08, 249)},
        1024: {4096: (147.97, 77), 16384: (402.98, 124)},
        4096: {16384: (135.77, 70)}},
}


def paper_case(example: int, n_fine: int, coarse: int, p: int, seed: int = 17) -> Problem:
    """The paper's experimental regime: T_HH = T_h (every cell its own subdomain),
    Voronoi fine mesh of n_fine cells on (0,1)^2, rho = 1, q = p, C_sigma = 10.
    example 2: nested agglomerates with H = coarse * h_bar (h_bar = h of the 4096-cell mesh, so the
               coarse mesh has 4096 / coarse^2 RCB agglomerates);
    example 4: an independently generated Voronoi coarse mesh of `coarse` cells.
    The paper never states f; BASELINE's f = 2 pi^2 sin sin is used (R21)."""
    if example == 2:
        n_coarse = max(1, 4096 // (coarse * coarse))
        return generate(1, n_fine, seed=seed, lloyd=5, sub_mode=1, n_sub=n_fine, coarse_mode=1, n_coarse=n_coarse,
                        name=f"ex2_h{n_fine}_H{coarse}_p{p}", p=p, q=p, f_kind=F_SINSIN)
    if example == 4:
        return generate(1, n_fine, seed=seed, lloyd=5, sub_mode=1, n_sub=n_fine, coarse_mode=4, n_coarse=coarse,
                        name=f"ex4_h{n_fine}_H{coarse}_p{p}", p=p, q=p, f_kind=F_SINSIN)
    raise ValueError(example)


PAPER_EX1 = {  # Tables tab:RhoAlignedAndNotAligned / ...NonCOnvex: K vs rho_e = 10..1e6
    "convex": {("aligned", 1): [231, 233, 234, 234, 234, 234], ("aligned", 2): [612, 614, 614, 612, 611, 610],
               ("not_aligned", 1): [292, 1.04e3, 7.73e3, 7.42e4, 7.39e5, 7.38e6],
               ("not_aligned", 2): [654, 2.26e3, 1.71e4, 1.65e5, 1.64e6, 1.64e7]},
    "nonconvex": {("aligned", 1): [965, 1.15e3, 1.20e3, 1.21e3, 1.21e3, 1.21e3],
                  ("aligned", 2): [2.47e3, 2.86e3, 3.18e3, 3.25e3, 3.26e3, 3.26e3],
                  ("not_aligned", 1): [802, 2.09e3, 1.68e4, 1.65e5, 1.64e6, 1.64e7],
                  ("not_aligned", 2): [2.36e3, 6.10e3, 4.74e4, 4.62e5, 4.61e6, 4.61e7]},
}


def paper_case_ex1(variant: str, aligned: bool, rho_e: float, p: int, levels: int = 3, n_fine: int = 2000,
                   n_coarse: int = 16, seed: int = 11) -> Problem:
    """Ex.1: L-shaped domain, T_HH = T_h, q = p, rho_o = 1 and rho_e on even-indexed
    elements. variant "convex": a Voronoi coarse mesh of 16 convex cells on the L, fine mesh by `levels`
    centroid-midpoint refinements (nested); variant "nonconvex": a Voronoi fine mesh of n_fine cells on the
    L with RCB agglomerates (METIS is out of scope; R33). aligned: rho_e on coarse elements D_j
    with even 1-based index j; not aligned: rho_e on fine elements with even 1-based index."""
    if variant == "convex":
        # the cell around the re-entrant corner splits into two convex cells (gen.cpp clip_L), so fewer
        # seeds may be needed for exactly n_coarse coarse cells
        for ns in (n_coarse, n_coarse - 1, n_coarse - 2):
            P = generate(2, levels, seed=seed, lloyd=5, sub_mode=2, coarse_mode=5, n_coarse=ns,
                         name=f"ex1c_l{levels}_{'al' if aligned else 'na'}_p{p}", p=p, q=p, f_kind=F_SINSIN)
            if P.n_coarse == n_coarse:
                break
    elif variant == "nonconvex":
        P = generate(3, n_fine, seed=seed, lloyd=5, sub_mode=2, coarse_mode=1, n_coarse=n_coarse,
                     name=f"ex1n_{n_fine}_{'al' if aligned else 'na'}_p{p}", p=p, q=p, f_kind=F_SINSIN)
    else:
        raise ValueError(variant)
    idx = P.parent if aligned else np.arange(P.n_cells)
    P.kappa = np.where(idx % 2 == 1, float(rho_e), 1.0)
    P.meta.update(rho_e=rho_e, aligned=aligned, variant=variant)
    return P
