"""Oracle pins P3-P6 for the SIPDG assembly (PAPER.md eq:Ah P:83-98, face form P:467-469).

P3/P3b are hand-derived worked examples (closed forms in tests/golden/sipg_worked_examples.txt);
P4 symmetry/SPD (Lemma 5.1); P5 exact reproduction of a polynomial solution in V_h;
P6 DG-norm / L2 convergence rates (eq:DGnorm_2 P:240-241, Lemma 5.3)."""
import copy
import os

import numpy as np
import pytest

import dgas_gen as g
import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "sipg_worked_examples.txt")


def _golden():
    vals = {}
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if not line:
            continue
        k, v = line.split("=", 1)
        vals[k.strip()] = eval(v, {"sqrt": np.sqrt})  # closed-form expressions
    return vals


def _square(n=1):
    return g.generate(0, n, sub_mode=0, sub_tile=n, coarse_mode=0, p=1, q=1)


def test_P3_single_cell_closed_form():
    G = _golden()
    for s_n in (1, 4):
        P = _square(1)
        P.xy = P.xy / s_n  # side s = 1/s_n
        o = O.Oracle(P)
        B, _ = o.block(0, 0)
        s = 1.0 / s_n
        ref = np.diag(G["P3_diag"]) / s ** 2
        assert np.abs(B - ref).max() <= 1e-13 * np.abs(ref).max()
        # ||1||_DG^2 = sigma * perimeter (constant has no volume term; boundary jump = 1)
        c = np.array([s, 0, 0])  # coefficient of v = 1 in the orthonormal basis {1/s, ...}
        assert abs(c @ B @ c - G["P3_sigma_perimeter"]) < 1e-12


def test_P3b_interior_face_block():
    G = _golden()
    P = _square(1)
    P2 = copy.copy(P)
    P2.xy = np.array([[0, 0], [1, 0], [2, 0], [0, 1], [1, 1], [2, 1]], float)
    P2.cell_ptr = np.array([0, 4, 8], np.int32)
    P2.cell_vtx = np.array([0, 1, 4, 3, 1, 2, 5, 4], np.int32)
    P2.part = np.zeros(2, np.int32); P2.kappa = np.ones(2); P2.parent = np.zeros(2, np.int32)
    o = O.Oracle(P2)
    Bpm, ok = o.block(0, 1)
    Bmp, _ = o.block(1, 0)
    assert ok
    ref = np.array(G["P3b_Bpm"])
    assert np.abs(Bpm - ref).max() < 1e-13
    assert np.abs(Bmp - ref.T).max() < 1e-13
    # kappa+ diagonal block = boundary part (3 faces) + shared-face part
    Bpp, _ = o.block(0, 0)
    face_pp = np.array(G["P3b_face_pp"])
    # volume + 3 boundary faces of the unit square (x=0, y=0, y=1), computed independently below
    vol = np.diag([0, 12, 12.0])
    sig = 10 / np.sqrt(2)
    # boundary x=0 (n=(-1,0)), y=0 (n=(0,-1)), y=1 (n=(0,1)) with phi = {1, sqrt3(2x-1), sqrt3(2y-1)}
    xs, ws = np.polynomial.legendre.leggauss(4)
    t = 0.5 * (xs + 1); w = 0.5 * ws
    bnd = np.zeros((3, 3))
    r3 = np.sqrt(3)
    for (X, Y, n) in [(0 * t, t, (-1, 0)), (t, 0 * t, (0, -1)), (t, 0 * t + 1, (0, 1))]:
        phi = np.stack([np.ones_like(t), r3 * (2 * X - 1), r3 * (2 * Y - 1)])
        dn = np.array([0, 2 * r3 * n[0], 2 * r3 * n[1]])[:, None] * np.ones_like(t)
        bnd += (sig * phi[:, None] * phi[None] - dn[None] * phi[:, None] - dn[:, None] * phi[None]) @ w
    assert np.abs(Bpp - (vol + bnd + face_pp)).max() < 1e-12


def test_P3c_harmonic_h_and_rho_unequal_cells():
    """Unit square next to a 2x1 rectangle: the off-diagonal block pins <h> and <rho> as HARMONIC
    averages over the face (eq:Sigma P:94-98; R1), which the equal-square P3b cannot."""
    G = _golden()
    P = _square(1)
    P2 = copy.copy(P)
    P2.xy = np.array([[0, 0], [1, 0], [3, 0], [0, 1], [1, 1], [3, 1]], float)
    P2.cell_ptr = np.array([0, 4, 8], np.int32)
    P2.cell_vtx = np.array([0, 1, 4, 3, 1, 2, 5, 4], np.int32)
    P2.part = np.zeros(2, np.int32); P2.parent = np.zeros(2, np.int32)
    for rho, key in (([1.0, 1.0], "P3c_rho1_Bpm"), ([1.0, 3.0], "P3c_rho13_Bpm")):
        P2.kappa = np.array(rho)
        o = O.Oracle(P2)
        Bpm, ok = o.block(0, 1)
        Bmp, _ = o.block(1, 0)
        ref = np.array(G[key])
        assert ok
        assert np.abs(Bpm - ref).max() < 1e-13, (key, Bpm, ref)
        assert np.abs(Bmp - ref.T).max() < 1e-13


@pytest.mark.parametrize("cfg", [1, 2])
def test_P4_symmetric_spd(cfg):
    P = g.config(cfg, scale="small")
    o = O.Oracle(P)
    A = o.dense_A()
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max() * 10
    ev = np.linalg.eigvalsh(0.5 * (A + A.T))
    assert ev[0] > 0


def test_P4_spd_jumps():
    # rho = 10^U(-4,4) per subdomain (config-4 style): still SPD
    P = g.generate(1, 256, seed=4, lloyd=5, sub_mode=1, n_sub=16, coarse_mode=0, kappa_mode=1, p=2, q=1)
    assert P.kappa.max() / P.kappa.min() > 1e3
    o = O.Oracle(P)
    A = o.dense_A()
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    assert np.linalg.eigvalsh(0.5 * (A + A.T))[0] > 0


@pytest.mark.parametrize("p", [4, 5])
def test_P5_polynomial_reproduction(p):
    # u = x(1-x)y(1-y) is in V_h (p>=4) and in H^1_0 with no jumps: the SIPG solution equals u
    # for any admissible sigma (consistency of eq:Ah). f = 2[x(1-x)+y(1-y)].
    P = g.generate(1, 40, seed=9, lloyd=3, sub_mode=1, n_sub=4, coarse_mode=0, p=p, q=1, f_kind=g.F_POLY)
    o = O.Oracle(P)
    o.setup_schwarz()
    b = o.rhs()
    res = o.pcg(b, rtol=1e-13)
    u = o.project(1)
    assert res["status"] == 0
    assert np.linalg.norm(res["x"] - u) <= 1e-9 * np.linalg.norm(u)


def _rates(meshes, p):
    errs, hs = [], []
    for P in meshes:
        o = O.Oracle(P, p=p)
        o.setup_schwarz(use_coarse=False)
        res = o.pcg(o.rhs(g.F_SINSIN), rtol=1e-13)
        errs.append(o.errors(res["x"]))
        hs.append(1.0 / np.sqrt(P.n_cells))
    errs = np.array(errs)
    h = np.array(hs)
    sl2 = np.polyfit(np.log(h), np.log(errs[:, 0]), 1)[0]
    sdg = np.polyfit(np.log(h), np.log(errs[:, 1]), 1)[0]
    return sl2, sdg


@pytest.mark.parametrize("p", [1, 2, 3])
def test_P6_convergence_cartesian(p):
    meshes = [g.generate(0, n, sub_mode=0, sub_tile=4, coarse_mode=0, p=p, q=1) for n in (8, 16, 32)]
    sl2, sdg = _rates(meshes, p)
    assert abs(sdg - p) < 0.25, sdg
    assert abs(sl2 - (p + 1)) < 0.3, sl2


@pytest.mark.parametrize("p", [1, 2])
def test_P6_convergence_voronoi(p):
    meshes = [g.generate(1, n, seed=21, lloyd=5, sub_mode=1, n_sub=n // 16, coarse_mode=0, p=p, q=1) for n in (64, 256, 1024)]
    sl2, sdg = _rates(meshes, p)
    assert abs(sdg - p) < 0.3, sdg
    assert abs(sl2 - (p + 1)) < 0.35, sl2


def test_rhs_constant_f_p0_like():
    # f = 1: b_0 for each cell = int phi_0 = |kappa| / sqrt(|kappa|) = sqrt(|kappa|) (phi_0 = 1/sqrt|kappa|)
    P = g.generate(1, 32, seed=1, lloyd=2, sub_mode=1, n_sub=2, coarse_mode=0, p=2, q=1)
    o = O.Oracle(P)
    b = o.rhs(g.F_ONE).reshape(P.n_cells, -1)
    for c in range(P.n_cells):
        poly = P.xy[P.cell_vtx[P.cell_ptr[c]:P.cell_ptr[c + 1]]]
        area = 0.5 * np.sum(poly[:, 0] * np.roll(poly[:, 1], -1) - np.roll(poly[:, 0], -1) * poly[:, 1])
        assert abs(abs(b[c, 0]) - np.sqrt(area)) < 1e-13
        assert np.abs(b[c, 1:]).max() < 1e-13
