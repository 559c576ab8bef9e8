"""Oracle pins P7-P10: prolongation R0^T (eq:R0T P:144-147, Remark 3.2 P:153-159), the additive
Schwarz operator (Lemma 5.8, Assumptions P:522-546, Thm TosWil),
PCG / Lanczos and the condition-number scaling laws (Remark 6.6 P:700-710)."""
import copy
import math

import numpy as np
import pytest

import dgas_gen as g
import oracle as O


def test_P7b_nested_Q_closed_form():
    # config 1: 8x8 coarse tiles of squares, q = 1, any p: Q block of fine cell at tile position (i,j):
    # [[1/m, sqrt3(2i+1-m)/m^2, sqrt3(2j+1-m)/m^2], [0, 1/m^2, 0], [0, 0, 1/m^2]]; rows >= 3 zero.
    for p in (1, 2):
        P = g.config(1)
        o = O.Oracle(P, p=p)
        o.setup_schwarz(q=None) if False else o.setup_schwarz()
        G = o.G()
        m = 8
        n = 16
        for cell in [0, 9, 63, 100, 255]:
            ci, cj = cell % n, cell // n
            i, j = ci % m, cj % m
            ref = np.zeros((o.np_, 3))
            ref[0] = [1 / m, math.sqrt(3) * (2 * i + 1 - m) / m ** 2, math.sqrt(3) * (2 * j + 1 - m) / m ** 2]
            ref[1, 1] = 1 / m ** 2
            ref[2, 2] = 1 / m ** 2
            assert np.abs(G[cell] - ref).max() < 1e-14, cell


def _Q_dense(o):
    f, c, _, _ = o._ov
    Q = np.zeros((o.N, o.N0))
    G = o.G()
    for k in range(o.n_ov):
        Q[f[k] * o.np_:(f[k] + 1) * o.np_, c[k] * o.nq_:(c[k] + 1) * o.nq_] += G[k]
    return Q


def _coarse_const(o):
    """coarse coefficients of the constant 1: (psi_b, 1)_{D_J} with psi orthonormal on D_J."""
    c1 = np.zeros(o.N0)
    f, c, ptr, xy = o._ov
    # (1, psi_J,b) = sum over pieces of int psi; psi_0 = 1/sqrt|D_J| and others orthogonal to 1
    areas = np.zeros(o.n_coarse)
    for k in range(o.n_ov):
        poly = xy[ptr[k]:ptr[k + 1]]
        areas[c[k]] += 0.5 * np.sum(poly[:, 0] * np.roll(poly[:, 1], -1) - np.roll(poly[:, 0], -1) * poly[:, 1])
    c1[0::o.nq_] = np.sqrt(areas)
    return c1, areas


@pytest.mark.parametrize("cfg", [2, 4])
def test_P7_constant_reproduction(cfg):
    # Q maps the coarse representation of 1 to the fine representation of 1 (nested and non-nested)
    P = g.config(cfg, scale="small")
    o = O.Oracle(P)
    o.setup_schwarz()
    Q = _Q_dense(o)
    c1, areas = _coarse_const(o)
    assert abs(areas.sum() - 1.0) < 1e-12
    one_h = o.project(1) * 0  # fine coefficients of 1: sqrt|kappa| in mode 0
    for c in range(P.n_cells):
        poly = P.xy[P.cell_vtx[P.cell_ptr[c]:P.cell_ptr[c + 1]]]
        one_h[c * o.np_] = np.sqrt(0.5 * np.sum(poly[:, 0] * np.roll(poly[:, 1], -1) - np.roll(poly[:, 0], -1) * poly[:, 1]))
    tol = 1e-12 if P.nested else 1e-10
    assert np.abs(Q @ c1 - one_h).max() < tol


def test_P7_nested_injection_and_split_pieces():
    # Remark 3.2: nested => R0^T = natural injection: Q c equals the exact re-expansion of the coarse
    # polynomial on each fine cell (pointwise). Also: splitting every fine cell into two pieces of the
    # same coarse element (a "non-nested" description of a nested pair) gives the same Q.
    P = g.config(2, scale="small")
    o = O.Oracle(P)
    o.setup_schwarz()
    Q = _Q_dense(o)
    rng = np.random.default_rng(3)
    cvec = rng.normal(size=o.N0)
    fine = Q @ cvec
    # evaluate both at random points inside some fine cells
    f, cc, ptr, xy = o._ov
    for cell in [0, 17, 100, 255]:
        poly = P.xy[P.cell_vtx[P.cell_ptr[cell]:P.cell_ptr[cell + 1]]]
        pts = poly.mean(0) + 0.2 * (poly[:2] - poly.mean(0))
        phi, _, _ = o.eval_basis(cell, pts)
        uh = phi @ fine[cell * o.np_:(cell + 1) * o.np_]
        J = P.parent[cell]
        Cc, bb = o.coarse_basis(J)
        xi = 2 * (pts[:, 0] - bb[0]) / (bb[1] - bb[0]) - 1
        eta = 2 * (pts[:, 1] - bb[2]) / (bb[3] - bb[2]) - 1
        L = np.polynomial.legendre.Legendre.basis
        graw = np.stack([L(1)(xi) * 0 + 1, L(1)(xi), L(1)(eta)], 1)  # q = 1 graded order
        uH = (graw @ Cc.T) @ cvec[J * o.nq_:(J + 1) * o.nq_]
        assert np.abs(uh - uH).max() < 1e-12
    # split pieces
    nf, ncf, nptr, nxy = [], [], [0], []
    for cell in range(P.n_cells):
        poly = P.xy[P.cell_vtx[P.cell_ptr[cell]:P.cell_ptr[cell + 1]]]
        k = len(poly)
        a = poly[:k // 2 + 1]
        b = np.concatenate([poly[k // 2:], poly[:1]])
        for piece in (a, b):
            nf.append(cell); ncf.append(P.parent[cell]); nxy.extend(piece.tolist()); nptr.append(len(nxy))
    o2 = O.Oracle(P)
    o2.setup_schwarz(coarse=(P.n_coarse, np.array(nf), np.array(ncf), np.array(nptr), np.array(nxy)))
    Q2 = _Q_dense(o2)
    assert np.abs(Q2 - Q).max() < 1e-12


def test_P8_schwarz_properties_cfg1():
    P = g.config(1)
    o = O.Oracle(P)
    o.setup_schwarz()
    A = o.dense_A()
    M = o.dense_precond()
    # (i) symmetry, (ii) SPD
    assert np.abs(M - M.T).max() <= 1e-12 * np.abs(M).max()
    assert np.linalg.eigvalsh(0.5 * (M + M.T))[0] > 0
    # (vi) trace identity: tr(P^-1 A) = N + N0 (each exact subspace solve is a projection of rank dim V_i)
    assert abs(np.trace(M @ A) - (o.N + o.N0)) < 1e-8 * o.N
    # (vii) 1 <= lambda_max(P^-1 A) <= 1 + rho(I + Adj_face); config 1's face graph is a 4-cycle => <= 4
    ev = np.sort(np.linalg.eigvals(M @ A).real)
    assert ev[-1] >= 1 - 1e-10 and ev[-1] <= 4 + 1e-10
    # projections: P_i E_i v = E_i v  (local parts are A-orthogonal projections)
    Pad = M @ A
    rng = np.random.default_rng(0)
    v = rng.normal(size=o.N)
    # apply of A v restricted to... linearity
    z1 = o.apply(v); z2 = o.apply(2 * v)
    assert np.abs(z2 - 2 * z1).max() < 1e-12 * np.abs(z1).max()
    # Lanczos K (rtol 1e-14) <= dense K and within 5%
    b = o.rhs()
    res = o.pcg(b, rtol=1e-14, maxit=2000)
    Kd = ev[-1] / ev[0]
    assert res["cond"] <= Kd * (1 + 1e-8)
    assert res["cond"] >= 0.95 * Kd


def test_P8_exactness_limits():
    P = g.config(1)
    # single subdomain, no coarse: P^-1 = A^-1 -> 1 iteration, K = 1
    o = O.Oracle(P, part=np.zeros(P.n_cells, np.int32), n_sub=1)
    o.setup_schwarz(use_coarse=False)
    res = o.pcg(o.rhs(), rtol=1e-8)
    assert res["iters"] == 1 and abs(res["cond"] - 1) < 1e-8
    # coarse space = fine space (T_H = T_h, q = p), coarse only -> A^-1
    P2 = copy.copy(P)
    P2.parent = np.arange(P.n_cells, dtype=np.int32)
    P2.n_coarse = P.n_cells
    o2 = O.Oracle(P2)
    o2.setup_schwarz(use_local=False)
    res2 = o2.pcg(o2.rhs(), rtol=1e-8)
    assert res2["iters"] == 1


def test_P8_decomposition_identity():
    # Lemma 5.8: unique non-overlapping decomposition => sum_i E_i E_i^T = I: with A_i = A restricted
    # and the coarse part off, P^-1 A v = v for block-diagonal A (one subdomain per cell-block)
    P = g.config(2, scale="small")
    o = O.Oracle(P)
    o.setup_schwarz(use_coarse=False)
    rng = np.random.default_rng(2)
    r = rng.normal(size=o.N)
    z = o.apply(r)
    # on each subdomain, A_i z_i = r_i exactly
    A = o.dense_A()
    for s in range(P.n_sub):
        idx = np.concatenate([np.arange(c * o.np_, (c + 1) * o.np_) for c in np.where(P.part == s)[0]])
        assert np.abs(A[np.ix_(idx, idx)] @ z[idx] - r[idx]).max() < 1e-9 * np.abs(r).max()


def test_P9_lanczos_diag14():
    # diag(1,4), b=(1,1), M=I: alpha0 = 0.4, beta0 = 0.36, alpha1 = 0.625 (hand-checked) -> Ritz {1,4}
    lmin, lmax, K = O.lanczos([0.4, 0.625], [0.36])
    assert abs(lmin - 1) < 1e-13 and abs(lmax - 4) < 1e-13 and abs(K - 4) < 1e-12


def test_P9_pcg_matches_dense_solve():
    P = g.config(1)
    o = O.Oracle(P)
    o.setup_schwarz()
    b = o.rhs()
    res = o.pcg(b, rtol=1e-12)
    x = np.linalg.solve(o.dense_A(), b)
    assert np.linalg.norm(res["x"] - x) <= 1e-9 * np.linalg.norm(x)
    # residual history decreases to below rtol, checked on the Euclidean norm
    assert res["resid"][-1] <= 1e-12


def test_R30_long_double_sensitivity_small_cfg4():
    # fp64 apply vs long-double apply (R30) on the config-4-style problem with rho jumps
    P = g.config(4, scale="small")
    o = O.Oracle(P)
    o.setup_schwarz(long_double=True)
    r = g.normal(11, o.N)
    z = o.apply(r); zl = o.apply(r, long_double=True)
    assert np.linalg.norm(z - zl) <= 1e-11 * np.linalg.norm(zl)


def _K(P, **kw):
    o = O.Oracle(P, part=np.arange(P.n_cells, dtype=np.int32), n_sub=P.n_cells)  # paper regime T_HH = T_h
    o.setup_schwarz(**kw)
    res = o.pcg(o.rhs(), rtol=1e-12, maxit=3000)
    return res["cond"]


def test_P10_scaling_fixed_H_refine_h():
    # nested Cartesian, p = q = 1, T_HH = T_h, fixed coarse 2x2 (H = 1/2): K = O(H^2/h^2)
    Ks, r = [], []
    for n in (8, 16, 32):
        P = g.generate(0, n, sub_mode=0, sub_tile=1, coarse_mode=2, coarse_tile=n // 2, p=1, q=1)
        Ks.append(_K(P)); r.append(n / 2)
    slope = np.polyfit(np.log(r), np.log(Ks), 1)[0]
    assert 1.4 <= slope <= 2.2, (Ks, slope)


def test_P10_scaling_fixed_ratio():
    # fixed H/h = 4: K approximately constant (diagonals of Table ASPCG_P1_poly), < 1.6x variation
    Ks = []
    for n in (8, 16, 32):
        P = g.generate(0, n, sub_mode=0, sub_tile=1, coarse_mode=2, coarse_tile=4, p=1, q=1)
        Ks.append(_K(P))
    assert max(Ks) / min(Ks) < 1.6, Ks


def test_P10_p_scaling_nested():
    # nested, q = p: K = O(p) for fixed meshes (Remark 6.6 p^2/q term, Ex.5 P:1040): slope in [0.6, 1.4]
    Ks, ps = [], []
    for p in (1, 2, 3, 4):
        P = g.generate(0, 8, sub_mode=0, sub_tile=1, coarse_mode=2, coarse_tile=2, p=p, q=p)
        Ks.append(_K(P)); ps.append(p)
    slope = np.polyfit(np.log(ps), np.log(Ks), 1)[0]
    assert 0.6 <= slope <= 1.4, (Ks, slope)


# ---------------------------------------------------------------- paper regime
def _paper_run(ex, nf, coarse, p):
    P = g.paper_case(ex, nf, coarse, p)
    o = O.Oracle(P)
    o.setup_schwarz()
    return o.pcg(o.rhs(), rtol=1e-8)  # rtol 1e-8, x0 = 0


@pytest.mark.parametrize("ex", [2, 4])
def test_paper_tables_p1_magnitude_and_trend(ex):
    """Tables tab:ASPCG_P1_poly and tab:ASPCG_Cond_Nest0_hHfine_HHcoarse_P1
    (PAPER.md:998-1002). Our seeded Voronoi meshes are not the paper's, so the printed values pin
    magnitude (K within [0.3, 1.5]x, iterations within [0.6, 1.2]x) and the stated trends: K grows like
    (H/h)^2 along a row (fitted slope in [1.4, 2.3]) and stays nearly constant along the diagonal H/h = 2."""
    tab = (g.PAPER_EX2 if ex == 2 else g.PAPER_EX4)[1]
    first = next(iter(tab))                  # coarsest coarse mesh: H = 16 h_bar / N_H = 16
    row, diag = [], []
    for coarse, cols in tab.items():
        for nf, (k_ref, it_ref) in cols.items():
            if nf > 1024:
                continue
            r = _paper_run(ex, nf, coarse, 1)
            assert 0.3 * k_ref <= r["cond"] <= 1.5 * k_ref, (coarse, nf, r["cond"], k_ref)
            assert 0.6 * it_ref <= r["iters"] <= 1.2 * it_ref, (coarse, nf, r["iters"], it_ref)
            if coarse == first:
                row.append((nf, r["cond"]))
            if nf == min(cols):
                diag.append(r["cond"])
    hh = np.sqrt([nf for nf, _ in row])      # H/h ~ sqrt(N_h) at fixed H
    slope = np.polyfit(np.log(hh), np.log([k for _, k in row]), 1)[0]
    assert 1.4 <= slope <= 2.3, (row, slope)
    assert max(diag) / min(diag) < 2.0, diag


def test_paper_table_p3_corner():
    """tab:ASPCG_P3_poly H = 16 h_bar, h = 8 h_bar: 88.63 (80)."""
    r = _paper_run(2, 64, 16, 3)
    assert 0.3 * 88.63 <= r["cond"] <= 1.5 * 88.63 and 0.6 * 80 <= r["iters"] <= 1.2 * 80


def _ex1(variant, aligned, rho_e, p, levels=3):
    P = g.paper_case_ex1(variant, aligned, rho_e, p, levels=levels)
    o = O.Oracle(P)
    o.setup_schwarz()
    return o.pcg(o.rhs(), rtol=1e-8, maxit=20000)


def test_paper_ex1_rho_dichotomy():
    """Table tab:RhoAlignedAndNotAligned and Remark 6.6: aligned with T_H, K does not
    depend on rho_e; not aligned, K grows linearly in rho_e. Values pin magnitude (p = 1, level-3
    refinement of a 16-cell convex Voronoi coarse mesh): within [0.5, 2]x of the printed K."""
    ref = g.PAPER_EX1["convex"]
    al = [_ex1("convex", True, r, 1)["cond"] for r in (10.0, 1e3, 1e6)]
    na = [_ex1("convex", False, r, 1)["cond"] for r in (10.0, 1e3, 1e6)]
    assert max(al) / min(al) < 1.15, al
    assert 500 <= na[2] / na[1] <= 2000, na
    for k, r in zip(al, (ref[("aligned", 1)][0], ref[("aligned", 1)][2], ref[("aligned", 1)][5])):
        assert 0.5 * r <= k <= 2 * r, (al, r)
    for k, r in zip(na, (ref[("not_aligned", 1)][0], ref[("not_aligned", 1)][2], ref[("not_aligned", 1)][5])):
        assert 0.5 * r <= k <= 2 * r, (na, r)


def test_paper_ex1_rho_one_identical():
    """rho_e = 1: the aligned and not-aligned problems are the same matrix (SPEC-style trivial case)."""
    a = _ex1("convex", True, 1.0, 1, levels=1)
    b = _ex1("convex", False, 1.0, 1, levels=1)
    assert a["iters"] == b["iters"] and np.array_equal(a["x"], b["x"])


@pytest.mark.parametrize("cfg", [2, 3])
def test_band_coarse_path_matches_dense(cfg):
    """The band-Cholesky coarse factor/solve (used by the oracle when N0 > dense_max, i.e. full-size
    config 3) against the dense Cholesky path (pinned by P8/P9 above): z = Q A0^-1 Q^T r + local
    solves, eq. P:160-165, must agree to rounding. Iterative refinement (R30) can only
    move the band solve closer to the dense one."""
    P = g.config(cfg, scale="small")
    od = O.Oracle(P)
    od.setup_schwarz()
    ob = O.Oracle(P)
    ob.setup_schwarz(dense_max=0)
    # the band path really ran: A0 is not stored densely
    with pytest.raises(O.OracleError):
        ob.A0()
    A0 = od.A0()
    kap = np.linalg.cond(A0)
    for seed in range(3):
        r = g.normal(70 + seed, od.N)
        zd = od.apply(r)
        zb = ob.apply(r)
        assert np.linalg.norm(zb - zd) <= max(1e-12, 10 * kap * 2.2e-16) * np.linalg.norm(zd), (seed, kap)
    # coarse part alone against numpy's dense solve of the same A0
    oc = O.Oracle(P)
    oc.setup_schwarz(dense_max=0, use_local=False)
    r = g.normal(80, od.N)
    Q = _Q_dense(od)
    zc_ref = Q @ np.linalg.solve(A0, Q.T @ r)
    zc = oc.apply(r)
    assert np.linalg.norm(zc - zc_ref) <= 10 * kap * 2.2e-16 * np.linalg.norm(zc_ref)
    oc.set_refine(1)
    zc1 = oc.apply(r)
    assert np.linalg.norm(zc1 - zc_ref) <= 2 * np.linalg.norm(zc - zc_ref) + 1e-14 * np.linalg.norm(zc_ref)


@pytest.mark.parametrize("cfg", [2, 4])
def test_apply_sampled_is_full_apply_restricted(cfg):
    """or_apply_sampled (full-size sampled parity) is the full apply P^-1 r restricted to the
    cells of the sampled subdomains, and zero elsewhere: equal to the full apply there, bit for bit
    (same coarse solve, same local solves), whether or not the other subdomains were factored."""
    P = g.config(cfg, scale="small")
    sample = [0, P.n_sub // 2, P.n_sub - 1]
    of = O.Oracle(P)
    of.setup_schwarz()
    os_ = O.Oracle(P)
    os_.setup_schwarz(sample=sample)
    r = g.normal(90, of.N)
    z = of.apply(r)
    zs = os_.apply_sampled(r, sample)
    zs2 = of.apply_sampled(r, sample)
    mask = np.repeat(np.isin(P.part, sample), of.np_)
    assert mask.any() and (~mask).any()
    assert np.array_equal(zs[mask], z[mask])
    assert np.array_equal(zs2[mask], z[mask])
    assert not zs[~mask].any() and not zs2[~mask].any()
    # the unsampled setup really lacks the other factors
    with pytest.raises(O.OracleError):
        os_.apply(r)


def test_long_double_sampled_apply_and_band():
    """The long-double sampled apply (the exact reference of the full-size GPU apply check, Z30 / R30) is
    the long-double full apply restricted to the sample; with the band coarse path (no long-double band
    factor: fp64 band solve refined with long-double residuals) it agrees with the dense long-double
    apply to ~1e-15 once refined."""
    P = g.config(3, scale="small")
    sample = [0, P.n_sub - 1]
    od = O.Oracle(P)
    od.setup_schwarz(long_double=True)
    r = g.normal(95, od.N)
    zl = od.apply(r, long_double=True)
    mask = np.repeat(np.isin(P.part, sample), od.np_)
    assert np.array_equal(od.apply_sampled(r, sample, long_double=True)[mask], zl[mask])
    ob = O.Oracle(P)
    ob.setup_schwarz(long_double=True, dense_max=0, sample=sample)
    ob.set_refine(2)
    zb = ob.apply_sampled(r, sample, long_double=True)
    assert np.linalg.norm(zb[mask] - zl[mask]) <= 1e-14 * np.linalg.norm(zl[mask])


def test_perturb_A_probe_is_symmetric_and_bounded():
    """The A-perturbation sensitivity probe (R22/R30) keeps A symmetric and moves every entry by at
    most eps relative (and really moves them)."""
    P = g.config(1)
    o = O.Oracle(P)
    A = o.dense_A()
    o2 = O.Oracle(P)
    o2.perturb_A(1e-6, 3)
    A2 = o2.dense_A()
    # same factor on (i,j) and (j,i): the asymmetry of assembly rounding is only scaled, never added to
    assert np.abs(A2 - A2.T).max() <= np.abs(A - A.T).max() * (1 + 2e-6)
    nz = A != 0
    rel = np.abs(A2[nz] - A[nz]) / np.abs(A[nz])
    assert rel.max() <= 1e-6 * (1 + 1e-12) and rel.max() > 1e-7
