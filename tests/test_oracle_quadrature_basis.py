"""Oracle pins P1 (quadrature) and P2 (basis) — checked against closed forms and numpy routines,
never against the oracle itself. DESIGN.md readings R6 (basis), R10 (quadrature)."""
import math

import numpy as np
import pytest

import dgas_gen as g
import oracle as O


def test_gauss_legendre_matches_numpy():
    # Golub–Welsch (oracle) vs numpy.polynomial.legendre.leggauss (independent library routine)
    for m in range(1, 13):
        x, w = O.gauss_legendre(m)
        xr, wr = np.polynomial.legendre.leggauss(m)
        assert np.allclose(x, xr, atol=1e-14, rtol=0)
        assert np.allclose(w, wr, atol=1e-14, rtol=0)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 6, 8])
def test_triangle_rule_monomials(m):
    # P1: int_{ref triangle} u^a v^b = a! b! / (a+b+2)!, exact for a+b <= 2m-2
    r = O.triangle_rule(m)
    assert np.all(r[:, 2] > 0)
    for a in range(0, 2 * m - 1):
        for b in range(0, 2 * m - 1 - a):
            exact = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
            got = np.sum(r[:, 2] * r[:, 0] ** a * r[:, 1] ** b)
            assert abs(got - exact) <= 1e-14 * max(1.0, exact) + 1e-16, (m, a, b)


def _green_monomial(poly, a, b):
    """int_P x^a y^b dA = 1/(a+1) \\oint x^{a+1} y^b dy, each edge integrated exactly by numpy leggauss."""
    xs, ws = np.polynomial.legendre.leggauss(a + b + 3)
    t = 0.5 * (xs + 1); w = 0.5 * ws
    s = 0.0
    n = len(poly)
    for i in range(n):
        (x0, y0), (x1, y1) = poly[i], poly[(i + 1) % n]
        x = x0 + t * (x1 - x0); y = y0 + t * (y1 - y0)
        s += np.sum(w * x ** (a + 1) * y ** b) * (y1 - y0)
    return s / (a + 1)


def test_polygon_monomials_green():
    rng = np.random.default_rng(7)
    for trial in range(30):
        # random convex polygon: sorted angles on a perturbed circle
        k = rng.integers(3, 9)
        ang = np.sort(rng.uniform(0, 2 * np.pi, k))
        rad = rng.uniform(0.5, 1.0)
        c = rng.uniform(-1, 1, 2)
        poly = np.stack([c[0] + rad * np.cos(ang), c[1] + rad * np.sin(ang)], 1)
        for (a, b) in [(0, 0), (1, 0), (0, 1), (2, 3), (4, 2), (5, 5)]:
            m = (a + b + 2) // 2 + 1
            ex = _green_monomial(poly, a, b)
            for fan in (0, 1):
                got = O.poly_monomial(poly, a, b, m, fan)
                assert abs(got - ex) <= 1e-12 * max(1, abs(ex)), (trial, a, b, fan)


def test_signed_fan_nonconvex():
    # L-shape (non-convex): signed vertex-0 fan stays exact (used for overlap pieces)
    L = np.array([[0, 0], [2, 0], [2, 1], [1, 1], [1, 2], [0, 2]], float)
    for (a, b) in [(0, 0), (1, 0), (2, 1), (3, 3)]:
        m = (a + b + 2) // 2 + 1
        assert abs(O.poly_monomial(L, a, b, m, 1) - _green_monomial(L, a, b)) < 1e-12
    # and a rotation of the vertex list (fan apex at a reflex-adjacent vertex)
    L2 = np.roll(L, 3, axis=0)
    assert abs(O.poly_monomial(L2, 2, 2, 4, 1) - _green_monomial(L, 2, 2)) < 1e-12


def _numpy_cell_rule(poly, m):
    """Independent (numpy) centroid-fan Duffy rule."""
    xs, ws = np.polynomial.legendre.leggauss(m)
    c = poly.mean(0)
    pts, wts = [], []
    for i in range(len(poly)):
        a, b = poly[i], poly[(i + 1) % len(poly)]
        det = (a[0] - c[0]) * (b[1] - c[1]) - (b[0] - c[0]) * (a[1] - c[1])
        for xi, wi in zip(xs, ws):
            u = 0.5 * (1 + xi)
            for xj, wj in zip(xs, ws):
                v = (1 - u) * 0.5 * (1 + xj)
                pts.append(c + u * (a - c) + v * (b - c)); wts.append(wi * wj * (1 - u) * 0.25 * det)
    return np.array(pts), np.array(wts)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6])
def test_basis_orthonormal_voronoi(p):
    # P2: Gram = I on random Voronoi cells, with an independent (numpy) quadrature
    P = g.generate(1, 64, seed=11, lloyd=2, sub_mode=1, n_sub=1, coarse_mode=0, p=p, q=1)
    o = O.Oracle(P)
    for cell in [0, 7, 33, 63]:
        poly = P.xy[P.cell_vtx[P.cell_ptr[cell]:P.cell_ptr[cell + 1]]]
        pts, w = _numpy_cell_rule(poly, p + 2)
        phi, _, _ = o.eval_basis(cell, pts)
        G = (phi * w[:, None]).T @ phi
        assert np.abs(G - np.eye(o.np_)).max() < 1e-12


def test_basis_square_closed_form():
    # P2 on a square of side s: phi_(a,b) = sqrt((2a+1)(2b+1))/s L_a(xi) L_b(eta) (R6)
    P = g.generate(0, 4, sub_mode=0, sub_tile=4, coarse_mode=0, p=3, q=1)
    o = O.Oracle(P)
    s = 0.25
    cell = 5  # i=1, j=1 -> [0.25,0.5]^2
    rng = np.random.default_rng(0)
    pts = 0.25 + 0.25 * rng.uniform(size=(20, 2))
    phi, px, py = o.eval_basis(cell, pts)
    xi = (pts[:, 0] - 0.25) / s * 2 - 1; eta = (pts[:, 1] - 0.25) / s * 2 - 1
    k = 0
    for d in range(4):
        for a in range(d, -1, -1):
            b = d - a
            La = np.polynomial.legendre.Legendre.basis(a)(xi); Lb = np.polynomial.legendre.Legendre.basis(b)(eta)
            ref = math.sqrt((2 * a + 1) * (2 * b + 1)) / s * La * Lb
            assert np.allclose(phi[:, k], ref, atol=1e-12), (a, b)
            dLa = np.polynomial.legendre.Legendre.basis(a).deriv()(xi) * 2 / s
            assert np.allclose(px[:, k], math.sqrt((2 * a + 1) * (2 * b + 1)) / s * dLa * Lb, atol=1e-10)
            k += 1


def test_basis_spans_Pp():
    # projection of a random degree-p polynomial reproduces it pointwise (span = P_p(kappa), eq:Vh)
    p = 3
    P = g.generate(1, 16, seed=3, lloyd=1, sub_mode=1, n_sub=1, coarse_mode=0, p=p, q=1)
    o = O.Oracle(P)
    rng = np.random.default_rng(1)
    coef = rng.normal(size=(p + 1, p + 1))
    f = lambda x, y: sum(coef[i, j] * x ** i * y ** j for i in range(p + 1) for j in range(p + 1 - i))
    cell = 4
    poly = P.xy[P.cell_vtx[P.cell_ptr[cell]:P.cell_ptr[cell + 1]]]
    pts, w = _numpy_cell_rule(poly, p + 2)
    phi, _, _ = o.eval_basis(cell, pts)
    cvec = (phi * w[:, None]).T @ f(pts[:, 0], pts[:, 1])
    test = poly.mean(0) + 0.01 * rng.normal(size=(5, 2))
    phit, _, _ = o.eval_basis(cell, test)
    assert np.allclose(phit @ cvec, f(test[:, 0], test[:, 1]), atol=1e-10)
