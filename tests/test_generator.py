"""Input-generator invariants (SPEC-style mesh checks)."""
import numpy as np
import pytest

import dgas_gen as g


def _areas(xy, ptr, vtx):
    out = []
    for c in range(len(ptr) - 1):
        p = xy[vtx[ptr[c]:ptr[c + 1]]]
        out.append(0.5 * np.sum(p[:, 0] * np.roll(p[:, 1], -1) - np.roll(p[:, 0], -1) * p[:, 1]))
    return np.array(out)


def _edges(P):
    from collections import Counter
    cnt = Counter()
    for c in range(P.n_cells):
        v = P.cell_vtx[P.cell_ptr[c]:P.cell_ptr[c + 1]]
        for k in range(len(v)):
            a, b = v[k], v[(k + 1) % len(v)]
            cnt[(min(a, b), max(a, b))] += 1
    return cnt


@pytest.mark.parametrize("k", [1, 2, 5])
def test_mesh_invariants(k):
    P = g.config(k)
    a = _areas(P.xy, P.cell_ptr, P.cell_vtx)
    assert np.all(a > 0)
    assert abs(a.sum() - 1) < 1e-12
    cnt = _edges(P)
    assert max(cnt.values()) <= 2
    # boundary edges lie on the boundary of the unit square
    for (u, v), n in cnt.items():
        if n == 1:
            pu, pv = P.xy[u], P.xy[v]
            on = lambda p: min(p[0], p[1], 1 - p[0], 1 - p[1]) < 1e-13
            assert on(pu) and on(pv)
            assert abs(pu[0] - pv[0]) < 1e-13 or abs(pu[1] - pv[1]) < 1e-13


def test_rcb_exact_counts_and_nesting():
    P = g.config(2)
    assert np.all(np.bincount(P.part, minlength=16) == 64)
    assert np.all(np.bincount(P.parent, minlength=64) == 16)
    # RCB(64) refines RCB(16): each agglomerate lies in one subdomain
    for J in range(64):
        assert len(set(P.part[P.parent == J])) == 1


def test_cartesian_tiles():
    P = g.config(1)
    assert np.all(np.bincount(P.part) == 64)
    assert np.array_equal(P.parent, P.part)
    P3 = g.config(3, scale="small")
    assert P3.n_coarse == (32 // 4) ** 2 and P3.n_sub == (32 // 8) ** 2


def test_nonnested_overlaps_complete():
    P = g.config(4, scale="small")
    assert not P.nested
    a_cell = _areas(P.xy, P.cell_ptr, P.cell_vtx)
    a_piece = _areas(P.ov_xy, P.ov_ptr, np.arange(P.ov_xy.shape[0]))
    s = np.zeros(P.n_cells)
    np.add.at(s, P.ov_fine, a_piece)
    assert np.abs(s - a_cell).max() <= 1e-10 * a_cell.max()
    # coarse areas sum to 1 and pieces of each coarse element add up to its polygon area
    a_coarse = _areas(P.cpoly_xy, P.cpoly_ptr, np.arange(P.cpoly_xy.shape[0]))
    assert abs(a_coarse.sum() - 1) < 1e-12
    sc = np.zeros(P.n_coarse)
    np.add.at(sc, P.ov_coarse, a_piece)
    assert np.abs(sc - a_coarse).max() < 1e-10
    # genuinely non-nested: some fine cell is cut by a coarse boundary
    assert len(P.ov_fine) > P.n_cells


def test_kappa_per_subdomain():
    P = g.config(4, scale="small")
    for s in range(P.n_sub):
        assert len(set(P.kappa[P.part == s])) == 1
    assert P.kappa.min() >= 1e-4 and P.kappa.max() <= 1e4


def test_determinism():
    a = g.config(2); b = g.config(2)
    assert np.array_equal(a.xy, b.xy) and np.array_equal(a.cell_vtx, b.cell_vtx)
    assert np.array_equal(g.normal(5, 100), g.normal(5, 100))
    x = g.normal(5, 200000)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01


def test_independent_coarse_mesh_overlaps():
    """Ex.4: an independently generated Voronoi coarse mesh; the pieces kappa ∩ D_J tile
    every fine cell and every coarse polygon."""
    P = g.paper_case(4, 256, 16, 1)
    assert not P.nested and P.n_coarse == 16 and P.n_sub == P.n_cells == 256
    assert np.array_equal(np.sort(P.part), np.arange(256))
    a_cell = _areas(P.xy, P.cell_ptr, P.cell_vtx)
    a_piece = _areas(P.ov_xy, P.ov_ptr, np.arange(P.ov_xy.shape[0]))
    assert a_piece.min() > 0
    s = np.zeros(P.n_cells)
    np.add.at(s, P.ov_fine, a_piece)
    assert np.abs(s - a_cell).max() <= 1e-10 * a_cell.max()
    a_coarse = _areas(P.cpoly_xy, P.cpoly_ptr, np.arange(P.cpoly_xy.shape[0]))
    assert abs(a_coarse.sum() - 1) < 1e-12
    sc = np.zeros(P.n_coarse)
    np.add.at(sc, P.ov_coarse, a_piece)
    assert np.abs(sc - a_coarse).max() < 1e-10
    assert len(P.ov_fine) > P.n_cells
    # Ex.2 nested hierarchy: H = 8 h_bar -> 4096 / 64 = 64 agglomerates of the fine cells
    P2 = g.paper_case(2, 256, 8, 1)
    assert P2.nested and P2.n_coarse == 64 and len(np.unique(P2.parent)) == 64


@pytest.mark.parametrize("variant", ["convex", "nonconvex"])
def test_lshape_meshes(variant):
    """Ex.1 L-shaped domain: area 3/4, conforming (every edge shared by at most two cells,
    unshared edges on the boundary of L), convex cells, nested coarse map with consecutive children."""
    P = g.paper_case_ex1(variant, True, 10.0, 1, levels=2)
    a = _areas(P.xy, P.cell_ptr, P.cell_vtx)
    assert a.min() > 0 and abs(a.sum() - 0.75) < 1e-12
    cnt = _edges(P)
    assert max(cnt.values()) == 2
    for (i, j), c in cnt.items():
        if c == 1:  # boundary edge: on x = 0, x = 1, y = 0, y = 1, x = 1/2 (y <= 1/2) or y = 1/2 (x >= 1/2)
            (x0, y0), (x1, y1) = P.xy[i], P.xy[j]
            on = [abs(x0) + abs(x1) < 1e-12, abs(x0 - 1) + abs(x1 - 1) < 1e-12, abs(y0) + abs(y1) < 1e-12,
                  abs(y0 - 1) + abs(y1 - 1) < 1e-12,
                  abs(x0 - .5) + abs(x1 - .5) < 1e-12 and max(y0, y1) <= .5 + 1e-12,
                  abs(y0 - .5) + abs(y1 - .5) < 1e-12 and min(x0, x1) >= .5 - 1e-12]
            assert any(on), (P.xy[i], P.xy[j])
    for c in range(P.n_cells):  # convex: every cross product of consecutive edges >= 0 (collinear allowed)
        q = P.xy[P.cell_vtx[P.cell_ptr[c]:P.cell_ptr[c + 1]]]
        e = np.roll(q, -1, axis=0) - q
        cr = e[:, 0] * np.roll(e, -1, axis=0)[:, 1] - e[:, 1] * np.roll(e, -1, axis=0)[:, 0]
        assert cr.min() >= -1e-14
    assert P.nested and P.n_coarse == 16 and P.n_sub == P.n_cells
    if variant == "convex":
        assert np.all(np.diff(P.parent) >= 0)  # children consecutive
        # not aligned: rho alternates within every coarse element, so max/min = rho_e in each D_j
        Q = g.paper_case_ex1(variant, False, 10.0, 1, levels=2)
        for J in range(16):
            k = Q.kappa[Q.parent == J]
            assert k.max() / k.min() == 10.0
        assert np.array_equal(np.unique(P.kappa[P.parent % 2 == 1]), [10.0])
