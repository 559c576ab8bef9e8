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
