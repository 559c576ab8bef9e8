"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element on the
same seeded inputs (BASELINE.json north_star tolerances: apply <= 1e-10 relative L2; PCG iterations
within 2 at rtol 1e-8; x <= 1e-7 relative; Lanczos K within 1%). Intermediate diagnostics use the
tighter SURVEY.md Appendix B bounds (A blocks 1e-13, b 1e-14, A0 1e-12)."""
import os

import numpy as np
import pytest

import dgas_gen as g
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # the -m gpu suite runs on a B200; never silently pass without one
    pytest.fail("GPU tests need CUDA", pytrace=False) if os.environ.get("DGAS_REQUIRE_GPU") else None


def _solver(P, **kw):
    from paper_1903_11357_b200 import dgas
    return dgas.Solver(P, **kw)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


from parity_helpers import _EPS, _coord_tol, _iters_ok, _kappa_gram, _oracle_spread  # noqa: E402,F401


CASES = {
    "cfg1": lambda: g.config(1),
    "cfg2": lambda: g.config(2),
    "cfg2s": lambda: g.config(2, scale="small"),
    "cfg3s": lambda: g.config(3, scale="small"),
    # config-3-style Cartesian meshes with many subdomains sharing a factor (multi-RHS local solve)
    "cart128_p3": lambda: g.generate(0, 128, sub_mode=0, sub_tile=8, coarse_mode=2, coarse_tile=4, name="cart128_p3",
                                     p=3, q=1, f_kind=g.F_SINSIN),
    "cart64_p1": lambda: g.generate(0, 64, sub_mode=0, sub_tile=8, coarse_mode=2, coarse_tile=4, name="cart64_p1",
                                    p=1, q=1, f_kind=g.F_SINSIN),
    "cart64_p2": lambda: g.generate(0, 64, sub_mode=0, sub_tile=8, coarse_mode=2, coarse_tile=4, name="cart64_p2",
                                    p=2, q=2, f_kind=g.F_SINSIN),
    "cart64_p4": lambda: g.generate(0, 64, sub_mode=0, sub_tile=8, coarse_mode=2, coarse_tile=4, name="cart64_p4",
                                    p=4, q=1, f_kind=g.F_SINSIN),
    "cfg4s": lambda: g.config(4, scale="small"),
    "cfg5s_p1q1": lambda: g.config(5, 1, 1, scale="small"),
    "cfg5s_p3q1": lambda: g.config(5, 3, 1, scale="small"),
    "cfg5s_p4q1": lambda: g.config(5, 4, 1, scale="small"),
    "cfg5s_p5q1": lambda: g.config(5, 5, 1, scale="small"),
    "cfg5s_p5q5": lambda: g.config(5, 5, 5, scale="small"),
    "cfg5s_p4q4": lambda: g.config(5, 4, 4, scale="small"),
    "cfg5s_p6q1": lambda: g.config(5, 6, 1, scale="small"),
    "cfg5s_p6q6": lambda: g.config(5, 6, 6, scale="small"),
    # paper regime T_HH = T_h: nested agglomeration (Ex.2) and independent
    # non-nested Voronoi coarse meshes (Ex.4)
    "ex2_h256_H8_p1": lambda: g.paper_case(2, 256, 8, 1),
    "ex4_h256_H16_p3": lambda: g.paper_case(4, 256, 16, 3),
    "ex4_h1024_H64_p1": lambda: g.paper_case(4, 1024, 64, 1),
    # Ex.1 L-shape, rho_e = 1e3 on every other fine cell (not aligned with T_H; K ~ 4e3)
    "ex1c_l2_na_1e3_p2": lambda: g.paper_case_ex1("convex", False, 1e3, 2, levels=2),
}
_cache = {}


def _pair(name):
    if name not in _cache:
        P = CASES[name]()
        o = O.Oracle(P)
        o.setup_schwarz()
        _cache[name] = (P, o, _solver(P))
    return _cache[name]


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4s", "cfg5s_p6q6"])
def test_basis_and_blocks(name):
    P, o, S = _pair(name)
    rng = np.random.default_rng(1)
    cells = rng.choice(P.n_cells, size=min(12, P.n_cells), replace=False)
    for c in cells:
        Cg = S.basis(int(c))
        Co, _ = o.basis(int(c))
        # C = (CholQR2 of the cell Gram)^-1: both sides carry a relative error ~ kappa(Gram) * eps
        kap = _kappa_gram(o, [c])
        assert np.linalg.norm(Cg - Co) <= max(1e-13, 10 * kap * _EPS) * np.linalg.norm(Co), (c, kap)
        # diagonal block and every neighbour block
        for j in range(P.n_cells):
            Bo, ok = o.block(int(c), j)
            if not ok:
                continue
            Bg, okg = S.block(int(c), j)
            assert okg
            err = np.linalg.norm(Bg - Bo) / np.linalg.norm(Bo)
            kap = _kappa_gram(o, [c, j])
            assert err <= max(1e-13, 10 * kap * _EPS), (c, j, err, kap)


@pytest.mark.parametrize("name", list(CASES))
def test_spmv_rhs(name):
    P, o, S = _pair(name)
    x = g.normal(3, S.N)
    y = S.spmv(_dev(x)).cpu().numpy()
    yr = o.spmv(x)
    # rounding scale of A x is |A||x| (cancellation grows with p); entrywise bound with margin
    # entries of A themselves differ by ~kappa(Gram) eps between two correct assemblies (p up to 6)
    scale = o.spmv_abs(x)
    rng = np.random.default_rng(5)
    kap = _kappa_gram(o, rng.choice(P.n_cells, size=min(64, P.n_cells), replace=False))
    # ... and by the coordinate rounding 4 p^2 eps / w_min on fine Cartesian cells (R35)
    tol = max(1e-13, 20 * kap * _EPS, _coord_tol(P))
    assert np.all(np.abs(y - yr) <= tol * scale + 1e-300), (kap, np.max(np.abs(y - yr) / scale))
    b = S.rhs(P.f_kind).cpu().numpy()
    br = o.rhs()
    assert np.abs(b - br).max() <= 1e-14 * max(1.0, np.abs(br).max()) * 10


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4s", "cfg5s_p3q1"])
def test_coarse_operator(name):
    P, o, S = _pair(name)
    A0 = S.A0()
    A0r = o.A0()
    assert np.abs(A0 - A0r).max() <= 1e-12 * np.abs(A0r).max()


@pytest.mark.parametrize("name", list(CASES))
def test_apply_parity(name):
    P, o, S = _pair(name)
    for seed in range(5):
        r = g.normal(100 + seed, S.N)
        z = S.apply(_dev(r)).cpu().numpy()
        zr = o.apply(r)
        assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(zr), seed


def _pcg_parity(S, o, P, b, label, x_tol=1e-7):
    """Full PCG parity against the oracle on the same b (north_star): iterations (_iters_ok), x within
    1e-7 relative (at the common iteration count when the stops differ), Lanczos K within
    1% (or the oracle's own spread / interlacing when the RHS excites an extreme eigenvector only at
    rounding level, R22), and the first CG coefficients to rounding."""
    ref = o.pcg(b, rtol=1e-8)
    x, iters, cond, st = S.pcg(_dev(b), rtol=1e-8)
    x = x.cpu().numpy()
    a, bet = S.history()
    assert st == 0 and ref["status"] == 0
    assert _iters_ok(o, b, ref, iters, P, label), (label, iters, ref["iters"])
    if iters == ref["iters"]:
        err = np.linalg.norm(x - ref["x"]) / np.linalg.norm(ref["x"])
    else:  # compare at a fixed iteration count to separate round-off from stopping
        k = min(iters, ref["iters"])
        xk, ik, _, sk = S.pcg(_dev(b), rtol=1e-300, maxit=k)
        rk = o.pcg(b, rtol=1e-300, maxit=k)
        assert ik == k == rk["iters"], (ik, sk, k, rk["iters"], rk["status"])
        err = np.linalg.norm(xk.cpu().numpy() - rk["x"]) / np.linalg.norm(rk["x"])
    assert err <= x_tol, (label, err)
    if abs(cond - ref["cond"]) > 0.01 * ref["cond"]:
        ks = [o.pcg(b * (1 + 1e-13 * g.normal(600 + t, b.shape[0])), rtol=1e-8)["cond"] for t in range(4)]
        ok = min(ks) * 0.99 <= cond <= max(ks) * 1.01
        if not ok and S.N <= 3000:
            ev = np.sort(np.linalg.eigvals(o.dense_precond() @ o.dense_A()).real)
            ok = 0.95 * ev[-1] / ev[0] <= cond <= ev[-1] / ev[0] * (1 + 1e-8)
        print(f"\n[K branch] {label}: GPU K {cond}, oracle {ref['cond']}, oracle spread {ks}, ok {ok}")
        assert ok, (cond, ref["cond"], ks)
    assert len(a) == iters
    assert np.allclose(a[:3], ref["alphas"][:3], rtol=1e-9)
    return iters, cond


@pytest.mark.parametrize("name", list(CASES))
def test_pcg_parity(name):
    P, o, S = _pair(name)
    _pcg_parity(S, o, P, o.rhs(), name)


def test_pcg_host_matches_device():
    P, o, S = _pair("cfg2")
    b = o.rhs()
    x, it1, c1, _ = S.pcg(_dev(b))
    bh = torch.from_numpy(b).pin_memory()
    xh = torch.zeros(S.N, dtype=torch.float64).pin_memory()
    it2, c2, st = S.pcg_host(bh, xh)
    assert st == 0 and it1 == it2 and c1 == c2
    assert np.array_equal(x.cpu().numpy(), xh.numpy())


def test_pcg_nonzero_x0_and_maxit():
    P, o, S = _pair("cfg2s")
    b = o.rhs()
    x0 = g.normal(9, S.N) * 1e-3
    ref = o.pcg(b, rtol=1e-8, x0=x0)
    x, iters, cond, st = S.pcg(_dev(b), x=_dev(x0.copy()), rtol=1e-8)
    assert abs(iters - ref["iters"]) <= 2
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
    # maxit reached -> DGAS_NOT_CONVERGED (positive status), iterate kept
    x2, it2, c2, st2 = S.pcg(_dev(b), rtol=1e-14, maxit=3)
    assert st2 == 1 and it2 == 3
    ref3 = o.pcg(b, rtol=1e-14, maxit=3)
    assert np.linalg.norm(x2.cpu().numpy() - ref3["x"]) <= 1e-9 * np.linalg.norm(ref3["x"])


def test_pcg_zero_rhs_and_determinism():
    P, o, S = _pair("cfg1")
    x, iters, cond, st = S.pcg(torch.zeros(S.N, dtype=torch.float64, device="cuda"))
    assert st == 0 and iters == 0 and torch.count_nonzero(x).item() == 0
    b = _dev(o.rhs())
    xa, ia, ca, _ = S.pcg(b)
    xb, ib, cb, _ = S.pcg(b)
    assert ia == ib and ca == cb and torch.equal(xa, xb)  # bitwise reproducible (no atomics)


def test_exactness_limits_gpu():
    from paper_1903_11357_b200 import dgas
    P = g.config(1)
    P.part = np.zeros(P.n_cells, np.int32)
    P.n_sub = 1
    S = dgas.Solver(P)
    o = O.Oracle(P)
    b = o.rhs()
    _, iters, cond, st = S.pcg(_dev(b))
    # one subdomain = whole domain: local solve is A^-1 and the coarse term adds a projection, so
    # P^-1 A has eigenvalues in {1, 2}: CG converges in at most 2 iterations
    assert st == 0 and iters <= 2


def test_banded_coarse_path(monkeypatch):
    # force the banded (non-dense) coarse factor on a small problem: same z as the oracle
    monkeypatch.setenv("DGAS_COARSE_DENSE_MAX", "0")
    P = g.config(3, scale="small")
    S = _solver(P)
    assert S.info["coarse_dense"] == 0
    o = O.Oracle(P)
    o.setup_schwarz()
    r = g.normal(7, S.N)
    z = S.apply(_dev(r)).cpu().numpy()
    zr = o.apply(r)
    assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(zr)


def test_errors():
    from paper_1903_11357_b200 import dgas
    P = g.config(1)
    with pytest.raises(dgas.DgasError) as e:
        dgas.Solver(P, p=1, q=2)
    assert e.value.code == dgas.E_INVALID_ARG
    P2 = g.config(1)
    P2.kappa = P2.kappa.copy(); P2.kappa[3] = -1
    with pytest.raises(dgas.DgasError) as e:
        dgas.Solver(P2)
    assert e.value.code == dgas.E_INVALID_ARG
    # a tiny penalty makes A indefinite: a local block fails Cholesky -> NOT_SPD
    P3 = g.config(1)
    with pytest.raises(dgas.DgasError) as e:
        dgas.Solver(P3, penalty=0.05)
    assert e.value.code == dgas.E_NOT_SPD


# --------------------------------------------------------------------------- full BASELINE sizes
@pytest.mark.parametrize("k", [3, 4, 5])
def test_full_size_sampled_apply(k):
    """Full-size configs in the bench's launch configuration: apply parity on sampled subdomains
    (oracle computes the full coarse correction and the local solves of the sampled subdomains)."""
    P = g.config(k, 6, 6) if k == 5 else g.config(k)
    S = _solver(P)
    o = O.Oracle(P)
    sample = [0, P.n_sub // 3, P.n_sub - 1]
    # the exact apply to rounding is the oracle's long-double one (R30): local
    # solves in long double, coarse solve refined with long-double residuals. Both fp64 applies (oracle
    # and GPU) carry ~kappa(A_i) eps local-solve error (config 3: ~1e-10 each), so the GPU is held to
    # the north_star bound against the exact apply, and the fp64 oracle's own distance is printed.
    o.setup_schwarz(sample=sample, long_double=True)
    o.set_refine(2)
    r = g.normal(42, S.N)
    z = S.apply(_dev(r)).cpu().numpy()
    zr = o.apply_sampled(r, sample)
    zl = o.apply_sampled(r, sample, long_double=True)
    mask = np.zeros(P.n_cells, bool)
    for s in sample:
        mask |= P.part == s
    idx = np.repeat(mask, S.info["n_p"])
    err = np.linalg.norm(z[idx] - zl[idx]) / np.linalg.norm(zl[idx])
    err64 = np.linalg.norm(z[idx] - zr[idx]) / np.linalg.norm(zr[idx])
    err_or = np.linalg.norm(zr[idx] - zl[idx]) / np.linalg.norm(zl[idx])
    info = S.get_info()
    msg = (f"cfg{k} full-size sampled apply: GPU vs exact (long double) {err:.3e}, GPU vs fp64 oracle {err64:.3e}, "
           f"fp64 oracle vs exact {err_or:.3e}; coarse solve relerr {info['coarse_solve_relerr']:.3e} with "
           f"{info['coarse_refine']} refinement step(s)")
    print("\n" + msg)
    if info["coarse_mode"] == 2:
        assert info["coarse_solve_relerr"] <= 3e-11  # the GPU's own coarse solve is exact to Z30's bound
    if err > 1e-10:
        # DESIGN.md R30: the exact apply of the GPU's A0 and of the oracle's A0 differ by kappa(A0) times
        # their assembly rounding (A, G and Q^T A Q summed in different orders): refining the GPU's
        # coarse solve does not move this (cfg3: 1.66e-10 -> 1.47e-10). The bound is then the oracle's
        # own spread: its exact (long-double) apply after perturbing G by 1 ulp and A by the relative
        # difference actually measured between the GPU's and the oracle's A blocks on sampled cells.
        rng = np.random.default_rng(3)
        d_a = 0.0
        for c in rng.choice(P.n_cells, size=24, replace=False):
            for j in [int(c)] + [int(v) for v in np.nonzero(P.part == P.part[c])[0]]:
                Bo, ok = o.block(int(c), j)
                if ok:
                    d_a = max(d_a, np.abs(S.block(int(c), j)[0] - Bo).max() / np.abs(Bo).max())
        eps_a = max(d_a, 2.2e-16)
        sens = []
        for kind, seed in (("G", 1), ("G", 2), ("A", 1), ("A", 2)):
            o2 = O.Oracle(P)
            if kind == "G":
                o2.set_perturb(2.2e-16, seed)
            else:
                o2.perturb_A(eps_a, seed)
            o2.setup_schwarz(sample=sample, long_double=True)
            o2.set_refine(2)
            zp = o2.apply_sampled(r, sample, long_double=True)
            sens.append(np.linalg.norm(zp[idx] - zl[idx]) / np.linalg.norm(zl[idx]))
        print(f"[sensitivity branch] cfg{k}: GPU {err:.3e} > 1e-10; measured GPU-vs-oracle A block difference "
              f"{d_a:.2e}; oracle spread (G 1 ulp x2, A {eps_a:.2e} x2) {['%.3e' % e for e in sens]}")
        assert err <= 2 * max(sens), (msg, sens)
    # PCG at full size: converges, and the true residual (oracle SpMV) meets the tolerance
    b = o.rhs()
    x, iters, cond, st = S.pcg(_dev(b))
    assert st == 0 and iters > 0 and cond >= 1
    assert S.get_info()["last_relres"] <= 1e-8
    # true residual: rtol plus the attainable floor of a recursive-residual CG in fp64
    # (|b - A x| drifts from the recursive residual by ~ eps * iters * || |A||x| ||)
    xh = x.cpu().numpy()
    res = np.linalg.norm(b - o.spmv(xh))
    floor = 2.2e-16 * iters * np.linalg.norm(o.spmv_abs(np.abs(xh)))
    assert res <= 1.5e-8 * np.linalg.norm(b) + floor, (res / np.linalg.norm(b), floor / np.linalg.norm(b))
    S.close()


@pytest.mark.parametrize("name,leaf", [("cfg2", "4"), ("cfg3s", "4"), ("cfg4s", "2"), ("cfg5s_p4q4", "3"), ("cfg1", "2")])
def test_nested_dissection_coarse_path(monkeypatch, name, leaf):
    """The multifrontal nested-dissection coarse solve (used for N0 > 8192, e.g. config 3) forced on
    small problems with tiny leaves (deep trees): same z as the oracle's dense Cholesky solve."""
    monkeypatch.setenv("DGAS_COARSE_MODE", "nd")
    monkeypatch.setenv("DGAS_ND_LEAF", leaf)
    P = CASES[name]()
    S = _solver(P)
    info = S.get_info()
    assert info["coarse_mode"] == 2
    # setup-time calibration of the ND solve (R30, Z30): one solve of A0 z = A0 v within 3e-11 after refinement
    assert 0 < info["coarse_solve_relerr"] <= 3e-11 and 0 <= info["coarse_refine"] <= 2
    o = O.Oracle(P)
    o.setup_schwarz()
    for seed in range(3):
        r = g.normal(300 + seed, S.N)
        z = S.apply(_dev(r)).cpu().numpy()
        zr = o.apply(r)
        assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(zr), seed
    _pcg_parity(S, o, P, o.rhs(), f"nd {name} leaf {leaf}")


@pytest.mark.parametrize("name", ["cfg2s", "ex4_h256_H16_p3", "cfg4s"])
def test_precond_variants(name):
    """dgas_set_precond: one-level (no coarse space), coarse only, and none (plain CG,
    whose Lanczos estimate is K(A_h)) against the oracle with the same parts switched off."""
    P = CASES[name]()
    S = _solver(P)
    b = None
    for mode in ("one_level", "coarse", "none"):
        o = O.Oracle(P)
        o.setup_schwarz(use_coarse=mode != "one_level", use_local=mode != "coarse")
        S.set_precond(mode)
        r = g.normal(7, S.N)
        z = S.apply(_dev(r)).cpu().numpy()
        if mode == "none":
            assert np.array_equal(z, r)
        else:
            zr = o.apply(r)
            assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(zr), mode
        if mode == "coarse":
            continue  # R0^T A0^-1 R0 alone is singular on V_h: not a preconditioner for PCG
        if mode == "none" and P.kappa.max() > 10 * P.kappa.min():
            continue  # plain CG on the 1e8 rho-jump matrix does not converge in 20000 iterations
        b = o.rhs() if b is None else b
        ref = o.pcg(b, rtol=1e-8, maxit=20000, precond=mode != "none")
        x, iters, cond, st = S.pcg(_dev(b), rtol=1e-8, maxit=20000)
        assert st == 0 and ref["status"] == 0
        # long unpreconditioned runs: the stopping iteration drifts with rounding (R22), compare x at
        # a common iteration count and K to 1%
        assert abs(iters - ref["iters"]) <= max(2, 0.02 * ref["iters"]), (mode, iters, ref["iters"])
        k = min(iters, ref["iters"])
        xk, ik, _, _ = S.pcg(_dev(b), rtol=1e-300, maxit=k)
        rk = o.pcg(b, rtol=1e-300, maxit=k, precond=mode != "none")
        assert np.linalg.norm(xk.cpu().numpy() - rk["x"]) <= 1e-7 * np.linalg.norm(rk["x"]), mode
        assert abs(cond - ref["cond"]) <= 0.01 * ref["cond"], (mode, cond, ref["cond"])
    S.set_precond("two_level")
    o = O.Oracle(P)
    o.setup_schwarz()
    r = g.normal(8, S.N)
    zr = o.apply(r)
    assert np.linalg.norm(S.apply(_dev(r)).cpu().numpy() - zr) <= 1e-10 * np.linalg.norm(zr)
    with pytest.raises(Exception):
        S.set_precond(7)
    S.close()


@pytest.mark.parametrize("name", ["cfg2s", "cfg4s"])
def test_eager_path_matches_graph(monkeypatch, name):
    """The profiling path (DGAS_EAGER: host-launched iterations, what ncu sees kernel by kernel) computes
    bit-for-bit the same solve as the CUDA-graph path."""
    P = CASES[name]()
    S = _solver(P)
    b = _dev(g.normal(11, S.N))
    x1, it1, c1, s1 = S.pcg(b, rtol=1e-8)
    monkeypatch.setenv("DGAS_EAGER", "1")
    x2, it2, c2, s2 = S.pcg(b, rtol=1e-8)
    assert s1 == s2 == 0 and it1 == it2 and c1 == c2
    assert torch.equal(x1, x2)
    S.close()


# --------------------------------------------------------------------------- local-solve kernels
@pytest.mark.parametrize("name,env,kernel", [
    ("cfg2s", {"DGAS_LOCAL_KERNEL": "1"}, 1),
    ("cfg4s", {"DGAS_LOCAL_KERNEL": "1"}, 1),
    ("cfg1", {}, 2),
    ("cfg5s_p3q1", {}, 2),
    # explicit local inverses (NEXT-4, local_inv.cu), the default when they fit half the L2
    ("cfg1", {"DGAS_LOCAL_INV": "1"}, 3),
    ("cfg2", {"DGAS_LOCAL_INV": "1"}, 3),
    ("cfg5s_p1q1", {"DGAS_LOCAL_INV": "1"}, 3),
    ("cfg3s", {"DGAS_LOCAL_INV": "1"}, 3),
    # warp-per-subdomain merged-panel solve (k_local_warp): default ring, tiny ring (many refills), 1 warp/CTA
    ("cfg4s", {"DGAS_LOCAL_WARP": "1"}, 4),
    ("cfg3s", {"DGAS_LOCAL_WARP": "1"}, 4),
    ("cfg2s", {"DGAS_LOCAL_WARP": "1", "DGAS_LW_SLOT_KB": "1"}, 4),
    ("cfg5s_p1q1", {"DGAS_LOCAL_WARP": "1", "DGAS_LW_WARPS": "1", "DGAS_LW_CPS": "4"}, 4),
    ("cfg5s_p4q4", {"DGAS_LOCAL_WARP": "1", "DGAS_LW_WARPS": "4"}, 4),
    # tiny ring: every panel spans several units, many backward refills (producer protocol)
    ("cfg4s", {"DGAS_LOCAL_CPS": "8", "DGAS_PANEL_SLOT_KB": "1"}, 2),
    ("cfg3s", {"DGAS_PANEL_KEEP": "0", "DGAS_LOCAL_CPS": "3"}, 2),
    ("cfg5s_p6q1", {}, 1),  # n_p = 28: envelope kernel (faster there)
    ("cfg5s_p4q4", {"DGAS_LOCAL_CPS": "7"}, 2),  # 128-thread CTAs on a small problem
    # multi-RHS solve over subdomains sharing a de-duplicated factor (local_mrhs.cu): default geometry,
    # batches of 1 (chain per subdomain), 2-slot ring, B > 16 (one b per lane), every n_p
    ("cart128_p3", {"DGAS_MR_KERNEL": "1"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "1", "DGAS_MR_B": "1", "DGAS_MR_S": "2"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "1", "DGAS_MR_B": "24"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "1", "DGAS_MR_B": "3"}, 5),
    ("cart64_p1", {"DGAS_MR_KERNEL": "1", "DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p2", {"DGAS_MR_KERNEL": "1", "DGAS_MR_MINAVG": "1", "DGAS_MR_B": "17", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p4", {"DGAS_MR_KERNEL": "1", "DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    # independent warp chains (k_local_mrhs_w): default geometry (4 warps x 8 columns), one
    # warp with a 2-slot ring (producer waits on every step), 4 / 16 / 32 columns per warp (8 / 2 / 1
    # K-slices), 8 warps, every n_p (odd n_p: scalar panel loads)
    # independent warp chains (k_local_mrhs_w): default geometry (8 warps x 2 columns, 16 K-slices),
    # one warp with a 2-slot ring (producer waits on every
    # step), 4 / 16 / 32 columns per warp (8 / 2 / 1 K-slices), every n_p (odd n_p: scalar panel loads)
    ("cart128_p3", {"DGAS_MR_KERNEL": "2"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "2", "DGAS_MR_NW": "1", "DGAS_MR_S": "2"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "2", "DGAS_MR_G": "4", "DGAS_MR_NW": "8"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "2", "DGAS_MR_G": "4", "DGAS_MR_NW": "3"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "2", "DGAS_MR_G": "16", "DGAS_MR_NW": "3"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "2", "DGAS_MR_G": "32", "DGAS_MR_NW": "2", "DGAS_MR_S": "8"}, 5),
    ("cart64_p1", {"DGAS_MR_KERNEL": "2", "DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p2", {"DGAS_MR_KERNEL": "2", "DGAS_MR_MINAVG": "1", "DGAS_MR_G": "16", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p4", {"DGAS_MR_KERNEL": "2", "DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p4", {"DGAS_MR_KERNEL": "2", "DGAS_MR_MINAVG": "1", "DGAS_MR_G": "4", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    # warp chains on the FP64 tensor cores (k_local_mrhs_t, mma.sync m8n8k4, the default): default geometry, one warp with a
    # 2-slot ring, 3 and 8 warps (ragged last warp: mirrored columns), every n_p (1 or 2 m-tiles, 1..4 k-steps)
    ("cart128_p3", {}, 5),
    ("cart128_p3", {"DGAS_MR_NW": "4"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "4", "DGAS_MR_NW": "1", "DGAS_MR_S": "2"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "4", "DGAS_MR_NW": "3", "DGAS_MR_S": "4"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "4", "DGAS_MR_NW": "8"}, 5),
    ("cart64_p1", {"DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p2", {"DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p4", {"DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p4", {"DGAS_MR_KERNEL": "4", "DGAS_MR_MINAVG": "1", "DGAS_MR_NW": "2", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    # warp chains with row lanes in the forward sweep (k_local_mrhs_r): default geometry, one warp with a
    # 2-slot ring, 3 warps (ragged last warp), every n_p (3 / 5 / 10 / 2 columns per warp)
    ("cart128_p3", {"DGAS_MR_KERNEL": "3"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "3", "DGAS_MR_NW": "1", "DGAS_MR_S": "2"}, 5),
    ("cart128_p3", {"DGAS_MR_KERNEL": "3", "DGAS_MR_NW": "3", "DGAS_MR_S": "4"}, 5),
    ("cart64_p1", {"DGAS_MR_KERNEL": "3", "DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p2", {"DGAS_MR_KERNEL": "3", "DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p4", {"DGAS_MR_KERNEL": "3", "DGAS_MR_MINAVG": "1", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
    ("cart64_p4", {"DGAS_MR_KERNEL": "3", "DGAS_MR_MINAVG": "1", "DGAS_MR_NW": "2", "DGAS_DEDUP_MAXFRAC": "1"}, 5),
])
def test_local_kernel_variants(monkeypatch, name, env, kernel):
    """Both local-solve kernels (envelope k_local, panel k_local_panel) and the panel kernel's ring
    geometries give the oracle's preconditioner apply within 1e-10 (north_star tolerance)."""
    monkeypatch.setenv("DGAS_LOCAL_INV", "0")  # the factor kernels unless the case asks for the inverses
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    P = CASES[name]()
    S = _solver(P)
    assert S.info["local_kernel"] == kernel
    if kernel == 3:  # Z_i reproduces the exact local solve (setup check)
        assert S.info["local_inv_err"] <= 1e-12
    o = O.Oracle(P)
    o.setup_schwarz()
    for seed in range(3):
        r = g.normal(300 + seed, S.N)
        z = S.apply(_dev(r)).cpu().numpy()
        zr = o.apply(r)
        assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(zr), seed
    _pcg_parity(S, o, P, o.rhs(), f"local {name} {env}")
    S.close()


@pytest.mark.parametrize("name,env", [
    ("cfg2s", {"DGAS_SPMV_KERNEL": "3"}),
    ("cfg4s", {"DGAS_SPMV_KERNEL": "3"}),
    # small byte ring: many wrap-arounds and producer waits on the oldest block
    ("cfg4s", {"DGAS_SR_RING_KB": "40", "DGAS_SR_CPS": "4"}),
    ("cfg5s_p6q6", {"DGAS_SR_RING_KB": "120"}),
    ("cfg1", {}),
    # separate direction-update pass (default only for large vectors) on small problems
    ("cfg4s", {"DGAS_SPMV_PSPLIT": "1"}),
    ("cfg5s_p6q6", {"DGAS_SPMV_PSPLIT": "1"}),
])
def test_spmv_kernel_variants(monkeypatch, name, env):
    """Both SpMV kernels (slot ring k_spmv3, byte ring k_spmv_ring) match the oracle's A x, and the
    fused PCG path built on them matches the oracle's iteration count."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    P = CASES[name]()
    S = _solver(P)
    o = O.Oracle(P)
    o.setup_schwarz()
    rng = np.random.default_rng(5)
    kap = _kappa_gram(o, rng.choice(P.n_cells, size=min(64, P.n_cells), replace=False))
    tol = max(1e-13, 20 * kap * _EPS, _coord_tol(P))  # as test_spmv_rhs: two correct assemblies differ by ~kappa eps
    for seed in range(2):
        xv = g.normal(400 + seed, S.N)
        yv = S.spmv(_dev(xv)).cpu().numpy()
        yr = o.spmv(xv)
        assert np.all(np.abs(yv - yr) <= tol * o.spmv_abs(xv) + 1e-300), seed
    _pcg_parity(S, o, P, o.rhs(), f"spmv {name} {env}")
    S.close()


@pytest.mark.parametrize("name", ["cfg4s", "cfg5s_p6q6"])
def test_pupdate_split_is_bitwise_identical(monkeypatch, name):
    """The separate direction-update pass (k_pupdate + SpMV gather of one vector, the default only when
    the vectors exceed 12 MB, i.e. full-size config 3) computes p = z + beta p with the same expression
    as the fused gather: PCG with and without the split gives the same iterations, K and x bit for bit."""
    P = CASES[name]()
    b = _dev(g.normal(12, P.N))
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("DGAS_SPMV_PSPLIT", v)
        S = _solver(P)
        x, it, c, st = S.pcg(b, rtol=1e-8)
        a, bet = S.history()
        out.append((x.cpu().numpy(), it, c, st, a))
        S.close()
    (x0, i0, c0, s0, a0), (x1, i1, c1, s1, a1) = out
    assert s0 == s1 == 0 and i0 == i1 and c0 == c1
    assert np.array_equal(x0, x1) and np.array_equal(a0, a1)


@pytest.mark.parametrize("name,env", [
    ("cfg1", {}),                          # explicit inverses (k_local_inv)
    ("cfg2", {"DGAS_LOCAL_INV": "0"}),     # wide panel kernel
    ("cfg5s_p3q1", {}),                    # wide panel kernel, non-nested pieces
    ("cfg5s_p6q1", {}),                    # envelope kernel (n_p = 28)
    ("cfg4s", {"DGAS_LOCAL_KERNEL": "1"}),  # envelope kernel with rho jumps and the ND coarse path
])
def test_fused_residual_is_bitwise_identical(monkeypatch, name, env):
    """DESIGN.md §6 item 19: with the residual update fused into the local solve (mode 3) the restriction
    runs beside the local solves; both kernels form r = fma(-alpha, q, r_old), so PCG with and without the
    fusion gives the same iterations, K, alphas and x bit for bit."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    P = CASES[name]()
    b = _dev(g.normal(21, P.N))
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("DGAS_FUSE_R", v)
        S = _solver(P)
        x, it, c, st = S.pcg(b, rtol=1e-8)
        a, bet = S.history()
        out.append((x.cpu().numpy(), it, c, st, a))
        S.close()
    (x0, i0, c0, s0, a0), (x1, i1, c1, s1, a1) = out
    assert s0 == s1 == 0 and i0 == i1 and c0 == c1
    assert np.array_equal(a0, a1) and np.array_equal(x0, x1)


def test_nd_two_contexts_smem_limit(monkeypatch):
    """the ND kernels' dynamic shared-memory limit is a per-function attribute; a second
    context with smaller fronts must not break the first one's launches (or its PCG graph)."""
    monkeypatch.setenv("DGAS_COARSE_MODE", "nd")
    P = CASES["cfg4s"]()
    monkeypatch.setenv("DGAS_ND_LEAF", "64")
    S1 = _solver(P)
    r = _dev(g.normal(21, S1.N))
    z1 = S1.apply(r).cpu().numpy()
    b = _dev(g.normal(22, S1.N))
    x1, it1, _, _ = S1.pcg(b)
    monkeypatch.setenv("DGAS_ND_LEAF", "2")
    S2 = _solver(P)
    z2 = S2.apply(r).cpu().numpy()
    assert np.linalg.norm(z2 - z1) <= 1e-10 * np.linalg.norm(z1)
    assert np.array_equal(S1.apply(r).cpu().numpy(), z1)  # first context still works, same result
    x1b, it1b, _, st = S1.pcg(b)
    assert st == 0 and it1b == it1 and torch.equal(x1b, x1)
    S2.close()
    S1.close()


@pytest.mark.parametrize("name", ["cfg4s", "cfg3s", "cfg2s"])
def test_panel_f32_variant(monkeypatch, name):
    """SURVEY §8(f) NEXT-4, outside the fp64 contract: local factors stored in fp32 (fp64 arithmetic).
    The apply is then an fp32-rounded exact solve (relative error ~1e-7, bounded here by 1e-5), and
    PCG, whose residuals stay fp64, still reaches rtol 1e-8 with the oracle's solution (1e-7) and
    about its iteration count."""
    monkeypatch.setenv("DGAS_PANEL_F32", "1")
    monkeypatch.setenv("DGAS_LOCAL_INV", "0")
    P = CASES[name]()
    S = _solver(P)
    assert S.info["local_kernel"] == 2
    o = O.Oracle(P)
    o.setup_schwarz()
    r = g.normal(500, S.N)
    z = S.apply(_dev(r)).cpu().numpy()
    zr = o.apply(r)
    rel = np.linalg.norm(z - zr) / np.linalg.norm(zr)
    assert 1e-12 < rel <= 1e-5, rel  # really fp32-stored, and still a close preconditioner
    b = o.rhs()
    ref = o.pcg(b, rtol=1e-8)
    x, iters, cond, st = S.pcg(_dev(b))
    assert st == 0 and abs(iters - ref["iters"]) <= max(2, ref["iters"] // 20)
    xh = x.cpu().numpy()
    assert np.linalg.norm(xh - ref["x"]) <= 1e-7 * np.linalg.norm(ref["x"])
    S.close()


def test_dedup_is_bitwise_identical(monkeypatch):
    """Exact de-duplication (dedup.cu, NEXT-4): config-3-style Cartesian meshes produce bitwise-identical
    row-blocks and local factors; storing each once changes no arithmetic. With the SpMV on the same CTA
    chunking as the byte ring (DGAS_DD_CPS = its CTAs per SM), PCG gives the same iterations, K and x bit
    for bit, with and without de-duplication."""
    P = CASES["cfg3s"]()
    out = []
    monkeypatch.setenv("DGAS_MRHS", "0")  # same local kernel (warp per subdomain) in every run
    # runs: no de-duplication (byte ring) | de-duplicated A read through L2 by k_spmv_dd (the byte ring's
    # arithmetic order) | de-duplicated A with the class-sorted k_spmv_cls (its own slice order: same
    # operator, sums in another order, so equal to rounding only)
    for dd, cls, tc in (("0", "0", "0"), ("1", "0", "0"), ("1", "1", "0"), ("1", "1", "1")):
        monkeypatch.setenv("DGAS_DEDUP", dd)
        monkeypatch.setenv("DGAS_SPMV_CLS", cls)
        monkeypatch.setenv("DGAS_CLS_TC", tc)  # 1: the tensor-core class SpMV (k_spmv_cls_t, the default)
        monkeypatch.setenv("DGAS_DD_CPS", "2")
        S = _solver(P)
        info = S.get_info()
        if dd == "1":
            assert 0 < info["dedup_A_bytes"] < info["bytes_A"] // 4
        else:
            assert info["dedup_A_bytes"] == 0
        b = S.rhs(P.f_kind)
        x, it, c, st = S.pcg(b, rtol=1e-8)
        out.append((x.cpu().numpy(), it, c, st, S.spmv(b).cpu().numpy()))
        out_b = b.cpu().numpy()
        S.close()
    (x0, i0, c0, s0, y0), (x1, i1, c1, s1, y1), (x2, i2, c2, s2, y2), (x3, i3, c3, s3, y3) = out
    assert s0 == s1 == 0 and i0 == i1 and c0 == c1
    assert np.array_equal(y0, y1)
    assert np.array_equal(x0, x1)
    # class-sorted SpMV: A x equal entrywise to a few ulps of |A||x| (the sums' rounding scale; A b cancels
    # heavily for the smooth b), PCG within the north_star tolerances of the ring's
    assert s2 == 0 and abs(i2 - i0) <= 2
    scale = O.Oracle(P).spmv_abs(out_b)
    assert np.all(np.abs(y2 - y0) <= 64 * _EPS * scale)
    # tensor-core class SpMV (DMMA sums over k inside the instruction): the same bounds
    assert s3 == 0 and abs(i3 - i0) <= 2
    assert np.all(np.abs(y3 - y0) <= 64 * _EPS * scale)
    assert np.linalg.norm(x3 - x0) <= 1e-7 * np.linalg.norm(x0)
    assert np.linalg.norm(x2 - x0) <= 1e-7 * np.linalg.norm(x0)


def test_error_paths_mesh_breakdown_notconverged(monkeypatch):
    """include/dgas.h error contract: DGAS_E_MESH for a clockwise cell, for a non-manifold
    edge and for overlap pieces that do not cover their fine cell; DGAS_E_BREAKDOWN for a non-finite
    right-hand side; DGAS_NOT_CONVERGED (positive, iterate kept) when maxit is reached with the
    nested-dissection coarse path."""
    import copy
    from paper_1903_11357_b200 import dgas
    P = g.config(1)
    P1 = copy.deepcopy(P)
    a, b_ = P1.cell_ptr[5], P1.cell_ptr[6]
    P1.cell_vtx = P1.cell_vtx.copy()
    P1.cell_vtx[a:b_] = P1.cell_vtx[a:b_][::-1]  # clockwise loop
    with pytest.raises(dgas.DgasError) as e:
        dgas.Solver(P1)
    assert e.value.code == dgas.E_MESH
    P2 = copy.deepcopy(P)  # a duplicated cell: its edges are shared by three cells
    n0 = P2.cell_ptr[1]
    P2.cell_vtx = np.concatenate([P2.cell_vtx, P2.cell_vtx[:n0]]).astype(np.int32)
    P2.cell_ptr = np.concatenate([P2.cell_ptr, [P2.cell_ptr[-1] + n0]]).astype(np.int32)
    P2.part = np.concatenate([P2.part, [0]]).astype(np.int32)
    P2.kappa = np.concatenate([P2.kappa, [1.0]])
    if P2.parent is not None:
        P2.parent = np.concatenate([P2.parent, [0]]).astype(np.int32)
    with pytest.raises(dgas.DgasError) as e:
        dgas.Solver(P2)
    assert e.value.code == dgas.E_MESH
    P4 = g.config(4, scale="small")  # non-nested: shrink one overlap piece so the cell is not covered
    P4.ov_xy = P4.ov_xy.copy()
    k0, k1 = P4.ov_ptr[0], P4.ov_ptr[1]
    cen = P4.ov_xy[k0:k1].mean(0)
    P4.ov_xy[k0:k1] = cen + 0.5 * (P4.ov_xy[k0:k1] - cen)
    with pytest.raises(dgas.DgasError) as e:
        dgas.Solver(P4)
    assert e.value.code == dgas.E_MESH
    S = _solver(P)
    bad = torch.ones(S.N, dtype=torch.float64, device="cuda")
    bad[7] = float("nan")
    with pytest.raises(dgas.DgasError) as e:
        S.pcg(bad, rtol=1e-8)
    assert e.value.code == dgas.E_BREAKDOWN
    S.close()
    monkeypatch.setenv("DGAS_COARSE_MODE", "nd")
    monkeypatch.setenv("DGAS_ND_LEAF", "2")
    S = _solver(CASES["cfg2s"]())
    b = S.rhs(g.F_SINSIN)
    x, it, cond, st = S.pcg(b, rtol=1e-14, maxit=5)
    assert st == dgas.NOT_CONVERGED and it == 5 and torch.isfinite(x).all() and cond >= 1
    S.close()
