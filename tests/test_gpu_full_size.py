"""Full-size parity: dgas_pcg on the BASELINE workloads at their full sizes (configs 3, 4 and all 11
config-5 (p,q) pairs, BASELINE.json configs[2..4]) against reference outputs the ORACLE wrote
(tests/golden/full_*.npz, tools/make_golden.py; nothing in them comes from the CUDA path).

ASPCG protocol (R11/R12): x0 = 0, Euclidean relative residual <= 1e-8,
Lanczos estimate from the same run's CG coefficients. north_star tolerances, applied strictly:
  * iterations within 2 of the oracle's, or (where tools/golden_spread.py stored it) inside the oracle's
    own spread under last-bit perturbations of A, G and b (R22) -- one allowance, never both stacked;
  * x within 1e-7 relative (L2 over the sampled dofs, and element by element against max |x|) at
    the GPU's own iteration count, which the oracle also stored (it ran 2 iterations past its stop),
    else at the nearest stored iteration (the GPU re-run to exactly that count);
  * Lanczos K within 1%.
The sampled dofs are those of >= 8 fixed subdomains (first/last, spread interior ids, and for
config 4 the subdomains of extreme rho). The GPU computes its own b (dgas_rhs); it is checked
against the oracle's b on the same dofs and by norm/sum checksums first.

The CPU test at the bottom checks the golden files themselves (consistency, and that K is the
Lanczos estimate of the stored alpha/beta history) without a GPU."""
import glob
import os

import numpy as np
import pytest

import dgas_gen as g
import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FILES = sorted(glob.glob(os.path.join(GOLD, "full_*.npz")))
NAMES = [os.path.basename(f)[5:-4] for f in FILES]


def _problem(name):
    if name == "cfg3":
        return g.config(3)
    if name == "cfg4":
        return g.config(4)
    return g.config(5, int(name[6]), int(name[8]))


def _load(name):
    return np.load(os.path.join(GOLD, f"full_{name}.npz"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_full_size_pcg_golden(name):
    torch = pytest.importorskip("torch")
    from paper_1903_11357_b200 import dgas
    d = _load(name)
    P = _problem(name)
    S = dgas.Solver(P)
    assert S.N == int(d["N"])
    idx = torch.from_numpy(d["idx"]).cuda()
    b = S.rhs(P.f_kind)
    bh = b.cpu().numpy()
    # b: the oracle's on the sampled dofs (1e-14) and its checksums
    b_ref = d["b_idx"]
    assert np.abs(bh[d["idx"]] - b_ref).max() <= 1e-13 * np.abs(b_ref).max()
    assert abs(np.linalg.norm(bh) - float(d["bnorm"])) <= 1e-13 * float(d["bnorm"])
    assert abs(np.abs(bh).sum() - float(d["b_abs_sum"])) <= 1e-13 * float(d["b_abs_sum"])
    x, iters, cond, st = S.pcg(b, rtol=1e-8, maxit=5000)
    it_ref, k_ref = int(d["iters"]), float(d["cond"])
    xs = x[idx].cpu().numpy()
    a, _ = S.history()
    print(f"\n{name}: iters {iters} (oracle {it_ref}), K {cond:.6f} (oracle {k_ref:.6f})")
    assert st == 0
    if abs(iters - it_ref) > 2:
        # R22: where the residual plateaus near rtol the stopping iteration is not unique under rounding;
        # tools/golden_spread.py stored the ORACLE's own counts under last-bit perturbations of A, G and b.
        # One allowance or the other: within 2 of the oracle, or inside its own spread.
        assert "spread_iters" in d, (iters, it_ref)
        sp = [it_ref] + [int(v) for v in d["spread_iters"]]
        print(f"[spread branch] {name}: GPU {iters}, oracle {it_ref}, oracle spread {min(sp)}..{max(sp)} "
              f"({list(d['spread_probes'])})")
        assert min(sp) <= iters <= max(sp), (iters, sp)
    hist_iters = list(d["hist_iters"])
    if iters not in hist_iters:  # spread branch beyond the stored window: compare at the nearest stored one
        k = min(max(iters, hist_iters[0]), hist_iters[-1])
        xs = S.pcg(b, rtol=1e-300, maxit=k)[0][idx].cpu().numpy()
        iters = k
    xr = d["hist"][hist_iters.index(iters)]
    rel = np.linalg.norm(xs - xr) / np.linalg.norm(xr)
    ew = np.abs(xs - xr).max() / np.abs(xr).max()
    print(f"{name}: x at iteration {iters}: rel L2 {rel:.3e}, max elementwise {ew:.3e}")
    assert rel <= 1e-7 and ew <= 1e-7, (rel, ew)
    assert abs(cond - k_ref) <= 0.01 * k_ref, (cond, k_ref)
    # first CG coefficients: same arithmetic up to rounding
    assert np.allclose(a[:3], d["alphas"][:3], rtol=1e-9)
    S.close()


def test_golden_files_consistent():
    """The golden files are what make_golden.py writes: K is the Lanczos estimate (R12)
    of the stored alpha/beta history (recomputed here by the oracle's Sturm bisection), the history
    covers iters-2..iters+2 and the residual history crosses rtol exactly at `iters`."""
    if not FILES:
        pytest.skip("no golden files")
    for name in NAMES:
        d = _load(name)
        it = int(d["iters"])
        assert d["alphas"].shape[0] == it and d["betas"].shape[0] == it - 1
        lmin, lmax, K = O.lanczos(d["alphas"], d["betas"])
        assert abs(K - float(d["cond"])) <= 1e-12 * K and lmin > 0
        assert list(d["hist_iters"]) == list(range(it - 2, it + 3)), name
        res = d["resid"]
        assert res[it - 1] <= 1e-8 < res[it - 2], name
        assert d["hist"].shape == (5, d["idx"].shape[0])
        assert "b_idx" in d and d["b_idx"].shape == d["idx"].shape
