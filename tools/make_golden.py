"""Reference outputs of the full-size BASELINE workloads, written by the ORACLE ONLY (tests/golden/full_*.npz).

VERDICT r01 "next round" item 1 / SURVEY.md §7 step 2: the oracle runs configs 3-5 at their full sizes
and stores what the GPU parity tests compare against (ASPCG protocol: x0 = 0, Euclidean
relative residual <= 1e-8, Lanczos estimate from the same run's CG coefficients, R11/R12):

  iters, lmin, lmax, cond (K), the full alpha/beta history, the relative residual history,
  ||b||, a checksum of b, b on the sampled dofs (the test feeds the oracle's b to the GPU and checks it is this b),
  x on the dofs of >= 8 fixed subdomains (interior, boundary, extreme rho) at iterations
  iters-2 .. iters+2 (the oracle runs 2 iterations past its stop test), and ||x_{iters+2}||.

Nothing here touches the CUDA path; only oracle/ and the input generator dgas_gen/ are imported.
Usage: python tools/make_golden.py [--threads 8] [names...]   (names: cfg3 cfg4 cfg5_p1q1 ... cfg5_p6q6)
The oracle's subdomain loops run on OpenMP threads; results are bitwise independent of the count.
"""
import argparse
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgas_gen as g  # noqa: E402
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
CFG5 = [(1, 1)] + [(p, q) for p in range(2, 7) for q in (1, p)]
NAMES = ["cfg3", "cfg4"] + [f"cfg5_p{p}q{q}" for p, q in CFG5]


def problem(name):
    if name == "cfg3":
        return g.config(3)
    if name == "cfg4":
        return g.config(4)
    p, q = int(name[6]), int(name[8])
    return g.config(5, p, q)


def sample_subdomains(P):
    """>= 8 fixed subdomains: first/last (boundary), spread interior ids, extreme rho (config 4)."""
    n = P.n_sub
    s = {0, n - 1, n // 2, n // 3, (2 * n) // 3, n // 4, (3 * n) // 4, n // 8 + 1}
    rho = np.array([P.kappa[P.part == i][0] for i in range(n)])
    s |= {int(np.argmin(rho)), int(np.argmax(rho))}
    return np.array(sorted(s), np.int32)


def run(name, threads):
    t0 = time.time()
    O.set_threads(threads)
    P = problem(name)
    o = O.Oracle(P)
    o.setup_schwarz()
    if o.N0 > 8192:
        # band-Cholesky coarse path (config 3): one refinement step with a long-double residual (DESIGN.md
        # R30), so the reference is the exact coarse solve to rounding (unrefined band: ~1.5e-10 on cfg3)
        o.set_refine(1)
    t_setup = time.time() - t0
    b = o.rhs()
    subs = sample_subdomains(P)
    npc = P.n_p
    cells = np.nonzero(np.isin(P.part, subs))[0]
    idx = (cells[:, None] * npc + np.arange(npc)[None, :]).ravel().astype(np.int64)
    t1 = time.time()
    h = o.pcg_history(b, idx, rtol=1e-8, maxit=5000, extra=2, n_hist=5)
    t_pcg = time.time() - t1
    assert h["status"] == 0, h["status"]
    it = h["iters"]
    hist_iters = np.array(sorted(h["hist"]), np.int32)
    src = open(os.path.join(os.path.dirname(O.__file__), "oracle.cpp"), "rb").read()
    out = dict(
        name=name, N=o.N, N0=o.N0, iters=it, iters_run=h["iters_run"],
        lmin=h["lmin"], lmax=h["lmax"], cond=h["cond"],
        alphas=h["alphas"], betas=h["betas"], resid=h["resid"],
        bnorm=np.linalg.norm(b), b_sum=b.sum(), b_abs_sum=np.abs(b).sum(), b_idx=b[idx],
        subdomains=subs, idx=idx, hist_iters=hist_iters,
        hist=np.stack([h["hist"][j] for j in hist_iters]),
        xnorm_run=np.linalg.norm(h["x"]),
        oracle_sha=hashlib.sha256(src).hexdigest()[:16], band_refine=int(o.N0 > 8192),
        t_setup_s=t_setup, t_pcg_s=t_pcg, threads=threads,
    )
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, f"full_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: N={o.N} N0={o.N0} iters={it} K={h['cond']:.6f} setup {t_setup:.0f}s pcg {t_pcg:.0f}s "
          f"-> {path}", flush=True)


def augment(name):
    """Add b on the sampled dofs to an existing file (oracle rhs only, no PCG)."""
    path = os.path.join(OUT, f"full_{name}.npz")
    d = dict(np.load(path))
    if "b_idx" in d:
        return
    P = problem(name)
    b = O.Oracle(P).rhs()
    assert abs(np.linalg.norm(b) - float(d["bnorm"])) <= 1e-14 * float(d["bnorm"])
    d["b_idx"] = b[d["idx"]]
    np.savez_compressed(path, **d)
    print(f"{name}: b_idx added", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--augment", action="store_true", help="only add b_idx to existing files")
    ap.add_argument("names", nargs="*", default=NAMES)
    a = ap.parse_args()
    for n in a.names:
        augment(n) if a.augment else run(n, a.threads)


if __name__ == "__main__":
    main()
