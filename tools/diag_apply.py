"""Diagnostic (test infrastructure): split the full-size sampled apply error of a config into its
local and coarse parts against the oracle's long-double apply (R30).
  python tools/diag_apply.py cfg3 [env=value ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    os.environ[k] = v
import torch  # noqa: E402

import dgas_gen as g  # noqa: E402
import oracle as O  # noqa: E402
from paper_1903_11357_b200 import dgas  # noqa: E402

name = sys.argv[1]
P = g.config(int(name[3])) if len(name) == 4 else g.config(5, int(name[6]), int(name[8]))
S = dgas.Solver(P)
sample = [0, P.n_sub // 3, P.n_sub - 1]
mask = np.repeat(np.isin(P.part, sample), P.n_p)
r = g.normal(42, S.N)
info = S.get_info()
print(f"{name}: coarse relerr (calibration) {info['coarse_solve_relerr']:.3e}, refine {info['coarse_refine']}")
for mode, uc, ul in (("two_level", True, True), ("one_level", False, True), ("coarse", True, False)):
    o = O.Oracle(P)
    o.setup_schwarz(sample=sample, long_double=True, use_coarse=uc, use_local=ul)
    o.set_refine(2)
    S.set_precond(mode)
    z = S.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    zl = o.apply_sampled(r, sample, long_double=True)
    zr = o.apply_sampled(r, sample)
    e = np.linalg.norm(z[mask] - zl[mask]) / np.linalg.norm(zl[mask])
    e64 = np.linalg.norm(zr[mask] - zl[mask]) / np.linalg.norm(zl[mask])
    print(f"  {mode:10s}: GPU vs exact {e:.3e}   fp64 oracle vs exact {e64:.3e}   |z| {np.linalg.norm(zl[mask]):.3e}")
