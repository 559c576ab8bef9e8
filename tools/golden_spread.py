"""The oracle's own stopping-iteration spread at full size (R22/R30), added to the golden files.

Two correct fp64 assemblies differ in their last bits (A: ~kappa(Gram) eps, G: ~1 ulp, b: ~1e-13), and
where the PCG residual plateaus near rtol the stopping iteration is not unique under such rounding. This
runs the ORACLE's PCG (oracle/ only, like make_golden.py) under those perturbations and stores the
iteration counts as `spread_iters` (probes in `spread_probes`), so a GPU count is accepted within 2 of the
oracle's or inside [min, max] of its own spread -- one allowance, not both.
  python tools/golden_spread.py [--threads 8] cfg4 ..."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgas_gen as g  # noqa: E402
import oracle as O  # noqa: E402
from make_golden import OUT, problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("names", nargs="+")
    a = ap.parse_args()
    O.set_threads(a.threads)
    for name in a.names:
        path = os.path.join(OUT, f"full_{name}.npz")
        d = dict(np.load(path))
        P = problem(name)
        o = O.Oracle(P)
        b = o.rhs()
        kap = max(np.linalg.cond(o.basis(int(c))[0]) ** 2 for c in range(0, P.n_cells, max(1, P.n_cells // 64)))
        probes, its = [], []
        for kind, seed in (("A", 1), ("A", 2), ("G", 1), ("G", 2), ("b", 1)):
            o2 = O.Oracle(P)
            if kind == "A":
                o2.perturb_A(kap * 2.220446049250313e-16, seed)
            elif kind == "G":
                o2.set_perturb(2.220446049250313e-16, seed)
            o2.setup_schwarz()
            if o2.N0 > 8192:
                o2.set_refine(1)
            bb = b * (1 + 1e-13 * g.normal(500 + seed, b.shape[0])) if kind == "b" else b
            it = o2.pcg(bb, rtol=1e-8)["iters"]
            probes.append(f"{kind}{seed}")
            its.append(it)
            print(f"{name}: probe {kind}{seed} (kappa_gram {kap:.3g}) -> {it} iterations", flush=True)
        d["spread_probes"] = np.array(probes)
        d["spread_iters"] = np.array(its, np.int32)
        np.savez_compressed(path, **d)
        print(f"{name}: oracle {int(d['iters'])}, spread {min(its)}..{max(its)}", flush=True)


if __name__ == "__main__":
    main()
