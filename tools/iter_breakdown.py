"""Per-iteration time of the PCG graph on one config under the preconditioner variants of
dgas_set_precond (two-level, one-level, coarse-only, none): the differences show what each part of
the apply costs inside the graph (where the coarse solve overlaps the local solves).
  python tools/iter_breakdown.py cfg4"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1903_11357_b200 import dgas  # noqa: E402


def main(name):
    P = bench._problem(name)
    S = dgas.Solver(P)
    b = S.rhs(P.f_kind)
    for mode, label in ((0, "two-level"), (1, "one-level"), (2, "coarse-only"), (3, "none")):
        S.set_precond(mode)
        x = torch.zeros_like(b)
        S.pcg(b, x, maxit=200)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0
        e0.record()
        for _ in range(3):
            x.zero_()
            _, it, _, _ = S.pcg(b, x, maxit=200)
            tot += it
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} {label:12s} iters {tot // 3:5d}  us/iter {e0.elapsed_time(e1) * 1e3 / tot:8.1f}", flush=True)
    S.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
