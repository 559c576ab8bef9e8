"""Time the coarse solve (dgas_bench_kernels which=4), the local solves (3) and the SpMV (0) on paper-regime
cases, for the coarse-solver choice (DGAS_COARSE_MODE=dense|nd)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dgas_gen as g  # noqa: E402
from paper_1903_11357_b200 import dgas  # noqa: E402


def t(S, which, reps=20):
    S.bench_kernels(which, 3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    S.bench_kernels(which, reps)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


cases = [(4, 4096, 1024, 3), (4, 16384, 1024, 3), (4, 16384, 4096, 3), (4, 16384, 256, 3), (4, 16384, 4096, 1),
         (2, 4096, 2, 3)]
for ex, nf, c, p in cases:
    P = g.paper_case(ex, nf, c, p)
    S = dgas.Solver(P)
    i = S.get_info()
    b = S.rhs(0)
    x, it, cond, st = S.pcg(b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x, it, cond, st = S.pcg(b); e1.record(); torch.cuda.synchronize()
    print(f"ex{ex} Nh={nf} NH={c} p={p} N0={i['N0']} mode={i['coarse_mode']} refine={i['coarse_refine']} "
          f"relerr={i['coarse_solve_relerr']:.2e} coarse {t(S, 4):.1f}us local {t(S, 3):.1f}us spmv {t(S, 0):.1f}us "
          f"apply {t(S, 1):.1f}us iter {e0.elapsed_time(e1) / it * 1e3:.1f}us launches/iter {i['launches_per_iter']}",
          flush=True)
    S.close()
