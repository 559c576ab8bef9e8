"""compute-sanitizer target: one setup, 3 applies and one PCG solve of a small config through the C ABI
(every per-iteration kernel: ring SpMV, chunked restriction, coarse solve (dense or ND), local solves,
prolongation, Lanczos).  python tools/sanitize_run.py cfg1|cfg2s|cfg4s|cfg4s_nd|cfg3s_nd [maxit]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name = sys.argv[1]
if name.endswith("_nd"):
    os.environ["DGAS_COARSE_MODE"] = "nd"
    os.environ["DGAS_ND_LEAF"] = "4"
    name = name[:-3]
import torch  # noqa: E402

import dgas_gen as g  # noqa: E402
from paper_1903_11357_b200 import dgas  # noqa: E402

k = int(name[3])
P = g.config(k, scale="small") if name.endswith("s") else g.config(k)
S = dgas.Solver(P)
r = torch.from_numpy(g.normal(1, S.N)).cuda()
for _ in range(3):
    z = S.apply(r)
b = S.rhs(P.f_kind)
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
x, it, cond, st = S.pcg(b, maxit=maxit)
torch.cuda.synchronize()
print(f"{sys.argv[1]}: iters {it} cond {cond:.4f} status {st} info {S.get_info()['coarse_mode']}")
S.close()
