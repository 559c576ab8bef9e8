import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, torch, dgas_gen as g, oracle as O
from paper_1903_11357_b200 import dgas
P = g.config(1); o = O.Oracle(P); o.setup_schwarz(); b0 = o.rhs()
S = dgas.Solver(P)
for s in range(6):
    b = b0 if s == 0 else (b0 * (1 + 1e-13 * g.normal(700 + s, b0.shape[0])) if s < 4 else g.normal(900 + s - 4, b0.shape[0]))
    x, it, cond, st = S.pcg(torch.from_numpy(b).cuda())
    inf = S.get_info()
    ref = o.pcg(b)
    print('case', s, 'gpu', it, round(cond, 5), inf['last_lmin'], inf['last_lmax'], '| oracle', ref['iters'], round(ref['cond'], 5), ref['lmin'], ref['lmax'])
