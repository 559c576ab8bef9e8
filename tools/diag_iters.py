import os, sys, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import dgas_gen as g, oracle as O
from paper_1903_11357_b200 import dgas
P = g.config(4, scale="small")
o = O.Oracle(P); o.setup_schwarz()
b = o.rhs(); ref = o.pcg(b, rtol=1e-8)
print("oracle", ref["iters"])
its = [o.pcg(b * (1 + 1e-13 * g.normal(500 + s, b.shape[0])), rtol=1e-8)["iters"] for s in range(3)]
print("oracle b 1e-13", its)
its = [o.pcg(b * (1 + 1e-10 * g.normal(700 + s, b.shape[0])), rtol=1e-8)["iters"] for s in range(3)]
print("oracle b 1e-10", its)
for seed in (1, 2, 3):
    o2 = O.Oracle(P); o2.set_perturb(2.2e-16, seed); o2.setup_schwarz()
    print("oracle G 1ulp seed", seed, o2.pcg(b, rtol=1e-8)["iters"])
for env in [{}, {"DGAS_ORDER_RCM": "1"}, {"DGAS_COARSE_MODE": "nd", "DGAS_ND_LEAF": "2"}, {"DGAS_COARSE_MODE": "nd", "DGAS_ND_LEAF": "2", "DGAS_ORDER_RCM": "1"}, {"DGAS_SPMV_KERNEL": "3"}, {"DGAS_SPMV_KERNEL": "3", "DGAS_ORDER_RCM": "1"}]:
    for k in ["DGAS_ORDER_RCM", "DGAS_COARSE_MODE", "DGAS_ND_LEAF", "DGAS_SPMV_KERNEL"]: os.environ.pop(k, None)
    os.environ.update(env)
    S = dgas.Solver(P)
    x, it, cond, st = S.pcg(torch.from_numpy(b).cuda())
    r = np.random.default_rng(1).normal(size=S.N)
    z = S.apply(torch.from_numpy(r).cuda()).cpu().numpy(); zr = o.apply(r)
    print("gpu", env, "iters", it, "apply rel", np.linalg.norm(z - zr) / np.linalg.norm(zr))
    S.close()
