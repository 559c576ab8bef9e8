"""GPU diagnostic: SpMV entrywise error against the oracle, per SpMV kernel variant (class-sorted, de-duplicated
L2 path, byte ring), on the Cartesian test cases. Test infrastructure (calls oracle/)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import dgas_gen as g  # noqa: E402
import oracle as O  # noqa: E402
from paper_1903_11357_b200 import dgas  # noqa: E402
from test_gpu_parity import CASES  # noqa: E402

for name in sys.argv[1:] or ["cart128_p3", "cfg3s"]:
    P = CASES[name]()
    o = O.Oracle(P)
    x = g.normal(3, P.N)
    yr = o.spmv(x)
    scale = o.spmv_abs(x)
    ys = {}
    for tag, env in (("cls", {}), ("dd", {"DGAS_SPMV_CLS": "0"}), ("ring", {"DGAS_DEDUP": "0"})):
        for k in ("DGAS_SPMV_CLS", "DGAS_DEDUP"):
            os.environ.pop(k, None)
        os.environ.update(env)
        S = dgas.Solver(P)
        y = S.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
        ys[tag] = y
        r = np.abs(y - yr) / scale
        print(f"{name} {tag}: max |y - y_oracle| / (|A||x|) = {r.max():.3e}, median {np.median(r):.3e}, "
              f"99.9% {np.quantile(r, 0.999):.3e}", flush=True)
        # worst cell's blocks against the oracle
        c = int(np.argmax(r)) // S.info["n_p"]
        worst = 0.0
        for j in range(P.n_cells):
            Bo, ok = o.block(c, j)
            if not ok:
                continue
            Bg, _ = S.block(c, j)
            worst = max(worst, float(np.abs(Bg - Bo).max() / np.abs(Bo).max()))
        print(f"   worst cell {c}: max entry difference of its blocks / max entry = {worst:.3e}", flush=True)
        S.close()
    for a in ("dd", "ring"):
        d = np.abs(ys["cls"] - ys[a]) / scale
        print(f"{name} cls vs {a}: max {d.max():.3e}; bitwise equal: {np.array_equal(ys['cls'], ys[a])}")
