"""Print the ND coarse-solve calibration (refinement steps, measured relative error) per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgas_gen as g  # noqa: E402
from paper_1903_11357_b200 import dgas  # noqa: E402

for name, P in [("cfg3", g.config(3)), ("cfg4", g.config(4)), ("cfg5_p6q6", g.config(5, 6, 6)),
                ("cfg5_p4q4", g.config(5, 4, 4)), ("cfg5_p3q3", g.config(5, 3, 3))]:
    S = dgas.Solver(P)
    i = S.get_info()
    print(name, "N0", i["N0"], "mode", i["coarse_mode"], "refine", i["coarse_refine"],
          "relerr %.3e" % i["coarse_solve_relerr"], flush=True)
    S.close()
