import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import golden_cases as gc
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb
from oracle import frb_oracle as orc
case = gc.load(sys.argv[1] if len(sys.argv) > 1 else "lat8_seed5")
T = int(sys.argv[2]) if len(sys.argv) > 2 else 512
for k in (1, 2, 3, 4, 6, 10, 30, 100):
    cfg = frb.SolverConfig(max_iters=k)
    batch = frb.pack_batch([case.network], [frb.AffineBC(case.F)])
    dres = batch.to_device().solve(cfg, frb.TeamBatched(team_size=T))
    r = fb.results_to_solve_results(batch, dres)[0]
    o = orc.solve(case.network, case.F, cfg)
    du = np.abs(r.u - o.u)
    bad = np.flatnonzero(r.u != o.u)
    print(k, "res", r.final_residual == o.residual, r.final_residual, o.residual, "u diff", du.max(), "first bad dofs", bad[:10], flush=True)
