import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import golden_cases as gc
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb
case = gc.load(sys.argv[1])
T = int(sys.argv[2])
cfg = frb.SolverConfig(max_iters=int(sys.argv[3]))
batch = frb.pack_batch([case.network], [frb.AffineBC(case.F)])
for rep in range(3):
    dres = batch.to_device().solve(cfg, frb.TeamBatched(team_size=T))
    u = dres.u.cpu().numpy()[:648]; f = dres.f.cpu().numpy()[:648]
    z = np.flatnonzero(u == 0)
    print("u zeros", len(z), z[:5], z[-5:] if len(z) else None, "f zeros", np.count_nonzero(f == 0), "iters", dres.host_results()["iters"])
