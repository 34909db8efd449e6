import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import golden_cases as gc
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb
case = gc.load(sys.argv[1] if len(sys.argv) > 1 else "lat8_seed5")
batch = frb.pack_batch([case.network], [frb.AffineBC(case.F)])
print("groups", batch.groups)
for T in (224, 256, 320, 512, 544, 672, 1024):
    try:
        r = fb.results_to_solve_results(batch, batch.to_device().solve(case.cfg, frb.TeamBatched(team_size=T)))[0]
        print(T, r.iters, int(case.data["iters"]), np.abs(r.u - case.data["u"]).max())
    except Exception as e:
        print(T, "err", e)
