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
cfg = frb.SolverConfig(max_iters=1)
batch = frb.pack_batch([case.network], [frb.AffineBC(case.F)])
dres = batch.to_device().solve(cfg, frb.TeamBatched(team_size=T))
us = dres.u.cpu().numpy()
o = orc.solve(case.network, case.F, cfg)
order = batch.problems[0].node_order
uo = o.u.reshape(-1, 3)[order].reshape(-1)
bad = np.flatnonzero(us != uo)
print("nf", 3 * batch.problems[0].n_free_nodes, "bad solver dofs", bad.min() if len(bad) else None, bad.max() if len(bad) else None, len(bad))
print("ratios", (us[bad] / uo[bad])[:12])
print("gpu", us[bad][:6], "orc", uo[bad][:6])
