import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import golden_cases as gc
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb
from oracle import frb_oracle as orc
case = gc.load(sys.argv[1]); T = int(sys.argv[2])
batch = frb.pack_batch([case.network], [frb.AffineBC(case.F)])
dres = batch.to_device().solve(frb.SolverConfig(), frb.TeamBatched(team_size=T))
nf = 3 * batch.problems[0].n_free_nodes
f = dres.f.cpu().numpy()[:nf]; v = dres.u.cpu().numpy()[:nf]
s = orc.setup(case.network, case.F, 0.5)
u0 = np.zeros((s.n_nodes, 3)); u0[s.nfn:] = s.u_presc
f0, _ = orc.forces(s, u0)
f0 = f0.reshape(-1)[:nf]
a0 = -f0 / np.repeat(s.mass[:s.nfn], 3); v0 = 0.0 + (0.5 * s.dt) * a0; a = v; a0 = v0
bf = np.flatnonzero(f != f0); ba = np.flatnonzero(a != a0)
print("T", T, "f bad", len(bf), bf[:8], "a bad", len(ba), ba[:8])
