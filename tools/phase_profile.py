"""Per-phase SM cycles of the persistent kernel (clock64 marks by thread 0)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import _native as nat

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=15)
ap.add_argument("--P", type=int, default=256)
ap.add_argument("--teams", default="512")
a = ap.parse_args()
nets = [frb.generate_lattice(a.n, a.n, a.n, 0.3, s) for s in range(a.P)]
batch = frb.pack_batch(nets, [frb.AffineBC(np.diag([1.1, 1, 1]))] * a.P)
db = batch.to_device()
for T in [int(x) for x in a.teams.split(",")]:
    L = db.prepare(frb.SolverConfig(), frb.TeamBatched(team_size=T), phase_profile=True)
    L.run(); torch.cuda.synchronize()
    L.phase.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); L.run(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    cyc = L.phase.cpu().numpy().reshape(-1, nat.PHASES)
    iters = L.out.host_results()["iters"].sum()
    C = int(batch.groups["cluster"].max())
    tot = cyc.sum(axis=0)
    print(f"T={T}: {ms:.2f} ms, {iters} network-iterations, cluster {C}, grid {int((cyc.sum(axis=1) > 0).sum())} CTAs")
    for k in range(nat.PHASES):
        print(f"   {nat.PHASE_NAMES[k]:12s} {tot[k] / iters / C:9.0f} cycles per rank-iteration ({100 * tot[k] / tot.sum():5.1f}%)")
