"""Kernel time of parts of the c2 batch: full waves on 2-CTA clusters, the 34-network tail on 2- and 4-CTA
clusters, one wave, the whole batch (the measurement behind dropping last-wave rebalancing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fbm

nets = [frb.generate_lattice(15, 15, 15, 0.3, s) for s in range(256)]
bc = frb.AffineBC(np.diag([1.1, 1, 1]))

def timed(batch, label):
    db = batch.to_device()
    L = db.prepare(frb.SolverConfig(), frb.TeamBatched())
    L.run(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); L.run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"{label}: {min(ts):.2f} ms  groups {[(int(g['cluster']), int(g['count']), int(g['block_threads'])) for g in batch.groups]}", flush=True)

timed(frb.pack_batch(nets[:222], [bc] * 222), "222 x C2")
timed(fbm._pack(nets[222:], [bc] * 34, [fbm.build_problem(n, bc) for n in nets[222:]], cluster=4), "34 x C4")
timed(frb.pack_batch(nets[222:], [bc] * 34), "34 x C2")
timed(frb.pack_batch(nets[:74], [bc] * 74), "74 x C2")
timed(frb.pack_batch(nets, [bc] * 256), "256 no split")
