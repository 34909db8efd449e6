"""Kernel-time sweep of cluster size (FRB_DOFS_PER_RANK) x CTA size on a C2-like batch."""
import os, sys, time, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fbm

n = int(os.environ.get("N", "15")); P = int(os.environ.get("P", "256"))
nets = [frb.generate_lattice(n, n, n, 0.3, s) for s in range(P)]
bcs = [frb.AffineBC(np.diag([1.1, 1, 1]))] * P
for dpr in [int(x) for x in os.environ.get("DPR", "3400,1700").split(",")]:
    fbm.DOFS_PER_RANK = dpr
    batch = frb.pack_batch(nets, bcs)
    db = batch.to_device()
    for T in [int(x) for x in os.environ.get("TEAMS", "256,512,768,1024").split(",")]:
        try:
            L = db.prepare(frb.SolverConfig(), frb.TeamBatched(team_size=T))
            L.run(); torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); L.run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            it = L.out.host_results()["iters"]
            print(f"dpr={dpr} C={int(batch.groups['cluster'].max())} T={T} smem={int(batch.groups['smem_bytes'].max())} ms={min(ts):.2f} iters={it.mean():.1f}", flush=True)
        except Exception as ex:
            print(f"dpr={dpr} T={T} failed: {ex}", flush=True)
