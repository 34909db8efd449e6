"""c2 networks on one CTA each with f_prev in global memory (lean mode), vs team size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fbm
from paper_2305_07030_b200.partition import partition_smem_bytes
P = 256
nets = [frb.generate_lattice(15, 15, 15, 0.3, s) for s in range(P)]
probs = [fbm.build_problem(n, frb.AffineBC(np.diag([1.1, 1, 1]))) for n in nets]
batch = fbm._pack(nets, [frb.AffineBC(np.diag([1.1, 1, 1]))] * P, probs, cluster=1)
batch.groups[0]["fprv_global"] = 1
batch.groups[0]["smem_bytes"] = partition_smem_bytes(probs[0].topo.partition(1), True)
db = batch.to_device()
for T in [int(x) for x in os.environ.get("TEAMS", "512,768,1024").split(",")]:
    batch.groups[0]["block_threads"] = T
    L = db.prepare(frb.SolverConfig())
    L.run(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); L.run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"C=1 lean T={T} ms={min(ts):.2f} iters={L.out.host_results()['iters'].mean():.1f}", flush=True)
