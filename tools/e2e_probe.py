"""Where the c2 end-to-end step goes: upload, solve, download + result conversion."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb

nets = [frb.generate_lattice(15, 15, 15, 0.3, s) for s in range(256)]
batch = frb.pack_batch(nets, [frb.AffineBC(np.diag([1.1, 1, 1]))] * 256)
cfg, strat = frb.SolverConfig(), frb.TeamBatched()
dev = torch.device("cuda:0")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    db = batch.to_device(dev); torch.cuda.synchronize(); t1 = time.perf_counter()
    dres = db.solve(cfg, strat); torch.cuda.synchronize(); t2 = time.perf_counter()
    res = fb.results_to_solve_results(batch, dres); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"to_device {1e3*(t1-t0):.1f} ms  solve {1e3*(t2-t1):.1f} ms  results {1e3*(t3-t2):.1f} ms  total {1e3*(t3-t0):.1f}")
