"""Where the end-to-end step goes: upload, solve, download + result conversion
(python tools/e2e_probe.py [config])."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb
import bench

config = sys.argv[1] if len(sys.argv) > 1 else "c2"
n_total, _ = bench.layout_of(config, 1, None)
pairs = [bench.network_spec(config, i) for i in range(n_total)]
nets = [frb.generate_lattice(*lat) for lat, _ in pairs]
batch = frb.pack_batch(nets, [frb.AffineBC(F) for _, F in pairs]).pin()
cfg, strat = frb.SolverConfig(), frb.TeamBatched()
dev = torch.device("cuda:0")
res = None
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    db = batch.to_device(dev); torch.cuda.synchronize(); t1 = time.perf_counter()
    launch = db.prepare(cfg, strat); t2 = time.perf_counter()
    launch.run(); torch.cuda.synchronize(); t3 = time.perf_counter()
    res = fb.results_to_solve_results(batch, launch.out); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"{config}: to_device {1e3*(t1-t0):.1f} ms  prepare {1e3*(t2-t1):.1f} ms  run {1e3*(t3-t2):.1f} ms  "
          f"results {1e3*(t4-t3):.1f} ms  total {1e3*(t4-t0):.1f} ms", flush=True)
