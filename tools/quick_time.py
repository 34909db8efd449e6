"""Quick device timing of the persistent kernel on synthetic lattice batches."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb

def run(n, P, reps=3):
    nets = [frb.generate_lattice(n, n, n, 0.3, s) for s in range(P)]
    t0 = time.time()
    batch = frb.pack_batch(nets, [frb.AffineBC(np.diag([1.1, 1, 1]))] * P)
    t_pack = time.time() - t0
    db = batch.to_device()
    cfg = frb.SolverConfig()
    db.solve(cfg); torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dres = db.solve(cfg); e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    rec = dres.host_results()
    iters = rec["iters"].astype(np.int64)
    N = n ** 3
    ms = min(times)
    node_upd = float((iters * N).sum()) / (ms / 1e3)
    print(f"n={n} P={P} pack={t_pack:.2f}s ms={ms:.2f} (all {[round(t,2) for t in times]}) iters mean={iters.mean():.0f} "
          f"nets/s={P/(ms/1e3):.1f} node-upd/s={node_upd/1e9:.3f}G smem={batch.smem_bytes}", flush=True)

for n, P in [(8, 1), (8, 512), (15, 1), (15, 256)]:
    run(n, P)
