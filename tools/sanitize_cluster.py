"""A single network on an 8- or 16-CTA cluster for compute-sanitizer runs
(racecheck / synccheck / memcheck), `iters` iterations, compared with the
oracle afterwards so a sanitizer-perturbed schedule must still be exact."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2305_07030_b200 as frb
n, iters = int(sys.argv[1]), int(sys.argv[2])
net = frb.generate_lattice(n, n, n, 0.3, 3)
F = np.eye(3) + 0.2 * np.outer([1, 0, 0], [0, 1, 0])
cfg = frb.SolverConfig(max_iters=iters)
batch = frb.pack_batch([net], [frb.AffineBC(F)])
print("cluster", int(batch.desc[0]["cluster"]), "threads", int(batch.groups[0]["block_threads"]), flush=True)
r = frb.solve_batch(batch, config=cfg)[0]
if "--check" in sys.argv:
    from oracle import frb_oracle as orc
    o = orc.solve(net, F, cfg)
    assert r.iters == o.iters and np.array_equal(r.u, o.u), "differs from the oracle"
    print("bit-equal to the oracle")
print("iters", r.iters, "residual", r.final_residual)
