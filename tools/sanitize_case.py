"""Small solves for compute-sanitizer runs: one CTA, a 2-CTA cluster, the
energy ledger with the ramp, and a singular element."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2305_07030_b200 as frb
import golden_cases as gc
nets = [frb.generate_lattice(6, 6, 6, 0.3, 1), frb.generate_lattice(14, 14, 15, 0.3, 2)]
F = np.diag([1.1, 1.0, 1.0])
r = frb.solve_batch(frb.pack_batch(nets, [frb.AffineBC(F)] * 2), config=frb.SolverConfig(max_iters=30))
print("plain", [x.iters for x in r])
r = frb.solve_batch(frb.pack_batch(nets, [frb.AffineBC(F)] * 2),
                    config=frb.SolverConfig(max_iters=12, energy_check_interval=1, bc_ramp_iters=5))
print("ledger", [round(x.energy_residual, 6) for x in r])
bad = gc.load("bar_singular")
try:
    frb.dynamic_relaxation_solve(bad.network, frb.AffineBC(bad.F), bad.cfg)
except frb.SingularElementError as e:
    print("singular", e)
