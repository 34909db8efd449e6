import sys; sys.path.insert(0, '.')
import numpy as np, paper_2305_07030_b200 as frb
net = frb.generate_lattice(20, 20, 20, 0.3, 3)
F = np.eye(3) + 0.2 * np.outer([1, 0, 0], [0, 1, 0])
r = frb.solve_batch(frb.pack_batch([net], [frb.AffineBC(F)]), config=frb.SolverConfig(max_iters=3))[0]
print(r.iters)
