"""Wall time of homogenized_tangent (19 solves per network, one device batch) on c2 networks."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb

P = int(os.environ.get("P", "16"))
nets = [frb.generate_lattice(15, 15, 15, 0.3, s) for s in range(P)]
Fs = [np.diag([1.1, 1.0, 1.0])] * P
frb.homogenized_tangent(nets[:1], Fs[:1], h=1e-6)  # warm-up (library load, first pack)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = frb.homogenized_tangent(nets, Fs, h=1e-6)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{P} c2 networks x 19 solves: {dt:.2f} s wall incl. packing and transfers -> {P / dt:.1f} tangents/s; "
      f"all converged {all(r.converged for r in res)}; C_1111 {res[0].tangent[0, 0, 0, 0]:.6g}")
