"""The paper's Figs. 2-4 measurement on the B200 (SPEC.md bench module):
self-speedup of the team kernel and of the naive per-operation strategy for a
~1k-DOF (7x7x8) and a ~10k-DOF (15^3) network, plus the team-over-naive
speedup.  Writes profiles/r02_self_speedup{,.summary}.csv and an SVG of each
metric (cli plot).  Wall clock per SPEC.md:444 (packing + upload + solve +
download); a device-only column is measured separately for the team kernel
(CUDA events around the persistent-kernel launch on a resident batch)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import cli
from paper_2305_07030_b200.benchmark import RAW_HEADER, SUMMARY_HEADER, emit_csv, run_benchmark, summarize

out = os.path.join(ROOT, "gpurun_out", "r02_self_speedup")
sizes = [(7, 7, 8), (15, 15, 15)]
recs = run_benchmark(sizes, [1, 4, 16, 64, 148], strategies=("team", "naive"), reps=3)
recs += run_benchmark(sizes, [256, 1024], strategies=("team",), reps=3)
open(out + ".csv", "w").write(emit_csv(recs, RAW_HEADER))
rows = summarize(recs)
open(out + ".summary.csv", "w").write(emit_csv(rows, SUMMARY_HEADER))
cli.main(["plot", "--input", out + ".summary.csv", "-o", out + ".svg"])
cli.main(["plot", "--input", out + ".summary.csv", "--metric", "speedup_over_naive", "-o", out + "_over_naive.svg"])
# device-only team kernel time on a resident batch
lines = ["strategy,n_dofs,n_problems,device_seconds"]
for size in sizes:
    net = frb.generate_lattice(*size, 0.3, 0)
    for N in (1, 4, 16, 64, 148, 256, 1024):
        b = frb.pack_batch([net] * N, [frb.AffineBC(np.diag([1.1, 1, 1]))] * N)
        L = b.to_device().prepare(frb.SolverConfig())
        L.run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            e0.record(); L.run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 1e3)
        lines.append(f"team,{3 * net.n_nodes},{N},{float(np.mean(ts))!r}")
open(out + "_device.csv", "w").write("\n".join(lines) + "\n")
for r in rows:
    print(r.strategy, r.n_dofs, r.n_problems, round(r.mean_seconds, 4), r.self_speedup and round(r.self_speedup, 2),
          r.speedup_over_naive and round(r.speedup_over_naive, 1))
print("\n".join(lines))
