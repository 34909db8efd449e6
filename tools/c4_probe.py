"""Where c4's makespan goes: the whole heterogeneous batch, its 16-CTA-cluster
networks alone, and the rest alone (kernel time, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07030_b200 as frb
import bench

n_total, _ = bench.layout_of("c4", 1, None)
specs = [bench.network_spec("c4", i) for i in range(n_total)]
nets = [frb.generate_lattice(*lat) for lat, _ in specs]
bcs = [frb.AffineBC(F) for _, F in specs]
full = frb.pack_batch(nets, bcs)
big = [i for i in range(n_total) if int(full.desc["cluster"][i]) >= 16]
rest = [i for i in range(n_total) if int(full.desc["cluster"][i]) < 16]


def timed(batch, label):
    L = batch.to_device().prepare(frb.SolverConfig(), frb.TeamBatched())
    L.run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); L.run(); e1.record(); torch.cuda.synchronize()
    g = [(int(x["cluster"]), int(x["count"]), int(x["block_threads"])) for x in batch.groups]
    print(f"{label}: {e0.elapsed_time(e1):.1f} ms  groups {g}", flush=True)


timed(full, "c4 all")
timed(frb.pack_batch([nets[i] for i in big], [bcs[i] for i in big]), f"c4 C16 only ({len(big)})")
timed(frb.pack_batch([nets[i] for i in rest], [bcs[i] for i in rest]), f"c4 rest ({len(rest)})")

# each smaller group alone (is the concurrent phase 1 better than one after another?)
if os.environ.get("C4_GROUPS"):
    for C in (8, 4, 2, 1):
        ids = [i for i in rest if int(full.desc["cluster"][i]) == C]
        timed(frb.pack_batch([nets[i] for i in ids], [bcs[i] for i in ids]), f"c4 C{C} alone ({len(ids)})")
