#!/usr/bin/env python
"""Benchmark: batched dynamic relaxation of fiber networks on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
    python bench.py --impl reference ...      # CPU reference arm (oracle port)

A *step* is one solve of the whole batch (every network relaxed to
convergence) by one persistent-kernel launch.  Default workload is
BASELINE.json configs[1] (c2): 256 networks generate_lattice(15,15,15,0.3,s)
s = 0..255 (10,125 DOF, 9,450 fibers each) under uniaxial F=diag(1.1,1,1),
default SolverConfig, FP64.  Under torchrun each rank solves its own 256
networks (seeds offset by rank; weak scaling) and the per-network stresses
are gathered to rank 0 with NCCL at the end of every step.

Printed JSON (rank 0): value = networks/s for the whole job (device-resident
batch, kernel + result gather), e2e = the same through the public API from
pinned host buffers (upload, solve, download, unpermute), roofline of the
kernel against the measured HBM copy bandwidth using the algorithmic bytes
B_iter = 48 N + 48 nf + 24 M per network-iteration, and a
CPU baseline: the oracle port timed on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # CPU arm: one BLAS thread per worker
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

METRIC = "networks solved/sec and DR node-updates/sec per GPU at 1/2/4/8 B200; % HBM roofline"
UNIAX = np.diag([1.1, 1.0, 1.0])
BIAX = np.diag([1.1, 1.1, 1.0])
SHEAR = np.eye(3) + 0.2 * np.outer([1, 0, 0], [0, 1, 0])
L2_FLUSH_BYTES = 256 << 20


C5_TOTAL = 16384


def shard_indices(name: str, rank: int, world: int) -> list[int]:
    """Network indices a rank solves: c2 is weak-scaled (256 per
    GPU), c3/c4 are strided (iteration counts vary by size/load), c5 is split
    into contiguous shards of the FE2 macro-step's 16,384 networks."""
    if name == "c1":
        return [0]
    if name == "c2":
        return list(range(rank * 256, (rank + 1) * 256))
    if name == "c3":
        return list(range(rank, 1024, world))
    if name == "c4":
        return list(range(rank, 1024, world))
    if name == "c5":
        per = -(-C5_TOTAL // world)
        return list(range(rank * per, min(C5_TOTAL, (rank + 1) * per)))
    raise SystemExit(f"unknown --config {name}")


def c5_gradient(i: int) -> np.ndarray:
    """Random macro deformation gradient of FE2 network i."""
    rng = np.random.default_rng(10 ** 6 + i)
    diag = rng.uniform(0.0, 0.1, 3)
    off = rng.uniform(-0.05, 0.05, (3, 3))
    np.fill_diagonal(off, 0.0)
    return np.eye(3) + np.diag(diag) + off


def config_networks(name: str, rank: int, world: int, limit: int | None = None):
    """(workload description, networks, deformation gradients) for one rank."""
    import paper_2305_07030_b200 as frb
    idx = shard_indices(name, rank, world)
    n_all = len(idx)  # limit=0: the description only (names the whole shard)
    if limit is not None:
        idx = idx[:limit]
        n_all = n_all if limit == 0 else len(idx)
    if name == "c1":
        return ("c1: 1 x generate_lattice(7,7,8,0.3,seed=0), uniaxial F=diag(1.1,1,1)",
                [frb.generate_lattice(7, 7, 8, 0.3, 0)], [UNIAX])
    if name == "c2":
        return (f"c2: {n_all} x generate_lattice(15,15,15,0.3,seed=s) per GPU (10,125 DOF, 9,450 fibers), "
                "uniaxial F=diag(1.1,1,1)",
                [frb.generate_lattice(15, 15, 15, 0.3, s) for s in idx], [UNIAX] * len(idx))
    if name == "c3":
        return (f"c3: 1024 x generate_lattice(32,32,32,0.3,seed=s) (98,304 DOF, 95,232 fibers), uniaxial, "
                f"strided shards ({n_all} on this GPU)",
                [frb.generate_lattice(32, 32, 32, 0.3, s) for s in idx], [UNIAX] * len(idx))
    if name == "c4":
        nets, Fs = [], []
        for i in idx:
            n = 7 + (i % 26)
            nets.append(frb.generate_lattice(n, n, n, 0.3, i))
            Fs.append([UNIAX, BIAX, SHEAR][i % 3])
        return ("c4: 1024 heterogeneous lattices n=7+(i mod 26) (1k-100k DOF), "
                "loads uniax/biax/shear by i mod 3, strided shards", nets, Fs)
    return (f"c5: FE2 macro-step, {C5_TOTAL} x 15^3 networks, random F, contiguous shards",
            [frb.generate_lattice(15, 15, 15, 0.3, i) for i in idx], [c5_gradient(i) for i in idx])


def gather_stresses(sig, world: int, dist):
    """Final homogenized-stress gather of the macro step: every rank's
    [P, 9] float64 block to every rank (NCCL on the GPU box, gloo in tests)."""
    import torch
    P = sig.shape[0]
    counts = torch.tensor([P], dtype=torch.int64, device=sig.device)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts)
    Pmax = int(max(c.item() for c in all_counts))
    pad = torch.zeros((Pmax, 9), dtype=sig.dtype, device=sig.device)
    pad[:P] = sig
    out = torch.empty((world, Pmax, 9), dtype=sig.dtype, device=sig.device)
    if sig.is_cuda:
        dist.all_gather_into_tensor(out.view(world * Pmax, 9), pad)
    else:  # gloo has no all_gather_into_tensor
        dist.all_gather(list(out.unbind(0)), pad)
    return torch.cat([out[r, :int(all_counts[r].item())] for r in range(world)])


def b_iter(N: int, nf: int, M: int) -> int:
    """Algorithmic bytes per network-iteration."""
    return 48 * N + 48 * nf + 24 * M


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


# --------------------------------------------------------------------- CPU arm

def _oracle_solve(args):
    cfgname, i = args
    sys.path.insert(0, ROOT)
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import paper_2305_07030_b200 as frb
    from oracle import frb_oracle as orc
    if cfgname == "warm":
        net, F = frb.generate_lattice(3, 3, 3, 0.3, 0), UNIAX
    else:
        _, nets, Fs = config_networks(cfgname, 0, 1, limit=None) if cfgname == "c1" else \
            _one_network(cfgname, i)
        net, F = nets[0], Fs[0]
    t0 = time.perf_counter()
    r = orc.solve(net, F, frb.SolverConfig())
    return time.perf_counter() - t0, r.iters, net.n_nodes


def _one_network(cfgname: str, i: int):
    """Network i of a workload (the CPU sample takes the first ones)."""
    import paper_2305_07030_b200 as frb
    if cfgname == "c2":
        return "", [frb.generate_lattice(15, 15, 15, 0.3, i)], [UNIAX]
    if cfgname == "c3":
        return "", [frb.generate_lattice(32, 32, 32, 0.3, i)], [UNIAX]
    if cfgname == "c4":
        n = 7 + (i % 26)
        return "", [frb.generate_lattice(n, n, n, 0.3, i)], [[UNIAX, BIAX, SHEAR][i % 3]]
    return "", [frb.generate_lattice(15, 15, 15, 0.3, i)], [c5_gradient(i)]


def cpu_sample(config: str, cores: int, per_core: int = 1):
    """Time the oracle port on `cores` worker processes over a bounded sample
    of the workload: its first cores * per_core networks (networks/s over the
    sample; generation excluded)."""
    import multiprocessing as mp
    jobs = [(config, i) for i in range(cores * per_core)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_oracle_solve, [("warm", 0)] * cores)  # warm the workers (imports)
        t0 = time.perf_counter()
        out = pool.map(_oracle_solve, jobs)
        wall = time.perf_counter() - t0
    node_upd = sum(it * n for _, it, n in out)
    return dict(networks=len(jobs), wall_s=wall, nets_per_s=len(jobs) / wall,
                node_updates_per_s=node_upd / wall, cpu_s=sum(t for t, _, _ in out))


def run_reference_arm(args, rank: int):
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(args.config, cores)
    samples = [cpu_sample(args.config, cores) for _ in range(args.steps)]
    value = sum(s["networks"] for s in samples) / sum(s["wall_s"] for s in samples)
    ms = 1e3 * statistics.mean(s["wall_s"] for s in samples)
    sample = (f"{samples[0]['networks']} networks of the {args.config} workload per step "
              f"(one per core, fork pool, OPENBLAS_NUM_THREADS=1)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "networks/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generate_lattice inputs)",
        "config": {"workload": config_networks(args.config, 0, 1, limit=0)[0],
                   "arm": "oracle/frb_oracle.py (numpy restatement of fibrelax, bit-exact)"},
        "node_updates_per_s": statistics.mean(s["node_updates_per_s"] for s in samples),
        "cpu_baseline": {"value": value, "unit": "networks/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "networks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--limit", type=int, default=None, help="networks per rank (c3/c4/c5 samples)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--team-size", type=int, default=None, help="CTA size override (TeamBatched)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2305_07030_b200 as frb
    from paper_2305_07030_b200 import batch as fb

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    workload, nets, Fs = config_networks(args.config, rank, world, args.limit)
    cfg = frb.SolverConfig()
    t0 = time.perf_counter()
    batch = frb.pack_batch(nets, [frb.AffineBC(F) for F in Fs])
    setup_s = time.perf_counter() - t0
    batch.pin()
    dbatch = batch.to_device(dev)
    strategy = frb.TeamBatched(team_size=args.team_size)
    launch = dbatch.prepare(cfg, strategy)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    P = batch.n_problems
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        flush.zero_()
        if ev is not None:
            ev[0].record(stream)
        launch.run(stream)
        if ev is not None:
            ev[1].record(stream)
        if world > 1:  # final homogenized-stress gather (C1 result gather)
            sig = launch.out.results.view(torch.float64).view(P, -1)[:, 5:14]
            gather_stresses(sig, world, dist)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize(dev)
        t_start.record(stream)
        for k in range(args.steps):
            step(kev[k])
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    elapsed = t_start.elapsed_time(t_end) / 1e3
    kern = [a.elapsed_time(b) / 1e3 for a, b in kev]
    if world > 1:
        t = torch.tensor([elapsed, statistics.mean(kern)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, kern_mean = t.tolist()
    else:
        kern_mean = statistics.mean(kern)

    rec = launch.out.host_results()
    iters = rec["iters"].astype(np.int64)
    Ns = np.array([p.n_nodes for p in batch.problems], dtype=np.int64)
    nfs = np.array([3 * p.n_free_nodes for p in batch.problems], dtype=np.int64)
    Ms = np.array([p.network.n_elements for p in batch.problems], dtype=np.int64)
    alg_bytes = float((iters * (48 * Ns + 48 * nfs + 24 * Ms)).sum())
    node_updates = float((iters * Ns).sum())
    assert (rec["status"] == 0).all(), "not every network converged"

    # ---- e2e through the public API (pinned host buffers -> results) ----
    def e2e_step():
        return fb.results_to_solve_results(batch, batch.to_device(dev).solve(cfg, strategy))
    for _ in range(1):
        e2e_step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e_steps = max(1, min(args.steps, 3))
    te = time.perf_counter()
    for _ in range(e_steps):
        res = e2e_step()
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - te) / e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = t.item()
    h2d = sum(a.nbytes for a in batch.arrays.values()) + batch.desc.nbytes
    d2h = 3 * int(batch.node_base[-1]) * 8 + P * 144
    assert all(r.converged for r in res)

    ms_per_step = 1e3 * elapsed / args.steps
    value = world * P / (elapsed / args.steps)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as fh:
            peak, peak_src = float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    achieved = alg_bytes / kern_mean / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get(args.config)

    line = {
        "metric": METRIC, "value": value, "unit": "networks/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generate_lattice jittered lattices, same generator as the reference)",
        "config": {"workload": workload, "networks_per_gpu": P, "parallelism": f"shard{world}",
                   "l2": "flushed (256 MiB memset before every step)",
                   "setup_s_per_rank": round(setup_s, 3), "cta_threads": launch.threads},
        "node_updates_per_s": world * node_updates / (elapsed / args.steps),
        "iters_mean": float(iters.mean()),
        "e2e": {"value": world * P / e2e_s, "unit": "networks/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": args.steps * int((launch.groups["count"] > 0).sum()),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "frb_relax_kernel", "kernel_ms": 1e3 * kern_mean,
                     "alg_bytes_per_launch": alg_bytes},
        "clocks": clocks.summary(),
        "kernel_ms_per_step": [round(1e3 * k, 3) for k in kern],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        s = cpu_sample(args.config, cores)
        line["cpu_baseline"] = {
            "value": s["nets_per_s"], "unit": "networks/s", "cores": cores, "kind": "port",
            "sample": f"{s['networks']} networks of the {args.config} workload, one per core "
                      f"({s['wall_s']:.1f} s wall, {s['cpu_s']:.1f} s CPU)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
