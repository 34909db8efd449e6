#!/usr/bin/env python
"""Benchmark: batched dynamic relaxation of fiber networks on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
    python bench.py --impl reference ...   # the reference's CPU path on this host

A *step* is one solve of the whole batch (every network relaxed to
convergence) by one persistent-kernel launch per launch group.  The default
workload is BASELINE.json configs[2] (c3), the largest single-GPU
configuration and the one the north-star target is quoted on: 1,024 networks
generate_lattice(32,32,32,0.3,s), s = 0..1023 (98,304 DOF, 95,232 fibers
each; the 16-CTA cluster path) under uniaxial F = diag(1.1,1,1), default
SolverConfig, FP64.  Under torchrun the 1,024 networks are sharded by index
over the GPUs (strided shards, paper_2305_07030_b200.distributed; strong
scaling) and every step ends with the NCCL gather of all networks' result
records.  --config c1/c2/c4/c5 select the other BASELINE configs (c2: 256
networks per GPU, weak scaling; c5: the 16,384-network FE2 macro step in
contiguous shards).

Printed JSON (rank 0): value = networks/s for the whole job (device-resident
batch: kernel + result gather), e2e = the same through the public API
(solve_batch: upload of the packed batch from pinned host memory, solve,
download, unpermute) timed over the same number of steps, the roofline of
the relaxation kernel against the measured HBM copy bandwidth using the
algorithmic bytes B_iter = 48 N + 48 nf + 24 M per network-iteration
(SURVEY.md 8d), a bench-side parity spot check of the timed batch against
the real reference's golden records (tests/golden), and a CPU baseline: the
reference's own solver (fibrelax.dynamic_relaxation_solve from baseline/_ref
when installed, else the bit-exact oracle port) on this host's cores.
"""

from __future__ import annotations

import argparse
import hashlib
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
TOTAL = {"c1": 1, "c3": 1024, "c4": 1024, "c5": C5_TOTAL}
SCALING = {"c1": "weak", "c2": "weak", "c3": "strong", "c4": "strong", "c5": "strong"}
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def shard_indices(name: str, rank: int, world: int) -> list[int]:
    """Network indices a rank solves (through the product's
    distributed.shard_indices): c2 is weak-scaled (256 per GPU), c3/c4 are
    strided shards of 1,024 (iteration counts vary by size / load), c5 is
    split into contiguous shards of the FE2 macro step's 16,384 networks."""
    from paper_2305_07030_b200.distributed import shard_indices as shard
    if name == "c1":
        return [0]
    if name == "c2":
        return list(range(rank * 256, (rank + 1) * 256))
    if name in ("c3", "c4"):
        return [int(i) for i in shard(1024, rank, world, "strided")]
    if name == "c5":
        return [int(i) for i in shard(C5_TOTAL, rank, world, "contiguous")]
    raise SystemExit(f"unknown --config {name}")


def c5_gradient(i: int) -> np.ndarray:
    """Random macro deformation gradient of FE2 network i."""
    rng = np.random.default_rng(10 ** 6 + i)
    diag = rng.uniform(0.0, 0.1, 3)
    off = rng.uniform(-0.05, 0.05, (3, 3))
    np.fill_diagonal(off, 0.0)
    return np.eye(3) + np.diag(diag) + off


def network_spec(name: str, i: int):
    """(lattice args, F) of network i of a workload (same recipe on the GPU
    and the CPU arm, and in tests/golden/make_golden.py)."""
    if name == "c1":
        return (7, 7, 8, 0.3, 0), UNIAX
    if name == "c2":
        return (15, 15, 15, 0.3, i), UNIAX
    if name == "c3":
        return (32, 32, 32, 0.3, i), UNIAX
    if name == "c4":
        n = 7 + (i % 26)
        return (n, n, n, 0.3, i), [UNIAX, BIAX, SHEAR][i % 3]
    return (15, 15, 15, 0.3, i), c5_gradient(i)


def describe(name: str, n_here: int) -> str:
    return {
        "c1": "c1: 1 x generate_lattice(7,7,8,0.3,seed=0), uniaxial F=diag(1.1,1,1)",
        "c2": f"c2: {n_here} x generate_lattice(15,15,15,0.3,seed=s) per GPU (10,125 DOF, 9,450 fibers), "
              "uniaxial F=diag(1.1,1,1)",
        "c3": f"c3: 1024 x generate_lattice(32,32,32,0.3,seed=s) (98,304 DOF, 95,232 fibers), uniaxial "
              f"F=diag(1.1,1,1), strided shards ({n_here} on this GPU)",
        "c4": f"c4: 1024 heterogeneous lattices n=7+(i mod 26) (1k-100k DOF), loads uniax/biax/shear by "
              f"i mod 3, strided shards ({n_here} on this GPU)",
        "c5": f"c5: FE2 macro-step, {C5_TOTAL} x 15^3 networks, random F, contiguous shards ({n_here} on this GPU)",
    }[name]


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

_REF = {}


def reference_module():
    """The reference's own package (fibrelax 0.1.0, pip-installed from
    /root/reference/pkg into baseline/_ref) if it is present on this host,
    else None (the CPU arm then times the bit-exact oracle port)."""
    if "mod" not in _REF:
        _REF["mod"] = None
        if os.path.isdir(os.path.join(REF_PATH, "fibrelax")):
            sys.path.insert(0, REF_PATH)
            try:
                import fibrelax  # noqa: F401
                _REF["mod"] = sys.modules["fibrelax"]
            except ImportError:
                _REF["mod"] = None
    return _REF["mod"]


def _cpu_solve(args):
    """One network of a workload through the reference's public solver (or
    the oracle port); returns (seconds, iterations, nodes).  Network
    generation is outside the timed call, setup inside."""
    cfgname, i = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ref = reference_module()
    if cfgname == "warm":
        lat, F = (3, 3, 3, 0.3, 0), UNIAX
    else:
        lat, F = network_spec(cfgname, i)
    if ref is not None:
        net = ref.generate_lattice(*lat)
        t0 = time.perf_counter()
        r = ref.dynamic_relaxation_solve(net, ref.AffineBC(F), ref.SolverConfig())
        return time.perf_counter() - t0, r.iters, net.n_nodes
    import paper_2305_07030_b200 as frb
    from oracle import frb_oracle as orc
    net = frb.generate_lattice(*lat)
    t0 = time.perf_counter()
    r = orc.solve(net, F, frb.SolverConfig())
    return time.perf_counter() - t0, r.iters, net.n_nodes


def cpu_arm_name() -> tuple[str, str]:
    if reference_module() is not None:
        return "reference", "fibrelax.dynamic_relaxation_solve (the reference package, baseline/_ref)"
    return "port", "oracle/frb_oracle.py (bit-exact numpy restatement of fibrelax; reference not installed)"


class CpuPool:
    """A fork pool of one worker per host core (OPENBLAS_NUM_THREADS=1), warmed
    by one tiny solve per worker (imports, allocator)."""

    def __init__(self, cores: int):
        import multiprocessing as mp
        reference_module()  # imported before the fork: workers inherit it
        self.cores = cores
        self.pool = mp.get_context("fork").Pool(cores)
        self.pool.map(_cpu_solve, [("warm", 0)] * cores)

    def step(self, config: str, k: int) -> dict:
        """Step k: the workload's networks k*cores .. (k+1)*cores - 1 (mod its
        size), one per core."""
        n_total = TOTAL.get(config, 256)
        jobs = [(config, (k * self.cores + j) % n_total) for j in range(self.cores)]
        t0 = time.perf_counter()
        out = self.pool.map(_cpu_solve, jobs, chunksize=1)
        wall = time.perf_counter() - t0
        return dict(networks=len(jobs), wall_s=wall, cpu_s=sum(t for t, _, _ in out),
                    node_updates=sum(it * n for _, it, n in out), first=jobs[0][1], last=jobs[-1][1])

    def close(self):
        self.pool.terminate()


def summarize_cpu(config: str, samples: list, cores: int) -> dict:
    nets = sum(s["networks"] for s in samples)
    wall = sum(s["wall_s"] for s in samples)
    kind, arm = cpu_arm_name()
    per_net = sum(s["cpu_s"] for s in samples) / nets
    return {
        "value": nets / wall, "unit": "networks/s", "cores": cores, "kind": kind,
        "sample": (f"{nets} networks of the {config} workload ({len(samples)} step(s) of {cores}, one network "
                   f"per core per step, networks {samples[0]['first']}..{samples[-1]['last']}); {wall:.1f} s wall, "
                   f"{per_net:.2f} s per network per core; {arm}; OPENBLAS_NUM_THREADS=1 fork pool"),
        "single_core": {"value": 1.0 / per_net, "unit": "networks/s",
                        "note": "mean per-network solve time of the same sample on one core"},
        "node_updates_per_s": sum(s["node_updates"] for s in samples) / wall,
    }


def run_reference_arm(args, rank: int):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    pool = CpuPool(cores)
    try:
        for _ in range(args.warmup):  # light warm-ups: one tiny solve per worker
            pool.pool.map(_cpu_solve, [("warm", 0)] * cores)
        samples = [pool.step(args.config, k) for k in range(args.steps)]
    finally:
        pool.close()
    cb = summarize_cpu(args.config, samples, cores)
    n_here = len(shard_indices(args.config, 0, 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "networks/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(s["wall_s"] for s in samples),
        "higher_is_better": True, "scaling": SCALING[args.config], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generate_lattice inputs)",
        "config": {"workload": describe(args.config, n_here), "arm": cpu_arm_name()[1],
                   "per_step": f"{cores} networks (one per host core)"},
        "node_updates_per_s": cb["node_updates_per_s"],
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "networks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- parity spot check

def spot_check(config: str, indices: list, results) -> dict:
    """Networks of the timed batch that have a golden record of the real
    reference (tests/golden): iterations, residual and u must match exactly.
    results: the public-API SolveResults of this rank's shard."""
    gdir = os.path.join(ROOT, "tests", "golden")
    checks = []
    big = {}
    if os.path.exists(os.path.join(gdir, "big_index.json")):
        with open(os.path.join(gdir, "big_index.json")) as fh:
            big = json.load(fh)
    pos = {g: k for k, g in enumerate(indices)}
    for name, rec in big.items():
        lat = tuple(rec["lattice"])
        for g, k in pos.items():
            spec, F = network_spec(config, g)
            if tuple(spec) == (lat[0], lat[1], lat[2], lat[3], lat[4]) and np.array_equal(F, np.array(rec["F"])):
                r = results[k]
                ok = (r.iters == rec["iters"] and r.final_residual == float.fromhex(rec["final_residual"])
                      and hashlib.sha256(np.ascontiguousarray(r.u, "<f8").tobytes()).hexdigest() == rec["u_sha256"])
                checks.append({"network": g, "golden": name, "iters": r.iters, "bit_equal": bool(ok)})
    if config in ("c1", "c2") and 0 in pos:
        name = "c1_7x7x8_uniax" if config == "c1" else "c2_15cube_seed0"
        z = np.load(os.path.join(gdir, f"{name}.npz"))
        r = results[pos[0]]
        ok = r.iters == int(z["iters"]) and np.array_equal(r.u, z["u"]) and r.final_residual == float(z["final_residual"])
        checks.append({"network": 0, "golden": name, "iters": r.iters, "bit_equal": bool(ok)})
    return {"checked": len(checks), "all_bit_equal": all(c["bit_equal"] for c in checks), "cases": checks}


# --------------------------------------------------------------------- GPU arm

def layout_of(name: str, world: int, limit: int | None):
    """(n_total, shard mode) of a workload at `world` ranks."""
    n_total, mode = {"c1": (world, "contiguous"), "c2": (256 * world, "contiguous"), "c3": (1024, "strided"),
                     "c4": (1024, "strided"), "c5": (C5_TOTAL, "contiguous")}[name]
    if limit is not None:
        n_total = min(n_total, limit * world)
    return n_total, mode


def traffic_per_launch(config: str, n_networks: int):
    """DRAM bytes (read + write) of the relaxation kernel from the committed
    ncu --set full capture of this config (profiles/traffic.json), scaled to
    this launch's network count; None when no capture exists."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as fh:
        t = json.load(fh).get(config)
    if not isinstance(t, dict):
        return None, None
    return t["bytes"] * n_networks / t["networks"], t["source"]


def pipe_utilisation(config: str):
    """FP64-pipe, issue and warp occupancy percentages of the relaxation
    kernel from the same committed ncu capture (the compute side of the
    roofline: the streaming fraction is an effective bandwidth)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        t = json.load(fh).get(config)
    if not isinstance(t, dict) or "fp64_pipe_pct" not in t:
        return None
    return {k: t[k] for k in ("fp64_pipe_pct", "issue_active_pct", "warps_active_pct")} | {"source": t["source"].split(":")[0] + " (ncu --set full)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--limit", type=int, default=None, help="networks per rank (ncu captures)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (profiling runs)")
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
    from paper_2305_07030_b200.distributed import ShardedBatch, decode_records

    # FRB_BENCH_GPUS_PER_NODE=1 with FRB_DIST_BACKEND=gloo runs several ranks
    # on one GPU (a functional check of the multi-rank path; not a measurement)
    local_gpu = local % int(os.environ.get("FRB_BENCH_GPUS_PER_NODE", str(max(1, torch.cuda.device_count()))))
    torch.cuda.set_device(local_gpu)
    dev = torch.device("cuda", local_gpu)
    if world > 1:
        backend = os.environ.get("FRB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def make(i):
        lat, F = network_spec(args.config, i)
        return frb.generate_lattice(*lat), frb.AffineBC(F)

    n_total, mode = layout_of(args.config, world, args.limit)
    t0 = time.perf_counter()
    sb = ShardedBatch(make, n_total, mode, device=dev, rank=rank, world=world)
    build_s = time.perf_counter() - t0   # generation + host setup + upload
    batch = sb.batch
    batch.pin()
    cfg = frb.SolverConfig()
    strategy = frb.TeamBatched(team_size=args.team_size)
    launch = sb.prepare(cfg, strategy)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    P = batch.n_problems
    stream = torch.cuda.current_stream(dev)
    gathered = [None]

    def step(ev=None):
        flush.zero_()
        if ev is not None:
            ev[0].record(stream)
        launch.run(stream)
        if ev is not None:
            ev[1].record(stream)
        if world > 1:  # every network's result record to every rank (NCCL, no host sync)
            gathered[0] = sb.gather(launch.out.results)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_gpu) as clocks:
        torch.cuda.synchronize(dev)
        t_start.record(stream)
        for k in range(args.steps):
            step(kev[k])
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    elapsed = t_start.elapsed_time(t_end) / 1e3
    kern = [a.elapsed_time(b) / 1e3 for a, b in kev]

    rec = launch.out.host_results()
    iters = rec["iters"].astype(np.int64)
    Ns = np.array([p.n_nodes for p in batch.problems], dtype=np.int64)
    nfs = np.array([3 * p.n_free_nodes for p in batch.problems], dtype=np.int64)
    Ms = np.array([p.network.n_elements for p in batch.problems], dtype=np.int64)
    alg_bytes = float((iters * (48 * Ns + 48 * nfs + 24 * Ms)).sum())
    node_updates = float((iters * Ns).sum())
    converged_local = int((rec["status"] == 0).sum())
    if world > 1:
        t = torch.tensor([elapsed, statistics.mean(kern)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, kern_mean = t.tolist()
        s = torch.tensor([alg_bytes, node_updates, float(converged_local)], dtype=torch.float64, device=dev)
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        alg_all, node_updates_all, converged_all = s.tolist()
        all_rec = decode_records(gathered[0])
        assert len(all_rec) == n_total and (all_rec["status"] == 0).all(), "not every network converged"
    else:
        kern_mean = statistics.mean(kern)
        alg_all, node_updates_all, converged_all = alg_bytes, node_updates, converged_local
    assert converged_all == n_total, "not every network converged"

    # ---- e2e through the public API: pinned host batch -> results ----
    e2e = None
    spot = None
    if not args.no_e2e:
        def e2e_step():
            dres = batch.to_device(dev).solve(cfg, strategy)
            out = fb.results_to_solve_results(batch, dres)
            if world > 1:
                sb.gather(dres.results)
            return out
        for _ in range(max(2, min(args.warmup, 3))):  # steady state: two result buffers in the host cache
            res = e2e_step()
        res = None
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        te = time.perf_counter()
        for _ in range(args.steps):
            res = e2e_step()
        torch.cuda.synchronize(dev)
        e2e_s = (time.perf_counter() - te) / args.steps
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = t.item()
        h2d = sum(a.nbytes for a in batch.arrays.values())
        d2h = 3 * int(batch.node_base[-1]) * 8 + P * nat_result_bytes()
        assert all(r.converged for r in res)
        e2e = {"value": n_total / e2e_s, "unit": "networks/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "note": "solve_batch path per step: upload of the packed batch from pinned memory, solve, "
                       "download of u and the result records, unpermute to the original node order; "
                       "host setup (pack_batch) excluded, reported as setup_s_per_rank"}
        if rank == 0:
            spot = spot_check(args.config, sb.indices.tolist(), res)
            assert spot["all_bit_equal"], f"parity spot check failed: {spot}"

    ms_per_step = 1e3 * elapsed / args.steps
    value = n_total / (elapsed / args.steps)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as fh:
            peak, peak_src = float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    achieved = alg_all / world / kern_mean / 1e9
    traffic, traffic_src = traffic_per_launch(args.config, P)

    line = {
        "metric": METRIC, "value": value, "unit": "networks/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": SCALING[args.config], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generate_lattice jittered lattices, same generator as the reference)",
        "config": {"workload": describe(args.config, P), "networks_total": n_total, "networks_per_gpu": P,
                   "parallelism": f"shard{world} ({mode})",
                   "l2": "flushed (256 MiB memset before every step)",
                   "setup_s_per_rank": round(batch.setup_s, 3),
                   "build_s_per_rank": round(build_s, 3),
                   "cta_threads": launch.threads,
                   "clusters": sorted({int(c) for c in batch.desc["cluster"]})},
        "node_updates_per_s": node_updates_all / (elapsed / args.steps),
        "iters_mean": float(iters.mean()),
        "e2e": e2e,
        "gpu_launches": args.steps * launch.kernel_launches,  # frb_solve_launches() per step
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src, "compute": pipe_utilisation(args.config),
                     "kernel": "frb_relax_kernel", "kernel_ms": 1e3 * kern_mean,
                     "alg_bytes_per_launch": alg_all / world,
                     "alg_bytes_model": "sum over networks of iters * (48 N + 48 nf + 24 M) (SURVEY.md 8d)"},
        "parity_spot_check": spot,
        "clocks": clocks.summary(),
        "kernel_ms_per_step": [round(1e3 * k, 3) for k in kern],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        pool = CpuPool(cores)
        try:
            line["cpu_baseline"] = summarize_cpu(args.config, [pool.step(args.config, 0)], cores)
        finally:
            pool.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def nat_result_bytes() -> int:
    from paper_2305_07030_b200 import _native as nat
    return nat.RESULT_DTYPE.itemsize


if __name__ == "__main__":
    main()
