"""Self-speedup benchmark of batched solves (the spec'd ``bench`` module,
reference ``SPEC.md:396-455``; the reference package has no bench code).

It reproduces the paper's measurement (``PAPER.md:84-114``, Figs. 2-4): the
runtime of N concurrent copies of one sub-problem against one copy,
``self_speedup = N * t1 / tN`` -- 1 means runtime grows linearly with N (no
batching benefit), N means a flat runtime.  On the B200 the strategies are
``TeamBatched`` (one persistent kernel, a work queue, one CTA cluster per
network -- the paper's team kernel), ``SerialReference`` (the same kernel
with a single team: problems strictly one after another) and ``NaiveLoop``
(the paper's naive baseline: one kernel launch per line of the Fig. 1 loop,
problems in sequence, the host checking convergence every iteration), so
``speedup_over_naive`` reproduces the team-vs-naive comparison of Fig. 4.

Timing boundary: wall clock of ``solve_batch`` including batch
packing, host->device upload, the solve and the download of the results;
network generation is excluded.  One discarded warm-up run per cell, then the
mean of ``reps`` runs (the paper's "mean of three analysis runs").
"""

from __future__ import annotations

import csv
import io
import time
from dataclasses import dataclass, fields
from typing import Iterable, Sequence

import numpy as np

RAW_HEADER = ["strategy", "n_dofs", "n_problems", "rep", "wall_seconds"]
SUMMARY_HEADER = ["strategy", "n_dofs", "n_problems", "mean_seconds", "self_speedup", "speedup_over_naive"]
NAIVE = "naive"


@dataclass(frozen=True)
class BenchRecord:
    strategy: str
    n_dofs: int
    n_problems: int
    rep: int
    wall_seconds: float

    def __post_init__(self):
        if not self.wall_seconds > 0:
            raise ValueError("wall_seconds must be > 0")


@dataclass(frozen=True)
class SpeedupRow:
    strategy: str
    n_dofs: int
    n_problems: int
    mean_seconds: float
    self_speedup: float | None
    speedup_over_naive: float | None


def self_speedup(t1: float, tN: float, N: int) -> float:
    """N * t1 / tN."""
    if not (t1 > 0 and tN > 0) or N < 1:
        raise ValueError("self_speedup needs t1 > 0, tN > 0 and N >= 1")
    return t1 / (tN / N)


def _strategy(name: str, team_size: int | None):
    from .batch import NaiveLoop, SerialReference, TeamBatched
    if name == "team":
        return TeamBatched(team_size=team_size)
    if name == "serial":
        return SerialReference()
    if name == NAIVE:
        return NaiveLoop()
    raise ValueError(f"unknown strategy {name!r} (team, serial, naive)")


def run_benchmark(sizes: Sequence[tuple[int, int, int]], counts: Sequence[int],
                  strategies: Sequence[str] = ("team",), reps: int = 3, config=None, load=None,
                  seed: int = 0, team_size: int | None = None) -> list[BenchRecord]:
    """Time solve_batch over a grid of lattice sizes x batch counts x
    strategies.  Every cell solves N identical copies of
    generate_lattice(*size, 0.3, seed) under `load` (default uniaxial
    F = diag(1.1, 1, 1)); a non-converged cell raises."""
    from .batch import pack_batch, results_to_solve_results
    from .microsolver import SolverConfig
    from .network import AffineBC, generate_lattice
    import torch
    if reps < 1:
        raise ValueError("reps must be >= 1")
    cfg = config or SolverConfig()
    F = np.diag([1.1, 1.0, 1.0]) if load is None else np.asarray(load, dtype=np.float64)
    records = []
    for size in sizes:
        net = generate_lattice(*size, 0.3, seed)
        n_dofs = 3 * net.n_nodes
        for name in strategies:
            strat = _strategy(name, team_size)
            for N in counts:
                nets, bcs = [net] * N, [AffineBC(F)] * N

                def once():
                    t0 = time.perf_counter()
                    batch = pack_batch(nets, bcs)
                    res = results_to_solve_results(batch, batch.to_device().solve(cfg, strat))
                    torch.cuda.synchronize()
                    dt = time.perf_counter() - t0
                    if not all(r.converged for r in res):
                        raise RuntimeError(f"non-converged cell {name} {size} N={N}")
                    return dt

                once()  # warm-up, discarded
                for rep in range(reps):
                    records.append(BenchRecord(name, n_dofs, N, rep, once()))
    return records


def summarize(records: Iterable[BenchRecord]) -> list[SpeedupRow]:
    """Mean over reps, self-speedup against the same strategy's N = 1 mean,
    speedup over the naive strategy where a naive cell exists.
    Independent of record order."""
    cells: dict[tuple[str, int, int], list[float]] = {}
    for r in records:
        cells.setdefault((r.strategy, r.n_dofs, r.n_problems), []).append(r.wall_seconds)
    mean = {k: float(np.mean(sorted(v))) for k, v in cells.items()}
    rows = []
    for (s, d, n) in sorted(mean):
        m = mean[(s, d, n)]
        t1 = mean.get((s, d, 1))
        naive = mean.get((NAIVE, d, n))
        rows.append(SpeedupRow(s, d, n, m, None if t1 is None else self_speedup(t1, m, n),
                               None if naive is None else naive / m))
    return rows


def _fmt(x) -> str:
    if x is None:
        return ""
    return repr(x) if isinstance(x, float) else str(x)


def emit_csv(rows, header: Sequence[str]) -> str:
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(header)
    for r in rows:
        w.writerow([_fmt(getattr(r, h)) for h in header])
    return out.getvalue()


def parse_csv(text: str, kind: type) -> list:
    """Inverse of emit_csv for BenchRecord or SpeedupRow."""
    types = {f.name: f.type for f in fields(kind)}
    rd = csv.reader(io.StringIO(text))
    header = next(rd)
    out = []
    for row in rd:
        vals = {}
        for h, v in zip(header, row):
            t = types[h]
            if v == "":
                vals[h] = None
            elif t in ("int", int):
                vals[h] = int(v)
            elif t in ("str", str):
                vals[h] = v
            else:
                vals[h] = float(v)
        out.append(kind(**vals))
    return out
