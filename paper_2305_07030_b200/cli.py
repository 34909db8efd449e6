"""Command line (the spec's ``cli`` module, reference ``SPEC.md:457-512``; the
reference's pyproject names a ``fibrelax`` script whose module is absent,
``pyproject.toml:20-21``).

    python -m paper_2305_07030_b200 gen   --lattice 3,3,3 [--jitter 0.3] [--seed 0] -o net.txt
    python -m paper_2305_07030_b200 solve --network net.txt --deform f11 f12 ... f33
                                          [--tol 1e-6] [--max-iters N] [--strategy team|serial|naive]
                                          [--teams T] [--team-size S] [-o result.json]
    python -m paper_2305_07030_b200 bench --sizes 4,4,4 6,6,6 --counts 1 2 4 [--strategies team naive]
                                          [--reps 3] [--team-size 512] -o raw.csv   (+ raw.summary.csv)
    python -m paper_2305_07030_b200 plot  --input raw.summary.csv -o speedup.svg

Exit codes: 0 success, 1 usage / IO / validation error, 2 a
solve that did not converge.  Solves run on the B200 (no CPU fallback).
"""

from __future__ import annotations

import argparse
import math
import sys

import numpy as np

EXIT_OK, EXIT_ERROR, EXIT_NOT_CONVERGED = 0, 1, 2


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # unknown flag / bad value -> exit 1
        raise UsageError(message)


def _lattice(text: str) -> tuple[int, int, int]:
    try:
        nx, ny, nz = (int(x) for x in text.split(","))
    except ValueError:
        raise UsageError(f"--lattice wants nx,ny,nz, got {text!r}") from None
    if min(nx, ny, nz) < 2:
        raise UsageError(f"--lattice counts must be >= 2, got {text}")
    return nx, ny, nz


def cmd_gen(a) -> int:
    from .network import generate_lattice, save_network
    net = generate_lattice(*_lattice(a.lattice), a.jitter, a.seed)
    with open(a.output, "w") as fh:
        fh.write(save_network(net))
    return EXIT_OK


def _strategy(a):
    from .batch import NaiveLoop, SerialReference, TeamBatched
    if a.strategy == "team":
        return TeamBatched(teams=a.teams, team_size=a.team_size)
    if a.strategy == "serial":
        return SerialReference()
    return NaiveLoop()


def cmd_solve(a) -> int:
    from .batch import pack_batch, solve_batch
    from .microsolver import SolverConfig
    from .network import AffineBC, load_network
    with open(a.network) as fh:
        net = load_network(fh)
    F = np.array(a.deform, dtype=np.float64).reshape(3, 3)
    kw = {}
    if a.tol is not None:
        kw["tol_rel"] = a.tol
    if a.max_iters is not None:
        kw["max_iters"] = a.max_iters
    res = solve_batch(pack_batch([net], [AffineBC(F)]), strategy=_strategy(a), config=SolverConfig(**kw))[0]
    text = res.to_json()
    if a.output:
        with open(a.output, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text + "\n")
    return EXIT_OK if res.converged else EXIT_NOT_CONVERGED


def cmd_bench(a) -> int:
    from .benchmark import RAW_HEADER, SUMMARY_HEADER, emit_csv, run_benchmark, summarize
    sizes = [_lattice(s) for s in a.sizes]
    records = run_benchmark(sizes, a.counts, strategies=a.strategies, reps=a.reps, team_size=a.team_size)
    with open(a.output, "w") as fh:
        fh.write(emit_csv(records, RAW_HEADER))
    base = a.output[:-4] if a.output.endswith(".csv") else a.output
    with open(base + ".summary.csv", "w") as fh:
        fh.write(emit_csv(summarize(records), SUMMARY_HEADER))
    return EXIT_OK


def render_svg(rows, metric: str = "self_speedup") -> str:
    """Deterministic SVG line chart: log2-x = concurrent sub-problems, y =
    `metric`, one polyline per (strategy, n_dofs) (the paper's Figs. 2-4)."""
    W, H, M = 640, 400, 60
    series: dict[tuple[str, int], list[tuple[int, float]]] = {}
    for r in rows:
        y = getattr(r, metric)
        if y is not None:
            series.setdefault((r.strategy, r.n_dofs), []).append((r.n_problems, float(y)))
    xs = [n for pts in series.values() for n, _ in pts] or [1]
    ys = [y for pts in series.values() for _, y in pts] or [1.0]
    x0, x1 = math.log2(min(xs)), math.log2(max(xs))
    y1 = max(ys) * 1.1 if max(ys) > 0 else 1.0
    sx = lambda n: M + (W - 2 * M) * ((math.log2(n) - x0) / (x1 - x0) if x1 > x0 else 0.5)  # noqa: E731
    sy = lambda y: H - M - (H - 2 * M) * (y / y1)  # noqa: E731
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" viewBox="0 0 {W} {H}">',
           f'<line x1="{M}" y1="{H - M}" x2="{W - M}" y2="{H - M}" stroke="black"/>',
           f'<line x1="{M}" y1="{M}" x2="{M}" y2="{H - M}" stroke="black"/>',
           f'<text x="{W / 2:.1f}" y="{H - 15}" text-anchor="middle">concurrent sub-problems (log2)</text>',
           f'<text x="15" y="{H / 2:.1f}" transform="rotate(-90 15 {H / 2:.1f})" text-anchor="middle">'
           f'{metric}</text>']
    colors = ["#1f77b4", "#d62728", "#2ca02c", "#9467bd", "#ff7f0e", "#8c564b"]
    for k, key in enumerate(sorted(series)):
        pts = sorted(series[key])
        path = " ".join(f"{sx(n):.2f},{sy(y):.2f}" for n, y in pts)
        out.append(f'<polyline fill="none" stroke="{colors[k % len(colors)]}" points="{path}">'
                   f'<title>{key[0]} {key[1]} DOF</title></polyline>')
    out.append("</svg>")
    return "\n".join(out) + "\n"


def cmd_plot(a) -> int:
    from .benchmark import SpeedupRow, parse_csv
    with open(a.input) as fh:
        rows = parse_csv(fh.read(), SpeedupRow)
    with open(a.output, "w") as fh:
        fh.write(render_svg(rows, a.metric))
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="paper_2305_07030_b200", description="B200 batched dynamic relaxation of fiber networks")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    g = sub.add_parser("gen", help="write a jittered lattice network")
    g.add_argument("--lattice", required=True)
    g.add_argument("--jitter", type=float, default=0.3)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("-o", "--output", required=True)
    s = sub.add_parser("solve", help="solve one network, write the SolveResult JSON")
    s.add_argument("--network", required=True)
    s.add_argument("--deform", type=float, nargs=9, required=True, metavar="F")
    s.add_argument("--tol", type=float)
    s.add_argument("--max-iters", type=int)
    s.add_argument("--strategy", choices=["team", "serial", "naive"], default="team")
    s.add_argument("--teams", type=int)
    s.add_argument("--team-size", type=int)
    s.add_argument("-o", "--output")
    b = sub.add_parser("bench", help="self-speedup benchmark, raw + summary CSV")
    b.add_argument("--sizes", nargs="+", required=True)
    b.add_argument("--counts", type=int, nargs="+", required=True)
    b.add_argument("--strategies", nargs="+", choices=["team", "serial", "naive"], default=["team"])
    b.add_argument("--reps", type=int, default=3)
    b.add_argument("--team-size", type=int)
    b.add_argument("-o", "--output", required=True)
    q = sub.add_parser("plot", help="SVG of a summary CSV")
    q.add_argument("--input", required=True)
    q.add_argument("--metric", choices=["self_speedup", "speedup_over_naive"], default="self_speedup")
    q.add_argument("-o", "--output", required=True)
    return p


def main(argv=None) -> int:
    try:
        a = build_parser().parse_args(argv)
        return {"gen": cmd_gen, "solve": cmd_solve, "bench": cmd_bench, "plot": cmd_plot}[a.cmd](a)
    except UsageError as e:
        sys.stderr.write(f"usage error: {e}\n")
        return EXIT_ERROR
    except (OSError, ValueError, RuntimeError) as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
