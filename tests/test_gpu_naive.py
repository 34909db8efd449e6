"""NaiveLoop (one kernel launch per Fig. 1 line) on the B200:
bit-identical to the team kernel and to the reference's golden vectors, and
slower than the team kernel on a batch (the paper's Fig. 4 trend,
SPEC.md:522-523)."""

import numpy as np
import pytest

import golden_cases as gc
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb

pytestmark = pytest.mark.gpu

CASES = ["c1_7x7x8_uniax", "lat5_shear", "lat5_ramp10", "lat6_fixed1", "lat6_maxiter", "lat4_identity",
         "lat2_allfixed", "lat4x5x6_tolabs", "random90_fixed", "lat6_general_F"]


@pytest.mark.parametrize("name", CASES)
def test_naive_matches_reference(cuda_device, name):
    case = gc.load(name)
    batch = frb.pack_batch([case.network], [frb.AffineBC(case.F)])
    r = fb.results_to_solve_results(batch, batch.to_device().solve(case.cfg, frb.NaiveLoop()))[0]
    d = case.data
    assert r.iters == int(d["iters"]) and r.converged == bool(d["converged"])
    assert np.array_equal(r.u, d["u"])
    assert r.final_residual == float(d["final_residual"])
    scale = max(np.abs(d["avg_stress"]).max(), 1e-300)
    assert np.abs(r.avg_stress - d["avg_stress"]).max() <= 1e-13 * scale


def test_naive_equals_team_on_a_batch(cuda_device):
    nets = [frb.generate_lattice(6, 6, 7, 0.3, s) for s in range(3)] + [gc.load("random60").network]
    Fs = [np.diag([1.1, 1, 1]), np.diag([1.1, 1.1, 1]), np.eye(3) + 0.2 * np.outer([1, 0, 0], [0, 1, 0]),
          np.diag([1.1, 1, 1])]
    batch = frb.pack_batch(nets, [frb.AffineBC(F) for F in Fs])
    team = frb.solve_batch(batch)
    naive = frb.solve_batch(batch, strategy=frb.NaiveLoop())
    for a, b in zip(team, naive):
        assert a.iters == b.iters and np.array_equal(a.u, b.u) and np.array_equal(a.avg_stress, b.avg_stress)


def test_naive_singular_element(cuda_device):
    case = gc.load("bar_singular")
    with pytest.raises(frb.SingularElementError, match="element 0"):
        frb.solve_batch(frb.pack_batch([case.network], [frb.AffineBC(case.F)]), strategy=frb.NaiveLoop())


def test_team_beats_naive_on_a_batch(cuda_device):
    """Fig. 4 trend: on a batch of 16 copies the team kernel is faster than
    per-operation dispatch (speedup_over_naive > 1)."""
    from paper_2305_07030_b200.benchmark import run_benchmark, summarize
    rows = summarize(run_benchmark([(6, 6, 6)], [1, 16], strategies=("naive", "team"), reps=1))
    by = {(r.strategy, r.n_problems): r for r in rows}
    assert by[("team", 16)].speedup_over_naive > 1.0
    assert by[("naive", 16)].self_speedup < 1.5   # strictly sequential: runtime grows ~linearly
