"""The spec'd bench module: self-speedup arithmetic,
summaries, CSV round trip (CPU) and a small timed grid on the B200."""

import random

import pytest

from paper_2305_07030_b200 import benchmark as bm


def test_self_speedup_examples():
    assert bm.self_speedup(1.0, 2.0, 8) == 4.0
    assert bm.self_speedup(0.7, 0.7 * 5, 5) == pytest.approx(1.0)
    assert bm.self_speedup(0.5, 0.5, 8) == 8.0
    with pytest.raises(ValueError):
        bm.self_speedup(0.0, 1.0, 2)
    with pytest.raises(ValueError):
        bm.self_speedup(1.0, 1.0, 0)


def _records():
    R = bm.BenchRecord
    return [R("team", 300, 1, 0, 1.0), R("team", 300, 1, 1, 1.1), R("team", 300, 1, 2, 0.9),
            R("team", 300, 4, 0, 1.0), R("naive", 300, 4, 0, 5.0), R("naive", 300, 1, 0, 1.25)]


def test_summarize_means_speedups_and_order_invariance():
    rows = bm.summarize(_records())
    by = {(r.strategy, r.n_problems): r for r in rows}
    assert by[("team", 1)].mean_seconds == pytest.approx(1.0)     # mean of {1.0, 1.1, 0.9}
    assert by[("team", 1)].self_speedup == pytest.approx(1.0)
    assert by[("team", 4)].self_speedup == pytest.approx(4.0)
    assert by[("team", 4)].speedup_over_naive == pytest.approx(5.0)
    assert by[("naive", 4)].self_speedup == pytest.approx(1.0)
    shuffled = _records()
    random.Random(3).shuffle(shuffled)
    assert bm.summarize(shuffled) == rows
    only = bm.summarize([bm.BenchRecord("team", 9, 2, 0, 1.0)])  # no N = 1 baseline: empty field
    assert only[0].self_speedup is None


def test_csv_round_trip_and_headers():
    recs = _records()
    raw = bm.emit_csv(recs, bm.RAW_HEADER)
    assert raw.splitlines()[0] == "strategy,n_dofs,n_problems,rep,wall_seconds"
    assert bm.parse_csv(raw, bm.BenchRecord) == recs
    rows = bm.summarize(recs)
    summ = bm.emit_csv(rows, bm.SUMMARY_HEADER)
    assert summ.splitlines()[0] == "strategy,n_dofs,n_problems,mean_seconds,self_speedup,speedup_over_naive"
    assert bm.parse_csv(summ, bm.SpeedupRow) == rows


def test_record_validation():
    with pytest.raises(ValueError):
        bm.BenchRecord("team", 1, 1, 0, 0.0)


@pytest.mark.gpu
def test_team_batching_beats_serial_on_b200(cuda_device):
    """Fig. 3 vs Fig. 2 on the B200: the team kernel's runtime is nearly
    flat in N (self-speedup well above 1), the single-team serial strategy
    grows linearly (self-speedup ~ 1)."""
    recs = bm.run_benchmark([(6, 6, 6)], [1, 16], strategies=("team", "serial"), reps=2)
    assert len(recs) == 2 * 2 * 2
    rows = {(r.strategy, r.n_problems): r for r in bm.summarize(recs)}
    assert rows[("team", 16)].self_speedup > 4.0
    assert 0.5 < rows[("serial", 16)].self_speedup < 2.0
