"""Full-length parity on the large BASELINE configs (B200).

Golden records in ``tests/golden/big_index.json`` were produced by running the
REAL reference (``make_golden.py --big``: ``fibrelax`` 0.1.0,
``dynamic_relaxation_solve`` path, microsolver.py:567-574) on:

* C3: generate_lattice(32,32,32,0.3,0), uniaxial (2,519 iterations) -- the
  16-CTA cluster path with f_prev in global memory;
* c4 recipe networks: i=77 (32^3 shear, 6,407 iterations, 16 CTAs), i=71
  (26^3 shear, 8 CTAs), i=13 (20^3 biaxial);
* a 24^3 shear network (8-CTA cluster, 3,777 iterations);
* c5 networks 0 and 1 (15^3 under the FE2 random F).

Every network runs to convergence through the public batch API; u and f are
compared bit for bit through SHA-256 digests of their exact bytes (original
node order, like the reference), residual and r_ref bit for bit, iterations
and convergence exactly, sigma within 1e-13 of max|sigma|.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2305_07030_b200 as frb

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
BIG = json.load(open(os.path.join(HERE, "golden", "big_index.json")))
SAMPLE_STRIDE = 97


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def _case(name):
    rec = BIG[name]
    net = frb.generate_lattice(*rec["lattice"][:3], float(rec["lattice"][3]), int(rec["lattice"][4]))
    return net, np.array(rec["F"], dtype=np.float64), rec


def _check(name, rec, r, f):
    assert r.iters == rec["iters"], f"{name}: iters {r.iters} != {rec['iters']}"
    assert r.converged == rec["converged"], name
    u_s = [float.fromhex(x) for x in rec["u_sample"]]
    if _digest(r.u) != rec["u_sha256"]:
        d = np.abs(r.u[::SAMPLE_STRIDE] - u_s).max()
        pytest.fail(f"{name}: u differs from the reference (sampled max |du| {d:.3e})")
    assert np.array_equal(r.u[::SAMPLE_STRIDE], u_s), name
    if f is not None:
        assert _digest(f) == rec["f_sha256"], f"{name}: final f differs from the reference"
    assert r.final_residual == float.fromhex(rec["final_residual"]), name
    assert r.r_ref == float.fromhex(rec["r_ref"]), name
    sig = np.array([float.fromhex(x) for x in rec["avg_stress"]]).reshape(3, 3)
    assert np.abs(r.avg_stress - sig).max() <= 1e-13 * np.abs(sig).max(), name


def _forces(batch, dres, i):
    """Final internal force of problem i in original node order."""
    p = batch.problems[i]
    b0, b1 = int(batch.node_base[i]), int(batch.node_base[i + 1])
    f_solver = dres.f[3 * b0:3 * b1].cpu().numpy().reshape(-1, 3)
    f = np.empty_like(f_solver)
    f[p.node_order] = f_solver
    return f.reshape(-1)


def test_big_cases_are_the_baseline_configs():
    """The records name the inputs the bench uses (CPU-side sanity, runs in -m gpu)."""
    assert BIG["c3_32cube_seed0"]["lattice"] == [32, 32, 32, 0.3, 0]
    assert BIG["c3_32cube_seed0"]["iters"] == 2519


def test_full_length_heterogeneous_batch(cuda_device):
    """All large cases in ONE batch (c4's execution mode: the 8- and 2-CTA
    groups concurrently, then the 16-CTA groups), each to convergence."""
    from paper_2305_07030_b200 import batch as fb
    names = sorted(BIG)
    cases = [_case(n) for n in names]
    batch = frb.pack_batch([c[0] for c in cases], [frb.AffineBC(c[1]) for c in cases])
    assert {int(c) for c in batch.desc["cluster"]} >= {2, 8, 16}
    dres = batch.to_device().solve(frb.SolverConfig())
    res = fb.results_to_solve_results(batch, dres)
    for i, (name, (_, _, rec), r) in enumerate(zip(names, cases, res)):
        _check(name, rec, r, _forces(batch, dres, i))


@pytest.mark.parametrize("name", ["c3_32cube_seed0", "lat24_shear_seed3"])
def test_cluster_path_alone(cuda_device, name):
    """The 16-CTA (C3) and 8-CTA paths with the whole GPU to themselves,
    through dynamic_relaxation_solve (a batch of one)."""
    net, F, rec = _case(name)
    r = frb.dynamic_relaxation_solve(net, frb.AffineBC(F), frb.SolverConfig())
    _check(name, rec, r, None)


def test_c3_batch_replicas(cuda_device):
    """Eight copies of the C3 network next to each other (every cluster of the
    persistent grid busy, the work queue handing out networks): all equal the
    reference."""
    from paper_2305_07030_b200 import batch as fb
    net, F, rec = _case("c3_32cube_seed0")
    batch = frb.pack_batch([net] * 8, [frb.AffineBC(F)] * 8)
    dres = batch.to_device().solve(frb.SolverConfig())
    for i, r in enumerate(fb.results_to_solve_results(batch, dres)):
        _check(f"c3 copy {i}", rec, r, _forces(batch, dres, i))


def test_heterogeneous_batch_with_virtual_clusters(cuda_device):
    """Nine C3 networks next to 8- and 2-CTA networks: the smaller groups run
    concurrently, then the 16-CTA group alone on 7 hardware + 2 virtual
    clusters (9 networks: the virtual clusters get work).  Two kernels for the
    16-CTA group, one per smaller group; every network equals the reference."""
    from paper_2305_07030_b200 import batch as fb
    names = ["c3_32cube_seed0"] * 9 + sorted(n for n in BIG if n != "c3_32cube_seed0" and BIG[n]["lattice"][0] < 26)
    cases = [_case(n) for n in names]
    batch = frb.pack_batch([c[0] for c in cases], [frb.AffineBC(c[1]) for c in cases])
    launch = batch.to_device().prepare(frb.SolverConfig(), frb.TeamBatched())
    launch.run()
    n_groups = int((batch.groups["count"] > 0).sum())
    assert launch.kernel_launches == n_groups + 1  # + the virtual clusters of the 16-CTA group
    res = fb.results_to_solve_results(batch, launch.out)
    for i, (name, (_, _, rec), r) in enumerate(zip(names, cases, res)):
        _check(f"{name} #{i}", rec, r, _forces(batch, launch.out, i))
