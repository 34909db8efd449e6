"""Generate golden fixtures by running the REAL reference (``fibrelax`` from
/root/reference/pkg/src) in the build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py --big   # big_index.json

Each case is written to ``tests/golden/<name>.npz`` with the inputs (so the
GPU box can rebuild the network without the reference) and the reference's
outputs: converged, iters, final_residual, r_ref, u (original order), the
final internal force f (original order, from the reference's own state),
avg_stress and energy_residual.  The reference is driven through its own
seams (build_problem -> make_state -> _Scratch -> _Run -> run_lanes(_relax)
-> finalize_result, microsolver.py:567-574) so f can be captured; the public
dynamic_relaxation_solve result is checked to be identical.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import fibrelax as fr  # noqa: E402
from fibrelax import microsolver as ms  # noqa: E402
from fibrelax._lanes import run_lanes  # noqa: E402

UNIAX = np.diag([1.1, 1.0, 1.0])
BIAX = np.diag([1.1, 1.1, 1.0])
SHEAR = np.eye(3) + 0.2 * np.outer([1, 0, 0], [0, 1, 0])


def random_network(seed, n_nodes=60, n_edges=200, n_mat=3, boundary_frac=0.3):
    """Irregular network: random nodes, random unique edges, mixed materials."""
    rng = np.random.default_rng(seed)
    coords = rng.uniform(0.0, 1.0, (n_nodes, 3))
    pairs = set()
    edges = []
    # spanning chain so no node is isolated, then random extras
    perm = rng.permutation(n_nodes)
    for a, b in zip(perm[:-1], perm[1:]):
        key = (min(a, b), max(a, b))
        pairs.add(key)
        edges.append((int(a), int(b)))
    while len(edges) < n_edges:
        a, b = rng.integers(0, n_nodes, 2)
        if a == b:
            continue
        key = (min(a, b), max(a, b))
        if key in pairs:
            continue
        pairs.add(key)
        edges.append((int(a), int(b)))
    order = rng.permutation(len(edges))
    mats = rng.integers(0, n_mat, len(edges))
    elements = np.array([[edges[i][0], edges[i][1], mats[k]] for k, i in enumerate(order)], dtype=np.int64)
    materials = [fr.Material(float(rng.uniform(0.5, 2.0)), float(rng.uniform(0.5, 2.0)),
                             float(rng.uniform(0.5, 2.0))) for _ in range(n_mat)]
    boundary = frozenset(int(x) for x in rng.choice(n_nodes, int(boundary_frac * n_nodes), replace=False))
    return fr.FiberNetwork(coords, elements, materials, boundary)


def bar3():
    return fr.FiberNetwork(np.array([[0.0, 0, 0], [0.5, 0, 0], [1.0, 0, 0]]),
                           np.array([[0, 1, 0], [1, 2, 0]]), [fr.Material(1, 1, 1)],
                           frozenset({0, 2}))


def bar3_bc():
    # ends fixed at u=0 and u_x=0.1: F=diag(1.1,1,1) maps X=1 -> u_x=0.1, X=0 -> 0
    return UNIAX


def cases():
    C = fr.SolverConfig
    yield "c1_7x7x8_uniax", fr.generate_lattice(7, 7, 8, 0.3, 0), UNIAX, C()
    yield "lat5_shear", fr.generate_lattice(5, 5, 5, 0.3, 1), SHEAR, C()
    yield "lat5_biax", fr.generate_lattice(5, 5, 5, 0.3, 2), BIAX, C()
    yield "lat5_ramp10", fr.generate_lattice(5, 5, 5, 0.3, 3), UNIAX, C(bc_ramp_iters=10)
    yield "lat5_ramp1", fr.generate_lattice(5, 5, 5, 0.3, 3), UNIAX, C(bc_ramp_iters=1)
    yield "lat6_fixed1", fr.generate_lattice(6, 6, 6, 0.3, 4), UNIAX, C(damping=fr.FixedDamping(1.0))
    yield "lat5_energy", fr.generate_lattice(5, 5, 5, 0.3, 5), UNIAX, C(energy_check_interval=1)
    yield "lat5_energy_ramp", fr.generate_lattice(5, 5, 5, 0.3, 5), BIAX, C(energy_check_interval=3, bc_ramp_iters=7)
    yield "lat6_maxiter", fr.generate_lattice(6, 6, 6, 0.3, 6), UNIAX, C(max_iters=50)
    yield "lat4_identity", fr.generate_lattice(4, 4, 4, 0.3, 7), np.eye(3), C()
    yield "lat2_allfixed", fr.generate_lattice(2, 2, 2, 0.0, 0), UNIAX, C()
    yield "lat3_one_free", fr.generate_lattice(3, 3, 3, 0.3, 8), SHEAR, C()
    yield "lat8_seed5", fr.generate_lattice(8, 8, 8, 0.3, 5), UNIAX, C()
    yield "lat4x5x6_tolabs", fr.generate_lattice(4, 5, 6, 0.2, 9), BIAX, C(tol_rel=0.0, tol_abs=1e-7)
    yield "lat5_dtsafe", fr.generate_lattice(5, 5, 5, 0.1, 10), SHEAR, C(dt_safety=0.9, tol_rel=1e-10)
    rot = np.array([[0.98, -0.17, 0.05], [0.17, 0.97, 0.02], [-0.04, 0.0, 1.03]])
    yield "lat6_general_F", fr.generate_lattice(6, 5, 7, 0.35, 11), rot, C()
    yield "random60", random_network(12), UNIAX, C()
    yield "random90_fixed", random_network(13, n_nodes=90, n_edges=400), SHEAR, C(damping=fr.FixedDamping(0.5), max_iters=4000)
    yield "bar3_adaptive", bar3(), bar3_bc(), C()
    yield "bar3_fixed05", bar3(), bar3_bc(), C(damping=fr.FixedDamping(0.5))
    yield "c2_15cube_seed0", fr.generate_lattice(15, 15, 15, 0.3, 0), UNIAX, C()
    # singular: collapse the bar along x (reference Appendix B error path)
    yield "bar_singular", fr.FiberNetwork(np.array([[0.0, 0, 0], [1.0, 0, 0]]), np.array([[0, 1, 0]]),
                                          [fr.Material(1, 1, 1)], frozenset({0, 1})), \
        np.diag([1e-13, 1.0, 1.0]), C()


def c5_gradient(i):
    """Random macro deformation gradient of FE2 network i."""
    rng = np.random.default_rng(10 ** 6 + i)
    diag = rng.uniform(0.0, 0.1, 3)
    off = rng.uniform(-0.05, 0.05, (3, 3))
    np.fill_diagonal(off, 0.0)
    return np.eye(3) + np.diag(diag) + off


def big_cases():
    """Full-length cases of the BASELINE configs that run on 8- and 16-CTA
    clusters (and the c4 / c5 recipes).  Stored compactly: the lattice
    parameters (the product's generate_lattice is bit-identical to the
    reference's, tests/test_packing.py) and SHA-256 digests of the exact u / f
    bytes plus a strided sample, so a multi-megabyte network costs a few KB."""
    C = fr.SolverConfig
    yield "c3_32cube_seed0", (32, 32, 32, 0.3, 0), UNIAX, C()                 # C3 (16-CTA cluster)
    yield "c4_i77_32cube_shear", (32, 32, 32, 0.3, 77), SHEAR, C()           # c4 i=77: 32^3 shear
    yield "c4_i71_26cube_shear", (26, 26, 26, 0.3, 71), SHEAR, C()           # c4 i=71: 26^3 shear
    yield "c4_i13_20cube_biax", (20, 20, 20, 0.3, 13), BIAX, C()             # c4 i=13: 20^3 biax
    yield "lat24_shear_seed3", (24, 24, 24, 0.3, 3), SHEAR, C()              # 8-CTA cluster
    yield "c5_i0_15cube_randF", (15, 15, 15, 0.3, 0), c5_gradient(0), C()    # c5 network 0
    yield "c5_i1_15cube_randF", (15, 15, 15, 0.3, 1), c5_gradient(1), C()    # c5 network 1


def digest(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


SAMPLE_STRIDE = 97


def main_big(only=None):
    import time
    path = os.path.join(HERE, "big_index.json")
    for name, lat, F, cfg in big_cases():
        if only and name not in only:
            continue
        net = fr.generate_lattice(*lat)
        t0 = time.perf_counter()
        out, err = run_reference(net, F, cfg)
        assert err is None, err
        res, f = out
        rec = dict(lattice=list(lat), F=np.asarray(F, dtype=np.float64).tolist(), cfg=cfg_dict(cfg),
                   converged=bool(res.converged), iters=int(res.iters),
                   final_residual=float(res.final_residual).hex(), r_ref=float(res.r_ref).hex(),
                   avg_stress=[float(x).hex() for x in res.avg_stress.reshape(-1)],
                   u_sha256=digest(res.u), f_sha256=digest(f),
                   u_sample=[float(x).hex() for x in res.u[::SAMPLE_STRIDE]],
                   f_sample=[float(x).hex() for x in f[::SAMPLE_STRIDE]],
                   n_nodes=net.n_nodes, n_elements=net.n_elements,
                   reference_seconds=round(time.perf_counter() - t0, 1))
        import fcntl
        with open(path + ".lock", "w") as lk:  # several generators may run at once
            fcntl.flock(lk, fcntl.LOCK_EX)
            index = json.load(open(path)) if os.path.exists(path) else {}
            index[name] = rec
            with open(path, "w") as fh:
                json.dump(dict(sorted(index.items())), fh, indent=0)
        print(name, rec["iters"], rec["converged"], rec["reference_seconds"], "s", flush=True)


def cfg_dict(cfg):
    return dict(tol_rel=cfg.tol_rel, tol_abs=cfg.tol_abs, max_iters=cfg.max_iters,
                dt_safety=cfg.dt_safety,
                damping_c=(cfg.damping.c if isinstance(cfg.damping, fr.FixedDamping) else None),
                energy_check_interval=cfg.energy_check_interval, bc_ramp_iters=cfg.bc_ramp_iters)


def run_reference(net, F, cfg):
    bc = fr.AffineBC(F)
    setup = ms.build_problem(net, bc)
    run = ms._Run(setup=setup, state=ms.make_state(setup), scratch=ms._Scratch(setup, cfg), cfg=cfg)
    try:
        run_lanes(1, lambda lane: ms._relax(lane, run))
    except fr.SingularElementError as exc:
        return None, str(exc)
    res = ms.finalize_result(run)
    pub = fr.dynamic_relaxation_solve(net, bc, cfg)
    assert pub.iters == res.iters and np.array_equal(pub.u, res.u)
    f = setup.dofmap.unpermute(run.state.f_int)
    return (res, f), None


def main(only=None):
    index = {}
    for name, net, F, cfg in cases():
        if only and name not in only:
            continue
        out, err = run_reference(net, F, cfg)
        mats = np.array([[m.elastic_modulus, m.cross_section_area, m.density] for m in net.materials])
        data = dict(coords=net.node_coords, elements=net.elements, materials=mats,
                    boundary=np.array(sorted(net.boundary_nodes), dtype=np.int64),
                    rve_volume=np.float64(math.nan if net.rve_volume is None else net.rve_volume),
                    F=np.asarray(F, dtype=np.float64), cfg=json.dumps(cfg_dict(cfg)))
        if err is not None:
            data.update(singular=np.bool_(True), error=err)
            index[name] = dict(error=err)
        else:
            res, f = out
            data.update(singular=np.bool_(False), converged=np.bool_(res.converged),
                        iters=np.int64(res.iters), final_residual=np.float64(res.final_residual),
                        r_ref=np.float64(res.r_ref), u=res.u, f=f, avg_stress=res.avg_stress,
                        energy_residual=np.float64(math.nan if res.energy_residual is None
                                                   else res.energy_residual))
            index[name] = dict(iters=res.iters, converged=bool(res.converged),
                               n_nodes=net.n_nodes, n_elements=net.n_elements)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
        print(name, index[name], flush=True)
    if not only:
        with open(os.path.join(HERE, "index.json"), "w") as fh:
            json.dump(dict(numpy=np.__version__, fibrelax=fr.__version__, cases=index), fh, indent=1)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--big"]:
        main_big(sys.argv[2:] or None)
    else:
        main(sys.argv[1:] or None)
