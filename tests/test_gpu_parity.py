"""CUDA path vs the reference golden vectors and the CPU oracle (B200).

Bar: u, f, final_residual, r_ref bit-equal; iters and
converged equal; avg_stress within 1e-13 of max|sigma| (BLAS order in the
reference).  Every call goes through the C-ABI library.
"""

import math

import numpy as np
import pytest

import golden_cases as gc
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb
from oracle import frb_oracle as orc

pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-13
NAMES = [n for n in gc.names() if n != "bar_singular"]


def assert_matches(r, u_ref, iters, converged, residual, r_ref, sigma, label=""):
    assert r.iters == iters, f"{label}: iters {r.iters} != {iters}"
    assert r.converged == converged, label
    assert np.array_equal(r.u, u_ref), f"{label}: u differs (max {np.abs(r.u - u_ref).max():.3e})"
    assert r.final_residual == residual or (math.isnan(r.final_residual) and math.isnan(residual)), label
    assert r.r_ref == r_ref or (math.isnan(r.r_ref) and math.isnan(r_ref)), label
    scale = max(np.abs(sigma).max(), 1e-300)
    assert np.abs(r.avg_stress - sigma).max() <= SIGMA_RTOL * scale, label


def golden_expect(case):
    d = case.data
    return (d["u"], int(d["iters"]), bool(d["converged"]), float(d["final_residual"]),
            float(d["r_ref"]), d["avg_stress"])


@pytest.mark.parametrize("name", NAMES)
def test_single_solve_matches_reference(cuda_device, name):
    case = gc.load(name)
    r = frb.dynamic_relaxation_solve(case.network, frb.AffineBC(case.F), case.cfg)
    assert_matches(r, *golden_expect(case), label=name)
    if case.cfg.energy_check_interval > 0:
        e = float(case.data["energy_residual"])
        assert abs(r.energy_residual - e) <= 1e-10 * max(abs(e), 1e-30)


def test_final_forces_bit_equal(cuda_device):
    for name in ("c1_7x7x8_uniax", "lat6_general_F", "random90_fixed"):
        case = gc.load(name)
        batch = frb.pack_batch([case.network], [frb.AffineBC(case.F)])
        dres = batch.to_device().solve(case.cfg)
        f_solver = dres.f.cpu().numpy().reshape(-1, 3)
        f = np.empty_like(f_solver)
        f[batch.problems[0].node_order] = f_solver
        assert np.array_equal(f.reshape(-1), case.data["f"]), name


def test_heterogeneous_batch_equals_single(cuda_device):
    """All golden cases with the default config in one launch (mixed sizes,
    loads, topologies); each must equal its reference result."""
    cases = [gc.load(n) for n in NAMES]
    cases = [c for c in cases if c.cfg == frb.SolverConfig()]
    res = frb.solve_batch(frb.pack_batch([c.network for c in cases], [frb.AffineBC(c.F) for c in cases]))
    for c, r in zip(cases, res):
        assert_matches(r, *golden_expect(c), label=c.name)


def test_singular_element_raises(cuda_device):
    case = gc.load("bar_singular")
    with pytest.raises(frb.SingularElementError, match="element 0: current length collapsed"):
        frb.dynamic_relaxation_solve(case.network, frb.AffineBC(case.F), case.cfg)


def test_singular_does_not_abort_siblings(cuda_device):
    good = gc.load("lat5_shear")
    bad = gc.load("bar_singular")
    batch = frb.pack_batch([good.network, bad.network, good.network],
                           [frb.AffineBC(good.F), frb.AffineBC(bad.F), frb.AffineBC(good.F)])
    dres = batch.to_device().solve(frb.SolverConfig())
    out = fb.results_to_solve_results(batch, dres, raise_singular=False)
    assert out[1] is None
    for r in (out[0], out[2]):
        assert_matches(r, *golden_expect(good), label="sibling")


@pytest.mark.parametrize("n,seed,load", [(6, 0, "uniax"), (7, 1, "biax"), (8, 2, "shear"),
                                         (9, 3, "uniax"), (5, 4, "shear")])
def test_random_lattices_vs_oracle(cuda_device, n, seed, load):
    F = {"uniax": np.diag([1.1, 1, 1]), "biax": np.diag([1.1, 1.1, 1]),
         "shear": np.eye(3) + 0.2 * np.outer([1, 0, 0], [0, 1, 0])}[load]
    net = frb.generate_lattice(n, n + 1, n, 0.3, seed)
    cfg = frb.SolverConfig()
    r = frb.dynamic_relaxation_solve(net, frb.AffineBC(F), cfg)
    o = orc.solve(net, F, cfg)
    assert_matches(r, o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label=f"{n}/{seed}")


def test_c2_batch_subset_vs_oracle(cuda_device):
    """Config 2 networks (15^3, uniaxial) inside a 16-network batch."""
    nets = [frb.generate_lattice(15, 15, 15, 0.3, s) for s in range(16)]
    F = np.diag([1.1, 1.0, 1.0])
    res = frb.solve_batch(frb.pack_batch(nets, [frb.AffineBC(F)] * 16))
    for s in (0, 7):
        o = orc.solve(nets[s], F, frb.SolverConfig())
        assert_matches(res[s], o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label=f"seed{s}")
    golden = gc.load("c2_15cube_seed0")
    assert_matches(res[0], *golden_expect(golden), label="golden c2")


def test_deterministic_rerun(cuda_device):
    nets = [frb.generate_lattice(8, 8, 8, 0.3, s) for s in range(40)]
    bcs = [frb.AffineBC(np.diag([1.1, 1.0, 1.0]))] * 40
    batch = frb.pack_batch(nets, bcs)
    a = frb.solve_batch(batch)
    b = frb.solve_batch(batch, strategy=frb.TeamBatched(teams=7))
    c = frb.solve_batch(batch, strategy=frb.SerialReference())
    for x, y, z in zip(a, b, c):
        assert x.iters == y.iters == z.iters
        assert np.array_equal(x.u, y.u) and np.array_equal(x.u, z.u)
        assert np.array_equal(x.avg_stress, y.avg_stress)


def test_internal_forces_matches_reference(cuda_device):
    case = gc.load("lat6_general_F")
    f = frb.internal_forces(case.network, case.data["u"])
    assert np.array_equal(f, case.data["f"])
    assert frb.force_residual(f, 0) == 0.0
    # translation invariance (SPEC.md invariants)
    t = np.tile([0.3, -0.2, 0.5], case.network.n_nodes)
    assert np.abs(frb.internal_forces(case.network, t)).max() < 1e-12


def test_identity_deformation_converges_in_one(cuda_device):
    net = frb.generate_lattice(6, 6, 6, 0.3, 1)
    r = frb.dynamic_relaxation_solve(net, frb.AffineBC(np.eye(3)))
    assert r.converged and r.iters == 1
    assert not r.u.any() and not r.avg_stress.any()


@pytest.mark.parametrize("n,iters", [(16, 20000), (24, 60), (32, 40)])
def test_cluster_paths_vs_oracle(cuda_device, n, iters):
    """Networks split over 2 / 8 / 16-CTA clusters (32^3: config 3's path,
    f_prev in global memory), bit-equal to the oracle.  The larger ones stop at
    max_iters so the CPU oracle stays fast; u, f, residual and the stress are
    compared at that iterate."""
    net = frb.generate_lattice(n, n, n, 0.3, 3)
    F = np.eye(3) + 0.2 * np.outer([1, 0, 0], [0, 1, 0])
    cfg = frb.SolverConfig(max_iters=iters)
    batch = frb.pack_batch([net], [frb.AffineBC(F)])
    assert int(batch.desc[0]["cluster"]) == {16: 2, 24: 8, 32: 16}[n]
    assert bool(batch.groups[0]["fprv_global"]) == (n == 32)
    r = frb.solve_batch(batch, config=cfg)[0]
    o = orc.solve(net, F, cfg)
    assert_matches(r, o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label=f"{n}^3")


def test_single_cta_global_fprev_vs_oracle(cuda_device):
    """The one-CTA kernel with f_prev in global memory (15^3 packed with
    cluster=1), bit-equal to the oracle."""
    net = frb.generate_lattice(15, 15, 15, 0.3, 4)
    F = np.diag([1.05, 1.1, 1.0])
    cfg = frb.SolverConfig(max_iters=200)
    p = fb.build_problem(net, frb.AffineBC(F))
    batch = fb._pack([net], [frb.AffineBC(F)], [p], cluster=1)
    from paper_2305_07030_b200.partition import partition_smem_bytes
    batch.groups[0]["fprv_global"] = 1
    batch.groups[0]["block_threads"] = 768
    batch.groups[0]["smem_bytes"] = partition_smem_bytes(p.topo.partition(1), True)
    r = fb.results_to_solve_results(batch, batch.to_device().solve(cfg))[0]
    o = orc.solve(net, F, cfg)
    assert_matches(r, o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label="15^3 one CTA")


@pytest.mark.parametrize("name", ["c1_7x7x8_uniax", "lat8_seed5", "random60", "lat6_general_F"])
def test_every_cta_size_matches_reference(cuda_device, name):
    """Each CTA size selects a different kernel instantiation (register-held
    DOFs per thread x thread bound); all of them must reproduce the
    reference bit for bit (guards against a miscompiled instantiation)."""
    case = gc.load(name)
    batch = frb.pack_batch([case.network], [frb.AffineBC(case.F)])
    nf = 3 * batch.problems[0].n_free_nodes
    for T in (64, 96, 128, 224, 256, 320, 416, 512, 544, 640, 768, 1024):
        if nf > fb.dofs_per_thread_cap(T) * T:
            continue
        r = fb.results_to_solve_results(batch, batch.to_device().solve(case.cfg, frb.TeamBatched(team_size=T)))[0]
        assert_matches(r, *golden_expect(case), label=f"{name} T={T}")


@pytest.mark.parametrize("n,ramp", [(6, 0), (6, 4), (16, 0), (16, 6)])
def test_energy_ledger_vs_oracle(cuda_device, n, ramp):
    """Work ledger on one CTA and on a 2-CTA cluster, with and without the BC
    ramp: same iterate bit for bit (the ledger never feeds back), energy
    residual within 1e-10 (the reference's np.dot is BLAS-ordered)."""
    net = frb.generate_lattice(n, n, n, 0.3, 2)
    F = np.diag([1.1, 1.0, 1.05])
    cfg = frb.SolverConfig(energy_check_interval=1, bc_ramp_iters=ramp, max_iters=400)
    r = frb.dynamic_relaxation_solve(net, frb.AffineBC(F), cfg)
    o = orc.solve(net, F, cfg)
    assert_matches(r, o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label=f"{n}/{ramp}")
    assert abs(r.energy_residual - o.energy_residual) <= 1e-10 * abs(o.energy_residual)


def test_fe2_macro_step_reuses_the_packed_batch(cuda_device):
    """DeviceBatch.set_deformation: a new F per network on the resident batch
    gives the same bits as packing afresh (the FE2 macro-step loop)."""
    nets = [frb.generate_lattice(6, 6, 7, 0.3, s) for s in range(4)]
    F0 = [np.diag([1.1, 1.0, 1.0])] * 4
    F1 = [np.eye(3) + 0.02 * (k + 1) * np.outer([1, 0, 0], [0, 1, 0]) for k in range(4)]
    batch = frb.pack_batch(nets, [frb.AffineBC(F) for F in F0])
    dev = batch.to_device()
    fb.results_to_solve_results(batch, dev.solve(frb.SolverConfig()))
    dev.set_deformation(F1)
    got = fb.results_to_solve_results(batch, dev.solve(frb.SolverConfig()))
    fresh = frb.solve_batch(frb.pack_batch(nets, [frb.AffineBC(F) for F in F1]))
    for a, b in zip(got, fresh):
        assert a.iters == b.iters and np.array_equal(a.u, b.u) and np.array_equal(a.avg_stress, b.avg_stress)


def test_tangent_matches_oracle_differences(cuda_device):
    """Homogenized tangent: the 19 solves per network run as one
    device batch; the result equals the oracle's central differences up to
    the σ bar propagated through the difference quotient."""
    from paper_2305_07030_b200.tangent import assemble_tangent, perturbed_gradients
    nets = [frb.generate_lattice(4, 4, 5, 0.3, s) for s in range(2)]
    Fs = [np.diag([1.05, 1.0, 1.0]), np.eye(3) + 0.1 * np.outer([1, 0, 0], [0, 1, 0])]
    h = 1e-5
    res = frb.homogenized_tangent(nets, Fs, h=h)
    for net, F, r in zip(nets, Fs, res):
        sig = [orc.solve(net, Fp, frb.SolverConfig()).sigma for Fp in perturbed_gradients(F, h)]
        C = assemble_tangent(sig, h)
        S = max(np.abs(s).max() for s in sig)
        assert r.converged and r.iters.shape == (19,)
        assert np.abs(r.sigma - sig[0]).max() <= SIGMA_RTOL * S
        assert np.abs(r.tangent - C).max() <= SIGMA_RTOL * S / h + 1e-15 * np.abs(C).max()
        assert np.array_equal(r.tangent, r.tangent.transpose(1, 0, 2, 3))


def test_two_slot_network_vs_oracle(cuda_device):
    """A lattice without its z-links has at most 2 slots per role: the
    padded (<= 3 slots) gather path, 400 iterations bit for bit."""
    net = frb.generate_lattice(5, 5, 4, 0.3, 0)
    X, E = net.node_coords, net.elements
    d = np.abs(X[E[:, 1]] - X[E[:, 0]])
    net2 = frb.FiberNetwork(X, E[d[:, 2] < 0.5 * np.maximum(d[:, 0], d[:, 1])], net.materials,
                            net.boundary_nodes, rve_volume=net.volume)
    part, _, _ = fb.build_problem(net2, frb.AffineBC(np.eye(3))).topo.choose_cluster()
    assert (part.slots_a, part.slots_b) == (2, 2)
    F = np.diag([1.1, 1.0, 1.0])
    cfg = frb.SolverConfig(max_iters=400)
    r = frb.dynamic_relaxation_solve(net2, frb.AffineBC(F), cfg)
    o = orc.solve(net2, F, cfg)
    assert_matches(r, o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label="2-slot")


def test_masses_in_global_memory_vs_oracle(cuda_device):
    """A 31^3 network (c4's n = 7 + 24) fills a 16-CTA cluster even with
    f_prev in global memory, so its node masses stay in global memory too
    (FRB_PF_MASS_GLOBAL); 60 iterations bit-equal to the oracle, and the same
    network to convergence on 2 of the shared code paths."""
    from paper_2305_07030_b200 import _native as nat
    net = frb.generate_lattice(31, 31, 31, 0.3, 76)
    F = np.eye(3) + 0.2 * np.outer([1, 0, 0], [0, 1, 0])
    cfg = frb.SolverConfig(max_iters=60)
    batch = frb.pack_batch([net], [frb.AffineBC(F)])
    assert int(batch.desc[0]["cluster"]) == 16 and int(batch.desc[0]["flags"]) & nat.PF_MASS_GLOBAL
    r = frb.solve_batch(batch, config=cfg)[0]
    o = orc.solve(net, F, cfg)
    assert_matches(r, o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label="31^3")


def test_randomly_renumbered_network_vs_oracle(cuda_device):
    """Node ids in random order (no slab locality): the 4 ranks keep hundreds
    of short halo runs each (odd starts and lengths widened to 16-byte bulk
    copies) and nodes are halo to up to 3 ranks; 100 iterations bit-equal."""
    net = frb.generate_lattice(16, 16, 16, 0.3, 1)
    perm = np.random.default_rng(0).permutation(net.n_nodes)
    el = net.elements.copy()
    el[:, :2] = perm[el[:, :2]]
    net2 = frb.FiberNetwork(net.node_coords[np.argsort(perm)], el, net.materials,
                            frozenset(int(perm[b]) for b in net.boundary_nodes))
    F = np.diag([1.1, 1.0, 1.05])
    cfg = frb.SolverConfig(max_iters=100)
    batch = frb.pack_batch([net2], [frb.AffineBC(F)])
    assert int(batch.desc[0]["cluster"]) > 1
    assert max(len(rt.runs) for rt in batch.problems[0].topo.chosen()[0].ranks) > 100
    r = frb.solve_batch(batch, config=cfg)[0]
    o = orc.solve(net2, F, cfg)
    assert_matches(r, o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label="renumbered 16^3")


def test_solve_reports_its_kernel_launches(cuda_device):
    """frb_solve_launches: one relaxation kernel per launch group (these
    groups have no virtual clusters: 1- and 2-CTA clusters)."""
    one = fb.pack_batch([frb.generate_lattice(6, 6, 6, 0.3, s) for s in range(3)],
                        [frb.AffineBC(np.diag([1.1, 1.0, 1.0]))] * 3)
    L = one.to_device().prepare(frb.SolverConfig(), frb.TeamBatched())
    L.run()
    assert L.kernel_launches == 1
    mixed = fb.pack_batch([frb.generate_lattice(6, 6, 6, 0.3, 0), frb.generate_lattice(15, 15, 15, 0.3, 0)],
                          [frb.AffineBC(np.diag([1.1, 1.0, 1.0]))] * 2)
    L = mixed.to_device().prepare(frb.SolverConfig(), frb.TeamBatched())
    L.run()
    assert len(mixed.groups) == 2 and L.kernel_launches == 2


def test_energy_ledger_heterogeneous_batch(cuda_device):
    """The ledger kernels on a batch of several cluster sizes (1- and 2-CTA
    groups launched concurrently): every network equals its own oracle run."""
    nets = [frb.generate_lattice(6, 6, 6, 0.3, 1), frb.generate_lattice(16, 16, 16, 0.3, 4),
            frb.generate_lattice(7, 6, 8, 0.3, 5)]
    Fs = [np.diag([1.1, 1.0, 1.05]), np.eye(3) + 0.05 * np.eye(3)[:, [1, 2, 0]], np.diag([1.05, 1.05, 1.0])]
    cfg = frb.SolverConfig(energy_check_interval=1, max_iters=300)
    batch = fb.pack_batch(nets, [frb.AffineBC(F) for F in Fs])
    assert len({int(c) for c in batch.desc["cluster"]}) >= 2
    res = frb.solve_batch(batch, config=cfg)
    for i, (net, F, r) in enumerate(zip(nets, Fs, res)):
        o = orc.solve(net, F, cfg)
        assert_matches(r, o.u, o.iters, o.converged, o.residual, o.r_ref, o.sigma, label=f"net {i}")
        assert abs(r.energy_residual - o.energy_residual) <= 1e-10 * abs(o.energy_residual)
