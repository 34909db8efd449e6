"""Host packing invariants (no GPU): incidence order equals the reference's
bincount summation order, slot tables mirror the CSR, cluster partitions are
consistent, SMEM mirrors agree with the library."""

import numpy as np
import pytest

import golden_cases as gc
import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import _native as nat
from paper_2305_07030_b200 import batch as fb
from paper_2305_07030_b200.partition import partition_smem_bytes, rank_smem_bytes
from paper_2305_07030_b200.plan import PlanView


def _nets():
    yield frb.generate_lattice(5, 6, 7, 0.3, 1)
    yield gc.load("random90_fixed").network
    yield gc.load("lat2_allfixed").network
    yield frb.generate_lattice(12, 12, 12, 0.3, 2)


NETS = list(_nets())


@pytest.mark.parametrize("net", NETS)
def test_csr_is_role_then_element_order(net):
    p = fb.build_problem(net, frb.AffineBC(np.eye(3)))
    t = p.topo
    rank = np.empty(net.n_nodes, dtype=np.int64)
    rank[p.node_order] = np.arange(net.n_nodes)
    ia, ib = rank[net.elements[:, 0]], rank[net.elements[:, 1]]
    for i in range(net.n_nodes):
        first, packed = t.inc_node[i]
        na, nb = packed & 0xffff, packed >> 16
        ent = t.inc[first:first + na + nb]
        ea = np.flatnonzero(ia == i)
        eb = np.flatnonzero(ib == i)
        assert list(ent[:na, 1]) == list(ea) and list(ent[:na, 0]) == list(ib[ea])
        assert list(ent[na:, 1]) == list(eb) and list(ent[na:, 0]) == list(ia[eb])


@pytest.mark.parametrize("net", NETS)
def test_slot_table_mirrors_csr(net):
    t = fb.build_problem(net, frb.AffineBC(np.eye(3))).topo
    for i in range(t.n_free_nodes):
        first, packed = t.inc_node[i]
        na, nb = packed & 0xffff, packed >> 16
        ent = t.inc[first:first + na + nb]
        a = [o for o in t.ell_other[:t.slots_a, i] if o >= 0]
        b = [o for o in t.ell_other[t.slots_a:, i] if o >= 0]
        assert a == list(ent[:na, 0]) and b == list(ent[na:, 0])
        col = t.ell_other[:t.slots_a, i]
        assert all(col[k] >= 0 for k in range(na)) and all(col[k] < 0 for k in range(na, t.slots_a))


@pytest.mark.parametrize("net", NETS)
@pytest.mark.parametrize("C", [1, 2, 4])
def test_partition_tables(net, C):
    t = fb.build_problem(net, frb.AffineBC(np.eye(3))).topo
    part = t.partition(C)
    NF = t.n_free_nodes
    ia, ib = t.elem_ab[:, 0], t.elem_ab[:, 1]
    starts = PlanView(t.plan).leaf_start
    nxt = 0
    leaf = 0
    for r, rt in enumerate(part.ranks):
        assert rt.node0 == nxt
        nxt += rt.n_own
        assert rt.leaf0 == leaf
        leaf += rt.n_leaves
        if rt.n_leaves:
            assert starts[rt.leaf0] == 3 * rt.node0   # leaf-aligned, node-aligned cut
        own = set(range(rt.node0, rt.node0 + rt.n_own))
        halo = list(rt.halo_g)

        def glob(l):
            if l < rt.n_own:
                return rt.node0 + l
            if l < rt.n_local:
                return halo[l - rt.n_own]
            return int(rt.fix_g[l - rt.n_local])

        act = set(np.flatnonzero(np.isin(ia, list(own)) | np.isin(ib, list(own))))
        assert set(rt.act_elem) == act
        ends = np.concatenate([ia[rt.act_elem], ib[rt.act_elem]])
        assert list(rt.fix_g) == sorted(set(ends[ends >= NF].tolist()))   # fixed ends of active elements
        w = rt.ell.astype(np.int64)[:, :rt.n_own]
        pad = rt.ell_o[:, :rt.n_own] < 0
        lo, lc = rt.ell_o[:, :rt.n_own], rt.ell_c[:, :rt.n_own]
        assert (w[~pad] >> 16 == lo[~pad]).all() and (w[~pad] & 0xFFFF == lc[~pad]).all()
        # padding points at the node itself (d = +0 exactly) and a real element of it
        assert ((w >> 16)[pad] == np.nonzero(pad)[1]).all()
        for k, i in zip(*np.nonzero(pad)):
            assert (w[k, i] & 0xFFFF) in set(lc[~pad[:, i], i].tolist())
        for e, (a, b) in zip(rt.act_elem, rt.act_ab):
            assert (glob(a), glob(b)) == (ia[e], ib[e])
        for i in range(rt.n_own):
            for k in range(part.slots_a + part.slots_b):
                o, c = rt.ell_o[k, i], rt.ell_c[k, i]
                go = t.ell_other[k, rt.node0 + i]
                assert (o < 0) == (go < 0)
                if o >= 0:
                    assert glob(o) == go
                    assert rt.act_elem[c] == t.ell_elem[k, rt.node0 + i]
        # every halo slot an element references is filled by exactly one bulk
        # copy of its owner's position (16-byte aligned addresses and sizes)
        used = {int(x) for x in rt.act_ab.reshape(-1) if rt.n_own <= x < rt.n_local}
        filled = {}
        recv = 0
        senders = 0
        for q, src in enumerate(part.ranks):
            for dst_rank, sb, db, nb in src.runs:
                assert sb % 16 == 0 and db % 16 == 0 and nb % 16 == 0 and nb > 0
                if dst_rank != r:
                    continue
                assert q != r
                senders |= 1 << q
                recv += nb
                for j in range(nb // 24):
                    d, sn = db // 24 + j, sb // 24 + j
                    assert d not in filled and rt.n_own <= d < rt.n_local
                    filled[d] = src.node0 + sn if sn < src.n_own else None
        assert recv == rt.halo_bytes and senders == rt.ack_from
        # interior elements (no halo endpoint) first, cut elements last
        is_halo = (rt.act_ab >= rt.n_own) & (rt.act_ab < rt.n_local)
        assert not is_halo[:rt.n_int].any() and is_halo[rt.n_int:].any(axis=1).all()
        for d in used:
            assert filled.get(d) == glob(d), (r, d)
    assert nxt == NF and leaf == t.n_leaves


def test_rank_smem_mirror_matches_library():
    from paper_2305_07030_b200.partition import smem_bytes
    for args in [(3375, 2197, 7098, 127, 700, 0), (1300, 1099, 3600, 80, 301, 1), (150, 150, 400, 7, 41, 0),
                 (0, 0, 0, 0, 14, 0), (1, 1, 0, 1, 15, 1), (63, 63, 400, 3, 20, 0), (3869, 1909, 6721, 482, 1302, 3)]:
        assert nat.lib().frb_rank_smem_bytes(*args) == smem_bytes(*args[:5], bool(args[5] & 1), bool(args[5] & 2))


def test_c2_networks_use_two_ranks_on_chip():
    """15^3 networks (config 2): a 2-CTA cluster keeps every array on chip
    (one CTA would need f_prev in global memory)."""
    t = fb.build_problem(frb.generate_lattice(15, 15, 15, 0.3, 0), frb.AffineBC(np.eye(3))).topo
    part, fglob, mglob = t.choose_cluster()
    assert part.C == 2 and not fglob and not mglob
    assert partition_smem_bytes(part, False) <= fb.SMEM_BUDGET < partition_smem_bytes(t.partition(1), False)


def test_c3_networks_fit_a_16_cluster_with_global_fprev():
    """100k-DOF networks (config 3): 16 ranks, f_prev in global memory."""
    t = fb.build_problem(frb.generate_lattice(32, 32, 32, 0.3, 0), frb.AffineBC(np.eye(3))).topo
    part, fglob, mglob = t.choose_cluster()
    assert part.C == 16 and fglob and mglob
    assert partition_smem_bytes(part, True) <= fb.SMEM_BUDGET


@pytest.mark.parametrize("n", [1, 7, 100, 129, 450, 1029, 6591, 24000])
@pytest.mark.parametrize("C", [1, 2, 3, 5, 16])
def test_tree_split_reproduces_numpy_sum(n, C):
    """The cluster split of the pairwise tree (local subtrees + exported
    roots + shared top program) gives np.sum's bits for any leaf split."""
    from paper_2305_07030_b200.plan import evaluate_split, reduction_plan, tree_split
    flat = reduction_plan(n)
    L = int(flat[0])
    if C > L:
        pytest.skip("more ranks than leaves")
    rng = np.random.default_rng(n * 31 + C)
    cuts = sorted(rng.choice(np.arange(1, L), C - 1, replace=False).tolist()) if C > 1 else []
    b = [0] + cuts + [L]
    ranges = list(zip(b[:-1], b[1:]))
    blocks = tree_split(flat, ranges)
    for _ in range(3):
        a = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
        assert evaluate_split(flat, blocks, ranges, a) == np.sum(a)
    assert len({int(bk[1]) for bk in blocks}) == 1 and len({int(bk[0]) for bk in blocks}) == 1


def test_pack_offsets_groups_and_dedup():
    nets = [frb.generate_lattice(6, 6, 6, 0.3, s) for s in range(4)] + [frb.generate_lattice(5, 5, 5, 0.3, 0)]
    b = frb.pack_batch(nets, [frb.AffineBC(np.eye(3))] * 5)
    assert list(b.node_base) == [0, 216, 432, 648, 864, 989]
    assert len({int(d["inc_base"]) for d in b.desc[:4]}) == 1      # shared topology tables
    assert b.arrays["inc"].shape[0] == 2 * (540 + 300)
    assert "act_EA" not in b.arrays                                  # uniform EA -> scalar
    assert all(d["flags"] & nat.PF_EA_UNIFORM for d in b.desc)
    assert len(b.groups) == 1 and b.groups[0]["cluster"] == 1 and b.groups[0]["count"] == 5
    assert sorted(b.arrays["order"].tolist()) == list(range(5))
    assert b.arrays["order"][-1] == 4                                # largest first
    g = b.groups[0]
    assert g["smem_bytes"] == max(partition_smem_bytes(p.topo.partition(1)) for p in b.problems)


def test_mixed_sizes_form_cluster_groups():
    nets = [frb.generate_lattice(16, 16, 16, 0.3, 0), frb.generate_lattice(6, 6, 6, 0.3, 0),
            frb.generate_lattice(32, 32, 32, 0.3, 0)]
    b = frb.pack_batch(nets, [frb.AffineBC(np.eye(3))] * 3)
    # groups: (cluster, f_prev in global memory); 32^3 needs both 16 ranks and global f_prev
    assert [(int(g["cluster"]), int(g["fprv_global"])) for g in b.groups] == [(1, 0), (2, 0), (16, 1)]
    assert [int(d["cluster"]) for d in b.desc] == [2, 1, 16]


def test_mixed_materials_carry_element_ea():
    net = gc.load("random90_fixed").network
    b = frb.pack_batch([net], [frb.AffineBC(np.eye(3))])
    assert "act_EA" in b.arrays and not (b.desc[0]["flags"] & nat.PF_EA_UNIFORM)


def test_pack_length_mismatch():
    with pytest.raises(ValueError):
        frb.pack_batch([frb.generate_lattice(3, 3, 3)], [])


def test_empty_batch():
    b = frb.pack_batch([], [])
    assert b.n_problems == 0
    assert frb.solve_batch(b) == []


def test_isolated_node_is_mass_error():
    net = frb.FiberNetwork(np.array([[0.0, 0, 0], [1, 0, 0], [2, 2, 2]]), np.array([[0, 1, 0]]),
                           [frb.Material(1, 1, 1)], frozenset({0}))
    with pytest.raises(frb.NetworkMassError):
        frb.pack_batch([net], [frb.AffineBC(np.eye(3))])


@pytest.mark.parametrize("name", ["random60", "random90_fixed", "lat6_general_F", "c1_7x7x8_uniax"])
def test_native_setup_bit_equal_to_numpy(name):
    """frb_setup_problem (native host setup, GIL-free) reproduces the numpy
    restatement of build_problem bit for bit: lengths, E*A, lumped masses in
    np.add.at order, dt base and volume (reference microsolver.py:170-193,
    302-335; network.py:154-172)."""
    import golden_cases as gc
    from paper_2305_07030_b200.microsolver import _lumped_node_mass
    net = gc.load(name).network
    p = fb.build_problem(net, frb.AffineBC(np.eye(3)))
    emod, area, rho = net.material_columns()
    L = net.reference_lengths()
    assert np.array_equal(p.L, L)
    assert np.array_equal(p.ea, emod * area)
    assert np.array_equal(p.node_mass, _lumped_node_mass(net)[p.node_order])
    assert np.array_equal(p.X, net.node_coords[p.node_order])
    assert p.dt_base == float(np.min(L * np.sqrt(rho / emod)))
    assert p.volume == net.volume


def test_packed_values_are_per_network_and_topology_tables_shared():
    """Networks of one lattice share the topology tables (inc_node / elem_ab
    stored once); coordinates, lengths and masses are per network."""
    nets = [frb.generate_lattice(5, 5, 5, 0.3, s) for s in range(3)]
    b = frb.pack_batch(nets, [frb.AffineBC(np.eye(3))] * 3)
    assert len(b.arrays["elem_ab"]) == nets[0].n_elements
    assert len(b.arrays["inc_node"]) == nets[0].n_nodes
    assert (b.desc["telem_base"] == 0).all() and (b.desc["tnode_base"] == 0).all()
    for i, net in enumerate(nets):
        eb = int(b.desc[i]["elem_base"])
        assert np.array_equal(b.arrays["elem_L"][eb:eb + net.n_elements], net.reference_lengths())


def test_zero_mass_node_raises_like_reference():
    X = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [5.0, 5, 5]])
    net = frb.FiberNetwork(X, np.array([[0, 1, 0], [1, 2, 0]]), [frb.Material(1, 1, 1)], frozenset({0}))
    with pytest.raises(frb.NetworkMassError, match="node 3 has zero mass"):
        frb.pack_batch([net], [frb.AffineBC(np.eye(3))])


@pytest.mark.parametrize("n,C", [(15, 2), (24, 8), (32, 16), (17, 3)])
def test_halo_runs_are_aligned_bulk_copies(n, C):
    """The BASELINE lattices' cluster partitions: every outgoing halo run is a
    legal cp.async.bulk (16-byte aligned source, destination and size) and
    the receiving ranks expect exactly the bytes that arrive."""
    t = fb.build_problem(frb.generate_lattice(n, n, n, 0.3, 1), frb.AffineBC(np.eye(3))).topo
    part = t.partition(C)
    recv = [0] * part.C
    for q, rt in enumerate(part.ranks):
        for dst, sb, db, nb in rt.runs:
            assert sb % 16 == 0 and db % 16 == 0 and nb % 16 == 0 and dst != q
            assert sb // 24 + nb // 24 <= rt.n_local + rt.n_fix + 1
            recv[dst] += nb
    assert recv == [rt.halo_bytes for rt in part.ranks]


def test_renumbered_network_packs_with_many_runs():
    """Random node numbering: nodes are halo to more than two ranks, which the
    run-based halo layout handles (round 1's two-target send table could not)."""
    net = frb.generate_lattice(16, 16, 16, 0.3, 1)
    perm = np.random.default_rng(0).permutation(net.n_nodes)
    el = net.elements.copy()
    el[:, :2] = perm[el[:, :2]]
    net2 = frb.FiberNetwork(net.node_coords[np.argsort(perm)], el, net.materials,
                            frozenset(int(perm[b]) for b in net.boundary_nodes))
    b = frb.pack_batch([net2], [frb.AffineBC(np.eye(3))])
    part = b.problems[0].topo.chosen()[0]
    assert part.C > 2
    assert sum(len(rt.runs) for rt in part.ranks) > 4 * part.C
