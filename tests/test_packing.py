"""Host packing invariants (no GPU): incidence order equals the reference's
bincount summation order, slot tables mirror the CSR, plans and SMEM sizes."""

import numpy as np
import pytest

import paper_2305_07030_b200 as frb
from paper_2305_07030_b200 import batch as fb
from paper_2305_07030_b200 import _native as nat
import golden_cases as gc


def _nets():
    yield frb.generate_lattice(5, 6, 7, 0.3, 1)
    yield gc.load("random90_fixed").network
    yield gc.load("lat2_allfixed").network


@pytest.mark.parametrize("net", list(_nets()))
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


@pytest.mark.parametrize("net", list(_nets()))
def test_slot_table_mirrors_csr(net):
    p = fb.build_problem(net, frb.AffineBC(np.eye(3)))
    t = p.topo
    for i in range(t.n_free_nodes):
        first, packed = t.inc_node[i]
        na, nb = packed & 0xffff, packed >> 16
        ent = t.inc[first:first + na + nb]
        a = [o for o in t.ell_other[:t.ell_slots_a, i] if o >= 0]
        b = [o for o in t.ell_other[t.ell_slots_a:, i] if o >= 0]
        assert a == list(ent[:na, 0]) and b == list(ent[na:, 0])
        # padding only at the end of each role block
        col = t.ell_other[:t.ell_slots_a, i]
        assert all(col[k] >= 0 for k in range(na)) and all(col[k] < 0 for k in range(na, t.ell_slots_a))


def test_pack_offsets_and_dedup():
    nets = [frb.generate_lattice(6, 6, 6, 0.3, s) for s in range(4)] + [frb.generate_lattice(5, 5, 5, 0.3, 0)]
    b = frb.pack_batch(nets, [frb.AffineBC(np.eye(3))] * 5)
    assert list(b.node_base) == [0, 216, 432, 648, 864, 989]
    # equal topologies share one incidence table
    assert len({int(d["inc_base"]) for d in b.desc[:4]}) == 1
    assert b.arrays["inc"].shape[0] == 2 * (540 + 300)
    assert b.smem_bytes == max(fb.cta_smem_bytes(p.n_free_nodes, len(p.topo.ff_elem), p.topo.n_leaves)
                               for p in b.problems)
    assert "ell_EA" not in b.arrays        # uniform EA -> scalar per problem
    assert all(d["flags"] & nat.PF_EA_UNIFORM for d in b.desc)
    assert b.desc.dtype.itemsize == 200


def test_mixed_materials_carry_slot_ea():
    net = gc.load("random90_fixed").network
    b = frb.pack_batch([net], [frb.AffineBC(np.eye(3))])
    assert "ell_EA" in b.arrays and not (b.desc[0]["flags"] & nat.PF_EA_UNIFORM)


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


@pytest.mark.parametrize("net", list(_nets()))
def test_free_free_coefficient_slots(net):
    p = fb.build_problem(net, frb.AffineBC(np.eye(3)))
    t = p.topo
    nfn = t.n_free_nodes
    for k in range(t.ell_slots_a + t.ell_slots_b):
        for i in range(nfn):
            o, c = t.ell_other[k, i], t.ell_c[k, i]
            if o < 0 or o >= nfn:
                assert c == -1
            else:
                a, b = t.ff_ab[c]
                assert {int(a), int(b)} == {i, int(o)}
                assert t.ff_elem[c] == t.ell_elem[k, i]
