"""Batch submit: pack many networks into one device batch and solve them with
persistent cluster-kernel launches.

Implements the spec'd ``batch`` module (reference ``SPEC.md:338-394``; there
is no batch code in the reference package itself):

* ``pack_batch(networks, bcs) -> Batch``
* ``solve_batch(batch, strategy, config) -> list[SolveResult]``
* strategies ``TeamBatched`` (the default: a device work queue, one team =
  one CTA cluster per network) and ``SerialReference`` (one team,
  problems in order).

Host setup per network restates ``build_problem`` (reference
``microsolver.py:302-335``) in vectorised form and adds what the kernel needs:
the per-node incidence lists (role a then role b, ascending element id -- the
summation order of ``np.bincount`` in ``_scatter_forces``, :214-218), the
pairwise-sum plan of the free-DOF count (plan.py), and the cluster partition
(partition.py).  Tables that depend only on topology are shared by every
network of that topology.

Layout is a PackedStorage in spirit (reference ``packed.py``): flat SoA arrays
with per-problem offsets, host space "a" (numpy) mirrored to device space "b"
(torch CUDA tensors) with explicit upload/download.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as nat
from .dofmap import build_dofmap
from .microsolver import (
    AdaptiveDamping, FixedDamping, SingularElementError, SolveResult, SolverConfig,
    _lumped_node_mass,
)
from .network import AffineBC, FiberNetwork
from .packed import PackedStorage
from .partition import RUN_WORDS, Partition, partition, partition_smem_bytes
from .plan import reduction_plan

__all__ = ["Batch", "DeviceBatch", "ExecutionStrategy", "NaiveLoop", "SerialReference",
           "TeamBatched", "pack_batch", "solve_batch", "build_problem", "DeviceResults"]

MAX_CTA_THREADS = 1024
CLUSTER_SIZES = (1, 2, 4, 8, 16)
# per-CTA dynamic SMEM budget (227 KB opt-in minus the kernel's static SMEM)
SMEM_BUDGET = 227 * 1024 - 4 * 1024
# most free DOFs per cluster rank before a larger cluster is considered; the
# SMEM budget usually decides first (15^3 networks need 2 ranks).  Fewer,
# fuller ranks win on heterogeneous batches: c4 156 -> 217 networks/s going
# from 3400 to 8000 (profiles/r01_configs.md), because large clusters cost
# SMs (a 16-CTA cluster fills a GPC) and exchange latency.
DOFS_PER_RANK = int(os.environ.get("FRB_DOFS_PER_RANK", "8000"))
# virtual clusters per launch group (frb200.h frb_group.gm_cap): groups of C
# plain CTAs exchanging through L2 on the SMs that hardware clusters of 8 or
# 16 CTAs leave idle (16-CTA clusters: 7 fit, 36 of 148 SMs idle -> 2 more).
# FRB_VIRTUAL=0 turns them off.
VIRTUAL_CAP = 4 if os.environ.get("FRB_VIRTUAL", "1") != "0" else 0


def dofs_per_thread_cap(threads: int, fprv_global: bool = False) -> int:
    """Register-resident DOFs per thread the kernel instantiates (frb200.h;
    24 exists only for the global-f_prev kernels of 256-thread CTAs)."""
    return 8 if threads > 768 else 12 if threads > 512 else 16 if (threads > 256 or not fprv_global) else 24


# ------------------------------------------------------------------ strategies

@dataclass(frozen=True)
class SerialReference:
    """Problems one after another on a single team."""


@dataclass(frozen=True)
class NaiveLoop:
    """Per-operation dispatch, the paper's naive baseline (SPEC.md:360,
    PAPER.md:71-74): problems strictly one after another, one kernel launch
    per line of the Fig. 1 loop with the kernel boundary as the cross-worker
    barrier, and the host checking convergence after every iteration
    (frb_naive_solve).  Bit-identical to TeamBatched.  On the device the
    workers of a line are all the GPU's threads; ``workers`` is kept for the
    spec's signature."""
    workers: int = 1

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")


@dataclass(frozen=True)
class TeamBatched:
    """Shared work queue; each team (a CTA cluster) runs whole solves
    (SPEC.md:361).  teams=None sizes the persistent grid by occupancy.

    team_size is the spec's lanes per team (any value >= 1).  On
    the device a lane is a thread and a team is one CTA per cluster rank, so
    the CTA gets ``cta_threads(team_size)`` threads: team_size rounded up to a
    whole number of 32-thread warps (at least 32, at most 1024).  The kernel
    template then runs the smallest of 256 / 512 / 768 / 1024 threads that
    holds it; results are bit-identical for every team size."""
    teams: int | None = None
    team_size: int | None = None

    def __post_init__(self):
        if self.teams is not None and self.teams < 1:
            raise ValueError("teams must be >= 1")
        if self.team_size is not None and not 1 <= self.team_size <= MAX_CTA_THREADS:
            raise ValueError(f"team_size must be in [1, {MAX_CTA_THREADS}] (lanes = CTA threads)")

    @staticmethod
    def cta_threads(team_size: int) -> int:
        return max(32, 32 * math.ceil(team_size / 32))


ExecutionStrategy = SerialReference | NaiveLoop | TeamBatched


# ------------------------------------------------------------------ host setup

@dataclass
class Topology:
    """Arrays that depend only on (elements, boundary) -- shared by every
    network of the same topology."""
    n_nodes: int
    n_free_nodes: int
    inc_node: np.ndarray         # (N, 2) int32: first entry, n_a | n_b << 16
    inc: np.ndarray              # (I, 2) int32: other endpoint, element id
    elem_ab: np.ndarray          # (M, 2) int32 solver node ids
    plan: np.ndarray             # int32 flat pairwise plan for nf
    n_leaves: int
    ell_other: np.ndarray        # (SA+SB, NF) int32 slot-major, -1 padding (solver ids)
    ell_elem: np.ndarray         # (SA+SB, NF) int32 element per slot (0 on padding)
    slots_a: int
    slots_b: int
    parts: dict = field(default_factory=dict)   # cluster size -> Partition
    _chosen: tuple | None = None

    def partition(self, C: int) -> Partition:
        if C not in self.parts:
            self.parts[C] = partition(self.n_nodes, self.n_free_nodes, self.elem_ab[:, 0].astype(np.int64),
                                      self.elem_ab[:, 1].astype(np.int64), self.ell_other, self.ell_elem,
                                      self.slots_a, self.slots_b, self.plan, C)
        return self.parts[C]

    def chosen(self) -> tuple[Partition, bool, bool]:
        """choose_cluster(), computed once per topology."""
        if self._chosen is None:
            self._chosen = self.choose_cluster()
        return self._chosen

    def choose_cluster(self) -> tuple[Partition, bool, bool]:
        """Smallest cluster with at most DOFS_PER_RANK free DOFs per rank whose
        ranks fit the SMEM budget (more ranks if SMEM demands it), keeping
        f_prev in SMEM whenever some cluster size allows it; otherwise the
        smallest cluster that fits with f_prev in global memory (32^3)."""
        nf = 3 * self.n_free_nodes
        want = max(1, math.ceil(nf / DOFS_PER_RANK))
        reasons = []
        # on-chip f_prev at any cluster size first; then f_prev (and the node
        # masses, frb_relax.cuh layout) in global memory
        for fprv_global, mass_global in ((False, False), (True, True)):
            for C in CLUSTER_SIZES:
                if C < want and C != CLUSTER_SIZES[-1]:
                    continue
                try:
                    part = self.partition(C)
                except ValueError as e:  # e.g. a node that is halo to more than two ranks
                    reasons.append(f"C={C}: {e}")
                    continue
                if partition_smem_bytes(part, fprv_global, mass_global) <= SMEM_BUDGET:
                    return part, fprv_global, mass_global
                reasons.append(f"C={C}{' (f_prev global)' if fprv_global else ''}"
                               f"{' (masses global)' if mass_global else ''}: "
                               f"{partition_smem_bytes(part, fprv_global, mass_global)} B of SMEM per rank")
        raise nat.NativeError(nat.FRB_E_TOO_LARGE,
                              f"network with {nf} free DOFs fits no cluster of {CLUSTER_SIZES} CTAs ("
                              + "; ".join(dict.fromkeys(reasons)) + ")")


def _topology(network: FiberNetwork, node_rank: np.ndarray, n_free_nodes: int) -> Topology:
    n = network.n_nodes
    m = network.n_elements
    ia = node_rank[network.elements[:, 0]]
    ib = node_rank[network.elements[:, 1]]
    na = np.bincount(ia, minlength=n)
    nb = np.bincount(ib, minlength=n)
    if m and max(na.max(), nb.max()) >= 1 << 15:
        raise ValueError("a node has more than 32767 incident elements in one role")
    node = np.concatenate([ia, ib])
    role = np.concatenate([np.zeros(m, np.int8), np.ones(m, np.int8)])
    elem = np.concatenate([np.arange(m), np.arange(m)])
    other = np.concatenate([ib, ia])
    order = np.lexsort((elem, role, node))
    inc = np.stack([other[order], elem[order]], axis=1).astype(np.int32)
    first = np.zeros(n, dtype=np.int64)
    np.cumsum((na + nb)[:-1], out=first[1:])
    inc_node = np.stack([first, na | (nb << 16)], axis=1).astype(np.int32)
    plan = reduction_plan(3 * n_free_nodes)
    # slot-major table of the free nodes: slot k < SA is the k-th role-a
    # incidence (ascending element), slot SA + k the k-th role-b incidence
    snode, srole = node[order], role[order]
    grp = snode.astype(np.int64) * 2 + srole
    starts = np.flatnonzero(np.r_[True, grp[1:] != grp[:-1]]) if len(grp) else np.zeros(0, np.int64)
    rank = np.arange(len(grp)) - np.repeat(starts, np.diff(np.r_[starts, len(grp)]))
    nfn = n_free_nodes
    sa = int(na[:nfn].max()) if nfn and m else 0
    sb = int(nb[:nfn].max()) if nfn and m else 0
    ell_other = np.full((sa + sb, nfn), -1, dtype=np.int32)
    ell_elem = np.zeros((sa + sb, nfn), dtype=np.int32)
    free = snode < nfn
    slot = np.where(srole == 0, rank, sa + rank)[free]
    ell_other[slot, snode[free]] = other[order][free]
    ell_elem[slot, snode[free]] = elem[order][free]
    return Topology(n_nodes=n, n_free_nodes=n_free_nodes, inc_node=inc_node, inc=inc,
                    elem_ab=np.stack([ia, ib], axis=1).astype(np.int32), plan=plan,
                    n_leaves=int(plan[0]), ell_other=ell_other, ell_elem=ell_elem,
                    slots_a=sa, slots_b=sb)


@dataclass
class _TopoEntry:
    """One cached topology: the connectivity it was built from (to verify a
    sampled-key hit), the DOF map's node order and the device tables."""
    elements: np.ndarray
    boundary: frozenset
    order: np.ndarray
    topo: Topology
    key: bytes
    elements_bytes: bytes = b""


_TOPO_CACHE: dict[bytes, list] = {}
_TOPO_LOCK = threading.Lock()
_TOPO_SERIAL = [0]


def _topo_entry(network: FiberNetwork) -> _TopoEntry:
    """The topology of a network, built once per distinct (connectivity,
    boundary set).  Lookup hashes a strided sample of the element rows and
    confirms a hit with a full comparison, so packing thousands of networks
    of one lattice costs one memcmp each instead of hashing megabytes."""
    n, el = network.n_nodes, network.elements
    m = len(el)
    h = hashlib.blake2b(digest_size=16)
    h.update(np.int64([n, m, len(network.boundary_nodes), hash(network.boundary_nodes)]).tobytes())
    h.update(el[::max(1, m // 256)].tobytes())
    k = h.digest()
    with _TOPO_LOCK:  # one build per topology even when networks are packed on several threads
        for ent in _TOPO_CACHE.get(k, ()):
            # confirm the sampled-key hit: byte comparison of the whole
            # element table (C-contiguous int64, FiberNetwork guarantees it)
            if ent.boundary == network.boundary_nodes and (
                    ent.elements is el or ent.elements_bytes == el.tobytes()):
                return ent
        dm = build_dofmap(n, network.boundary_nodes)
        order = dm.node_order
        rank = np.empty(n, dtype=np.int64)
        rank[order] = np.arange(n)
        topo = _topology(network, rank, dm.n_free // 3)
        if sum(len(v) for v in _TOPO_CACHE.values()) > 4096:
            _TOPO_CACHE.clear()
        _TOPO_SERIAL[0] += 1
        ent = _TopoEntry(elements=el, boundary=network.boundary_nodes, order=order, topo=topo,
                         key=k + _TOPO_SERIAL[0].to_bytes(8, "little"), elements_bytes=el.tobytes())
        _TOPO_CACHE.setdefault(k, []).append(ent)
        return ent


@dataclass
class HostProblem:
    """Solver-order setup of one network (ProblemSetup, microsolver.py:138-163).
    X / node_mass / L / ea are views into the packed batch arrays once packed."""
    network: FiberNetwork
    F: np.ndarray
    node_order: np.ndarray       # solver position -> original node
    topo_key: bytes
    topo: Topology
    check_mass: bool = True
    X: np.ndarray = None         # (N, 3) solver order
    node_mass: np.ndarray = None # (N,) solver order
    dt_base: float = math.nan    # min_e L sqrt(rho/E); dt = dt_safety * dt_base
    L: np.ndarray = None         # reference lengths, original element order
    ea: np.ndarray = None        # E*A per element
    volume: float = math.nan     # FiberNetwork.volume

    @property
    def n_nodes(self) -> int:
        return self.network.n_nodes

    @property
    def n_free_nodes(self) -> int:
        return self.topo.n_free_nodes


_MAT_CACHE: dict = {}


def _material_table(network: FiberNetwork) -> np.ndarray:
    """(n_materials, 3) float64 rows (E, A, rho), cached per material tuple."""
    key = tuple(network.materials)
    tab = _MAT_CACHE.get(key)
    if tab is None:
        tab = np.ascontiguousarray(np.array([[m.elastic_modulus, m.cross_section_area, m.density]
                                             for m in network.materials], dtype=np.float64).reshape(-1, 3))
        if len(_MAT_CACHE) > 1024:
            _MAT_CACHE.clear()
        _MAT_CACHE[key] = tab
    return tab


def _native_setup(p: HostProblem, X, mass, L, EA, act_elem=None, act_L=None, act_EA=None) -> int:
    """Fill one problem's packed values with frb_setup_problem (GIL released
    while it runs).  Returns the zero-mass node or -1; sets dt_base / volume."""
    net = p.network
    n, m = net.n_nodes, net.n_elements
    mats = _material_table(net)
    scal = np.empty(3)
    scratch = np.empty(max(n, 1))
    ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    n_act = 0 if act_elem is None else len(act_elem)
    nat.check(nat.lib().frb_setup_problem(
        n, m, ptr(net.node_coords), ptr(net.elements), ptr(mats), len(mats), ptr(p.node_order),
        ptr(act_elem), n_act, ptr(X), ptr(mass), ptr(L), ptr(EA), ptr(act_L), ptr(act_EA),
        ptr(scal), ptr(scratch)))
    p.dt_base = float(scal[0])
    p.volume = float(net.rve_volume) if net.rve_volume is not None else float(scal[1])
    p.X, p.node_mass, p.L, p.ea = X.reshape(n, 3), mass, L, EA
    return int(scal[2])


def _mass_error(node: int):
    """compute_lumped_mass's error (microsolver.py:179-181); node in original order."""
    from .microsolver import NetworkMassError
    return NetworkMassError(f"node {node} has zero mass (no incident elements)")


def _meta(network: FiberNetwork, bc: AffineBC, check_mass: bool = True) -> HostProblem:
    ent = _topo_entry(network)
    return HostProblem(network=network, F=np.asarray(bc.deformation_gradient, dtype=np.float64),
                       node_order=ent.order, topo_key=ent.key, topo=ent.topo, check_mass=check_mass)


def build_problem(network: FiberNetwork, bc: AffineBC, check_mass: bool = True) -> HostProblem:
    """Host setup for one network (reference build_problem, :302-335): the
    DOF map and device topology (cached per topology) plus the native
    per-network values (frb_setup_problem: lengths, lumped mass in np.add.at
    order, dt base, volume -- bit-identical to the reference's numpy).

    Raises NetworkMassError for a node without incident elements (like
    compute_lumped_mass, :179-181)."""
    p = _meta(network, bc, check_mass)
    n, m = network.n_nodes, network.n_elements
    bad = _native_setup(p, np.empty(3 * n), np.empty(n), np.empty(m), np.empty(m))
    if check_mass and bad >= 0:
        raise _mass_error(bad)
    if not check_mass:
        p.node_mass = np.ones(n)
    return p


def setup_threads() -> int:
    """Host threads for the per-network setup (FRB_SETUP_THREADS, default all
    cores): frb_setup_problem runs with the GIL released."""
    env = os.environ.get("FRB_SETUP_THREADS")
    return max(1, int(env)) if env else (os.cpu_count() or 1)


# ------------------------------------------------------------------ batch

@dataclass
class Batch:
    """Host-side packed batch (space "a").  ``packed_state`` exposes the
    spec's per-problem PackedStorage rows for u, v, a, f_int, m (built on
    first access).  ``setup_s`` is the host setup time of pack_batch."""
    networks: list
    bcs: list
    problems: list                     # HostProblem per network
    desc: np.ndarray                   # PROBLEM_DTYPE records (dt filled per solve)
    parts: np.ndarray                  # PART_DTYPE records
    groups: np.ndarray                 # GROUP_DTYPE records (host)
    arrays: dict                       # flat host arrays uploaded to the device
    node_base: np.ndarray              # (P+1,) int64 node offsets
    _packed_state: dict | None = field(default=None, repr=False)
    _orig_rows: np.ndarray | None = field(default=None, repr=False)  # solver -> original node rows
    _orig_rows_dev: dict = field(default_factory=dict, repr=False)    # the same per device
    pinned: dict | None = field(default=None, repr=False)
    setup_s: float = math.nan

    @property
    def n_problems(self) -> int:
        return len(self.problems)

    def pin(self) -> "Batch":
        """Page-lock the packed arrays once so uploads are pure DMA."""
        torch = _torch()
        self.pinned = {k: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                       for k, a in self.arrays.items()}
        return self

    @property
    def packed_state(self) -> dict:
        if self._packed_state is None:
            rows = [np.zeros(3 * p.n_nodes) for p in self.problems]
            st = {k: PackedStorage(rows) for k in ("u", "v", "a", "f_int")}
            st["m"] = PackedStorage([np.repeat(p.node_mass[np.argsort(p.node_order)], 3)
                                     for p in self.problems])
            self._packed_state = st
        return self._packed_state

    def to_device(self, device=None) -> "DeviceBatch":
        return DeviceBatch.upload(self, device)


def pack_batch(networks: Sequence[FiberNetwork], bcs: Sequence[AffineBC]) -> Batch:
    """Build the packed batch: topologies once (cached),
    then every network's values written straight into the packed arrays by
    the native setup on a pool of host threads."""
    import time
    if len(networks) != len(bcs):
        raise ValueError(f"networks and bcs differ in length ({len(networks)} vs {len(bcs)})")
    t0 = time.perf_counter()
    metas = [_meta(net, bc) for net, bc in zip(networks, bcs)]
    batch = _pack(list(networks), list(bcs), metas)
    batch.setup_s = time.perf_counter() - t0
    return batch


def _cat(parts, dtype, width=None):
    if not parts:
        return np.zeros((0,) if width is None else (0, width), dtype=dtype)
    return np.ascontiguousarray(np.concatenate(parts).astype(dtype, copy=False))


def _group_threads(max_own_dofs: int, max_rank_leaves: int, n_problems: int, cluster: int,
                   fprv_global: bool = False) -> int:
    """Threads per CTA for a group: 8 per pairwise leaf of a rank (one per
    accumulator chain) and at most 16 register-held DOFs per thread; more
    threads when too few problems fill the GPU (latency matters more than
    throughput then).  Measured on c2 (15^3, 2 ranks): 256 threads beat 512
    (82.9 vs 84.9 ms; tools/sweep_c2.py)."""
    need = max(64, min(8 * max_rank_leaves, 512), math.ceil(max_own_dofs / 16))  # more leaves: chain rounds
    if n_problems * cluster < 148:
        need = max(need, min(512, 32 * math.ceil(max_own_dofs / 32)))
    if fprv_global:  # 32^3 on 16 ranks: 768 threads 144.3 networks/s, 512 143.4, 256 ~20 % slower
        need = max(need, int(os.environ.get("FRB_FG_THREADS", "768")))
    threads = min(MAX_CTA_THREADS, 32 * math.ceil(need / 32))
    while max_own_dofs > dofs_per_thread_cap(threads, fprv_global) * threads and threads < MAX_CTA_THREADS:
        threads += 32
    return threads


def _pack(networks, bcs, probs, cluster: int | None = None) -> Batch:
    """Pack problems whose topology is known (HostProblem from _meta).

    Tables that depend only on the topology (incidence CSR, element
    endpoints, per-rank slot tables, trees) are stored once per topology;
    per-network values (coordinates, masses, lengths, E*A, active-element
    values) are written into the packed arrays by frb_setup_problem on a pool
    of host threads."""
    P = len(probs)
    desc = np.zeros(P, dtype=nat.PROBLEM_DTYPE)
    node_base = np.zeros(P + 1, dtype=np.int64)
    elem_base = np.zeros(P + 1, dtype=np.int64)
    actv_base = np.zeros(P + 1, dtype=np.int64)
    plan_slot: dict[int, int] = {}
    shared_slot: dict[tuple, list] = {}       # (topo, C) -> per-rank base offsets
    topo_slot: dict[bytes, tuple] = {}        # topo -> (inc base, topo node base, topo elem base)
    inc, plans, ell, act_ab, halo_g, runs, fix_g, trees, inc_node, elem_ab = ([] for _ in range(10))
    n_inc = n_plan = n_ell = n_act = n_halo = n_runs = n_fix = n_tree = n_tnode = n_telem = 0
    parts_rows = []
    part_of, fglob_of, mglob_of, act_of, cols = [], [], [], [], []
    n_parts = 0
    for i, p in enumerate(probs):
        t = p.topo
        part, fglob, mglob = (t.partition(cluster), False, False) if cluster else t.chosen()
        mglob_of.append(mglob)
        part_of.append(part)
        fglob_of.append(fglob)
        if p.topo_key not in topo_slot:
            topo_slot[p.topo_key] = (n_inc, n_tnode, n_telem)
            inc.append(t.inc)
            inc_node.append(t.inc_node)
            elem_ab.append(t.elem_ab)
            n_inc += len(t.inc)
            n_tnode += len(t.inc_node)
            n_telem += len(t.elem_ab)
        key = (p.topo_key, part.C)
        if key not in shared_slot:
            bases = []
            for rt in part.ranks:
                bases.append((n_ell, n_act, n_halo, n_runs, n_fix, n_tree))
                trees.append(rt.tree)
                n_tree += len(rt.tree)
                ell.append(rt.ell.reshape(-1))
                act_ab.append(rt.act_ab[:, 0].astype(np.uint32) | (rt.act_ab[:, 1].astype(np.uint32) << 16))
                halo_g.append(rt.halo_g)
                runs.append(rt.runs)
                fix_g.append(rt.fix_g)
                n_ell += rt.ell_o.size
                n_act += len(rt.act_ab)
                n_halo += len(rt.halo_g)
                n_runs += len(rt.runs)
                n_fix += rt.n_fix
            rows = np.zeros(len(part.ranks), dtype=nat.PART_DTYPE)  # identical for every network of (topo, C)
            off = 0
            for row, rt, (b_ell, b_act, b_halo, b_runs, b_fix, b_tree) in zip(rows, part.ranks, bases):
                row["ell_base"], row["act_base"], row["actv_off"] = b_ell, b_act, off
                row["halo_base"], row["runs_base"], row["fix_base"] = b_halo, b_runs, b_fix
                row["n_runs"], row["halo_bytes"], row["ack_from"] = len(rt.runs), rt.halo_bytes, rt.ack_from
                row["n_int"] = rt.n_int
                row["n_fix"] = rt.n_fix
                row["tree_base"], row["tree_len"] = b_tree, len(rt.tree)
                row["node0"], row["n_own"], row["n_local"], row["n_act"] = rt.node0, rt.n_own, rt.n_local, rt.n_act
                row["ell_stride"], row["slots_a"], row["slots_b"] = rt.stride, part.slots_a, part.slots_b
                row["leaf0"], row["n_leaves"] = rt.leaf0, rt.n_leaves
                off += rt.n_act
            shared_slot[key] = (rows, np.concatenate([rt.act_elem for rt in part.ranks]).astype(np.int64), off)
        rows, act_elem, n_actv = shared_slot[key]
        act_of.append(act_elem)
        nf = 3 * t.n_free_nodes
        if nf not in plan_slot:
            plan_slot[nf] = n_plan
            plans.append(t.plan)
            n_plan += len(t.plan)
        cols.append(topo_slot[p.topo_key] + (plan_slot[nf], n_parts, t.n_free_nodes, part.C))
        parts_rows.append(rows)
        n_parts += len(rows)
        actv_base[i + 1] = actv_base[i] + n_actv
        node_base[i + 1] = node_base[i] + p.n_nodes
        elem_base[i + 1] = elem_base[i] + p.network.n_elements
    if P:
        cv = np.array(cols, dtype=np.int64).reshape(P, 7)
        desc["node_base"], desc["elem_base"], desc["actv_base"] = node_base[:-1], elem_base[:-1], actv_base[:-1]
        desc["inc_base"], desc["tnode_base"], desc["telem_base"] = cv[:, 0], cv[:, 1], cv[:, 2]
        desc["plan_base"], desc["part_base"], desc["n_free_nodes"], desc["cluster"] = cv[:, 3], cv[:, 4], cv[:, 5], \
            cv[:, 6]
        desc["n_nodes"], desc["n_elems"] = np.diff(node_base), np.diff(elem_base)
        desc["F"] = np.array([p.F.reshape(9) for p in probs])

    # per-network values, native, straight into the packed arrays
    X = np.empty(3 * int(node_base[-1]))
    mass = np.empty(int(node_base[-1]))
    EL = np.empty(int(elem_base[-1]))
    EA = np.empty(int(elem_base[-1]))
    act_L = np.empty(int(actv_base[-1]))
    act_EA = np.empty(int(actv_base[-1]))

    items = np.zeros(P, dtype=nat.SETUP_ITEM_DTYPE)
    mats = [_material_table(p.network) for p in probs]
    it = items
    it["coords"] = [p.network.node_coords.ctypes.data for p in probs]
    it["elements"] = [p.network.elements.ctypes.data for p in probs]
    it["materials"] = [m.ctypes.data for m in mats]
    it["node_order"] = [p.node_order.ctypes.data for p in probs]
    it["act_elem"] = [a.ctypes.data for a in act_of]
    it["n_act"] = [len(a) for a in act_of]
    it["n_nodes"] = np.diff(node_base)
    it["n_elems"] = np.diff(elem_base)
    it["n_materials"] = [len(m) for m in mats]
    # output pointers: offsets into the packed arrays (vectorised)
    it["X_out"] = X.ctypes.data + 24 * node_base[:-1]
    it["mass_out"] = mass.ctypes.data + 8 * node_base[:-1]
    it["L_out"] = EL.ctypes.data + 8 * elem_base[:-1]
    it["EA_out"] = EA.ctypes.data + 8 * elem_base[:-1]
    it["act_L_out"] = act_L.ctypes.data + 8 * actv_base[:-1]
    it["act_EA_out"] = act_EA.ctypes.data + 8 * actv_base[:-1]
    nthr = min(setup_threads(), max(P, 1))
    scratch = np.empty(int(node_base[-1]) + 1)  # per-network original-order masses
    it["mass_scratch"] = scratch.ctypes.data + 8 * node_base[:-1]
    nat.check(nat.lib().frb_setup_batch(items.ctypes.data, P, nthr))
    for i, p in enumerate(probs):
        dt_base, vol, bad = items["scalars"][i]
        nb, eb, ab = int(node_base[i]), int(elem_base[i]), int(actv_base[i])
        p.dt_base = float(dt_base)
        p.volume = float(p.network.rve_volume) if p.network.rve_volume is not None else float(vol)
        p.X = X[3 * nb:3 * (nb + p.n_nodes)].reshape(-1, 3)
        p.node_mass = mass[nb:nb + p.n_nodes]
        p.L = EL[eb:eb + p.network.n_elements]
        p.ea = EA[eb:eb + p.network.n_elements]
        if not p.check_mass:
            p.node_mass[:] = 1.0
        elif bad >= 0:
            raise _mass_error(int(bad))
    uniform = [bool(p.ea.size == 0 or (p.ea == p.ea[0]).all()) for p in probs]
    any_nonuniform = not all(uniform)
    if P:
        desc["flags"] = np.where(uniform, nat.PF_EA_UNIFORM, 0) | np.where(mglob_of, nat.PF_MASS_GLOBAL, 0)  # informational
        desc["volume"] = [p.volume for p in probs]
        desc["ea"] = [p.ea[0] if p.ea.size else 0.0 for p in probs]

    parts = np.concatenate(parts_rows) if parts_rows else np.zeros(0, nat.PART_DTYPE)
    # launch groups by cluster size, longest problems first inside a group
    # (the work queue hands them out in this order: longest-first keeps the
    # tail short).  Cost estimate: N^(4/3) (nodes x iterations, which grow
    # with the network's linear size) x the load |F - I|, which sets how far
    # the relaxation has to travel (32^3: uniaxial 2,519, shear 6,805
    # iterations); it only orders the queue, results do not depend on it.
    if P:
        Fs = np.stack([np.asarray(p.F, dtype=np.float64).reshape(3, 3) for p in probs])
        load = np.maximum(np.linalg.norm(Fs - np.eye(3), axis=(1, 2)), 1e-3)
        est = np.array([p.n_nodes for p in probs], dtype=np.float64) ** (4.0 / 3.0) * load

    def cost(i):
        return -est[i]

    order, groups = [], []
    for C, fglob in sorted({(pt.C, fg) for pt, fg in zip(part_of, fglob_of)}):
        ids = [i for i in range(P) if part_of[i].C == C and fglob_of[i] == fglob]
        ids.sort(key=cost)
        smem = max(partition_smem_bytes(part_of[i], fglob, mglob_of[i]) for i in ids)
        own = max(3 * rt.n_own for i in ids for rt in part_of[i].ranks)
        leaves = max(rt.n_leaves for i in ids for rt in part_of[i].ranks)
        g = np.zeros((), dtype=nat.GROUP_DTYPE)
        g["cluster"], g["first"], g["count"] = C, len(order), len(ids)
        g["block_threads"] = _group_threads(own, leaves, len(ids), C, fglob)
        g["smem_bytes"], g["max_own_dofs"] = smem, own
        g["fprv_global"] = int(fglob)
        g["max_rank_leaves"] = leaves
        if C >= 8:  # virtual clusters may run on the SMs these clusters leave idle (frb200.h frb_group)
            pn = max(rt.n_local + rt.n_fix for i in ids for rt in part_of[i].ranks)
            ts = max(int(rt.tree[1]) for i in ids for rt in part_of[i].ranks)
            g["gm_cap"] = VIRTUAL_CAP if not os.environ.get("FRB_VIRTUAL_ONLY") else 9
            if os.environ.get("FRB_VIRTUAL_ONLY"):
                g["flags"] |= nat.GF_VIRTUAL_ONLY
            g["gm_ex_stride"] = 4 * math.ceil((3 * ts + 64) / 4)
            g["gm_mir_stride"] = 2 * (2 * math.ceil(3 * pn / 2))
        groups.append(g)
        order.extend(ids)
    arrays = dict(
        X=X, node_mass=mass,
        inc_node=_cat(inc_node, np.int32, 2), inc=_cat(inc, np.int32, 2),
        elem_ab=_cat(elem_ab, np.int32, 2), elem_L=EL,
        plans=_cat(plans, np.int32),
        ell=_cat(ell, np.uint32).view(np.int32), fix_g=_cat(fix_g, np.int32),
        act_ab=_cat(act_ab, np.uint32).view(np.int32), act_L=act_L,
        halo_g=_cat(halo_g, np.int32), runs=_cat(runs, np.int32, RUN_WORDS), trees=_cat(trees, np.int32),
        order=np.asarray(order, dtype=np.int32),
        problems=desc.view(np.uint8).copy(), parts=parts.view(np.uint8).copy(),
    )
    if any_nonuniform:  # otherwise E*A travels in the descriptor (FRB_PF_EA_UNIFORM)
        arrays["elem_EA"] = EA
        arrays["act_EA"] = act_EA
    return Batch(networks=networks, bcs=bcs, problems=probs, desc=desc, parts=parts,
                 groups=np.array(groups, dtype=nat.GROUP_DTYPE), arrays=arrays, node_base=node_base)


# ------------------------------------------------------------------ device

def _torch():
    import torch
    return torch


@dataclass
class DeviceResults:
    u: object            # torch float64 [3*sumN], solver order
    f: object
    results: object      # torch uint8 [P * 144]
    node_base: np.ndarray

    def host_results(self) -> np.ndarray:
        return self.results.cpu().numpy().view(nat.RESULT_DTYPE)


@dataclass
class DeviceBatch:
    """Device mirror (space "b") of a Batch; every array a torch CUDA tensor."""
    host: Batch
    device: object
    t: dict

    @classmethod
    def upload(cls, batch: Batch, device=None, pin: bool = True) -> "DeviceBatch":
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("solve_batch needs a CUDA device (no CPU fallback)")
        device = torch.device(device if device is not None else "cuda")
        t = {}
        for k, a in batch.arrays.items():
            if batch.pinned is not None:
                src = batch.pinned[k]
            else:
                src = torch.from_numpy(np.ascontiguousarray(a))
                if pin:
                    src = src.pin_memory()
            t[k] = src.to(device, non_blocking=True)
        return cls(host=batch, device=device, t=t)

    def set_deformation(self, Fs) -> None:
        """FE2 macro step: new deformation gradients for every network, the
        packed geometry and topology stay resident (only the per-problem
        descriptor changes; the prescribed displacements are formed on the
        device from F, microsolver.py:320-322).  Takes effect at the next
        prepare()/solve()."""
        h = self.host
        bcs = [b if isinstance(b, AffineBC) else AffineBC(np.asarray(b, dtype=np.float64)) for b in Fs]
        if len(bcs) != h.n_problems:
            raise ValueError(f"expected {h.n_problems} deformation gradients, got {len(bcs)}")
        for i, bc in enumerate(bcs):
            h.desc[i]["F"] = np.asarray(bc.deformation_gradient, dtype=np.float64).reshape(9)
            h.problems[i].F = np.asarray(bc.deformation_gradient, dtype=np.float64)
        h.bcs = bcs

    def prepare(self, cfg: SolverConfig, strategy=None, phase_profile: bool = False) -> "Launch":
        """Allocate outputs and build the launch arguments once; the
        returned Launch can be replayed (bench) or run once (solve)."""
        torch = _torch()
        strategy = strategy or TeamBatched()
        h = self.host
        groups = h.groups.copy()
        for g in groups:
            if isinstance(strategy, TeamBatched):
                if strategy.team_size is not None:
                    g["block_threads"] = TeamBatched.cta_threads(strategy.team_size)
                if strategy.teams is not None:
                    g["grid_clusters"] = strategy.teams
            elif isinstance(strategy, SerialReference):
                g["grid_clusters"] = 1
                g["flags"] |= nat.GF_SERIAL  # groups one after another on the caller's stream
            T = int(g["block_threads"])
            if int(g["max_own_dofs"]) > dofs_per_thread_cap(T, bool(g["fprv_global"])) * T:
                raise nat.NativeError(nat.FRB_E_TOO_LARGE,
                                      f"team_size {T} cannot hold {int(g['max_own_dofs'])} own DOFs")

        # exchange scratch of the virtual clusters, one slice per eligible group
        xoff = 0
        for g in groups:
            if int(g["gm_cap"]) > 0:
                cap, C = int(g["gm_cap"]), int(g["cluster"])
                g["xchg_off"] = xoff
                xoff += 4096 * cap + 8 * (cap * 2 * int(g["gm_ex_stride"]) + cap * C * int(g["gm_mir_stride"]))
                xoff = 256 * math.ceil(xoff / 256)
        n = int(h.node_base[-1])
        dev = self.device
        xchg = torch.empty(max(xoff, 1), dtype=torch.uint8, device=dev) if xoff else None
        u = torch.empty(3 * n, dtype=torch.float64, device=dev)
        f = torch.empty(3 * n, dtype=torch.float64, device=dev)
        work = torch.empty(3 * n + 1, dtype=torch.float64, device=dev)
        res = torch.zeros(h.n_problems * nat.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        queue = torch.zeros(max(len(groups), 1), dtype=torch.int32, device=dev)
        desc = h.desc.copy()
        desc["dt"] = [cfg.dt_safety * p.dt_base for p in h.problems]
        desc_t = torch.from_numpy(desc.view(np.uint8).copy()).to(dev)
        groups_c = np.ascontiguousarray(groups)
        fb = nat.FrbBatch()
        fb.n_problems = h.n_problems
        fb.n_groups = len(groups)
        fb.groups = groups_c.ctypes.data
        t = self.t
        for k in ("parts", "order", "X", "node_mass", "inc_node", "inc", "elem_ab", "elem_L", "elem_EA",
                  "plans", "ell", "act_ab", "act_L", "act_EA", "halo_g", "runs", "fix_g", "trees"):
            setattr(fb, k, t[k].data_ptr() if k in t and t[k].numel() else None)
        fb.problems = desc_t.data_ptr()
        fb.u, fb.f, fb.work = u.data_ptr(), f.data_ptr(), work.data_ptr()
        fb.results, fb.queue = res.data_ptr(), queue.data_ptr()
        fb.xchg = xchg.data_ptr() if xchg is not None else None
        phase = None
        if phase_profile:
            phase = torch.zeros(nat.PHASES * 148 * 16, dtype=torch.int64, device=dev)
            fb.phase_cycles = phase.data_ptr()
        naive = None
        if isinstance(strategy, NaiveLoop):
            need = max((int(nat.lib().frb_naive_scratch_doubles(p.n_nodes, p.network.n_elements, p.n_free_nodes))
                        for p in h.problems), default=1)
            naive = torch.empty(need, dtype=torch.float64, device=dev)
        return Launch(self, fb, config_struct(cfg), groups_c,
                      DeviceResults(u=u, f=f, results=res, node_base=h.node_base),
                      keep=(desc_t, queue, work, groups_c, xchg), phase=phase, naive=naive)

    def solve(self, cfg: SolverConfig, strategy=None, stream=None) -> DeviceResults:
        """Launch the persistent kernels; returns device-resident results
        (asynchronous on the current torch stream)."""
        launch = self.prepare(cfg, strategy)
        launch.run(stream)
        return launch.out


@dataclass
class Launch:
    dbatch: DeviceBatch
    fb: nat.FrbBatch
    fc: nat.FrbConfig
    groups: np.ndarray
    out: DeviceResults
    keep: tuple = ()
    phase: object = None
    naive: object = None          # NaiveLoop scratch (per-operation strategy)
    kernel_launches: int = 0      # relaxation kernels the last run() launched

    @property
    def threads(self) -> int:
        return int(self.groups["block_threads"].max()) if len(self.groups) else 0

    def run(self, stream=None):
        """One frb_solve_batch call (one kernel launch per group) on `stream`."""
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.dbatch.device)
        if self.naive is not None:  # NaiveLoop: problems one after another, one launch per line
            for p in range(self.fb.n_problems):
                nat.check(nat.lib().frb_naive_solve(C.byref(self.fb), C.byref(self.fc), p,
                                                    C.c_void_p(self.naive.data_ptr()), self.naive.numel(),
                                                    C.c_void_p(s.cuda_stream)))
            return
        nat.check(nat.lib().frb_solve_batch(C.byref(self.fb), C.byref(self.fc), C.c_void_p(s.cuda_stream)))
        self.kernel_launches = int(nat.lib().frb_solve_launches())  # hardware + virtual cluster kernels


def config_struct(cfg: SolverConfig) -> nat.FrbConfig:
    c = nat.FrbConfig()
    c.tol_rel, c.tol_abs, c.dt_safety = cfg.tol_rel, cfg.tol_abs, cfg.dt_safety
    if isinstance(cfg.damping, FixedDamping):
        c.damping, c.damping_c = nat.DAMPING_FIXED, float(cfg.damping.c)
    elif isinstance(cfg.damping, AdaptiveDamping):
        c.damping, c.damping_c = nat.DAMPING_ADAPTIVE, 0.0
    else:
        raise TypeError(f"unknown damping mode {cfg.damping!r}")
    c.max_iters = cfg.max_iters
    c.energy_check_interval = cfg.energy_check_interval
    c.bc_ramp_iters = cfg.bc_ramp_iters
    return c


def results_to_solve_results(batch: Batch, dres: DeviceResults, raise_singular: bool = True):
    """Download and unpermute (DofMap.unpermute, dofmap.py:33-38).

    The results' ``u`` are views of one page-locked buffer per call (no host
    copy); it is released when the last of them is dropped, so a caller that
    keeps a few results of a large batch should keep ``np.copy(r.u)``."""
    torch = _torch()
    rec = dres.host_results()
    # solver -> original node order as one row gather on the device, then one
    # pinned download and a copy the results own (the pinned buffer is reused)
    if batch._orig_rows is None:
        rows = np.empty(int(batch.node_base[-1]), dtype=np.int64)
        for i, p in enumerate(batch.problems):
            b0 = int(batch.node_base[i])
            rows[b0 + p.node_order] = b0 + np.arange(len(p.node_order))
        batch._orig_rows = rows
    key = str(dres.u.device)
    rows_t = batch._orig_rows_dev.get(key)
    if rows_t is None:
        rows_t = batch._orig_rows_dev[key] = torch.from_numpy(batch._orig_rows).to(dres.u.device)
    u_dev = dres.u.view(-1, 3).index_select(0, rows_t).view(-1)
    # one D2H into a fresh pinned buffer that the results own (their u are
    # views of it; torch's host allocator caches the block, so once the
    # previous call's results are dropped the next call reuses it: no host
    # copy and no page-locking per call)
    u_pin = torch.empty(u_dev.shape, dtype=u_dev.dtype, pin_memory=True)
    u_pin.copy_(u_dev)
    u_orig = u_pin.numpy()
    nb = (3 * batch.node_base).tolist()
    status = rec["status"].tolist()
    conv = rec["converged"].astype(bool).tolist()
    iters = rec["iters"].tolist()
    fres = rec["final_residual"].tolist()
    rref = rec["r_ref"].tolist()
    eres = rec["energy_residual"].tolist()
    stress = np.array(rec["avg_stress"], dtype=np.float64).reshape(-1, 3, 3)
    out = []
    first_bad = None
    for i in range(batch.n_problems):
        if status[i] == nat.STATUS_SINGULAR:
            if first_bad is None:
                first_bad = (i, int(rec["bad_element"][i]))
            out.append(None)
            continue
        e = eres[i]
        out.append(SolveResult(converged=conv[i], iters=iters[i], final_residual=fres[i], u=u_orig[nb[i]:nb[i + 1]],
                               avg_stress=stress[i], energy_residual=None if math.isnan(e) else e,
                               r_ref=rref[i]))
    if first_bad is not None and raise_singular:
        i, e = first_bad
        raise SingularElementError(f"element {e}: current length collapsed", element=e, problem=i)
    return out


def solve_batch(batch: Batch, strategy=None, config: SolverConfig | None = None):
    """Solve every problem of the batch on the B200.

    Returns one SolveResult per problem in batch order.  Non-convergence is
    reported per problem; a collapsed element raises SingularElementError
    (naming the element and the problem index) after all siblings finished.
    """
    cfg = config or SolverConfig()
    if batch.n_problems == 0:
        return []
    dres = batch.to_device().solve(cfg, strategy)
    return results_to_solve_results(batch, dres)


# ------------------------------------------------------------------ one-shot forces

def internal_forces_device(network: FiberNetwork, u: np.ndarray) -> np.ndarray:
    """f(u) for one network on the GPU, original DOF order."""
    torch = _torch()
    p = _meta(network, AffineBC(np.eye(3)), check_mass=False)
    batch = _pack([network], [None], [p], cluster=1)
    dbatch = batch.to_device()
    n = p.n_nodes
    launch = dbatch.prepare(SolverConfig())
    u_solver = np.asarray(u, dtype=np.float64).reshape(n, 3)[p.node_order].reshape(-1)
    u_t = torch.from_numpy(u_solver).to(dbatch.device)
    f_t = torch.empty_like(u_t)
    s = torch.cuda.current_stream(dbatch.device)
    nat.check(nat.lib().frb_internal_forces(C.byref(launch.fb), C.c_void_p(u_t.data_ptr()),
                                            C.c_void_p(f_t.data_ptr()), C.c_void_p(s.cuda_stream)))
    rec = launch.out.host_results()[0]
    if rec["status"] == nat.STATUS_SINGULAR:
        e = int(rec["bad_element"])
        raise SingularElementError(f"element {e}: current length collapsed", element=e)
    f = np.empty(3 * n)
    f.reshape(-1, 3)[p.node_order] = f_t.cpu().numpy().reshape(-1, 3)
    return f
