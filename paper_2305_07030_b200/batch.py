"""Batch submit: pack many networks into one device batch and solve them in a
single persistent-kernel launch.

Implements the spec'd ``batch`` module (reference ``SPEC.md:338-394``; there
is no batch code in the reference package itself):

* ``pack_batch(networks, bcs) -> Batch``
* ``solve_batch(batch, strategy, config) -> list[SolveResult]``
* strategies ``TeamBatched`` (the default: a device work queue, one CTA per
  network) and ``SerialReference`` (one team, problems in order,
  SPEC.md:359).

Host setup per network restates ``build_problem`` (reference
``microsolver.py:302-335``) in vectorised form and adds what the kernel
needs on top: the per-node incidence lists (role a then role b, ascending
element id -- the exact summation order of ``np.bincount`` in
``_scatter_forces``, :214-218) and the pairwise-sum plan for the free-DOF
count (plan.py).  Networks that share topology and materials share their
incidence / element arrays on the device.

Layout is a PackedStorage in spirit (reference ``packed.py``): flat SoA
arrays with per-problem offsets, host space "a" (numpy) mirrored to device
space "b" (torch CUDA tensors) with explicit upload/download.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
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
from .plan import PlanView, reduction_plan

__all__ = ["Batch", "DeviceBatch", "ExecutionStrategy", "NaiveLoop", "SerialReference",
           "TeamBatched", "pack_batch", "solve_batch", "build_problem", "DeviceResults"]

MAX_CTA_THREADS = 1024
MAX_DOFS_PER_THREAD = 8     # FRB_MAX_DOFS_PER_THREAD


# ------------------------------------------------------------------ strategies

@dataclass(frozen=True)
class SerialReference:
    """Problems one after another on a single team (one CTA)."""


@dataclass(frozen=True)
class NaiveLoop:
    """Per-operation dispatch (the paper's naive baseline).  Not provided on
    the device: the B200 build exists to remove per-operation launches."""
    workers: int = 1


@dataclass(frozen=True)
class TeamBatched:
    """Shared work queue; each team runs whole solves.
    teams=None sizes the persistent grid by occupancy; team_size=None picks
    the smallest CTA that covers the pairwise-sum chains."""
    teams: int | None = None
    team_size: int | None = None

    def __post_init__(self):
        if self.teams is not None and self.teams < 1:
            raise ValueError("teams must be >= 1")
        if self.team_size is not None and (self.team_size < 32 or self.team_size % 32):
            raise ValueError("team_size must be a positive multiple of 32")


ExecutionStrategy = SerialReference | NaiveLoop | TeamBatched


# ------------------------------------------------------------------ host setup

@dataclass
class HostProblem:
    """Solver-order setup of one network (ProblemSetup, microsolver.py:138-163)."""
    network: FiberNetwork
    F: np.ndarray
    node_order: np.ndarray       # solver position -> original node
    X: np.ndarray                # (N, 3)
    node_mass: np.ndarray        # (N,)
    dt_base: float               # min_e L sqrt(rho/E); dt = dt_safety * dt_base
    topo_key: bytes
    topo: "Topology"

    @property
    def n_nodes(self) -> int:
        return len(self.X)

    @property
    def n_free_nodes(self) -> int:
        return self.topo.n_free_nodes


@dataclass
class Topology:
    """Arrays that depend only on (elements, boundary, materials) -- shared
    by every network of the same topology."""
    n_nodes: int
    n_free_nodes: int
    inc_node: np.ndarray         # (N, 2) int32: first entry, n_a | n_b << 16
    inc: np.ndarray              # (I, 2) int32: other endpoint, element id
    elem_ab: np.ndarray          # (M, 2) int32 solver node ids
    plan: np.ndarray             # int32 flat pairwise plan for nf
    n_leaves: int
    max_own: int                 # most DOFs one chain thread owns
    ell_other: np.ndarray        # (SA+SB, S) int32 slot-major, -1 padding
    ell_elem: np.ndarray         # (SA+SB, S) int32 element per slot (0 on padding)
    ell_slots_a: int
    ell_slots_b: int
    ell_c: np.ndarray            # (SA+SB, S) int32 index into ff list, -1 fixed/padding
    ff_ab: np.ndarray            # (n_ff, 2) int32 endpoints of free-free elements
    ff_elem: np.ndarray          # (n_ff,) element ids


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
    # slot-major table for free nodes: slot k < SA is the k-th role-a
    # incidence (ascending element), slot SA + k the k-th role-b incidence
    snode, srole = node[order], role[order]
    grp = snode.astype(np.int64) * 2 + srole
    starts = np.flatnonzero(np.r_[True, grp[1:] != grp[:-1]])
    rank = np.arange(len(grp)) - np.repeat(starts, np.diff(np.r_[starts, len(grp)]))
    nfn = n_free_nodes
    sa = int(na[:nfn].max()) if nfn and m else 0
    sb = int(nb[:nfn].max()) if nfn and m else 0
    stride = max(32, 32 * ((nfn + 31) // 32))
    ell_other = np.full((sa + sb, stride), -1, dtype=np.int32)
    ell_elem = np.zeros((sa + sb, stride), dtype=np.int32)
    free = snode < nfn
    slot = np.where(srole == 0, rank, sa + rank)[free]
    ell_other[slot, snode[free]] = other[order][free]
    ell_elem[slot, snode[free]] = elem[order][free]
    sizes = PlanView(plan).leaf_size
    max_own = int(max(((z // 8) + (1 if z % 8 else 0)) if z >= 8 else 1 for z in sizes)) if len(sizes) else 1
    # elements between two free nodes: their coefficient is computed once per
    # iteration (fiber-parallel) and looked up by both endpoints' slots
    ff_mask = (ia < nfn) & (ib < nfn)
    ff_elem = np.flatnonzero(ff_mask)
    ff_index = np.full(m, -1, dtype=np.int64)
    ff_index[ff_elem] = np.arange(ff_elem.size)
    ell_c = np.where(ell_other >= 0, ff_index[ell_elem], -1)
    ell_c = np.where((ell_other >= 0) & (ell_other < nfn), ell_c, -1).astype(np.int32)
    return Topology(n_nodes=n, n_free_nodes=n_free_nodes, inc_node=inc_node, inc=inc,
                    elem_ab=np.stack([ia, ib], axis=1).astype(np.int32), plan=plan,
                    n_leaves=int(plan[0]), max_own=max_own, ell_other=ell_other,
                    ell_elem=ell_elem, ell_slots_a=sa, ell_slots_b=sb, ell_c=ell_c,
                    ff_ab=np.stack([ia[ff_elem], ib[ff_elem]], axis=1).astype(np.int32),
                    ff_elem=ff_elem.astype(np.int64))


_TOPO_CACHE: dict[bytes, Topology] = {}


def build_problem(network: FiberNetwork, bc: AffineBC, check_mass: bool = True) -> HostProblem:
    """Host setup for one network (reference build_problem, :302-335).

    Raises NetworkMassError for a node without incident elements (like
    compute_lumped_mass, :179-181)."""
    n = network.n_nodes
    dm = build_dofmap(n, network.boundary_nodes)
    order = dm.node_order
    rank = np.empty(n, dtype=np.int64)
    rank[order] = np.arange(n)
    nfn = dm.n_free // 3
    if check_mass:
        node_mass = _lumped_node_mass(network)[order]
    else:
        node_mass = np.ones(n)
    emod, area, rho = network.material_columns()
    L = network.reference_lengths()
    dt_base = float(np.min(L * np.sqrt(rho / emod))) if L.size else math.nan
    h = hashlib.blake2b(digest_size=16)
    h.update(np.int64([n, network.n_elements]).tobytes())
    h.update(network.elements.tobytes())
    h.update(np.asarray(sorted(network.boundary_nodes), dtype=np.int64).tobytes())
    key = h.digest()
    topo = _TOPO_CACHE.get(key)
    if topo is None:
        topo = _topology(network, rank, nfn)
        if len(_TOPO_CACHE) > 4096:
            _TOPO_CACHE.clear()
        _TOPO_CACHE[key] = topo
    return HostProblem(network=network, F=np.asarray(bc.deformation_gradient, dtype=np.float64),
                       node_order=order, X=np.ascontiguousarray(network.node_coords[order]),
                       node_mass=node_mass, dt_base=dt_base, topo_key=key, topo=topo)


def cta_smem_bytes(n_free_nodes: int, n_ff: int, n_leaves: int) -> int:
    """Mirror of frb_cta_smem_bytes (include/frb200.h): positions / sq, f,
    f_prev (8 B per free DOF each), sq2 / free-free coefficients, tree
    slots, and the tree's combine program (int32, bounded by a height of
    bit_length(L-1) + 1 levels)."""
    nf = 3 * n_free_nodes
    L = n_leaves
    slots = 2 * L - 1 if L > 0 else 1
    levels = (L - 1).bit_length() + 1 if L > 1 else 0
    prog = (levels + 1) + 3 * (L - 1 if L > 0 else 0)
    return 8 * (3 * nf + max(nf, n_ff) + 3 * slots) + 4 * ((prog + 1) & ~1)


# ------------------------------------------------------------------ batch

@dataclass
class Batch:
    """Host-side packed batch (space "a").  ``packed_state`` exposes the
    spec's per-problem PackedStorage rows for u, v, a, f_int, m (built on
    first access)."""
    networks: list
    bcs: list
    problems: list                     # HostProblem per network
    desc: np.ndarray                   # PROBLEM_DTYPE records (dt filled per solve)
    arrays: dict                       # flat host arrays
    node_base: np.ndarray              # (P+1,) int64 node offsets
    max_leaves: int
    smem_bytes: int
    max_nf: int
    _packed_state: dict | None = field(default=None, repr=False)
    pinned: dict | None = field(default=None, repr=False)

    def pin(self) -> "Batch":
        """Page-lock the packed arrays once so uploads are pure DMA."""
        torch = _torch()
        self.pinned = {k: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                       for k, a in self.arrays.items()}
        return self

    @property
    def n_problems(self) -> int:
        return len(self.problems)

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
    """Build the packed batch."""
    if len(networks) != len(bcs):
        raise ValueError(f"networks and bcs differ in length ({len(networks)} vs {len(bcs)})")
    probs = [build_problem(net, bc) for net, bc in zip(networks, bcs)]
    return _pack(list(networks), list(bcs), probs)


def _pack(networks, bcs, probs) -> Batch:
    P = len(probs)
    desc = np.zeros(P, dtype=nat.PROBLEM_DTYPE)
    node_base = np.zeros(P + 1, dtype=np.int64)
    topo_slot: dict[bytes, tuple[int, int]] = {}
    plan_slot: dict[int, int] = {}
    inc, plans, ell_other, ell_c, ff_ab = [], [], [], [], []
    n_inc = n_plan = n_ell = n_ffs = 0
    elem_base = ellv_base = ffv_base = 0
    ff_L, ff_EA = [], []
    X, mass, EL, EA, inc_node, elem_ab, ell_L, ell_EA = [], [], [], [], [], [], [], []
    any_nonuniform = False
    max_leaves = smem = max_nf = 0
    for i, p in enumerate(probs):
        t = p.topo
        if p.topo_key not in topo_slot:
            topo_slot[p.topo_key] = (n_inc, n_ell, n_ffs)
            inc.append(t.inc)
            ell_other.append(t.ell_other.reshape(-1))
            ell_c.append(t.ell_c.reshape(-1))
            ff_ab.append(t.ff_ab)
            n_inc += len(t.inc)
            n_ell += t.ell_other.size
            n_ffs += len(t.ff_ab)
        inc_b, ell_b, ff_b = topo_slot[p.topo_key]
        nf = 3 * t.n_free_nodes
        if nf not in plan_slot:
            plan_slot[nf] = n_plan
            plans.append(t.plan)
            n_plan += len(t.plan)
        emod, area, _ = p.network.material_columns()
        ea = emod * area
        L = p.network.reference_lengths()
        uniform = bool(ea.size == 0 or np.all(ea == ea[0]))
        d = desc[i]
        d["node_base"] = node_base[i]
        d["elem_base"] = elem_base
        d["inc_base"] = inc_b
        d["plan_base"] = plan_slot[nf]
        d["ell_base"] = ell_b
        d["ellv_base"] = ellv_base
        d["ff_base"] = ff_b
        d["ffv_base"] = ffv_base
        d["n_ff"] = len(t.ff_elem)
        d["n_nodes"] = p.n_nodes
        d["n_free_nodes"] = t.n_free_nodes
        d["n_elems"] = p.network.n_elements
        d["cluster"] = 1
        d["ell_stride"] = t.ell_other.shape[1]
        d["ell_slots_a"] = t.ell_slots_a
        d["ell_slots_b"] = t.ell_slots_b
        d["flags"] = nat.PF_EA_UNIFORM if uniform else 0
        d["volume"] = p.network.volume
        d["ea"] = ea[0] if ea.size else 0.0
        d["F"] = p.F.reshape(9)
        node_base[i + 1] = node_base[i] + p.n_nodes
        X.append(p.X.reshape(-1))
        mass.append(p.node_mass)
        EL.append(L)
        EA.append(ea)
        inc_node.append(t.inc_node)
        elem_ab.append(t.elem_ab)
        valid = t.ell_other.reshape(-1) >= 0
        eidx = t.ell_elem.reshape(-1)
        ell_L.append(np.where(valid, L[eidx] if L.size else 1.0, 1.0))
        if not uniform:
            any_nonuniform = True
        ell_EA.append(np.where(valid, ea[eidx] if ea.size else 0.0, 0.0))
        ellv_base += t.ell_other.size
        ff_L.append(L[t.ff_elem])
        ff_EA.append(ea[t.ff_elem])
        ffv_base += len(t.ff_elem)
        elem_base += p.network.n_elements
        max_leaves = max(max_leaves, t.n_leaves)
        max_nf = max(max_nf, 3 * t.n_free_nodes)
        smem = max(smem, cta_smem_bytes(t.n_free_nodes, len(t.ff_elem), t.n_leaves))

    def cat(parts, dtype, width=None):
        if not parts:
            return np.zeros((0,) if width is None else (0, width), dtype=dtype)
        return np.ascontiguousarray(np.concatenate(parts).astype(dtype, copy=False))

    arrays = dict(
        X=cat(X, np.float64), node_mass=cat(mass, np.float64),
        inc_node=cat(inc_node, np.int32, 2), inc=cat(inc, np.int32, 2),
        elem_ab=cat(elem_ab, np.int32, 2), elem_L=cat(EL, np.float64),
        elem_EA=cat(EA, np.float64), plans=cat(plans, np.int32),
        ell_other=cat(ell_other, np.int32), ell_L=cat(ell_L, np.float64),
        ell_c=cat(ell_c, np.int32), ff_ab=cat(ff_ab, np.int32, 2), ff_L=cat(ff_L, np.float64),
    )
    if any_nonuniform:
        arrays["ell_EA"] = cat(ell_EA, np.float64)
        arrays["ff_EA"] = cat(ff_EA, np.float64)
    # order: longest first (nodes as the work proxy) for the dynamic queue
    arrays["order"] = np.argsort(-node_base[1:] + node_base[:-1], kind="stable").astype(np.int32)
    return Batch(networks=networks, bcs=bcs, problems=probs, desc=desc, arrays=arrays,
                 node_base=node_base, max_leaves=max_leaves, smem_bytes=smem, max_nf=max_nf)


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
    desc_host: np.ndarray

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
        return cls(host=batch, device=device, t=t, desc_host=batch.desc.copy())

    def _desc_tensor(self, cfg: SolverConfig):
        torch = _torch()
        desc = self.desc_host
        desc["dt"] = [cfg.dt_safety * p.dt_base for p in self.host.problems]
        raw = torch.from_numpy(desc.view(np.uint8).copy())
        return raw.to(self.device, non_blocking=True)

    def default_threads(self) -> int:
        """Smallest CTA (multiple of 32, >= 64) that covers the pairwise
        chains and keeps <= MAX_DOFS_PER_THREAD DOFs per thread; large
        problems get 1024 threads for latency hiding."""
        h = self.host
        need = max(64, 8 * h.max_leaves, math.ceil(h.max_nf / MAX_DOFS_PER_THREAD))
        if h.max_nf > 2048:
            need = max(need, 1024)
        return min(MAX_CTA_THREADS, 32 * math.ceil(need / 32))

    @property
    def work(self):
        if getattr(self, "_work", None) is None:
            self._work = _torch().empty(3 * int(self.host.node_base[-1]) + 1, dtype=_torch().float64,
                                        device=self.device)
        return self._work

    def frb_batch(self, desc_t, u, f, results, queue) -> nat.FrbBatch:
        t = self.t
        b = nat.FrbBatch()
        b.n_problems = self.host.n_problems
        b.smem_bytes = self.host.smem_bytes
        b.max_nf = self.host.max_nf
        b.problems = desc_t.data_ptr()
        b.order = t["order"].data_ptr()
        for k in ("X", "node_mass", "inc_node", "inc", "elem_ab", "elem_L", "elem_EA", "plans",
                  "ell_other", "ell_L", "ell_EA", "ell_c", "ff_ab", "ff_L", "ff_EA"):
            setattr(b, k, t[k].data_ptr() if k in t and t[k].numel() else None)
        b.u, b.f = u.data_ptr(), f.data_ptr()
        b.work = self.work.data_ptr()
        b.results = results.data_ptr()
        b.queue = queue.data_ptr()
        return b

    def prepare(self, cfg: SolverConfig, strategy=None) -> "Launch":
        """Allocate outputs and build the launch arguments once; the
        returned Launch can be replayed (bench) or run once (solve)."""
        torch = _torch()
        strategy = strategy or TeamBatched()
        if isinstance(strategy, NaiveLoop):
            raise NotImplementedError("NaiveLoop per-operation dispatch is not provided on the B200 path")
        threads = self.default_threads()
        grid = 0
        if isinstance(strategy, TeamBatched):
            if strategy.team_size is not None:
                threads = strategy.team_size
            grid = strategy.teams or 0
        elif isinstance(strategy, SerialReference):
            grid = 1
        h = self.host
        if (threads < 8 * h.max_leaves or threads > MAX_CTA_THREADS
                or h.max_nf > MAX_DOFS_PER_THREAD * threads):
            raise nat.NativeError(nat.FRB_E_TOO_LARGE,
                                  f"team_size {threads} cannot hold {h.max_leaves} pairwise leaves / "
                                  f"{h.max_nf} free DOFs (cluster path needed)")
        n = int(self.host.node_base[-1])
        dev = self.device
        u = torch.empty(3 * n, dtype=torch.float64, device=dev)
        f = torch.empty(3 * n, dtype=torch.float64, device=dev)
        res = torch.zeros(self.host.n_problems * nat.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        queue = torch.zeros(1, dtype=torch.int32, device=dev)
        desc_t = self._desc_tensor(cfg)
        return Launch(self, self.frb_batch(desc_t, u, f, res, queue), config_struct(cfg), threads, grid,
                      DeviceResults(u=u, f=f, results=res, node_base=self.host.node_base),
                      keep=(desc_t, queue))

    def solve(self, cfg: SolverConfig, strategy=None, stream=None) -> DeviceResults:
        """Launch the persistent kernel; returns device-resident results
        (asynchronous on the current torch stream)."""
        launch = self.prepare(cfg, strategy)
        launch.run(stream)
        return launch.out


@dataclass
class Launch:
    dbatch: DeviceBatch
    fb: nat.FrbBatch
    fc: nat.FrbConfig
    threads: int
    grid: int
    out: DeviceResults
    keep: tuple = ()

    def run(self, stream=None):
        """One frb_solve_batch call (one kernel launch) on `stream`."""
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.dbatch.device)
        nat.check(nat.lib().frb_solve_batch(C.byref(self.fb), C.byref(self.fc), self.threads,
                                            self.grid, C.c_void_p(s.cuda_stream)))


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
    """Download and unpermute (DofMap.unpermute, dofmap.py:33-38)."""
    rec = dres.host_results()
    u_all = dres.u.cpu().numpy()
    out = []
    first_bad = None
    for i, p in enumerate(batch.problems):
        r = rec[i]
        if r["status"] == nat.STATUS_SINGULAR:
            if first_bad is None:
                first_bad = (i, int(r["bad_element"]))
            out.append(None)
            continue
        b0, b1 = 3 * int(batch.node_base[i]), 3 * int(batch.node_base[i + 1])
        u = np.empty(b1 - b0)
        u.reshape(-1, 3)[p.node_order] = u_all[b0:b1].reshape(-1, 3)
        e = float(r["energy_residual"])
        out.append(SolveResult(converged=bool(r["converged"]), iters=int(r["iters"]),
                               final_residual=float(r["final_residual"]), u=u,
                               avg_stress=np.array(r["avg_stress"], dtype=np.float64).reshape(3, 3),
                               energy_residual=None if math.isnan(e) else e,
                               r_ref=float(r["r_ref"])))
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
    dbatch = batch.to_device()
    dres = dbatch.solve(cfg, strategy)
    return results_to_solve_results(batch, dres)


# ------------------------------------------------------------------ one-shot forces

def internal_forces_device(network: FiberNetwork, u: np.ndarray) -> np.ndarray:
    """f(u) for one network on the GPU, original DOF order."""
    torch = _torch()
    p = build_problem(network, AffineBC(np.eye(3)), check_mass=False)
    batch = _pack([network], [None], [p])
    dbatch = batch.to_device()
    n = p.n_nodes
    u_solver = np.asarray(u, dtype=np.float64).reshape(n, 3)[p.node_order].reshape(-1)
    u_t = torch.from_numpy(u_solver).to(dbatch.device)
    f_t = torch.empty_like(u_t)
    res = torch.zeros(nat.RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dbatch.device)
    queue = torch.zeros(1, dtype=torch.int32, device=dbatch.device)
    desc_t = dbatch._desc_tensor(SolverConfig())
    fb = dbatch.frb_batch(desc_t, u_t, f_t, res, queue)
    s = torch.cuda.current_stream(dbatch.device)
    nat.check(nat.lib().frb_internal_forces(C.byref(fb), C.c_void_p(u_t.data_ptr()),
                                            C.c_void_p(f_t.data_ptr()), C.c_void_p(s.cuda_stream)))
    rec = res.cpu().numpy().view(nat.RESULT_DTYPE)[0]
    if rec["status"] == nat.STATUS_SINGULAR:
        e = int(rec["bad_element"])
        raise SingularElementError(f"element {e}: current length collapsed", element=e)
    f = np.empty(3 * n)
    f.reshape(-1, 3)[p.node_order] = f_t.cpu().numpy().reshape(-1, 3)
    return f
