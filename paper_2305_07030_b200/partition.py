"""Split one network's free DOFs over the CTAs of a thread-block cluster.

A network that outgrows one SM is solved by a cluster of C CTAs ("ranks")
exchanging data through distributed shared memory.  The split follows the
pairwise-sum plan (plan.py): rank r owns a contiguous run of leaves whose DOF
range [3*node0, 3*(node0 + n_own)) starts at a node boundary, so the
per-DOF work, the ordered chain sums and the force gather of a node all stay
on one rank.  Cuts are chosen among leaf starts that are multiples of 3,
nearest to the even split.

Per rank the kernel works in *local* node numbering; every local node's
position lives in the rank's shared memory (AoS, 3 doubles per node):
    [0, n_own)                 own free nodes (global solver ids node0 ...)
    [n_own, n_local)           halo: free neighbours owned by other ranks,
                               grouped by owner, plus alignment gap slots
    [n_local, n_local + n_fix) fixed nodes that end an active element
Tables built here (all int32, shared by networks of equal topology):
    ell_o / ell_c   slot-major incidence of the own nodes (other endpoint in
                    local numbering, index into the rank's active list); the
                    device gets them packed as one u32 per slot (``ell``)
    act_ab          active elements (>= 1 own endpoint) in local numbering
    act_elem        their global element ids (per-network L / EA lookups)
    halo_g          global solver id of each halo slot (gaps: a valid dummy)
    fix_g           global solver id of each local fixed node
    runs            the rank's outgoing halo copies: (dst rank, src byte, dst
                    byte, bytes) -- one bulk DSMEM copy (cp.async.bulk) per
                    run of consecutive own nodes that a peer keeps as
                    consecutive halo slots.  Bulk copies need 16-byte aligned
                    addresses and sizes, and a position is 24 bytes, so the
                    copy widens each run to even node bounds [lo, hi) at the
                    source and lands it at an even slot of the receiver's
                    halo layout; the extra nodes fill gap slots.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .plan import PlanView, tree_split

MAX_LOCAL = 0xFFFF            # local node ids and active-element ids are 16 bit
RUN_WORDS = 4                 # (dst rank, src byte, dst byte, bytes) per halo run


@dataclass
class RankTables:
    node0: int
    n_own: int
    n_local: int
    leaf0: int
    n_leaves: int
    ell_o: np.ndarray        # (SA+SB, stride) int32
    ell_c: np.ndarray        # (SA+SB, stride) int32
    act_ab: np.ndarray       # (n_act, 2) int32
    act_elem: np.ndarray     # (n_act,) int64
    halo_g: np.ndarray       # (n_local - n_own,) int32
    fix_g: np.ndarray = None # (n_fix,) int32
    tree: np.ndarray = None  # int32 block of plan.tree_split (local/top programs, exports)
    runs: np.ndarray = None  # (n_runs, RUN_WORDS) int32 outgoing bulk halo copies
    halo_bytes: int = 0      # bytes of halo copies this rank receives per iteration
    ack_from: int = 0        # bit q: rank q sends halo copies to this rank
    n_int: int = 0           # act_elem[:n_int] have no halo endpoint

    @property
    def stride(self) -> int:
        return self.ell_o.shape[1]

    @property
    def n_fix(self) -> int:
        return len(self.fix_g)

    @property
    def ell(self) -> np.ndarray:
        """Packed slot table for the device: (other << 16) | active index
        (uint32, same shape as ell_o).  A padding slot of own node i points
        at i itself and at the element of i's first slot: its d is exactly
        +0, so it adds a zero of either sign to the running sum.  The sums
        start at +0 and round to nearest, so they are never -0 and adding
        +-0 leaves them unchanged -- the gather needs no branch."""
        pad = self.ell_o < 0
        n_own = self.n_own
        w = (self.ell_o.astype(np.int64) << 16) | self.ell_c.astype(np.int64)
        if pad.any():
            valid = ~pad[:, :n_own]
            first = np.where(valid.any(axis=0), np.argmax(valid, axis=0), 0)
            c_first = np.where(valid.any(axis=0), self.ell_c[first, np.arange(n_own)], 0)
            self_w = (np.arange(n_own, dtype=np.int64) << 16) | c_first.astype(np.int64)
            w[:, :n_own] = np.where(pad[:, :n_own], self_w[None, :], w[:, :n_own])
            w[:, n_own:] = 0
        return w.astype(np.uint32)

    @property
    def n_act(self) -> int:
        return len(self.act_elem)


@dataclass
class Partition:
    C: int
    slots_a: int
    slots_b: int
    ranks: list


LEAVES_PER_ROUND = 64   # chain sums of 64 leaves take one round of a 512-thread CTA


def cut_points(plan: np.ndarray, nf: int, C: int) -> list[int]:
    """DOF cut offsets (0 = c_0 < ... < c_C = nf) at leaf starts that are
    multiples of 3 (node- and leaf-aligned), chosen to minimise the largest
    rank -- the one every other rank waits for at the tree exchange: the most
    own DOFs, and ranks of more than LEAVES_PER_ROUND leaves (an extra chain
    round) only when unavoidable.  Exact min-max over the candidate cuts by
    dynamic programming; fewer ranks when the plan has too few candidates."""
    p = PlanView(plan)
    starts = np.asarray(p.leaf_start, dtype=np.int64)
    if nf == 0 or C <= 1 or len(starts) == 0:
        return [0, nf]
    ok = (starts % 3 == 0) & (starts > 0) & (starts < nf)
    pos = np.r_[0, starts[ok], nf]                       # candidate cut DOFs
    leaf = np.r_[0, np.flatnonzero(ok), len(starts)]     # first leaf after each cut
    K = len(pos)
    C = min(C, K - 1)
    big = float(nf + 1)
    # cost[i, j] of a rank spanning candidates i < j
    span = pos[None, :] - pos[:, None]
    nleaf = leaf[None, :] - leaf[:, None]

    def solve(cost):
        best = cost[0].copy()                             # one rank covering [0, pos[j])
        back = [np.zeros(K, dtype=np.int64)]
        for _ in range(1, C):
            cand = np.maximum(best[:, None], cost)       # previous ranks end at i, the next spans i..j
            arg = np.argmin(cand, axis=0)
            best = cand[arg, np.arange(K)]
            back.append(arg)
        return best[K - 1], back

    plain = np.where(span > 0, span, np.inf).astype(np.float64)
    worst, back = solve(np.where(nleaf > LEAVES_PER_ROUND, plain + big, plain))
    if worst >= big:  # no split keeps every rank within one chain round: plain min-max
        worst, back = solve(plain)
    cuts = [K - 1]
    for k in range(C - 1, 0, -1):
        cuts.append(int(back[k][cuts[-1]]))
    cuts.append(0)
    return [int(pos[i]) for i in reversed(cuts)]


def partition(n_nodes: int, n_free: int, ia: np.ndarray, ib: np.ndarray, ell_other: np.ndarray,
              ell_elem: np.ndarray, slots_a: int, slots_b: int, plan: np.ndarray, C: int) -> Partition:
    """Build the per-rank tables of one topology for a cluster of C ranks.

    ia, ib: element endpoints in solver numbering; ell_other / ell_elem: the
    global slot-major table of the free nodes (batch._topology)."""
    nf = 3 * n_free
    p = PlanView(plan)
    cuts = cut_points(plan, nf, C)
    C = len(cuts) - 1
    leaf_start = np.asarray(p.leaf_start, dtype=np.int64)
    owner = np.full(n_nodes, -1, dtype=np.int64)
    local = np.full(n_nodes, -1, dtype=np.int64)
    ranks_nodes = []
    for r in range(C):
        n0, n1 = cuts[r] // 3, cuts[r + 1] // 3
        owner[n0:n1] = r
        local[n0:n1] = np.arange(n1 - n0)
        ranks_nodes.append((n0, n1))
    elem_ids = np.arange(len(ia))
    ns = slots_a + slots_b
    # pass 1: active elements, halo and fixed sets per rank
    acts, halos, fixes, n_ints = [], [], [], []
    for r, (n0, n1) in enumerate(ranks_nodes):
        own_a = (ia >= n0) & (ia < n1)
        own_b = (ib >= n0) & (ib < n1)
        act = elem_ids[own_a | own_b]
        ends = np.concatenate([ia[act], ib[act]])
        # interior elements (no halo endpoint) first: the kernel evaluates
        # them while the halo copies are in flight
        cut = np.zeros(len(act), dtype=bool)
        for e_end in (ia[act], ib[act]):
            cut |= (e_end < n_free) & ((e_end < n0) | (e_end >= n1))
        act = np.concatenate([act[~cut], act[cut]])
        n_ints.append(int((~cut).sum()))
        acts.append(act)
        halos.append(np.unique(ends[(ends < n_free) & ((ends < n0) | (ends >= n1))]))
        fixes.append(np.unique(ends[ends >= n_free]))
    # pass 2: halo layouts (runs of consecutive nodes per owner, parity-aligned)
    out_runs = [[] for _ in range(C)]
    layouts = []
    for r, (n0, n1) in enumerate(ranks_nodes):
        halo = halos[r]
        n_own = n1 - n0
        slot_of = np.empty(len(halo), dtype=np.int64)
        gids = []
        cur = n_own
        recv = 0
        ack = 0
        if len(halo):
            brk = np.flatnonzero(np.diff(halo) != 1) + 1
            starts = np.r_[0, brk]
            ends_ = np.r_[brk, len(halo)]
            for a0, a1 in zip(starts, ends_):
                # a run may span two owners only if their ranges touch: split there
                seg_owner = owner[halo[a0:a1]]
                sp = np.r_[0, np.flatnonzero(np.diff(seg_owner) != 0) + 1, a1 - a0]
                for c0, c1 in zip(sp[:-1], sp[1:]):
                    g0 = int(halo[a0 + c0])
                    q = int(owner[g0])
                    src = g0 - ranks_nodes[q][0]
                    n = int(c1 - c0)
                    # copy source nodes [lo, hi): both ends even (24-byte
                    # nodes, 16-byte aligned bulk copies), landing at an even
                    # slot; the extra nodes at either end fill gap slots
                    lo = src - (src % 2)
                    hi = src + n + ((src + n) % 2)
                    if cur % 2:
                        gids.append(g0)
                        cur += 1
                    if src > lo:
                        gids.append(g0)
                    slot_of[a0 + c0:a0 + c1] = cur + (src - lo) + np.arange(n)
                    gids.extend(int(g) for g in halo[a0 + c0:a0 + c1])
                    if hi > src + n:
                        gids.append(g0)
                    out_runs[q].append((r, 24 * lo, 24 * cur, 24 * (hi - lo)))
                    cur += hi - lo
                    recv += 24 * (hi - lo)
                    ack |= 1 << q
        layouts.append((slot_of, np.asarray(gids, dtype=np.int64), cur, recv, ack))
    ranks = []
    for r, (n0, n1) in enumerate(ranks_nodes):
        n_own = n1 - n0
        act, halo, fix = acts[r], halos[r], fixes[r]
        slot_of, gids, n_local, recv, ack = layouts[r]
        if n_local + len(fix) > MAX_LOCAL or len(act) > MAX_LOCAL:
            raise ValueError(f"rank {r} needs {n_local + len(fix)} local nodes / {len(act)} elements "
                             f"(limit {MAX_LOCAL}); use a larger cluster")

        def to_local(g, n0=n0, n1=n1, halo=halo, fix=fix, n_local=n_local, slot_of=slot_of):
            g = np.asarray(g, dtype=np.int64)
            out = np.empty_like(g)
            own = (g >= n0) & (g < n1)
            fixed = g >= n_free
            hal = ~own & ~fixed
            out[own] = g[own] - n0
            out[fixed] = n_local + np.searchsorted(fix, g[fixed])
            out[hal] = slot_of[np.searchsorted(halo, g[hal])]
            return out

        act_index = np.full(len(ia), -1, dtype=np.int64)
        act_index[act] = np.arange(len(act))
        stride = max(32, 32 * ((n_own + 31) // 32))
        ell_o = np.full((ns, stride), -1, dtype=np.int32)
        ell_c = np.full((ns, stride), -1, dtype=np.int32)
        if n_own and ns:
            go = ell_other[:, n0:n1]
            ge = ell_elem[:, n0:n1]
            valid = go >= 0
            lo = np.where(valid, to_local(np.where(valid, go, 0)), -1)
            ell_o[:, :n_own] = lo
            ell_c[:, :n_own] = np.where(valid, act_index[ge], -1)
        act_ab = np.stack([to_local(ia[act]), to_local(ib[act])], axis=1).astype(np.int32)
        lstarts = np.flatnonzero((leaf_start >= cuts[r]) & (leaf_start < cuts[r + 1]))
        ranks.append(RankTables(node0=n0, n_own=n_own, n_local=n_local,
                                leaf0=int(lstarts[0]) if len(lstarts) else 0,
                                n_leaves=len(lstarts), ell_o=ell_o, ell_c=ell_c, act_ab=act_ab,
                                act_elem=act.astype(np.int64), halo_g=gids.astype(np.int32),
                                fix_g=fix.astype(np.int32),
                                runs=np.asarray(out_runs[r], dtype=np.int32).reshape(-1, RUN_WORDS),
                                halo_bytes=recv, ack_from=ack, n_int=n_ints[r]))
    blocks = tree_split(plan, [(rt.leaf0, rt.leaf0 + rt.n_leaves) for rt in ranks])
    for rt, bk in zip(ranks, blocks):
        rt.tree = bk
    return Partition(C=C, slots_a=slots_a, slots_b=slots_b, ranks=ranks)


def rank_smem_bytes(rt: RankTables, fprv_global: bool = False, mass_global: bool = False) -> int:
    """Dynamic SMEM of one rank (mirror of frb_rank_smem_bytes):
    positions [n_local + n_fix][3] (a DOF's own position slot doubles as its
    sq entry between the force and update phases), f and -- unless it lives
    in global memory -- f_prev (8 B per own DOF each), coefficients / sq2
    max(own DOFs, n_act), local tree slots and two parity buffers of top
    tree slots (3 doubles each), two parity buffers of 64 cluster flag /
    ledger words plus 16 final ledger words and 16 halo-copy acknowledgement
    words, one refined reciprocal mass and the mass per
    own node and the int32 tree block (programs + exports)."""
    return smem_bytes(rt.n_local + rt.n_fix, rt.n_own, rt.n_act, int(rt.tree[0]) + 2 * int(rt.tree[1]),
                      int(rt.tree[2]), fprv_global, mass_global)


def partition_smem_bytes(part: "Partition", fprv_global: bool = False, mass_global: bool = False) -> int:
    """Dynamic SMEM of every rank of a partitioned problem: the kernel lays
    all ranks out identically (peers address each other's buffers by the same
    offsets), each region sized by its maximum over the ranks."""
    rs = part.ranks
    return smem_bytes(max(r.n_local + r.n_fix for r in rs), max(r.n_own for r in rs),
                      max(r.n_act for r in rs), int(rs[0].tree[0]) + 2 * int(rs[0].tree[1]), int(rs[0].tree[2]),
                      fprv_global, mass_global)


def smem_bytes(n_pos: int, n_own: int, n_act: int, n_slots: int, n_prog: int, fprv_global: bool = False,
               mass_global: bool = False) -> int:
    nf = 3 * n_own
    return 8 * (3 * n_pos + (1 if fprv_global else 2) * nf + max(nf, n_act) + (1 if mass_global else 2) * n_own +
                3 * n_slots + 160) + \
        4 * ((n_prog + 1) & ~1)
