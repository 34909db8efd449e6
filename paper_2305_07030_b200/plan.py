"""Reduction plans: NumPy's pairwise-sum tree as data for the device.

``np.sum`` over a contiguous float64 vector (reference ``microsolver.py:246,
479, 481, 494``) evaluates numpy 2.3's ``pairwise_sum``: a block of n <= 128
sums 8 stride-8 accumulator chains, folds them as
((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and adds the n%8 tail in order; a longer
block splits at n/2 rounded down to a multiple of 8 and adds the halves; n < 8
is a plain sequential sum from 0.0.  The tree depends only on n, so the host
builds it once per distinct free-DOF count and the kernel replays it:

* leaves (start, size): each device thread owns one (leaf, chain) pair and
  accumulates it in order; tail elements are added after the fold;
* combine ops (dst, left, right) over slots [leaves..., internal...], grouped
  by height so every op of one level is independent (one lane per op).

Flat int32 layout consumed by ``csrc/frb_relax.cuh`` (``PlanView``):
    [n_leaves, n_levels, root, pad,
     leaf_start[L], leaf_size[L], level_off[n_levels + 1],
     op_dst[K], op_left[K], op_right[K]]          K = L - 1
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

PW_BLOCK = 128
HEADER = 4


def _split(n: int) -> int:
    h = n // 2
    return h - h % 8


@lru_cache(maxsize=256)
def reduction_plan(n: int) -> np.ndarray:
    """Flat int32 plan for a length-n pairwise sum (read-only array)."""
    leaves: list[tuple[int, int]] = []
    ops: list[tuple[int, int, int, int]] = []      # (height, dst, left, right)
    n_internal = [0]

    def build(start: int, size: int):
        """Returns (slot, height); internal slots are renumbered later."""
        if size <= PW_BLOCK:
            leaves.append((start, size))
            return ("leaf", len(leaves) - 1), 0
        h = _split(size)
        left, hl = build(start, h)
        right, hr = build(start + h, size - h)
        n_internal[0] += 1
        me = ("node", n_internal[0] - 1)
        height = max(hl, hr) + 1
        ops.append((height, me, left, right))
        return me, height

    if n == 0:
        flat = np.zeros(HEADER + 1, dtype=np.int32)
        flat[:HEADER] = (0, 0, -1, 0)
        flat.setflags(write=False)
        return flat
    root, _ = build(0, n)
    L = len(leaves)

    def slot(ref):
        kind, i = ref
        return i if kind == "leaf" else L + i

    ops.sort(key=lambda o: o[0])          # stable: keeps post-order within a level
    heights = sorted({o[0] for o in ops})
    level_off = [0]
    for h in heights:
        level_off.append(level_off[-1] + sum(1 for o in ops if o[0] == h))
    parts = [
        np.array([L, len(heights), slot(root), 0], dtype=np.int32),
        np.array([s for s, _ in leaves], dtype=np.int32),
        np.array([z for _, z in leaves], dtype=np.int32),
        np.array(level_off, dtype=np.int32),
        np.array([slot(o[1]) for o in ops], dtype=np.int32),
        np.array([slot(o[2]) for o in ops], dtype=np.int32),
        np.array([slot(o[3]) for o in ops], dtype=np.int32),
    ]
    flat = np.concatenate(parts)
    flat.setflags(write=False)
    return flat


class PlanView:
    """Named access to a flat plan (host side; mirrors the device struct)."""

    def __init__(self, flat: np.ndarray):
        self.flat = flat
        self.n_leaves, self.n_levels, self.root = int(flat[0]), int(flat[1]), int(flat[2])
        L, H = self.n_leaves, self.n_levels
        K = max(L - 1, 0)
        o = HEADER
        self.leaf_start = flat[o:o + L]
        o += L
        self.leaf_size = flat[o:o + L]
        o += L
        self.level_off = flat[o:o + H + 1]
        o += H + 1
        self.op_dst = flat[o:o + K]
        o += K
        self.op_left = flat[o:o + K]
        o += K
        self.op_right = flat[o:o + K]


def evaluate(flat: np.ndarray, a) -> float:
    """Replay a plan on the host exactly as the kernel does (used by tests to
    prove the encoded plan reproduces np.sum; not a solver code path)."""
    p = PlanView(flat)
    a = [float(x) for x in np.asarray(a, dtype=np.float64)]
    if p.n_leaves == 0:
        return 0.0
    slots = [0.0] * (2 * p.n_leaves - 1)
    for l in range(p.n_leaves):
        start, size = int(p.leaf_start[l]), int(p.leaf_size[l])
        if size < 8:
            s, body = 0.0, 0
        else:
            body = size - size % 8
            r = []
            for j in range(8):
                acc = a[start + j]
                for t in range(start + j + 8, start + body, 8):
                    acc += a[t]
                r.append(acc)
            s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for t in range(start + body, start + size):
            s += a[t]
        slots[l] = s
    for lev in range(p.n_levels):
        for k in range(int(p.level_off[lev]), int(p.level_off[lev + 1])):
            slots[int(p.op_dst[k])] = slots[int(p.op_left[k])] + slots[int(p.op_right[k])]
    return slots[p.root]


# ---------------------------------------------------------------- cluster split

TREE_HEADER = 12


PROG_LANES = 32


def _program(ops: list[tuple[int, int, int, int]], scratch: int) -> np.ndarray:
    """Combine program as warp rounds: [n_rounds, 0, (n_rounds + 1) x 32 x 2
    words] (the pad keeps the word pairs 8-byte aligned on the device; the
    extra idle round lets the device prefetch the next round unconditionally).
    Ops (height, dst, left, right) of one height are independent; each round
    holds up to 32 of them, one per lane, as the pair (3 dst, 3 left |
    3 right << 16) -- slot indices premultiplied by the 3 components.  Idle
    lane l combines its own scratch slot `scratch + l` into itself, so the
    device loop has no branch and no two lanes touch the same slot.  Rounds
    run in order with a __syncwarp between them."""
    ops = sorted(ops, key=lambda o: o[0])
    assert 3 * (scratch + PROG_LANES - 1) < (1 << 16), "tree slot index exceeds 16 bits / 3"
    idle = [w for lane in range(PROG_LANES)
            for w in (3 * (scratch + lane), 3 * (scratch + lane) | (3 * (scratch + lane) << 16))]
    rounds = []
    for h in sorted({o[0] for o in ops}):
        level = [o for o in ops if o[0] == h]
        for i in range(0, len(level), PROG_LANES):
            words = list(idle)
            for lane, (_, d, a, b) in enumerate(level[i:i + PROG_LANES]):
                assert 3 * max(d, a, b) < (1 << 16), "tree slot index exceeds 16 bits / 3"
                words[2 * lane] = 3 * d
                words[2 * lane + 1] = 3 * a | (3 * b << 16)
            rounds.append(words)
    rounds.append(list(idle))
    return np.array([len(rounds) - 1, 0] + [w for r in rounds for w in r], dtype=np.int32)


MODE_QUAD = 4   # the rank's leaves fold in aligned quads inside the chain warps


def run_program(prog: np.ndarray, slots: list) -> None:
    """Host replay of a _program (test helper)."""
    n = int(prog[0])
    for r in range(n):
        words = prog[2 + 2 * PROG_LANES * r:2 + 2 * PROG_LANES * (r + 1)]
        new = {}
        for lane in range(PROG_LANES):
            d, w = int(words[2 * lane]), int(words[2 * lane + 1])
            new[d // 3] = slots[(w & 0xffff) // 3] + slots[(w >> 16) // 3]
        for d, v in new.items():
            slots[d] = v


def tree_split(flat: np.ndarray, ranges: list[tuple[int, int]]) -> list[np.ndarray]:
    """Split the pairwise tree over the cluster ranks that own the leaf
    ranges [a_r, b_r).  A node is *local* to rank r when all its leaves are
    r's; r evaluates its local nodes (the local program, over its own leaves
    numbered 0.. followed by its local internal nodes) and exports the
    maximal ones -- those whose parent is not local -- into a *top* slot
    array that every rank holds: exports first (ordered by leaf position),
    then the non-local internal nodes.  Every rank replays the same top
    program, so all ranks obtain the identical root.  The combine order is
    NumPy's throughout; only where each addition happens changes.

    Returns one int32 block per rank:
        [LS, TS, PI, lprog_off, tprog_off, exp_off, n_exp, root_top, E, mode, leaf_off, 0,
         local program, top program, exports (local slot, top slot) pairs,
         own leaves (start relative to the rank's first DOF, size) pairs]
    LS / PI are maxima over the ranks (uniform SMEM layout), TS = E + #top
    internal nodes, root_top = top slot of the root (-1: empty tree)."""
    p = PlanView(flat)
    L = p.n_leaves
    C = len(ranges)
    if L == 0:
        blocks = []
        for _ in range(C):
            empty = _program([], 0)
            blocks.append(np.concatenate([
                np.array([1, 1, TREE_HEADER + 2 * len(empty), TREE_HEADER, TREE_HEADER + len(empty),
                          TREE_HEADER + 2 * len(empty), 0, -1, 0, 0, TREE_HEADER + 2 * len(empty), 0],
                         dtype=np.int32), empty, empty]))
        return blocks
    n_slots = 2 * L - 1
    lo = np.zeros(n_slots, dtype=np.int64)
    hi = np.zeros(n_slots, dtype=np.int64)
    lo[:L] = np.arange(L)
    hi[:L] = np.arange(L) + 1
    parent = np.full(n_slots, -1, dtype=np.int64)
    K = L - 1
    for k in range(K):                         # ops are ordered by height
        d, a, b = int(p.op_dst[k]), int(p.op_left[k]), int(p.op_right[k])
        lo[d], hi[d] = lo[a], hi[b]
        parent[a] = parent[b] = d
    leaf_rank = np.empty(L, dtype=np.int64)
    for r, (a, b) in enumerate(ranges):
        leaf_rank[a:b] = r
    owner = np.where(leaf_rank[lo] == leaf_rank[hi - 1], leaf_rank[lo], -1)
    # every leaf range must be split exactly at rank boundaries
    for r, (a, b) in enumerate(ranges):
        if b > a:
            assert (leaf_rank[a:b] == r).all()
    exports = [s for s in range(n_slots)
               if owner[s] >= 0 and (parent[s] < 0 or owner[parent[s]] != owner[s])]
    exports.sort(key=lambda s: lo[s])
    E = len(exports)
    top_of = np.full(n_slots, -1, dtype=np.int64)
    for i, s in enumerate(exports):
        top_of[s] = i
    top_internal = [k for k in range(K) if owner[int(p.op_dst[k])] < 0]
    theight = {}
    top_ops = []
    for j, k in enumerate(top_internal):       # in height order
        d, a, b = int(p.op_dst[k]), int(p.op_left[k]), int(p.op_right[k])
        top_of[d] = E + j
        h = 1 + max(theight.get(a, 0), theight.get(b, 0))
        theight[d] = h
        top_ops.append((h, int(top_of[d]), int(top_of[a]), int(top_of[b])))
    TS = E + len(top_internal) + PROG_LANES   # + a scratch slot per lane for idle lanes
    root_top = int(top_of[p.root])
    tprog = _program(top_ops, TS - PROG_LANES)
    blocks = []
    children = {int(p.op_dst[k]): (int(p.op_left[k]), int(p.op_right[k])) for k in range(K)}
    pending = []
    for r, (a, b) in enumerate(ranges):
        nleaf = b - a
        # quad mode: every aligned group of 4 own leaves is the complete
        # subtree ((l0 + l1) + (l2 + l3)); the chain warps (4 leaves each)
        # fold it with shuffles and the local program starts at the quads
        quad_nodes, quad_roots = set(), []
        quad = nleaf > 0 and nleaf % 4 == 0
        if quad:
            for g in range(nleaf // 4):
                l0 = a + 4 * g
                p01, p23 = int(parent[l0]), int(parent[l0 + 2])
                q = int(parent[p01]) if p01 >= 0 else -1
                if (p01 < 0 or p23 < 0 or q < 0 or children.get(p01) != (l0, l0 + 1)
                        or children.get(p23) != (l0 + 2, l0 + 3) or children.get(q) != (p01, p23)
                        or owner[q] != r):
                    quad = False
                    break
                quad_nodes.update((l0, l0 + 1, l0 + 2, l0 + 3, p01, p23))
                quad_roots.append(q)
        if quad and any(owner[sl] == r and sl in quad_nodes for sl in exports):
            quad = False
        local_idx = np.full(n_slots, -1, dtype=np.int64)
        if quad:
            for g, q in enumerate(quad_roots):
                local_idx[q] = g
            nl = len(quad_roots)
        else:
            local_idx[a:b] = np.arange(nleaf)
            nl = nleaf
        below = set(quad_roots) | quad_nodes if quad else set()
        lheight = {}
        lops = []
        for k in range(K):
            d, x, y = int(p.op_dst[k]), int(p.op_left[k]), int(p.op_right[k])
            if owner[d] != r or d in below:
                continue
            local_idx[d] = nl
            nl += 1
            h = 1 + max(lheight.get(x, 0), lheight.get(y, 0))
            lheight[d] = h
            lops.append((h, int(local_idx[d]), int(local_idx[x]), int(local_idx[y])))
        exp = np.array([(int(local_idx[sl]), int(top_of[sl])) for sl in exports if owner[sl] == r],
                       dtype=np.int32).reshape(-1)
        mode = MODE_QUAD if quad else 0
        # the chain role of the rank's leaves (C phase): (start - the rank's
        # first DOF, size), read from shared memory instead of registers
        ls = np.asarray(p.leaf_start[a:b], dtype=np.int64)
        leaves = np.stack([ls - (ls[0] if len(ls) else 0), np.asarray(p.leaf_size[a:b], dtype=np.int64)],
                          axis=1).reshape(-1)
        pending.append((nl, lops, exp, mode, leaves))
    LS = max(nl for nl, _, _, _, _ in pending) + PROG_LANES   # + a scratch slot per lane for idle lanes
    for nl, lops, exp, mode, leaves in pending:
        lprog = _program(lops, LS - PROG_LANES)
        lprog_off = TREE_HEADER
        tprog_off = lprog_off + len(lprog)
        exp_off = tprog_off + len(tprog)
        leaf_off = exp_off + len(exp)
        leaf_off += leaf_off & 1  # 8-byte aligned pairs
        hdr = np.array([nl, TS, 0, lprog_off, tprog_off, exp_off, len(exp) // 2, root_top, E, mode, leaf_off, 0],
                       dtype=np.int32)
        blocks.append(np.concatenate([hdr, lprog, tprog, exp, np.zeros(leaf_off - exp_off - len(exp), np.int32),
                                      leaves]).astype(np.int32))
    PI = max(len(bk) for bk in blocks)
    for bk in blocks:
        bk[0] = LS
        bk[2] = PI
    return blocks


def evaluate_split(flat: np.ndarray, blocks: list[np.ndarray], ranges, a) -> float:
    """Replay the split tree on the host exactly as the kernel does (test
    helper proving tree_split preserves np.sum's result bit for bit)."""
    p = PlanView(flat)
    a = [float(x) for x in np.asarray(a, dtype=np.float64)]
    if p.n_leaves == 0:
        return 0.0
    leaf = []
    for l in range(p.n_leaves):
        start, size = int(p.leaf_start[l]), int(p.leaf_size[l])
        if size < 8:
            s, body = 0.0, 0
        else:
            body = size - size % 8
            r = []
            for j in range(8):
                acc = a[start + j]
                for t in range(start + j + 8, start + body, 8):
                    acc += a[t]
                r.append(acc)
            s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for t in range(start + body, start + size):
            s += a[t]
        leaf.append(s)

    run = run_program

    TS = int(blocks[0][1])
    top = [0.0] * max(TS, 1)
    for bk, (ra, rb) in zip(blocks, ranges):
        LS = int(bk[0])
        loc = [0.0] * max(LS, 1)
        if int(bk[9]) & MODE_QUAD:
            for g in range((rb - ra) // 4):
                l0 = ra + 4 * g
                loc[g] = (leaf[l0] + leaf[l0 + 1]) + (leaf[l0 + 2] + leaf[l0 + 3])
        else:
            loc[:rb - ra] = leaf[ra:rb]
        run(bk[int(bk[3]):int(bk[4])], loc)
        exp = bk[int(bk[5]):int(bk[5]) + 2 * int(bk[6])]
        for i in range(0, len(exp), 2):
            top[int(exp[i + 1])] = loc[int(exp[i])]
    bk = blocks[0]
    run(bk[int(bk[4]):int(bk[5])], top)
    return top[int(bk[7])]
