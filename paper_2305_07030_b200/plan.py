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

Flat int32 layout consumed by ``csrc/frb_kernels.cu`` (``PlanView``):
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
