"""CPU ORACLE for the batched dynamic-relaxation hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / the timed reference
arm.  The product (``paper_2305_07030_b200``) never imports it.

What it restates
----------------
The reference is the pure-NumPy package ``fibrelax`` 0.1.0
(``/root/reference/pkg/src/fibrelax``).  Its arithmetic lives in numpy 2.3.5
(pinned; einsum, bincount, add.at, pairwise ``np.sum``) and OpenBLAS 0.3.30
(the ``@`` for prescribed displacements).  This module restates the same
algorithm in the *device's* formulation, so it doubles as the proof that the
CUDA evaluation order reproduces the reference bit for bit:

* per-node role-split gather in element order instead of ``np.bincount``
  (reference ``microsolver.py:214-218``);
* the NumPy pairwise-sum tree written out (leaves of <=128 with 8 strided
  accumulators, split at n/2 rounded down to a multiple of 8) instead of
  ``np.sum`` (``microsolver.py:479, 481, 494``);
* lengths as ``sqrt((x*x + z*z) + y*y)`` (the einsum order,
  ``microsolver.py:205-206``, ``network.py:171-172``);
* the prescribed displacement as the FMA chain OpenBLAS evaluates for
  ``x_ref[nfn:] @ (F-I).T`` (``microsolver.py:320-322``), computed exactly
  with rationals so it does not depend on the host BLAS.

Parity pinning: ``tests/golden/`` holds outputs of the real reference run in
the build container (``tests/golden/make_golden.py``); ``tests/test_oracle.py``
checks this module against them bit for bit.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

COLLAPSE = 1e-12        # reference microsolver.py:30 LENGTH_COLLAPSE_FRACTION
ENERGY_FLOOR = 1e-30    # reference microsolver.py:29

STATUS_CONVERGED, STATUS_MAX_ITERS, STATUS_SINGULAR = 0, 1, 2


# ---------------------------------------------------------------- numerics

def seg_len(d: np.ndarray) -> np.ndarray:
    """Row norms in einsum's (x, z, y) order (reference microsolver.py:206)."""
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    return np.sqrt((x * x + z * z) + y * y)


def _split(n: int) -> int:
    h = n // 2
    return h - h % 8


def pairwise_scalar(a) -> float:
    """NumPy's pairwise_sum written out on Python floats (small n only)."""
    a = [float(x) for x in a]
    n = len(a)
    if n < 8:
        s = 0.0
        for x in a:
            s += x
        return s
    if n <= 128:
        r = a[:8]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] += a[i + j]
            i += 8
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for x in a[i:]:
            s += x
        return s
    h = _split(n)
    return pairwise_scalar(a[:h]) + pairwise_scalar(a[h:])


class PairwisePlan:
    """Vectorised evaluation of the pairwise tree for a fixed length n.

    Evaluates k independent sums at once (rows of a (k, n) array): the leaf
    chains run in lockstep across leaves, then the recursion combines leaf
    sums in the reference's split order.
    """

    def __init__(self, n: int):
        self.n = n
        self.leaves = []            # (start, size)
        self.tree = self._build(0, n)
        L = len(self.leaves)
        q = [s // 8 if s >= 8 else 0 for _, s in self.leaves]
        self.qmax = max(q) if q else 0
        self.chain_idx = np.zeros((max(L, 1), max(self.qmax, 1), 8), dtype=np.int64)
        self.chain_ok = np.zeros((max(L, 1), max(self.qmax, 1)), dtype=bool)
        self.tail_idx = np.zeros((max(L, 1), 8), dtype=np.int64)
        self.tail_ok = np.zeros((max(L, 1), 8), dtype=bool)
        self.small = np.zeros(max(L, 1), dtype=bool)
        for l, (start, size) in enumerate(self.leaves):
            if size < 8:
                self.small[l] = True
                body = 0
            else:
                body = size - size % 8
                for t in range(size // 8):
                    self.chain_idx[l, t] = start + 8 * t + np.arange(8)
                    self.chain_ok[l, t] = True
            for i, d in enumerate(range(start + body, start + size)):
                self.tail_idx[l, i] = d
                self.tail_ok[l, i] = True

    def _build(self, start, n):
        if n <= 128:
            self.leaves.append((start, n))
            return len(self.leaves) - 1
        h = _split(n)
        return (self._build(start, h), self._build(start + h, n - h))

    def __call__(self, a: np.ndarray) -> np.ndarray:
        a = np.atleast_2d(a)
        k = a.shape[0]
        if self.n == 0:
            return np.zeros(k)
        L = len(self.leaves)
        if self.qmax:
            r = a[:, self.chain_idx[:, 0, :]]                       # (k, L, 8)
            for t in range(1, self.qmax):
                ok = self.chain_ok[None, :L, t, None]
                r = np.where(ok, r + a[:, self.chain_idx[:, t, :]], r)
            leaf = ((r[..., 0] + r[..., 1]) + (r[..., 2] + r[..., 3])) + \
                   ((r[..., 4] + r[..., 5]) + (r[..., 6] + r[..., 7]))
            leaf = np.where(self.small[None, :L], 0.0, leaf)
        else:
            leaf = np.zeros((k, L))
        for i in range(8):
            ok = self.tail_ok[None, :L, i]
            if ok.any():
                leaf = np.where(ok, leaf + a[:, self.tail_idx[:L, i]], leaf)
        return self._eval(self.tree, leaf)

    def _eval(self, node, leaf):
        if isinstance(node, int):
            return leaf[:, node]
        return self._eval(node[0], leaf) + self._eval(node[1], leaf)


def fma_exact(a: float, b: float, c: float) -> float:
    """Correctly rounded a*b + c (Fraction -> float rounds to nearest-even)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def prescribed_displacement(x_fixed: np.ndarray, F: np.ndarray) -> np.ndarray:
    """u_presc = x_fixed @ (F - I).T as OpenBLAS's FMA chain evaluates it
    (reference microsolver.py:320-322): t = x0*g[j,0]; t = fma(x1, g[j,1], t);
    t = fma(x2, g[j,2], t)."""
    g = np.asarray(F, dtype=np.float64) - np.eye(3)
    out = np.empty((len(x_fixed), 3))
    for i, (x0, x1, x2) in enumerate(x_fixed.tolist()):
        for j in range(3):
            t = x0 * float(g[j, 0])
            t = fma_exact(x1, float(g[j, 1]), t)
            out[i, j] = fma_exact(x2, float(g[j, 2]), t)
    return out


def _role_slots(node_of_elem: np.ndarray, n_nodes: int) -> np.ndarray:
    """Padded (n_nodes, deg) matrix of element ids per node, ascending, -1 pad."""
    m = len(node_of_elem)
    if m == 0:
        return np.full((n_nodes, 0), -1, dtype=np.int64)
    order = np.argsort(node_of_elem, kind="stable")
    counts = np.bincount(node_of_elem, minlength=n_nodes)
    deg = int(counts.max())
    start = np.zeros(n_nodes + 1, dtype=np.int64)
    np.cumsum(counts, out=start[1:])
    slots = np.full((n_nodes, deg), -1, dtype=np.int64)
    rank = np.arange(m) - start[node_of_elem[order]]
    slots[node_of_elem[order], rank] = order
    return slots


def _gather_sum(values: np.ndarray, slots: np.ndarray, n_nodes: int) -> np.ndarray:
    """Per node: 0.0 + values[e1] + values[e2] + ... in slot order.

    Padding slots (-1) read an appended +0.0 row; adding +0.0 is exact here
    because a running sum that starts at +0.0 can never become -0.0."""
    padded = np.concatenate([values, np.zeros((1,) + values.shape[1:])])
    acc = np.zeros((n_nodes,) + values.shape[1:])
    for s in range(slots.shape[1]):
        acc = acc + padded[slots[:, s]]
    return acc


# ---------------------------------------------------------------- problem

@dataclass
class OracleSetup:
    n_nodes: int
    nfn: int
    order: np.ndarray          # solver position -> original node
    X: np.ndarray              # (N, 3) solver order
    ia: np.ndarray
    ib: np.ndarray
    ea: np.ndarray
    L: np.ndarray
    eps: np.ndarray
    dt: float
    mass: np.ndarray           # (N,) solver order
    u_presc: np.ndarray        # (N - nfn, 3)
    slots_a: np.ndarray
    slots_b: np.ndarray
    volume: float
    boundary_sorted: np.ndarray


def setup(network, F, dt_safety: float) -> OracleSetup:
    """build_problem restated (reference microsolver.py:302-335, 170-182)."""
    coords = np.asarray(network.node_coords, dtype=np.float64)
    elems = np.asarray(network.elements, dtype=np.int64).reshape(-1, 3)
    n = len(coords)
    fixed = np.zeros(n, dtype=bool)
    fixed[list(network.boundary_nodes)] = True
    order = np.concatenate([np.flatnonzero(~fixed), np.flatnonzero(fixed)])
    rank = np.empty(n, dtype=np.int64)
    rank[order] = np.arange(n)
    nfn = int((~fixed).sum())
    mats = np.array([[m.elastic_modulus, m.cross_section_area, m.density]
                     for m in network.materials], dtype=np.float64).reshape(-1, 3)
    E, A, rho = (mats[elems[:, 2], c] for c in range(3))
    L = seg_len(coords[elems[:, 1]] - coords[elems[:, 0]])
    # lumped mass: role a in element order, then role b (np.add.at, :177-178)
    half = rho * A * L / 2.0
    mass_orig = np.zeros(n)
    sa = _role_slots(elems[:, 0], n)
    sb = _role_slots(elems[:, 1], n)
    for slots in (sa, sb):
        for s in range(slots.shape[1]):
            col = slots[:, s]
            ok = col >= 0
            mass_orig[ok] = mass_orig[ok] + half[col[ok]]
    if np.any(mass_orig <= 0):
        raise ValueError(f"node {int(np.argmin(mass_orig))} has zero mass (no incident elements)")
    ia, ib = rank[elems[:, 0]], rank[elems[:, 1]]
    X = coords[order]
    dt = dt_safety * float(np.min(L * np.sqrt(rho / E))) if len(L) else math.nan
    return OracleSetup(
        n_nodes=n, nfn=nfn, order=order, X=X, ia=ia, ib=ib, ea=E * A, L=L,
        eps=COLLAPSE * L, dt=dt, mass=mass_orig[order],
        u_presc=prescribed_displacement(X[nfn:], F),
        slots_a=_role_slots(ia, n), slots_b=_role_slots(ib, n),
        volume=float(network.volume), boundary_sorted=np.sort(np.flatnonzero(fixed)))


def forces(s: OracleSetup, u: np.ndarray):
    """Element forces + per-node gather (reference microsolver.py:196-218).

    Returns (f (N,3), bad) where bad is the singular element index or -1.
    """
    P = s.X + u
    d = P[s.ib] - P[s.ia]
    l = seg_len(d)
    if np.any(l < s.eps):
        return None, int(np.argmin(l - s.eps))
    coef = s.ea * (l - s.L) / (s.L * l)
    nd = d * coef[:, None]
    fa = _gather_sum(-nd, s.slots_a, s.n_nodes)
    fb = _gather_sum(nd, s.slots_b, s.n_nodes)
    return fa + fb, -1


@dataclass
class OracleResult:
    status: int
    converged: bool
    iters: int
    residual: float
    r_ref: float
    u: np.ndarray              # original DOF order (3N,)
    f: np.ndarray              # original DOF order (3N,)
    sigma: np.ndarray          # (3, 3)
    energy_residual: float | None
    bad_element: int = -1
    energy: dict = field(default_factory=dict)


def _cfg(cfg):
    fixed_c = getattr(cfg.damping, "c", None)
    return (float(cfg.tol_rel), float(cfg.tol_abs), int(cfg.max_iters), float(cfg.dt_safety),
            fixed_c, int(cfg.energy_check_interval), int(cfg.bc_ramp_iters))


def solve(network, F, cfg, s: OracleSetup | None = None) -> OracleResult:
    """One dynamic-relaxation solve (reference microsolver.py:379-574)."""
    tol_rel, tol_abs, max_iters, dt_safety, fixed_c, energy_iv, ramp = _cfg(cfg)
    s = s or setup(network, F, dt_safety)
    n, nfn = s.n_nodes, s.nfn
    nf = 3 * nfn
    m = np.repeat(s.mass[:nfn], 3)
    plan = PairwisePlan(nf)
    energy_on = energy_iv > 0
    full_bc_iter = 0 if ramp == 0 else ramp - 1
    dt = s.dt
    hdt = 0.5 * dt

    u = np.zeros((n, 3))
    v = np.zeros(nf)
    alpha = 0.0 if ramp > 0 else 1.0
    d_alpha = 0.0
    c = float(fixed_c) if fixed_c is not None else 0.0
    w = dict(w_kin=0.0, w_int=0.0, w_damp=0.0, w_ext=0.0)
    if ramp == 0:
        u[nfn:] = s.u_presc
    f, bad = forces(s, u)
    if bad >= 0:
        return _singular(s, bad)
    if energy_on and ramp == 0:
        step = 0.5 * float(np.dot(f[nfn:].reshape(-1), s.u_presc.reshape(-1)))
        w["w_ext"] += step
        w["w_int"] += step
    a = -f[:nfn].reshape(-1) / m
    residual, r_ref, threshold = math.inf, math.nan, math.inf
    converged = False
    it = 0
    while True:
        v = v + hdt * a
        uf = u[:nfn].reshape(-1) + dt * v
        u[:nfn] = uf.reshape(-1, 3)
        if alpha < 1.0:
            new = min(1.0, (it + 1) / ramp)
            d_alpha = new - alpha
            alpha = new
            u[nfn:] = alpha * s.u_presc
        f_prev = f
        f, bad = forces(s, u)
        if bad >= 0:
            return _singular(s, bad)
        ff = f[:nfn].reshape(-1)
        fp = f_prev[:nfn].reshape(-1)
        if fixed_c is None:
            den = dt * v
            num = ff - fp
            kh = np.zeros_like(num)
            np.divide(num, den, out=kh, where=den != 0)
            kh = np.where((kh > 0.0) | np.isnan(kh), kh, 0.0)
            sums = plan(np.stack([(uf * kh) * uf, (uf * m) * uf, ff * ff]))
            mq = float(sums[1])
            if mq > 0.0:
                lam = float(sums[0]) / mq
                c = 2.0 * math.sqrt(lam) if lam > 0 else 0.0
            else:
                c = 0.0
            fsq = float(sums[2])
        else:
            fsq = float(plan(ff * ff)[0])
        residual = float(np.sqrt(fsq))
        if it == full_bc_iter:
            r_ref = residual
            t = tol_rel * r_ref
            threshold = t if t > tol_abs else tol_abs
        v_half = v
        a = (-ff) / m - c * v
        v = v + hdt * a
        if energy_on:
            _energy(w, s, f, f_prev, v_half, v, m, dt, c, d_alpha, nfn)
            d_alpha = 0.0
        iters = it + 1
        if it >= full_bc_iter and residual <= threshold:
            converged = True
            break
        if iters >= max_iters:
            break
        it += 1
    return _finish(s, u, f, converged, iters, residual, r_ref,
                   _balance(w) if energy_on else None, w)


def _energy(w, s, f, f_prev, vh, v, m, dt, c, d_alpha, nfn):
    """Trapezoidal work ledger (reference microsolver.py:533-546)."""
    ff, fp = f[:nfn].reshape(-1), f_prev[:nfn].reshape(-1)
    w["w_int"] += 0.5 * (dt * (float(np.dot(ff, vh)) + float(np.dot(fp, vh))))
    if d_alpha != 0.0:
        du = d_alpha * s.u_presc.reshape(-1)
        wfix = 0.5 * (float(np.dot(f[nfn:].reshape(-1), du)) + float(np.dot(f_prev[nfn:].reshape(-1), du)))
        w["w_int"] += wfix
        w["w_ext"] += wfix
    w["w_damp"] += c * dt * float(np.dot(m * vh, vh))
    w["w_kin"] = 0.5 * float(np.dot(m * v, v))


def _balance(w) -> float:
    defect = abs(w["w_ext"] - w["w_int"] - w["w_kin"] - w["w_damp"])
    return defect / max(abs(w["w_ext"]), abs(w["w_int"]), w["w_kin"], ENERGY_FLOOR)


def _to_original(s: OracleSetup, x: np.ndarray) -> np.ndarray:
    out = np.empty_like(x)
    out[s.order] = x
    return out


def average_stress(s: OracleSetup, u_orig: np.ndarray, f_orig: np.ndarray, coords) -> np.ndarray:
    """sym(sum_b r_b (x) x_b) / V over sorted boundary nodes (reference :285-299);
    BLAS order in the reference, so parity here is tolerance-only."""
    b = s.boundary_sorted
    if b.size == 0:
        return np.zeros((3, 3))
    r = f_orig[b]
    x = coords[b] + u_orig[b]
    S = r.T @ x
    return (S + S.T) / (2.0 * s.volume)


def _finish(s, u, f, converged, iters, residual, r_ref, e_res, w) -> OracleResult:
    u_o = _to_original(s, u)
    f_o = _to_original(s, f)
    coords = _to_original(s, s.X)
    sigma = average_stress(s, u_o, f_o, coords)
    return OracleResult(status=STATUS_CONVERGED if converged else STATUS_MAX_ITERS,
                        converged=converged, iters=iters, residual=residual, r_ref=r_ref,
                        u=u_o.reshape(-1), f=f_o.reshape(-1), sigma=sigma,
                        energy_residual=e_res, energy=dict(w))


def _singular(s, bad) -> OracleResult:
    z = np.zeros(3 * s.n_nodes)
    return OracleResult(status=STATUS_SINGULAR, converged=False, iters=0, residual=math.nan,
                        r_ref=math.nan, u=z, f=z, sigma=np.zeros((3, 3)),
                        energy_residual=None, bad_element=bad)


def internal_forces(network, u_orig) -> np.ndarray:
    """One-shot assembled force at u in original node order (reference
    microsolver.py:221-238).  Returns None-free; raises ValueError on a
    collapsed element."""
    coords = np.asarray(network.node_coords, dtype=np.float64)
    elems = np.asarray(network.elements, dtype=np.int64).reshape(-1, 3)
    n = len(coords)
    mats = np.array([[m.elastic_modulus, m.cross_section_area, m.density]
                     for m in network.materials], dtype=np.float64).reshape(-1, 3)
    E, A = mats[elems[:, 2], 0], mats[elems[:, 2], 1]
    L = seg_len(coords[elems[:, 1]] - coords[elems[:, 0]])
    s = OracleSetup(n_nodes=n, nfn=n, order=np.arange(n), X=coords, ia=elems[:, 0],
                    ib=elems[:, 1], ea=E * A, L=L, eps=COLLAPSE * L, dt=math.nan,
                    mass=np.zeros(n), u_presc=np.zeros((0, 3)),
                    slots_a=_role_slots(elems[:, 0], n), slots_b=_role_slots(elems[:, 1], n),
                    volume=1.0, boundary_sorted=np.zeros(0, dtype=np.int64))
    f, bad = forces(s, np.asarray(u_orig, dtype=np.float64).reshape(n, 3))
    if bad >= 0:
        raise ValueError(f"element {bad}: current length collapsed")
    return f.reshape(-1)
