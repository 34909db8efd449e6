"""Dynamic-relaxation solver API (drop-in for ``fibrelax.microsolver``,
reference ``pkg/src/fibrelax/microsolver.py``).

The relaxation loop itself (reference ``_relax``, ``microsolver.py:379-530``,
plus ``finalize_result`` ``:549-564``) runs on the B200 inside one persistent
CUDA kernel (``csrc/frb_relax.cuh``) reached through the C-ABI
``libfrb200.so``.  This module keeps the reference's public types, their
validation, and the small host-side helpers; ``dynamic_relaxation_solve`` is
a batch of one through ``batch.solve_batch``.  There is no CPU fallback: if
the CUDA library or a device is missing the call raises.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np
from numpy.typing import NDArray

from .network import AffineBC, FiberNetwork

__all__ = [
    "AdaptiveDamping", "EnergyLedger", "FixedDamping", "MicroState", "NetworkMassError",
    "SingularElementError", "SolveResult", "SolverConfig", "SolverError", "average_stress",
    "compute_lumped_mass", "critical_time_step", "damping_coefficient",
    "dynamic_relaxation_solve", "energy_balance", "force_residual", "internal_forces",
]

ENERGY_FLOOR = 1e-30
LENGTH_COLLAPSE_FRACTION = 1e-12


class SolverError(RuntimeError):
    pass


class SingularElementError(SolverError):
    """An element's current length collapsed below 1e-12 of its reference length."""

    def __init__(self, message: str, element: int | None = None, problem: int | None = None):
        super().__init__(message)
        self.element = element
        self.problem = problem


class NetworkMassError(ValueError):
    pass


@dataclass(frozen=True)
class FixedDamping:
    c: float

    def __post_init__(self):
        if self.c < 0:
            raise ValueError(f"fixed damping coefficient must be >= 0, got {self.c}")


@dataclass(frozen=True)
class AdaptiveDamping:
    """Rayleigh-quotient damping c = 2 sqrt(lambda), re-estimated every step."""


@dataclass(frozen=True)
class SolverConfig:
    """Solver knobs (reference ``microsolver.py:55-75``; same defaults and
    validation).  ``energy_check_interval`` > 0 switches the work ledger on;
    like the reference, the value is otherwise only used as a flag."""

    tol_rel: float = 1e-8
    tol_abs: float = 0.0
    max_iters: int = 20000
    dt_safety: float = 0.5
    damping: FixedDamping | AdaptiveDamping = AdaptiveDamping()
    energy_check_interval: int = 0
    bc_ramp_iters: int = 0

    def __post_init__(self):
        if not 0.0 < self.dt_safety <= 1.0:
            raise ValueError(f"dt_safety must be in (0, 1], got {self.dt_safety}")
        if self.tol_rel < 0 or self.tol_abs < 0:
            raise ValueError("tolerances must be >= 0")
        if self.tol_rel == 0 and self.tol_abs == 0:
            raise ValueError("tol_rel and tol_abs cannot both be zero")
        if self.max_iters <= 0:
            raise ValueError(f"max_iters must be > 0, got {self.max_iters}")
        if self.energy_check_interval < 0 or self.bc_ramp_iters < 0:
            raise ValueError("intervals must be >= 0")


@dataclass
class EnergyLedger:
    w_kin: float = 0.0
    w_int: float = 0.0
    w_damp: float = 0.0
    w_ext: float = 0.0


@dataclass
class MicroState:
    """Per-problem state in solver (free-prefix) DOF order."""

    u: NDArray[np.float64]
    v: NDArray[np.float64]
    a: NDArray[np.float64]
    f_int: NDArray[np.float64]
    m: NDArray[np.float64]
    n_free: int
    residual: float = math.inf
    iters: int = 0
    energy: EnergyLedger = field(default_factory=EnergyLedger)
    f_prev: NDArray[np.float64] | None = None
    dt: float = 0.0


@dataclass
class SolveResult:
    """Public result (reference ``microsolver.py:103-135``)."""

    converged: bool
    iters: int
    final_residual: float
    u: NDArray[np.float64]                 # original DOF order
    avg_stress: NDArray[np.float64]        # 3x3 symmetric
    energy_residual: float | None
    r_ref: float

    def to_json(self) -> str:
        return json.dumps({
            "converged": bool(self.converged),
            "iters": int(self.iters),
            "final_residual": float(self.final_residual),
            "avg_stress": [float(x) for x in np.asarray(self.avg_stress).reshape(9)],
            "energy_residual": None if self.energy_residual is None else float(self.energy_residual),
            "u": [float(x) for x in np.asarray(self.u)],
        })

    @classmethod
    def from_json(cls, text: str) -> "SolveResult":
        doc = json.loads(text)
        e = doc["energy_residual"]
        return cls(converged=bool(doc["converged"]), iters=int(doc["iters"]),
                   final_residual=float(doc["final_residual"]),
                   u=np.asarray(doc["u"], dtype=np.float64),
                   avg_stress=np.asarray(doc["avg_stress"], dtype=np.float64).reshape(3, 3),
                   energy_residual=None if e is None else float(e), r_ref=math.nan)


# --------------------------------------------------------------- host helpers

def _lumped_node_mass(network: FiberNetwork, columns=None, lengths=None) -> NDArray[np.float64]:
    """rho*A*L/2 to each end; role a in element order, then role b
    (reference ``microsolver.py:170-182``; np.add.at is sequential).
    columns / lengths: precomputed material_columns() / reference_lengths()."""
    _, area, rho = columns if columns is not None else network.material_columns()
    half = rho * area * (lengths if lengths is not None else network.reference_lengths()) / 2.0
    node_mass = np.zeros(network.n_nodes)
    np.add.at(node_mass, network.elements[:, 0], half)
    np.add.at(node_mass, network.elements[:, 1], half)
    if np.any(node_mass <= 0):
        raise NetworkMassError(
            f"node {int(np.argmin(node_mass))} has zero mass (no incident elements)")
    return node_mass


def compute_lumped_mass(network: FiberNetwork) -> NDArray[np.float64]:
    """Per-DOF lumped mass, original order."""
    return np.repeat(_lumped_node_mass(network), 3)


def critical_time_step(network: FiberNetwork, safety: float = 1.0) -> float:
    """safety * min_e L_e sqrt(rho_e / E_e) (reference ``microsolver.py:185-193``)."""
    if network.n_elements == 0:
        raise ValueError("network has no elements")
    emod, _, rho = network.material_columns()
    return float(safety * np.min(network.reference_lengths() * np.sqrt(rho / emod)))


def force_residual(f_int: NDArray, n_free: int) -> float:
    """L2 norm over the free prefix (reference ``microsolver.py:241-246``)."""
    f_int = np.asarray(f_int)
    if n_free > f_int.shape[0]:
        raise ValueError(f"n_free={n_free} exceeds vector length {f_int.shape[0]}")
    return float(np.sqrt(np.sum(np.square(f_int[:n_free]))))


def damping_coefficient(state: MicroState, mode: FixedDamping | AdaptiveDamping) -> float:
    """Fixed c, or the Rayleigh-quotient estimate 2 sqrt(lambda) with the
    clamped diagonal stiffness k_i = (f_i - f_prev_i) / (dt v_i)
    (reference ``microsolver.py:249-271``)."""
    if isinstance(mode, FixedDamping):
        return mode.c
    nf = state.n_free
    if nf == 0 or state.f_prev is None or state.dt == 0.0:
        return 0.0
    u = state.u[:nf]
    den = state.dt * state.v[:nf]
    num = state.f_int[:nf] - state.f_prev[:nf]
    khat = np.zeros_like(num)
    np.divide(num, den, out=khat, where=den != 0)
    np.maximum(khat, 0.0, out=khat)
    mass_quad = float(np.sum(u * state.m[:nf] * u))
    if mass_quad <= 0.0:
        return 0.0
    lam = float(np.sum(u * khat * u)) / mass_quad
    return 2.0 * math.sqrt(lam) if lam > 0 else 0.0


def energy_balance(state: MicroState) -> float:
    """|W_ext - W_int - W_kin - W_damp| / max(|W_ext|, |W_int|, W_kin, floor)."""
    e = state.energy
    defect = abs(e.w_ext - e.w_int - e.w_kin - e.w_damp)
    return defect / max(abs(e.w_ext), abs(e.w_int), e.w_kin, ENERGY_FLOOR)


def average_stress(network: FiberNetwork, u: NDArray, f_int: NDArray) -> NDArray[np.float64]:
    """sym(sum over sorted boundary nodes of r (x) x) / V
    (reference ``microsolver.py:285-299``)."""
    u = np.asarray(u, dtype=np.float64).reshape(network.n_nodes, 3)
    f = np.asarray(f_int, dtype=np.float64).reshape(network.n_nodes, 3)
    bound = sorted(network.boundary_nodes)
    if not bound:
        return np.zeros((3, 3))
    s = f[bound].T @ (network.node_coords[bound] + u[bound])
    return (s + s.T) / (2.0 * network.volume)


# --------------------------------------------------------------- device path

def internal_forces(network: FiberNetwork, u: NDArray) -> NDArray[np.float64]:
    """Assembled internal force at u (original order), evaluated on the GPU
    with the solver's exact gather order (reference ``microsolver.py:221-238``)."""
    from .batch import internal_forces_device
    u = np.asarray(u, dtype=np.float64)
    if u.shape[0] != 3 * network.n_nodes:
        raise ValueError(f"expected displacement vector of length {3 * network.n_nodes}, got {u.shape[0]}")
    return internal_forces_device(network, u)


def dynamic_relaxation_solve(network: FiberNetwork, bc: AffineBC,
                             config: SolverConfig | None = None) -> SolveResult:
    """Solve one network to static equilibrium on the B200 (batch of one).

    Same contract as reference ``microsolver.py:567-574``: non-convergence is
    reported via ``converged=False``; a collapsed element raises
    ``SingularElementError``.
    """
    from .batch import pack_batch, solve_batch
    return solve_batch(pack_batch([network], [bc]), config=config or SolverConfig())[0]
