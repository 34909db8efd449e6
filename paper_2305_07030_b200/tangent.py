"""Homogenized tangent dσ/dF by batched perturbed re-solves (SURVEY.md
§8 row f-2, the FE² macro solver's "tangent return" of BASELINE.json's
north star).

The reference has no tangent (``SPEC.md:332`` lists it as a non-goal), so
there is no reference output to pin it to.  What is pinned: every perturbed
solve is the bit-exact relaxation of ``microsolver.py:379-564`` on the
device, and the finite-difference assembly below is plain host arithmetic,
so the tangent equals the CPU oracle's finite differences of ``avg_stress``
up to the stress tolerance of the solver parity bar (σ agrees to 1e-13
relative; tests/test_gpu_parity.py::test_tangent_matches_oracle_differences).

All perturbations of all networks go to the device as ONE batch: a
network's 10 (forward) or 19 (central) copies share one host setup and one
set of topology tables (incidence, cluster partition, tree programs); only
the per-problem arrays (coordinates, masses, lengths) are repeated.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
from numpy.typing import NDArray

from .microsolver import SolverConfig
from .network import AffineBC, FiberNetwork

__all__ = ["TangentResult", "perturbed_gradients", "assemble_tangent", "homogenized_tangent"]

SCHEMES = ("forward", "central")


@dataclass
class TangentResult:
    """σ at F and C[i, j, k, l] = dσ_ij / dF_kl (finite differences of step h)."""

    sigma: NDArray[np.float64]      # 3x3
    tangent: NDArray[np.float64]    # 3x3x3x3
    converged: bool                 # every solve of this network converged
    iters: NDArray[np.int64]        # iterations of the base solve then each perturbation


def perturbed_gradients(F: NDArray, h: float, scheme: str = "central") -> list[NDArray[np.float64]]:
    """[F, F + h E_kl (k, l row-major), then F - h E_kl for the central scheme]."""
    if scheme not in SCHEMES:
        raise ValueError(f"scheme must be one of {SCHEMES}, got {scheme!r}")
    if not h > 0:
        raise ValueError(f"h must be > 0, got {h}")
    F = np.asarray(F, dtype=np.float64).reshape(3, 3)
    out = [F.copy()]
    signs = (1.0, -1.0) if scheme == "central" else (1.0,)
    for sgn in signs:
        for k in range(3):
            for l in range(3):
                Fp = F.copy()
                Fp[k, l] += sgn * h
                out.append(Fp)
    return out


def assemble_tangent(sigmas: Sequence[NDArray], h: float, scheme: str = "central") -> NDArray[np.float64]:
    """C[:, :, k, l] from the stresses in perturbed_gradients order:
    forward (σ(F + h E_kl) - σ(F)) / h, central (σ(F + h E_kl) - σ(F - h E_kl)) / 2h."""
    s = [np.asarray(x, dtype=np.float64).reshape(3, 3) for x in sigmas]
    need = 19 if scheme == "central" else 10
    if scheme not in SCHEMES or len(s) != need:
        raise ValueError(f"{scheme} differences need {need} stresses, got {len(s)}")
    C = np.empty((3, 3, 3, 3))
    for kl in range(9):
        k, l = divmod(kl, 3)
        if scheme == "central":
            C[:, :, k, l] = (s[1 + kl] - s[10 + kl]) / (2.0 * h)
        else:
            C[:, :, k, l] = (s[1 + kl] - s[0]) / h
    return C


def homogenized_tangent(networks: Sequence[FiberNetwork], Fs: Sequence[NDArray], h: float = 1e-6,
                        scheme: str = "central", config: SolverConfig | None = None,
                        strategy=None) -> list[TangentResult]:
    """σ(F) and dσ/dF for every network at its deformation gradient, all
    (1 + 9 or 1 + 18) solves per network in one device batch."""
    from dataclasses import replace
    from .batch import _pack, build_problem, solve_batch
    if len(networks) != len(Fs):
        raise ValueError(f"networks and Fs differ in length ({len(networks)} vs {len(Fs)})")
    per = 19 if scheme == "central" else 10
    nets, bcs, probs = [], [], []
    for net, F in zip(networks, Fs):
        base = None
        for Fp in perturbed_gradients(F, h, scheme):
            bc = AffineBC(Fp)
            # one host setup per network; the perturbed copies differ in F only
            base = build_problem(net, bc) if base is None else base
            nets.append(net)
            bcs.append(bc)
            probs.append(replace(base, F=np.asarray(Fp, dtype=np.float64)))
    res = solve_batch(_pack(nets, bcs, probs), strategy=strategy, config=config or SolverConfig())
    out = []
    for p in range(len(networks)):
        rs = res[p * per:(p + 1) * per]
        out.append(TangentResult(sigma=np.asarray(rs[0].avg_stress, dtype=np.float64),
                                 tangent=assemble_tangent([r.avg_stress for r in rs], h, scheme),
                                 converged=all(r.converged for r in rs),
                                 iters=np.array([r.iters for r in rs], dtype=np.int64)))
    return out
