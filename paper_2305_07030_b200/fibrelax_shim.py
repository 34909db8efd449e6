"""Drop-in dispatch for the reference package ``fibrelax``.

``install(fibrelax)`` routes the reference's solver entry points to the B200
build without touching any other code of the caller:

* ``fibrelax.dynamic_relaxation_solve`` / ``fibrelax.microsolver.
  dynamic_relaxation_solve`` (reference ``microsolver.py:567-574``) and
  ``internal_forces`` (``:221-238``) take and return the caller's own types
  (``fibrelax.FiberNetwork``, ``AffineBC``, ``SolverConfig``,
  ``SolveResult``); inputs are converted field for field.
* Errors are raised as the caller's classes: a collapsed element raises an
  exception that IS a ``fibrelax.SingularElementError`` (and
  ``fibrelax.SolverError`` / ``RuntimeError``) and also the B200 class, with
  the reference's message ``element <i>: current length collapsed``
  (``microsolver.py:207-209``); a massless node raises the caller's
  ``NetworkMassError`` (``:166-167``, ``:179-181``).
* ``uninstall(fibrelax)`` restores the originals.

When ``only_if_env`` is given, the dispatch is taken only while that
environment variable is ``"b200"`` (the INTEGRATION.md recipe,
``FIBRELAX_DEVICE=b200``); otherwise always.
"""

from __future__ import annotations

import os

import numpy as np

from . import batch as _batch
from . import microsolver as _ms
from . import network as _nw

_ORIGINALS = "_b200_originals"


def to_b200_network(net) -> _nw.FiberNetwork:
    mats = [_nw.Material(float(m.elastic_modulus), float(m.cross_section_area), float(m.density))
            for m in net.materials]
    return _nw.FiberNetwork(np.asarray(net.node_coords), np.asarray(net.elements), mats,
                            frozenset(int(b) for b in net.boundary_nodes), rve_volume=net.rve_volume)


def to_b200_config(fr, cfg) -> _ms.SolverConfig:
    if cfg is None:
        return _ms.SolverConfig()
    damping = (_ms.FixedDamping(float(cfg.damping.c)) if isinstance(cfg.damping, fr.FixedDamping)
               else _ms.AdaptiveDamping())
    return _ms.SolverConfig(tol_rel=cfg.tol_rel, tol_abs=cfg.tol_abs, max_iters=cfg.max_iters,
                            dt_safety=cfg.dt_safety, damping=damping,
                            energy_check_interval=cfg.energy_check_interval, bc_ramp_iters=cfg.bc_ramp_iters)


def error_classes(fr):
    """The caller's exception classes joined with the B200 ones (raised by the
    dispatch; an ``except fibrelax.SingularElementError`` catches them)."""
    ms = getattr(fr, "microsolver", fr)

    class SingularElementError(_ms.SingularElementError, fr.SingularElementError):
        def __init__(self, message, element=None, problem=None):
            _ms.SingularElementError.__init__(self, message, element=element, problem=problem)

    class NetworkMassError(_ms.NetworkMassError, ms.NetworkMassError):
        pass

    SingularElementError.__module__ = NetworkMassError.__module__ = fr.__name__
    return SingularElementError, NetworkMassError


def install(fr, only_if_env: str | None = None) -> None:
    """Route fibrelax's solver entry points to the B200 build."""
    if hasattr(fr, _ORIGINALS):
        return
    ms = getattr(fr, "microsolver", fr)
    orig = {"solve": fr.dynamic_relaxation_solve, "ms_solve": ms.dynamic_relaxation_solve,
            "forces": fr.internal_forces, "ms_forces": ms.internal_forces}
    Singular, Mass = error_classes(fr)

    def active():
        return only_if_env is None or os.environ.get(only_if_env) == "b200"

    def dynamic_relaxation_solve(network, bc, config=None):
        if not active():
            return orig["solve"](network, bc, config)
        try:
            r = _ms.dynamic_relaxation_solve(to_b200_network(network), _nw.AffineBC(bc.deformation_gradient),
                                             to_b200_config(fr, config))
        except _ms.SingularElementError as e:
            raise Singular(str(e), element=e.element, problem=e.problem) from None
        except _ms.NetworkMassError as e:
            raise Mass(str(e)) from None
        return fr.SolveResult(converged=r.converged, iters=r.iters, final_residual=r.final_residual, u=r.u,
                              avg_stress=r.avg_stress, energy_residual=r.energy_residual, r_ref=r.r_ref)

    def internal_forces(network, u):
        if not active():
            return orig["forces"](network, u)
        try:
            return _batch.internal_forces_device(to_b200_network(network), np.asarray(u, dtype=np.float64))
        except _ms.SingularElementError as e:
            raise Singular(str(e), element=e.element) from None

    fr.dynamic_relaxation_solve = ms.dynamic_relaxation_solve = dynamic_relaxation_solve
    fr.internal_forces = ms.internal_forces = internal_forces
    setattr(fr, _ORIGINALS, orig)


def uninstall(fr) -> None:
    orig = getattr(fr, _ORIGINALS, None)
    if orig is None:
        return
    ms = getattr(fr, "microsolver", fr)
    fr.dynamic_relaxation_solve, ms.dynamic_relaxation_solve = orig["solve"], orig["ms_solve"]
    fr.internal_forces, ms.internal_forces = orig["forces"], orig["ms_forces"]
    delattr(fr, _ORIGINALS)
