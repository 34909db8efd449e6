"""Homogenized tangent: finite-difference assembly on the host
and, against the CPU oracle, the symmetry the assembly must preserve."""

import numpy as np
import pytest

from paper_2305_07030_b200.tangent import assemble_tangent, perturbed_gradients
from oracle import frb_oracle as orc


def test_perturbations_are_row_major_unit_steps():
    F = np.diag([1.1, 1.0, 0.9])
    fw = perturbed_gradients(F, 1e-3, "forward")
    ce = perturbed_gradients(F, 1e-3, "central")
    assert len(fw) == 10 and len(ce) == 19
    assert np.array_equal(fw[0], F) and np.array_equal(ce[0], F)
    for kl in range(9):
        k, l = divmod(kl, 3)
        E = np.zeros((3, 3))
        E[k, l] = 1e-3
        assert np.array_equal(fw[1 + kl], F + E)
        assert np.array_equal(ce[1 + kl], F + E)
        assert np.array_equal(ce[10 + kl], F - E)


def test_assembly_is_exact_for_a_linear_stress():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((3, 3, 3, 3))
    F = np.eye(3) + 0.05 * rng.standard_normal((3, 3))
    h = 0.25  # power of two: every difference is exact
    for scheme in ("forward", "central"):
        sig = [np.einsum("ijkl,kl->ij", A, Fp) for Fp in perturbed_gradients(F, h, scheme)]
        assert np.allclose(assemble_tangent(sig, h, scheme), A, rtol=0, atol=1e-12)


def test_bad_arguments_raise():
    with pytest.raises(ValueError):
        perturbed_gradients(np.eye(3), 0.0)
    with pytest.raises(ValueError):
        perturbed_gradients(np.eye(3), 1e-6, "backward")
    with pytest.raises(ValueError):
        assemble_tangent([np.eye(3)] * 10, 1e-6, "central")


def test_oracle_tangent_is_symmetric_in_ij_and_near_linear_elastic_order():
    """Central differences of the oracle's avg_stress on a small lattice: C_ijkl
    = C_jikl exactly (σ is symmetrised per solve), and forward/central agree to
    O(h) (the FD schemes are consistent)."""
    import paper_2305_07030_b200 as frb
    net = frb.generate_lattice(3, 3, 4, 0.3, 1)
    F = np.diag([1.05, 1.0, 1.0])
    cfg = frb.SolverConfig()
    h = 1e-5
    sig_c = [orc.solve(net, Fp, cfg).sigma for Fp in perturbed_gradients(F, h, "central")]
    C = assemble_tangent(sig_c, h, "central")
    assert np.array_equal(C, C.transpose(1, 0, 2, 3))
    Cf = assemble_tangent(sig_c[:10], h, "forward")
    scale = np.abs(C).max()
    assert scale > 0 and np.abs(Cf - C).max() <= 1e-2 * scale
