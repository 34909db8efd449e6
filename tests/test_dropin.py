"""Drop-in conformance with the reference package ``fibrelax``.

* The reference's OWN test suite (``/root/reference/pkg/tests``: network
  construction and text I/O, DOF map, packed storage) runs against this
  package through a ``fibrelax`` module alias -- in the build container only
  (the reference is not on the GPU box).
* The INTEGRATION.md dispatch (``paper_2305_07030_b200.fibrelax_shim``):
  installing it on the real reference routes ``dynamic_relaxation_solve``
  to the B200 and raises the caller's own exception classes.
* File formats around the path: ``load_network`` / ``save_network`` round
  trips and the ``SolveResult`` JSON schema (reference ``network.py:186-309``,
  ``microsolver.py:113-135``).
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import golden_cases as gc
import paper_2305_07030_b200 as frb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
BASELINE_REF = os.path.join(ROOT, "baseline", "_ref")
need_ref_tests = pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tests not present (GPU box)")

ALIAS = """
import sys
sys.path.insert(0, {root!r})
import paper_2305_07030_b200 as p
from paper_2305_07030_b200 import network, dofmap, packed, microsolver
sys.modules["fibrelax"] = p
for name, mod in (("network", network), ("dofmap", dofmap), ("packed", packed), ("microsolver", microsolver)):
    sys.modules["fibrelax." + name] = mod
import pytest
sys.exit(pytest.main([{tests!r}, "-q", "-p", "no:cacheprovider", "-x"]))
"""


@need_ref_tests
def test_reference_suite_passes_against_this_package():
    """The reference's own 52 tests, unmodified, with `fibrelax` = this package."""
    proc = subprocess.run([sys.executable, "-c", ALIAS.format(root=ROOT, tests=REF_TESTS)],
                          capture_output=True, text=True, cwd="/tmp", timeout=600)
    tail = proc.stdout.strip().splitlines()[-1] if proc.stdout.strip() else proc.stderr[-2000:]
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-2000:]
    assert "passed" in tail and "failed" not in tail, tail


def _reference_module():
    for path in (REF_SRC, BASELINE_REF):
        if os.path.isdir(os.path.join(path, "fibrelax")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import fibrelax
            return fibrelax
    pytest.skip("the reference package is not present")


def test_shim_exceptions_are_the_callers_classes():
    fr = _reference_module()
    from paper_2305_07030_b200.fibrelax_shim import error_classes
    Singular, Mass = error_classes(fr)
    e = Singular("element 3: current length collapsed", element=3)
    assert isinstance(e, fr.SingularElementError) and isinstance(e, fr.SolverError)
    assert isinstance(e, frb.SingularElementError) and isinstance(e, RuntimeError) and e.element == 3
    assert isinstance(Mass("node 1 has zero mass"), fr.microsolver.NetworkMassError)
    assert isinstance(Mass("x"), ValueError)


def test_shim_install_and_uninstall_restore_the_reference():
    fr = _reference_module()
    from paper_2305_07030_b200 import fibrelax_shim
    orig = fr.dynamic_relaxation_solve
    fibrelax_shim.install(fr, only_if_env="FIBRELAX_DEVICE_TEST_UNSET")
    try:
        assert fr.dynamic_relaxation_solve is not orig
        assert fr.microsolver.dynamic_relaxation_solve is fr.dynamic_relaxation_solve
        # env var not "b200": the reference's own CPU path runs (tiny bar)
        net = fr.FiberNetwork(np.array([[0.0, 0, 0], [0.5, 0, 0], [1.0, 0, 0]]), np.array([[0, 1, 0], [1, 2, 0]]),
                              [fr.Material(1, 1, 1)], frozenset({0, 2}))
        r = fr.dynamic_relaxation_solve(net, fr.AffineBC(np.diag([1.1, 1, 1])))
        assert abs(r.u[3] - 0.05) < 1e-6
    finally:
        fibrelax_shim.uninstall(fr)
    assert fr.dynamic_relaxation_solve is orig


@pytest.mark.gpu
def test_shim_dispatch_on_the_gpu(cuda_device):
    """Through the installed shim the reference's public call returns the
    reference's own SolveResult type with the bit-exact B200 result, and a
    collapsed element raises the caller's SingularElementError."""
    fr = _reference_module()
    from paper_2305_07030_b200 import fibrelax_shim
    fibrelax_shim.install(fr)
    try:
        case = gc.load("c1_7x7x8_uniax")
        net = fr.generate_lattice(7, 7, 8, 0.3, 0)
        r = fr.dynamic_relaxation_solve(net, fr.AffineBC(case.F))
        assert type(r) is fr.SolveResult
        assert r.iters == int(case.data["iters"]) and np.array_equal(r.u, case.data["u"])
        bad = gc.load("bar_singular")
        fnet = fr.FiberNetwork(bad.network.node_coords, bad.network.elements, [fr.Material(1, 1, 1)],
                               bad.network.boundary_nodes)
        with pytest.raises(fr.SingularElementError, match="element 0: current length collapsed"):
            fr.dynamic_relaxation_solve(fnet, fr.AffineBC(bad.F))
    finally:
        fibrelax_shim.uninstall(fr)


@pytest.mark.parametrize("name", ["random90_fixed", "lat6_general_F", "bar3_adaptive"])
def test_network_text_round_trip(tmp_path, name):
    net = gc.load(name).network
    text = frb.save_network(net)
    back = frb.load_network(text)
    assert back == net
    assert np.array_equal(back.node_coords, net.node_coords) and np.array_equal(back.elements, net.elements)
    path = tmp_path / "net.txt"      # and through a file stream
    path.write_text(text)
    with open(path) as fh:
        assert frb.load_network(fh) == net


def test_load_network_reports_the_bad_line():
    with pytest.raises(frb.NetworkFormatError) as exc:
        frb.load_network("nodes 2\n0 0 0\n1 0 x\n")
    assert exc.value.line == 3


def test_solve_result_json_schema_round_trip():
    r = frb.SolveResult(converged=True, iters=12, final_residual=1.5e-9, u=np.arange(6.0),
                        avg_stress=np.eye(3) * 0.25, energy_residual=None, r_ref=0.1)
    doc = json.loads(r.to_json())
    assert set(doc) >= {"converged", "iters", "final_residual", "u", "avg_stress", "energy_residual"}
    back = frb.SolveResult.from_json(r.to_json())
    assert back.converged and back.iters == 12 and back.final_residual == 1.5e-9
    assert np.array_equal(back.u, r.u) and np.array_equal(back.avg_stress, r.avg_stress)
    assert back.energy_residual is None
