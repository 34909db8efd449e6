"""Load the committed reference fixtures (tests/golden/*.npz) into inputs.

Networks are rebuilt with the product's input classes (host-side data only),
so the GPU box never needs /root/reference.
"""

from __future__ import annotations

import glob
import json
import math
import os
from dataclasses import dataclass

import numpy as np

from paper_2305_07030_b200 import network as nw
from paper_2305_07030_b200.microsolver import AdaptiveDamping, FixedDamping, SolverConfig

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Case:
    name: str
    network: nw.FiberNetwork
    F: np.ndarray
    cfg: SolverConfig
    data: dict

    @property
    def singular(self) -> bool:
        return bool(self.data["singular"])


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load(name: str) -> Case:
    z = dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))
    mats = [nw.Material(*map(float, row)) for row in z["materials"]]
    vol = float(z["rve_volume"])
    net = nw.FiberNetwork(z["coords"], z["elements"], mats, frozenset(int(b) for b in z["boundary"]),
                          rve_volume=None if math.isnan(vol) else vol)
    c = json.loads(str(z["cfg"]))
    damping = AdaptiveDamping() if c["damping_c"] is None else FixedDamping(c["damping_c"])
    cfg = SolverConfig(tol_rel=c["tol_rel"], tol_abs=c["tol_abs"], max_iters=c["max_iters"],
                       dt_safety=c["dt_safety"], damping=damping,
                       energy_check_interval=c["energy_check_interval"],
                       bc_ramp_iters=c["bc_ramp_iters"])
    return Case(name, net, z["F"], cfg, z)
