"""ctypes binding of the C-ABI in ``include/frb200.h`` (``lib/libfrb200.so``).

The struct layouts below mirror the header field for field; ``tests/test_abi.py``
checks sizes and that every declared symbol is exported.  Loading fails
loudly: there is no CPU fallback for the solver.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FRB_LIB") or os.path.join(HERE, "lib", "libfrb200.so")

ABI_VERSION = 10
MAX_CLUSTER = 16
FRB_OK, FRB_E_INVALID, FRB_E_TOO_LARGE, FRB_E_CUDA, FRB_E_UNSUPPORTED = 0, -1, -2, -3, -4
STATUS_CONVERGED, STATUS_MAX_ITERS, STATUS_SINGULAR = 0, 1, 2
DAMPING_ADAPTIVE, DAMPING_FIXED = 0, 1
PF_EA_UNIFORM = 1
PF_MASS_GLOBAL = 2
PHASES = 12             # phase_cycles slots per CTA (frb200.h)
PHASE_NAMES = ("F1 coefs", "F2 gather", "A per-DOF", "C chains", "T local+exp", "T exch wait",
               "T top+scal", "U update", "epilogue", "prologue", "halo wait", "T local tree")

EXPORTS = ("frb_abi_version", "frb_last_error", "frb_solve_launches", "frb_device_info", "frb_rank_smem_bytes",
           "frb_max_dofs_per_thread", "frb_solve_batch", "frb_internal_forces",
           "frb_selftest_arith", "frb_setup_problem", "frb_setup_batch",
           "frb_naive_solve", "frb_naive_scratch_doubles")


class FrbConfig(C.Structure):
    _fields_ = [("tol_rel", C.c_double), ("tol_abs", C.c_double), ("dt_safety", C.c_double),
                ("damping_c", C.c_double), ("max_iters", C.c_int32), ("damping", C.c_int32),
                ("energy_check_interval", C.c_int32), ("bc_ramp_iters", C.c_int32)]


BATCH_POINTERS = ("groups", "problems", "parts", "order", "X", "node_mass", "inc_node", "inc",
                  "elem_ab", "elem_L", "elem_EA", "plans", "ell", "act_ab", "act_L",
                  "act_EA", "halo_g", "runs", "fix_g", "trees", "u", "f", "work", "results", "queue",
                  "xchg", "phase_cycles")


class FrbBatch(C.Structure):
    _fields_ = [("n_problems", C.c_int32), ("n_groups", C.c_int32)] + \
               [(name, C.c_void_p) for name in BATCH_POINTERS]


# frb_problem / frb_part / frb_group / frb_result as numpy record types
PROBLEM_DTYPE = np.dtype([
    ("node_base", "<i8"), ("elem_base", "<i8"), ("inc_base", "<i8"), ("plan_base", "<i8"),
    ("part_base", "<i8"), ("actv_base", "<i8"), ("tnode_base", "<i8"), ("telem_base", "<i8"),
    ("n_nodes", "<i4"), ("n_free_nodes", "<i4"), ("n_elems", "<i4"), ("cluster", "<i4"),
    ("flags", "<i4"), ("pad", "<i4"),
    ("dt", "<f8"), ("volume", "<f8"), ("ea", "<f8"), ("F", "<f8", (9,)),
])
PART_DTYPE = np.dtype([
    ("ell_base", "<i8"), ("act_base", "<i8"), ("actv_off", "<i8"), ("halo_base", "<i8"),
    ("runs_base", "<i8"), ("fix_base", "<i8"), ("tree_base", "<i8"),
    ("node0", "<i4"), ("n_own", "<i4"), ("n_local", "<i4"), ("n_act", "<i4"),
    ("ell_stride", "<i4"), ("slots_a", "<i4"), ("slots_b", "<i4"), ("leaf0", "<i4"),
    ("n_leaves", "<i4"), ("n_fix", "<i4"), ("tree_len", "<i4"), ("n_runs", "<i4"),
    ("halo_bytes", "<i4"), ("ack_from", "<u4"), ("n_int", "<i4"), ("pad", "<i4"),
])
GROUP_DTYPE = np.dtype([
    ("cluster", "<i4"), ("first", "<i4"), ("count", "<i4"), ("block_threads", "<i4"),
    ("smem_bytes", "<i4"), ("max_own_dofs", "<i4"), ("grid_clusters", "<i4"), ("fprv_global", "<i4"),
    ("max_rank_leaves", "<i4"), ("flags", "<i4"), ("xchg_off", "<i8"), ("gm_cap", "<i4"),
    ("gm_ex_stride", "<i4"), ("gm_mir_stride", "<i4"), ("pad", "<i4"),
])
GF_SERIAL = 1
GF_NO_VIRTUAL = 2
GF_VIRTUAL_ONLY = 4
SETUP_ITEM_DTYPE = np.dtype([
    ("coords", "<u8"), ("elements", "<u8"), ("materials", "<u8"), ("node_order", "<u8"), ("act_elem", "<u8"),
    ("X_out", "<u8"), ("mass_out", "<u8"), ("L_out", "<u8"), ("EA_out", "<u8"), ("act_L_out", "<u8"),
    ("act_EA_out", "<u8"), ("mass_scratch", "<u8"), ("n_act", "<i8"), ("n_nodes", "<i4"), ("n_elems", "<i4"),
    ("n_materials", "<i4"), ("rc", "<i4"), ("scalars", "<f8", (3,)),
])
RESULT_DTYPE = np.dtype([
    ("status", "<i4"), ("iters", "<i4"), ("bad_element", "<i4"), ("converged", "<i4"),
    ("final_residual", "<f8"), ("r_ref", "<f8"), ("energy_residual", "<f8"),
    ("avg_stress", "<f8", (9,)), ("energy", "<f8", (4,)),
])
assert PROBLEM_DTYPE.itemsize == 184 and PART_DTYPE.itemsize == 120
assert SETUP_ITEM_DTYPE.itemsize == 144 and GROUP_DTYPE.itemsize == 64 and RESULT_DTYPE.itemsize == 144


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"libfrb200 error {code}: {message}")
        self.code = code


_lib = None


def lib() -> C.CDLL:
    """Load libfrb200.so once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import "
                          "__graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    h = C.CDLL(LIB_PATH)
    h.frb_abi_version.restype = C.c_int
    h.frb_last_error.restype = C.c_char_p
    h.frb_solve_launches.restype = C.c_int
    h.frb_device_info.argtypes = [C.c_int] + [C.POINTER(C.c_int)] * 4
    h.frb_rank_smem_bytes.restype = C.c_int64
    h.frb_rank_smem_bytes.argtypes = [C.c_int32] * 6
    h.frb_max_dofs_per_thread.argtypes = [C.c_int, C.c_int]
    h.frb_solve_batch.argtypes = [C.POINTER(FrbBatch), C.POINTER(FrbConfig), C.c_void_p]
    h.frb_internal_forces.argtypes = [C.POINTER(FrbBatch), C.c_void_p, C.c_void_p, C.c_void_p]
    h.frb_selftest_arith.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    h.frb_setup_problem.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                    C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 8
    h.frb_setup_batch.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
    h.frb_naive_solve.argtypes = [C.POINTER(FrbBatch), C.POINTER(FrbConfig), C.c_int32, C.c_void_p, C.c_int64,
                                  C.c_void_p]
    h.frb_naive_scratch_doubles.restype = C.c_int64
    h.frb_naive_scratch_doubles.argtypes = [C.c_int32] * 3
    if h.frb_abi_version() != ABI_VERSION:
        raise ImportError("libfrb200.so ABI version mismatch (rebuild)")
    _lib = h
    return h


def check(rc: int):
    if rc != FRB_OK:
        raise NativeError(rc, lib().frb_last_error().decode(errors="replace"))


def device_info(device: int = 0):
    vals = [C.c_int() for _ in range(4)]
    check(lib().frb_device_info(device, *[C.byref(v) for v in vals]))
    return dict(n_sm=vals[0].value, smem_optin=vals[1].value, cc=(vals[2].value, vals[3].value))
