"""The C-ABI library loads without a GPU and exports every symbol that
include/frb200.h declares; the ctypes struct mirrors match the header."""

import ctypes as C
import os
import re

from paper_2305_07030_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "frb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(frb_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = nat.lib()
    names = declared_functions()
    assert set(names) == set(nat.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name
    assert lib.frb_abi_version() == nat.ABI_VERSION


def test_struct_layouts():
    assert C.sizeof(nat.FrbConfig) == 48
    assert C.sizeof(nat.FrbBatch) == 8 + 27 * 8
    assert nat.PROBLEM_DTYPE.itemsize == 184
    assert nat.PART_DTYPE.itemsize == 120
    assert nat.GROUP_DTYPE.itemsize == 64
    assert nat.RESULT_DTYPE.itemsize == 144


def test_dofs_per_thread_cap_matches_host():
    from paper_2305_07030_b200.batch import dofs_per_thread_cap
    for t in (64, 256, 512, 544, 768, 800, 1024):
        for fg in (0, 1):
            assert nat.lib().frb_max_dofs_per_thread(t, fg) == dofs_per_thread_cap(t, bool(fg))


def test_invalid_arguments_fail_loudly():
    lib = nat.lib()
    rc = lib.frb_solve_batch(None, None, None)
    assert rc == nat.FRB_E_INVALID
    assert b"null" in lib.frb_last_error()
