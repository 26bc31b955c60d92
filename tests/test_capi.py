"""The C-ABI library loads and exports every symbol include/srj.h declares.

No compute calls here (no GPU in the build container); srj_layout is pure host
arithmetic and is checked for the alignment contract of the padded layout.
"""

import ctypes
import os
import re

import pytest

from paper_1511_04292_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "srj.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(srj_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    names = declared_symbols()
    for must in ("srj_wj_dense", "srj_plan_create", "srj_plan_run",
                 "srj_plan_residual", "srj_layout", "srj_last_error"):
        assert must in names
    assert set(names) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.srj_abi_version() == _lib.ABI_VERSION
    assert lib.srj_max_fuse() >= 4


@pytest.mark.parametrize("shape", [(256, 256), (4096, 4096), (7, 100), (5, 6, 7), (512, 512, 512)])
def test_layout_alignment(shape):
    lib = _lib.load()
    nd = len(shape)
    n = (ctypes.c_int64 * 3)(*(list(shape) + [0] * (3 - nd)))
    lay = _lib.SrjLayout()
    assert lib.srj_layout(nd, n, 1, ctypes.byref(lay)) == 0
    assert lay.pitch % 16 == 0 and lay.plane % 16 == 0
    assert lay.pitch >= shape[-1] + 2 + 15
    # first interior element of every row is 128-byte aligned
    interior = lay.origin + lay.halo0 * lay.plane + (lay.pitch if nd == 3 else 0) + 1
    assert interior % 16 == 0
    assert lay.elems >= lay.rows0 * lay.plane + 64


def test_layout_rejects_bad_arguments():
    lib = _lib.load()
    lay = _lib.SrjLayout()
    n = (ctypes.c_int64 * 3)(8, 0, 0)
    assert lib.srj_layout(1, n, 1, ctypes.byref(lay)) == _lib.SRJ_EUNSUPPORTED
    n = (ctypes.c_int64 * 3)(8, 8, 0)
    assert lib.srj_layout(2, n, 0, ctypes.byref(lay)) == _lib.SRJ_EINVAL
    assert b"halo0" in lib.srj_last_error()
