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


def _desc(shape=(8, 8), **kw):
    """A plan descriptor with fake (never dereferenced) device pointers."""
    lib = _lib.load()
    nd = len(shape)
    n = (ctypes.c_int64 * 3)(*(list(shape) + [0] * (3 - nd)))
    d = _lib.SrjPlanDesc()
    assert lib.srj_layout(nd, n, 1, ctypes.byref(d.layout)) == 0
    d.coef_mode = 0
    d.coef[0] = 4.0
    for a in range(1, 1 + 2 * nd):
        d.coef[a] = -1.0
    d.source = 0x1000
    for key, val in kw.items():
        setattr(d, key, val)
    return d


def _create(d):
    lib = _lib.load()
    plan = ctypes.c_void_p()
    return lib.srj_plan_create(ctypes.byref(d), ctypes.byref(plan)), lib.srj_last_error()


def test_plan_create_validates_before_touching_the_device():
    """Descriptor errors come back as status codes with a message, before any
    CUDA call (so they are checkable without a GPU)."""
    lib = _lib.load()
    plan = ctypes.c_void_p()
    assert lib.srj_plan_create(None, ctypes.byref(plan)) == _lib.SRJ_EINVAL
    rc, msg = _create(_desc(source=0))
    assert rc == _lib.SRJ_EINVAL and b"source" in msg
    rc, msg = _create(_desc(coef_mode=2))
    assert rc == _lib.SRJ_EINVAL and b"coef_mode" in msg
    rc, msg = _create(_desc(coef_mode=1))
    assert rc == _lib.SRJ_EINVAL and b"coefficient array" in msg
    d = _desc()
    d.coef[0] = 0.0
    rc, msg = _create(d)
    assert rc == _lib.SRJ_EINVAL and b"center" in msg
    rc, msg = _create(_desc(own0_begin=3, own0_end=20))
    assert rc == _lib.SRJ_EINVAL and b"owned rows" in msg
    d = _desc()
    d.bc[0][0].kind = 7
    rc, msg = _create(d)
    assert rc == _lib.SRJ_EINVAL and b"boundary rule" in msg
    d = _desc()
    d.bc[2][0].kind = _lib.BC_KINDS["mirror"]  # axis 2 of a 2-D grid
    assert _create(d)[0] == _lib.SRJ_EINVAL
    d = _desc()
    d.bc[1][0].kind = _lib.BC_KINDS["periodic"]  # one-sided periodic
    rc, msg = _create(d)
    assert rc == _lib.SRJ_EINVAL and b"periodic" in msg
    d = _desc(physical_lo0=0, physical_hi0=1)
    d.bc[1][1].kind = _lib.BC_KINDS["mirror"]  # non-FIXED faces on a slab
    rc, msg = _create(d)
    assert rc == _lib.SRJ_EUNSUPPORTED and b"whole grid" in msg


def test_host_entry_points_reject_null_and_bad_arguments():
    lib = _lib.load()
    n = (ctypes.c_int64 * 3)(8, 8, 0)
    ptrs = (ctypes.c_void_p * 3)()
    assert lib.srj_wj_dense(4, n, None, None, None, None, ptrs, ptrs, None, 1.0, None,
                            None) == _lib.SRJ_EUNSUPPORTED
    assert lib.srj_wj_dense(2, n, None, None, None, None, ptrs, ptrs, None, 1.0, None,
                            None) == _lib.SRJ_EINVAL
    lay = _lib.SrjLayout()
    assert lib.srj_upload_field(None, None, None, None) == _lib.SRJ_EINVAL
    assert lib.srj_download_field(ctypes.byref(lay), None, None, None) == _lib.SRJ_EINVAL
    assert lib.srj_upload_interior(ctypes.byref(lay), ctypes.c_void_p(16), ctypes.c_void_p(16),
                                   4, None) == _lib.SRJ_EINVAL
    assert lib.srj_selftest_div(None, 1, 2.0, None, None, None) == _lib.SRJ_EINVAL
    assert lib.srj_plan_run(None, None, None, None, None, 1, 0, 1, 0, None,
                            None, None) == _lib.SRJ_EINVAL
    assert lib.srj_plan_residual(None, None, None, None) == _lib.SRJ_EINVAL
    assert lib.srj_plan_set_post_gather(None, None, None, 0) == _lib.SRJ_EINVAL
    assert lib.srj_plan_destroy(None) == _lib.SRJ_OK
    n = (ctypes.c_int64 * 3)(8, 1 << 31, 0)
    assert lib.srj_layout(2, n, 1, ctypes.byref(lay)) == _lib.SRJ_EINVAL
