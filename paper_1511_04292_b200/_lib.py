"""ctypes binding of libsrj.so (the C ABI declared in include/srj.h).

The product path has no CPU fallback: if the shared library is missing or was
built for another ABI, every entry point raises ``RuntimeError`` naming the
build command.  ``load()`` is the single gate.
"""

import ctypes
import os

__all__ = ["BC_KINDS", "LIB_PATH", "SrjFaceRule", "SrjLayout", "SrjPlanDesc", "SrjSlabPeer",
           "check", "load"]

# SRJ_LIB_PATH: load another build (A/B timing of kernel variants; development only)
LIB_PATH = os.environ.get("SRJ_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libsrj.so")

SRJ_OK = 0
SRJ_EINVAL = -1
SRJ_ECUDA = -2
SRJ_ENOMEM = -3
SRJ_EUNSUPPORTED = -4
ABI_VERSION = 7
SLAB_FLAG_WORDS = 8

BC_KINDS = {"fixed": 0, "mirror": 1, "periodic": 2, "face_dirichlet": 3}

_c_dp = ctypes.POINTER(ctypes.c_double)


class SrjLayout(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("halo0", ctypes.c_int32),
        ("n", ctypes.c_int64 * 3),
        ("pitch", ctypes.c_int64),
        ("plane", ctypes.c_int64),
        ("rows0", ctypes.c_int64),
        ("origin", ctypes.c_int64),
        ("elems", ctypes.c_int64),
    ]


class SrjFaceRule(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("value", ctypes.c_double),
        ("values", ctypes.c_void_p),
    ]


class SrjPlanDesc(ctypes.Structure):
    _fields_ = [
        ("layout", SrjLayout),
        ("coef_mode", ctypes.c_int32),
        ("coef", ctypes.c_double * 7),
        ("coef_arrays", ctypes.c_void_p * 7),
        ("act", ctypes.c_void_p),
        ("source", ctypes.c_void_p),
        ("kappa", ctypes.c_void_p),
        ("own0_begin", ctypes.c_int64),
        ("own0_end", ctypes.c_int64),
        ("physical_lo0", ctypes.c_int32),
        ("physical_hi0", ctypes.c_int32),
        ("bc", (SrjFaceRule * 2) * 3),
    ]


class SrjSlabPeer(ctypes.Structure):
    _fields_ = [
        ("bufs", ctypes.c_void_p * 3),
        ("flags", ctypes.c_void_p),
        ("dst_row", ctypes.c_int64),
    ]


_LIB = None

_SIGNATURES = {
    "srj_abi_version": (ctypes.c_int, []),
    "srj_last_error": (ctypes.c_char_p, []),
    "srj_max_fuse": (ctypes.c_int, []),
    "srj_layout": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.c_int32, ctypes.POINTER(SrjLayout)]),
    "srj_wj_dense": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p,
                                    ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
    "srj_plan_create": (ctypes.c_int, [ctypes.POINTER(SrjPlanDesc),
                                       ctypes.POINTER(ctypes.c_void_p)]),
    "srj_plan_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "srj_plan_set_post_gather": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_int64]),
    "srj_plan_set_coef_classes": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "srj_plan_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, _c_dp, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                    ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p]),
    "srj_plan_residual": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]),
    "srj_plan_residual_layers": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p]),
    "srj_slab_create": (ctypes.c_int, [ctypes.POINTER(SrjPlanDesc), ctypes.c_int32,
                                       ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p,
                                       ctypes.c_int32, ctypes.c_int32,
                                       ctypes.POINTER(ctypes.c_void_p)]),
    "srj_slab_connect": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32,
                                        ctypes.POINTER(SrjSlabPeer)]),
    "srj_slab_reset": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "srj_slab_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "srj_slab_plan": (ctypes.c_void_p, [ctypes.c_void_p]),
    "srj_slab_direct": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "srj_slab_depth": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "srj_slab_run": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                    ctypes.c_int32, _c_dp, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(ctypes.c_void_p)]),
    "srj_ipc_get_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.POINTER(ctypes.c_int64)]),
    "srj_ipc_open": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.POINTER(ctypes.c_void_p)]),
    "srj_ipc_close": (ctypes.c_int, [ctypes.c_void_p]),
    "srj_plan_gs": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                   ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "srj_upload_field": (ctypes.c_int, [ctypes.POINTER(SrjLayout), ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "srj_download_field": (ctypes.c_int, [ctypes.POINTER(SrjLayout), ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "srj_upload_interior": (ctypes.c_int, [ctypes.POINTER(SrjLayout), ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "srj_selftest_div": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "srj_copy_layers": (ctypes.c_int, [ctypes.POINTER(SrjLayout), ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_void_p]),
}

EXPORTS = tuple(_SIGNATURES)


def load():
    """Load libsrj.so; raise RuntimeError when it is missing (no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libsrj.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(the SRJ GPU path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.srj_abi_version() != ABI_VERSION:
        raise RuntimeError("libsrj.so ABI version mismatch; rebuild it")
    _LIB = lib
    return lib


def check(status, what="srj"):
    """Map a C status to the Python exception the reference would raise."""
    if status == SRJ_OK:
        return
    msg = (_LIB.srj_last_error() or b"").decode(errors="replace") if _LIB else ""
    text = f"{what}: {msg}" if msg else f"{what} failed ({status})"
    if status == SRJ_EINVAL:
        raise ValueError(text)
    if status == SRJ_EUNSUPPORTED:
        raise NotImplementedError(text)
    if status == SRJ_ENOMEM:
        raise MemoryError(text)
    raise RuntimeError(text)
