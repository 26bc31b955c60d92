"""Device-resident grid state and launch plan (torch owns memory, libsrj computes).

``DeviceGrid`` is the device half of the reference's ``_Sweeper``
(``grids.py:535-559``): it holds the field in HBM in the padded layout of
``include/srj.h`` -- three field buffers instead of the reference's two, so the
iterate at the start of a chunk survives as a snapshot and a solve can stop at
the exact step the stopping rule fires (see ``grids.srj_solve``) -- plus the
source / nonlinear factor, the stencil (scalars when constant, per-cell arrays
otherwise) and the mask.

torch is used only as the device allocator and stream provider.  There is no
CPU path: constructing a DeviceGrid without a CUDA device raises.
"""

import ctypes
import os
import warnings

import numpy as np

from . import _lib

__all__ = ["DeviceGrid", "coef_class", "constant_value", "require_cuda"]


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the SRJ GPU path needs a CUDA device (no CPU fallback)")
    return torch


def constant_value(a):
    """The scalar if every element of ``a`` has the same fp64 bit pattern."""
    a = np.asarray(a, dtype=np.float64)
    if a.size == 0:
        return None
    first = a.reshape(-1)[:1]
    if all(s == 0 for s in a.strides):
        return float(first[0])
    bits = a.view(np.int64) if a.flags.c_contiguous else np.ascontiguousarray(a).view(np.int64)
    if bool(np.all(bits == first.view(np.int64)[0])):
        return float(first[0])
    return None


def coef_class(a):
    """``SRJ_COEF_*`` class bits of an interior-shaped coefficient array
    (``srj_plan_set_coef_classes``, include/srj.h): 1 if every axis-0 slice
    equals the first, 2 if every value equals the first of its last-axis row,
    both bit for bit (so reading the representative changes no result).  The
    reference's problem builders broadcast such profiles over the grid
    (spherical_poisson, grad_shafranov: problems.py:489-560, :684-689)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim < 2 or a.size == 0:
        return 0
    bits = a.view(np.int64)
    cls = 0
    # a cheap test on two slices rejects most varying arrays before the full one
    if a.shape[0] >= 2 and np.array_equal(bits[1], bits[0]) and bool(np.all(bits == bits[:1])):
        cls |= 1
    if (a.shape[-1] >= 2 and np.array_equal(bits[..., 1], bits[..., 0])
            and bool(np.all(bits == bits[..., :1]))):
        cls |= 2
    return cls


def stencil_is_constant(center, lower, upper, active=None):
    """True when ``DeviceGrid`` would take the constant-stencil kernels: every
    coefficient array bitwise constant and no masked cell."""
    if active is not None and not bool(np.all(active)):
        return False
    return all(constant_value(c) is not None for c in [center, *lower, *upper])


def _contig(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


class DeviceGrid:
    """Field, coefficients and launch plan of one grid on one GPU.

    Parameters
    ----------
    u : ndarray
        Ghosted field (interior shape + 2 per axis), FIXED ghosts included.
    source, center, lower, upper, active :
        As the reference GridProblem (``grids.py:155-165``); ``active`` is the
        interior bool mask or None.
    kappa : ndarray, optional
        Nonlinear factor: the source becomes kappa * u^5 of the current
        iterate (``source`` is then ignored).
    halo0, own, physical : slab-decomposition knobs (``distributed.py``).
    """

    def __init__(self, u, source, center, lower, upper, active=None, kappa=None,
                 halo0=1, own=None, physical=(True, True), device=None, bc=None,
                 post_gather=None, pooled=False, allow_constant=True):
        torch = require_cuda()
        lib = _lib.load()
        self.torch = torch
        self.lib = lib
        nd = np.ndim(center)
        if nd not in (2, 3):
            raise NotImplementedError(
                "the GPU path supports 2- and 3-dimensional grids")
        self.shape = tuple(int(s) for s in np.shape(center))
        self.ndim = nd
        self.device = torch.device("cuda", torch.cuda.current_device()
                                   if device is None else device)
        n = (ctypes.c_int64 * 3)(*(list(self.shape) + [0] * (3 - nd)))
        self.layout = _lib.SrjLayout()
        _lib.check(lib.srj_layout(nd, n, int(halo0), ctypes.byref(self.layout)),
                   "srj_layout")
        elems = int(self.layout.elems)
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.current_stream(self.device)
            self._keep = []
            if pooled:
                # one allocation for the three fields + the slab exchange's
                # flag words, so a single CUDA IPC handle maps all of them
                # into the neighbour ranks (distributed.DeviceSlab)
                self.pool = torch.zeros(3 * elems + 16, dtype=torch.float64, device=self.device)
                self.fields = [self.pool[i * elems:(i + 1) * elems] for i in range(3)]
                self.flags = self.pool[3 * elems:3 * elems + 16].view(torch.int32)
            else:
                self.pool = None
                self.fields = [torch.zeros(elems, dtype=torch.float64, device=self.device)
                               for _ in range(3)]
            # one host->device copy; the other two buffers (whose ghost layers
            # the kernels never write) are device copies of it
            self.upload_field(_contig(u, np.float64), self.fields[0])
            with torch.cuda.stream(self.stream):
                for f in self.fields[1:]:
                    f.copy_(self.fields[0])

            desc = _lib.SrjPlanDesc()
            desc.layout = self.layout
            coefs = [center] + [x for ax in range(nd) for x in (lower[ax], upper[ax])]
            consts = [constant_value(c) for c in coefs]
            masked = active is not None and not bool(np.all(active))
            # allow_constant=False: the ranks of a slab decomposition agreed on
            # the per-cell kernels (another rank's rows are not constant)
            self.constant = (all(c is not None for c in consts) and not masked
                             and bool(allow_constant))
            if self.constant:
                desc.coef_mode = 0
                for i, c in enumerate(consts):
                    desc.coef[i] = c
            else:
                desc.coef_mode = 1
                for i, c in enumerate(coefs):
                    t = self._interior_array(c)
                    desc.coef_arrays[i] = t.data_ptr()
            if masked:
                m = torch.zeros(elems, dtype=torch.uint8, device=self.device)
                self._upload_interior(_contig(active, np.uint8), m, 1)
                self._keep.append(m)
                desc.act = m.data_ptr()
            # the source (or kappa) in the padded layout; kept for re-uploads
            self.f_dev = self._interior_array(kappa if kappa is not None else source)
            if kappa is not None:
                desc.kappa = self.f_dev.data_ptr()
            else:
                desc.source = self.f_dev.data_ptr()
            lo, hi = (0, self.shape[0]) if own is None else own
            desc.own0_begin = int(lo)
            desc.own0_end = int(hi)
            desc.physical_lo0 = int(bool(physical[0]))
            desc.physical_hi0 = int(bool(physical[1]))
            for ax, pair in enumerate(bc or ()):
                for side, rule in enumerate(pair):
                    self._set_face(desc.bc[ax][side], rule, ax)
            self.desc = desc
            plan = ctypes.c_void_p()
            _lib.check(lib.srj_plan_create(ctypes.byref(desc), ctypes.byref(plan)),
                       "srj_plan_create")
            self.plan = plan
            self.coef_classes = [0] * 7
            # coefficient classes: read by the 3D per-cell kernel (include/srj.h)
            if (not self.constant and nd == 3
                    and os.environ.get("SRJ_COEF_CLASSES", "1") != "0"):
                cls = [coef_class(c) for c in coefs] + [0] * (7 - len(coefs))
                if any(cls):
                    arr = (ctypes.c_int32 * 7)(*cls)
                    _lib.check(lib.srj_plan_set_coef_classes(plan, arr),
                               "srj_plan_set_coef_classes")
                    self.coef_classes = cls
            if post_gather is not None and len(post_gather[0]):
                self._set_post_gather(*post_gather)
            self.norms = torch.zeros(2, dtype=torch.float64, device=self.device)
            self.resid_out = torch.zeros(2, dtype=torch.float64, device=self.device)

    def _set_post_gather(self, dst, src):
        """Install a post-sweep gather given as flat indices of the ghosted
        field (C order, shape n+2 per axis); converted to padded offsets."""
        lay = self.layout
        gshape = tuple(n + 2 for n in self.shape)

        def offsets(flat):
            idx = np.unravel_index(np.asarray(flat, dtype=np.int64), gshape)
            off = int(lay.origin) + (int(lay.halo0) - 1 + idx[0]) * int(lay.plane)
            if self.ndim == 3:
                off = off + idx[1] * int(lay.pitch)
            return np.ascontiguousarray(off + idx[-1], dtype=np.int64)

        d, s = offsets(dst), offsets(src)
        _lib.check(self.lib.srj_plan_set_post_gather(
            self.plan, d.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
            len(d)), "srj_plan_set_post_gather")

    def _set_face(self, face, rule, ax):
        """Fill one srj_face_rule from a reference BoundaryRule (grids.py:73-112)."""
        face.kind = _lib.BC_KINDS[rule.kind]
        if rule.kind != "face_dirichlet":
            return
        vals = np.asarray(rule.values, dtype=np.float64)
        face_shape = self.shape[:ax] + self.shape[ax + 1:]
        if vals.ndim == 0:
            face.value = float(vals)
            return
        dense = np.ascontiguousarray(np.broadcast_to(vals, face_shape))
        t = self.torch.from_numpy(dense.copy()).to(self.device)
        self._keep.append(t)
        face.values = t.data_ptr()

    # ------------------------------------------------------------- transfers
    @property
    def _sp(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def _interior_array(self, a):
        t = self.torch.zeros(int(self.layout.elems), dtype=self.torch.float64,
                             device=self.device)
        self._upload_interior(_contig(a, np.float64), t, 8)
        self._keep.append(t)
        return t

    # Host <-> device copies of the padded layout (srj_layout, include/srj.h):
    # one contiguous transfer of the dense host array, then a device-side
    # scatter / gather through a strided view of the padded buffer.  The C
    # ABI's srj_upload_field / srj_upload_interior / srj_download_field do the
    # same with row-wise 2D copies (one per plane for 3D interiors), which the
    # copy engines run at well under the PCIe rate for 2-4 KB rows.
    def _field_view(self, t):
        l = self.layout
        last = int(l.n[l.ndim - 1]) + 2
        rows = (int(l.n[0]) + 2) * ((int(l.n[1]) + 2) if l.ndim == 3 else 1)
        off = int(l.origin) + (int(l.halo0) - 1) * int(l.plane)
        return t.as_strided((rows, last), (int(l.pitch), 1), t.storage_offset() + off)

    def _interior_view(self, t):
        l = self.layout
        if l.ndim == 2:
            off = int(l.origin) + int(l.halo0) * int(l.plane) + 1
            return t.as_strided((int(l.n[0]), int(l.n[1])), (int(l.pitch), 1),
                                t.storage_offset() + off)
        off = int(l.origin) + int(l.halo0) * int(l.plane) + int(l.pitch) + 1
        return t.as_strided((int(l.n[0]), int(l.n[1]), int(l.n[2])),
                            (int(l.plane), int(l.pitch), 1), t.storage_offset() + off)

    def _scatter(self, host, view):
        torch = self.torch
        with warnings.catch_warnings():  # read-only host arrays are only read
            warnings.simplefilter("ignore", UserWarning)
            src = torch.from_numpy(host).reshape(view.shape)
        with torch.cuda.stream(self.stream):
            staging = torch.empty(view.shape, dtype=view.dtype, device=self.device)
            staging.copy_(src, non_blocking=True)
            view.copy_(staging)
        self.stream.synchronize()  # host array may be a temporary

    def _upload_interior(self, host, dev, esize):
        self._scatter(host, self._interior_view(dev))

    def upload_field(self, host, dev):
        with self._on():
            self._upload_field(host, dev)

    def upload_source(self, host):
        """Re-upload the source (or kappa) from an interior-shaped host array."""
        with self._on():
            self._upload_interior(_contig(host, np.float64), self.f_dev, 8)

    def _upload_field(self, host, dev):
        self._scatter(host, self._field_view(dev))

    def download_field(self, idx, host):
        """Copy field buffer ``idx`` into the ghosted host array (in place)."""
        if not (host.flags.c_contiguous and host.dtype == np.float64):
            tmp = np.empty(host.shape, dtype=np.float64)
            self.download_field(idx, tmp)
            host[...] = tmp
            return
        torch = self.torch
        with self._on(), torch.cuda.stream(self.stream):
            dense = self._field_view(self.fields[idx]).contiguous()  # device gather
            torch.from_numpy(host).view(dense.shape).copy_(dense, non_blocking=True)
        self.stream.synchronize()

    # -------------------------------------------------------------- compute
    def ensure_norms(self, nsteps):
        if self.norms.numel() < 2 * nsteps:
            self.norms = self.torch.zeros(2 * nsteps, dtype=self.torch.float64,
                                          device=self.device)

    def _on(self):
        """The library launches on the current CUDA device: make it ours."""
        return self.torch.cuda.device(self.device)

    def run(self, src, weights, first, nsteps, fuse=0):
        """Run steps [first, first+nsteps) from buffer ``src``; returns the
        buffer index holding the result.  Norms land in ``self.norms``."""
        self.ensure_norms(max(nsteps, 1))
        a, b = [i for i in range(3) if i != src]
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = ctypes.c_int32(0)
        f = self.fields
        with self._on():
            _lib.check(self.lib.srj_plan_run(
                self.plan, ctypes.c_void_p(f[src].data_ptr()),
                ctypes.c_void_p(f[a].data_ptr()), ctypes.c_void_p(f[b].data_ptr()),
                w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(w), int(first),
                int(nsteps), int(fuse), ctypes.c_void_p(self.norms.data_ptr()),
                ctypes.byref(out), self._sp), "srj_plan_run")
        return (src, a, b)[out.value]

    def sub_plan(self, own_lo, own_hi):
        """A plan over the same fields that relaxes, stores and counts only
        local rows [own_lo, own_hi) (cached; the slab solver's edge / inner
        launches).  Rows outside the range are read, never written."""
        key = (int(own_lo), int(own_hi))
        plans = self.__dict__.setdefault("_sub_plans", {})
        if key not in plans:
            desc = _lib.SrjPlanDesc()
            ctypes.memmove(ctypes.byref(desc), ctypes.byref(self.desc), ctypes.sizeof(desc))
            desc.own0_begin, desc.own0_end = key
            plan = ctypes.c_void_p()
            with self._on():
                _lib.check(self.lib.srj_plan_create(ctypes.byref(desc), ctypes.byref(plan)),
                           "srj_plan_create")
            plans[key] = plan
        return plans[key]

    def run_single(self, plan, src, dst, weights, first, nsteps, norms):
        """One fused launch of ``plan``: buffer ``src`` -> buffer ``dst``
        (nsteps <= the plan's fused depth), per-step norms into the device
        tensor ``norms`` (2 * nsteps doubles)."""
        spare = [i for i in range(3) if i not in (src, dst)][0]
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = ctypes.c_int32(0)
        f = self.fields
        with self._on():
            _lib.check(self.lib.srj_plan_run(
                plan, ctypes.c_void_p(f[src].data_ptr()), ctypes.c_void_p(f[dst].data_ptr()),
                ctypes.c_void_p(f[spare].data_ptr()),
                w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(w), int(first),
                int(nsteps), int(nsteps), ctypes.c_void_p(norms.data_ptr()), ctypes.byref(out),
                self._sp), "srj_plan_run")
        if out.value != 1:
            raise RuntimeError("expected a single fused launch (fuse >= nsteps)")

    def gs(self, idx, omega, nsweeps):
        """``nsweeps`` in-place Gauss-Seidel / SOR sweeps of field buffer
        ``idx`` (srj_plan_gs); per-sweep (dmax, rmax) land in ``self.norms``."""
        self.ensure_norms(max(nsweeps, 1))
        with self._on():
            _lib.check(self.lib.srj_plan_gs(
                self.plan, ctypes.c_void_p(self.fields[idx].data_ptr()), float(omega),
                int(nsweeps), ctypes.c_void_p(self.norms.data_ptr()), self._sp), "srj_plan_gs")

    def copy_field(self, src, dst):
        """Device copy of field buffer ``src`` into ``dst`` (stream-ordered)."""
        with self._on(), self.torch.cuda.stream(self.stream):
            self.fields[dst].copy_(self.fields[src])

    def residual(self, idx):
        """(sum r^2, max|r|) of field buffer ``idx`` (synchronous)."""
        with self._on():
            _lib.check(self.lib.srj_plan_residual(
                self.plan, ctypes.c_void_p(self.fields[idx].data_ptr()),
                ctypes.c_void_p(self.resid_out.data_ptr()), self._sp), "srj_plan_residual")
        v = self.resid_out.cpu().numpy()
        return float(v[0]), float(v[1])

    def residual_layers(self, idx):
        """Per owned axis-0 layer (sum r^2, max|r|) of field buffer ``idx``
        as a host array [layers, 2] (srj_plan_residual_layers; synchronous)."""
        lo, hi = int(self.desc.own0_begin), int(self.desc.own0_end)
        n = max(hi - lo, 0)
        if getattr(self, "_layers", None) is None or self._layers.numel() < 2 * max(n, 1):
            self._layers = self.torch.zeros(2 * max(n, 1), dtype=self.torch.float64,
                                            device=self.device)
        with self._on():
            _lib.check(self.lib.srj_plan_residual_layers(
                self.plan, ctypes.c_void_p(self.fields[idx].data_ptr()),
                ctypes.c_void_p(self._layers.data_ptr()), self._sp), "srj_plan_residual_layers")
        return self._layers[:2 * n].view(n, 2).cpu().numpy()

    def close(self):
        subs = self.__dict__.pop("_sub_plans", {})
        if subs or getattr(self, "plan", None) is not None:
            with self._on():
                for plan in subs.values():
                    self.lib.srj_plan_destroy(plan)
                if getattr(self, "plan", None) is not None:
                    self.lib.srj_plan_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
