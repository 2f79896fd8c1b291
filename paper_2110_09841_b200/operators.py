"""Projector/backprojector pair — Python mirror of the reference operator API
(include/cbct/cvp.hpp:81-106, siddon.hpp:24-55) over libcvpb200's C-ABI.

Two ways in:

* :class:`DeviceScene` — the B200-native interface: one resident scene
  (geometry, per-view constants, pixel-scale images) per device; operators
  take float32 CUDA tensors and run asynchronously on the caller's stream.
* ``project_cvp_into`` & co. — the reference's call shapes. Device tensors
  dispatch to the device path; float64 numpy buffers go through the C-ABI's
  host entry points (H2D + kernels + D2H), which is the drop-in path for an
  existing reference caller.

There is no CPU implementation anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import enum
from collections import OrderedDict
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import InvalidArgument
from .geometry import (AttenuationVolume, DetectorGeometry, ProjectionStack, VolumeGeometry,
                       ViewGeometry, views_to_array)


class PixelScaling(enum.IntEnum):
    Cos = 0
    Exact = 1


class CvpPrecision(enum.IntEnum):
    Double = 0   # exact: float64 cut geometry + float64 voxel anchors
    Single = 1   # relaxed (same float64 column geometry)


class RadiusEstimate(enum.IntEnum):
    VoxelCenter = 0
    CutCentroid = 1


@dataclass
class CvpOptions:
    """cvp.hpp:17-22 (same defaults)."""
    scaling: PixelScaling = PixelScaling.Exact
    elevation_correction: bool = True
    precision: CvpPrecision = CvpPrecision.Double
    r_estimate: RadiusEstimate = RadiusEstimate.CutCentroid

    def _c(self):
        return N.cvpb_cvp_options(int(self.scaling), int(bool(self.elevation_correction)),
                                  int(self.precision), int(self.r_estimate))


@dataclass
class ExecPolicy:
    """exec.hpp:6-15."""
    threads: int = 0
    deterministic: bool = False
    allow_expensive: bool = False

    def _c(self):
        return N.cvpb_exec_policy(int(self.threads), int(bool(self.deterministic)),
                                  int(bool(self.allow_expensive)))


@dataclass
class PixelRoi:
    """siddon.hpp:28-33."""
    row_begin: int = 0
    row_end: int = -1
    col_begin: int = 0
    col_end: int = -1

    def _c(self):
        return N.cvpb_pixel_roi(self.row_begin, self.row_end, self.col_begin, self.col_end)


@dataclass
class TTOptions:
    amplitude: int = 1

    def _c(self):
        return N.cvpb_tt_options(int(self.amplitude))


@dataclass
class CutVolumeRecord:
    row: int
    column: int
    volume: float
    inv_r2: float


def _ptr(t, numel=None, device=None, at_least=False):
    """Device pointer of a contiguous float32 CUDA tensor; with numel / device
    the tensor must also hold exactly (at_least: at least) that many elements
    on that GPU (the kernels index the full scene, so a short or foreign buffer
    is refused here instead of being read or written out of bounds)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise InvalidArgument("expected a torch tensor")
    if not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise InvalidArgument("device buffers must be contiguous float32 CUDA tensors")
    if numel is not None and (t.numel() < numel if at_least else t.numel() != numel):
        raise InvalidArgument(f"device buffer holds {t.numel()} elements, the scene needs {numel}")
    if device is not None and (t.device.index if t.device.index is not None else 0) != device:
        raise InvalidArgument(f"device buffer lives on cuda:{t.device.index}, the scene on cuda:{device}")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class DeviceScene:
    """A scene resident on one GPU (libcvpb200 context + cvpb_set_geometry)."""

    def __init__(self, vol_geom: VolumeGeometry, det: DetectorGeometry,
                 views: Sequence[ViewGeometry], device: int = 0):
        L = N.lib()
        self.vol_geom, self.det = vol_geom, det
        self.views = list(views)
        self.device = int(device)
        h = C.c_void_p()
        N.check(L.cvpb_context_create(self.device, C.byref(h)))
        self._h = h
        arr = (N.cvpb_view * max(len(self.views), 1))()
        for i, v in enumerate(self.views):
            C.memmove(C.byref(arr[i]), C.byref(v._v), C.sizeof(N.cvpb_view))
        N.check(L.cvpb_set_geometry(h, C.byref(vol_geom._c()), C.byref(det._c()),
                                    len(self.views), arr))

    def close(self):
        if getattr(self, "_h", None):
            N.lib().cvpb_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_views(self):
        return len(self.views)

    def synchronize(self, stream=None):
        """Wait for the stream and raise the reference's exception for any
        geometry degeneracy an asynchronous device call flagged (cvpb_sync)."""
        N.check(N.lib().cvpb_sync(self._h, _stream(stream)))

    def _torch_device(self):
        import torch
        return torch.device("cuda", self.device)

    def new_volume(self):
        import torch
        return torch.zeros(self.vol_geom.shape(), dtype=torch.float32, device=self._torch_device())

    def new_stack(self, n_views=None):
        import torch
        n = self.n_views if n_views is None else n_views
        return torch.zeros((n, self.det.rows, self.det.cols), dtype=torch.float32,
                           device=self._torch_device())

    def _range(self, view_begin, view_count):
        if view_count is None:
            view_count = self.n_views - view_begin
        return int(view_begin), int(view_count)

    def _vol(self, t):
        return _ptr(t, self.vol_geom.voxel_count(), self.device)

    def _stk(self, t, n_views):
        # a stack argument points at the first view of the launch's range
        # (cvpb200.h); a longer buffer is fine, a shorter one is not
        return _ptr(t, self.det.pixel_count() * max(int(n_views), 0), self.device, at_least=True)

    # ---- CVP -------------------------------------------------------------
    def project_cvp(self, vol, out=None, opts: CvpOptions = None, exec: ExecPolicy = None,
                    view_begin=0, view_count=None, stream=None):
        opts = opts or CvpOptions()
        exec = exec or ExecPolicy()
        vb, vc = self._range(view_begin, view_count)
        if out is None:
            out = self.new_stack(vc)
        N.check(N.lib().cvpb_project_cvp(self._h, C.byref(opts._c()), C.byref(exec._c()),
                                         self._vol(vol), self._stk(out, vc), vb, vc, _stream(stream)))
        return out

    def backproject_cvp(self, proj, out=None, opts: CvpOptions = None, exec: ExecPolicy = None,
                        view_begin=0, view_count=None, accumulate=False, stream=None):
        opts = opts or CvpOptions()
        exec = exec or ExecPolicy()
        vb, vc = self._range(view_begin, view_count)
        if out is None:
            out = self.new_volume()
        N.check(N.lib().cvpb_backproject_cvp(self._h, C.byref(opts._c()), C.byref(exec._c()),
                                             self._stk(proj, vc), self._vol(out), vb, vc,
                                             int(bool(accumulate)), _stream(stream)))
        return out

    def backproject_cvp_scatter(self, proj, slabs, plane_begin, opts: CvpOptions = None,
                                exec: ExecPolicy = None, view_begin=0, view_count=None, stream=None,
                                store=False):
        """Backprojection fused with a reduce-scatter: planes
        [plane_begin[t], plane_begin[t+1]) are added (float atomics) into
        slabs[t] — a float32 CUDA tensor or a raw device address, on this or
        another GPU with peer access — as each brick finishes
        (cvpb_backproject_cvp_scatter). store=True overwrites the regions
        instead (plain stores; sum several ranks' regions with sum_slabs)."""
        opts = opts or CvpOptions()
        exec = exec or ExecPolicy()
        vb, vc = self._range(view_begin, view_count)
        n = len(slabs)
        if not 1 <= n <= 16 or len(plane_begin) != n + 1:
            raise InvalidArgument("slab targets: 1 to 16 slabs and n + 1 plane boundaries")
        plane = self.vol_geom.counts[0] * self.vol_geom.counts[1]
        tg = N.cvpb_slab_targets()
        tg.n = n
        tg.store = 1 if store else 0
        for t in range(n + 1):
            tg.plane_begin[t] = int(plane_begin[t])
        for t, sl in enumerate(slabs):
            cnt = (int(plane_begin[t + 1]) - int(plane_begin[t])) * plane
            if isinstance(sl, int):  # a raw device address (e.g. another process's buffer, CUDA IPC)
                tg.slab[t] = sl
            else:
                tg.slab[t] = _ptr(sl, cnt).value if cnt > 0 else None
        N.check(N.lib().cvpb_backproject_cvp_scatter(self._h, C.byref(opts._c()), C.byref(exec._c()),
                                                     self._stk(proj, vc), vb, vc, C.byref(tg),
                                                     _stream(stream)))
        return slabs

    def sum_slabs(self, sources, count, out, stream=None):
        """out[:count] = sum of the sources (device addresses or float32 CUDA
        tensors) in order, float64 accumulation (cvpb_sum_slabs); out float32
        or float64 CUDA tensor."""
        import torch
        n = len(sources)
        arr = (C.c_void_p * max(n, 1))()
        for h, src in enumerate(sources):
            arr[h] = src if isinstance(src, int) else _ptr(src, count, at_least=True).value
        if not out.is_cuda or not out.is_contiguous() or out.numel() < count:
            raise InvalidArgument("sum_slabs: out must be a contiguous CUDA tensor of at least count elements")
        o32 = C.c_void_p(out.data_ptr()) if out.dtype == torch.float32 else None
        o64 = C.c_void_p(out.data_ptr()) if out.dtype == torch.float64 else None
        if o32 is None and o64 is None:
            raise InvalidArgument("sum_slabs: out must be float32 or float64")
        N.check(N.lib().cvpb_sum_slabs(self._h, arr, n, int(count), o32, o64, _stream(stream)))
        return out

    def project_cvp_host(self, vol64: np.ndarray, out64: np.ndarray = None,
                         opts: CvpOptions = None, exec: ExecPolicy = None, view_seconds=None):
        """Reference-facing path: float64 host buffers, copies inside."""
        opts = opts or CvpOptions()
        exec = exec or ExecPolicy()
        vol64 = _host64(vol64, self.vol_geom.voxel_count())
        if out64 is None:
            out64 = np.zeros(self.det.pixel_count() * self.n_views)
        _check_host_out(out64, self.det.pixel_count() * self.n_views)
        vs = np.zeros(self.n_views) if view_seconds is not None else None
        N.check(N.lib().cvpb_project_cvp_host(self._h, C.byref(opts._c()), C.byref(exec._c()),
                                              C.c_void_p(vol64.ctypes.data),
                                              C.c_void_p(out64.ctypes.data),
                                              C.c_void_p(vs.ctypes.data) if vs is not None else None))
        if view_seconds is not None:
            view_seconds[:] = list(vs)
        return out64

    def backproject_cvp_host(self, proj64: np.ndarray, out64: np.ndarray = None,
                             opts: CvpOptions = None, exec: ExecPolicy = None, view_seconds=None):
        opts = opts or CvpOptions()
        exec = exec or ExecPolicy()
        proj64 = _host64(proj64, self.det.pixel_count() * self.n_views)
        if out64 is None:
            out64 = np.zeros(self.vol_geom.voxel_count())
        _check_host_out(out64, self.vol_geom.voxel_count())
        vs = np.zeros(self.n_views) if view_seconds is not None else None
        N.check(N.lib().cvpb_backproject_cvp_host(self._h, C.byref(opts._c()), C.byref(exec._c()),
                                                  C.c_void_p(proj64.ctypes.data),
                                                  C.c_void_p(out64.ctypes.data),
                                                  C.c_void_p(vs.ctypes.data) if vs is not None else None))
        if view_seconds is not None:
            view_seconds[:] = list(vs)
        return out64

    def cvp_view_weights(self, opts: CvpOptions = None, view_begin=0, view_count=None) -> np.ndarray:
        """Per-view share of a CVP launch's work (cut counts, sum 1): how the
        host calls split their measured time into view_seconds."""
        opts = opts or CvpOptions()
        vb, vc = self._range(view_begin, view_count)
        w = np.zeros(max(vc, 1))
        N.check(N.lib().cvpb_cvp_view_weights(self._h, C.byref(opts._c()), vb, vc,
                                              w.ctypes.data_as(C.POINTER(C.c_double))))
        return w[:vc]

    def collect_cut_records(self, opts: CvpOptions, view: int, i: int, j: int, k: int,
                            clamp=False, cap=256) -> List[CutVolumeRecord]:
        rows = (C.c_int * cap)()
        cols = (C.c_int * cap)()
        vol = (C.c_double * cap)()
        inv = (C.c_double * cap)()
        n = C.c_int()
        N.check(N.lib().cvpb_collect_cut_records(self._h, C.byref(opts._c()), view, i, j, k,
                                                 int(bool(clamp)), cap, rows, cols, vol, inv,
                                                 C.byref(n)))
        if n.value > cap:
            return self.collect_cut_records(opts, view, i, j, k, clamp, cap=n.value)
        return [CutVolumeRecord(rows[t], cols[t], vol[t], inv[t]) for t in range(n.value)]

    def scale_image(self, view: int, exact: bool = True) -> np.ndarray:
        out = np.zeros(self.det.pixel_count())
        N.check(N.lib().cvpb_scale_image(self._h, view, int(bool(exact)),
                                         out.ctypes.data_as(C.POINTER(C.c_double))))
        return out.reshape(self.det.rows, self.det.cols)

    # ---- Siddon-K ----------------------------------------------------------
    def project_siddon(self, vol, k_per_edge: int, out=None, roi: PixelRoi = None,
                       exec: ExecPolicy = None, view_begin=0, view_count=None, stream=None):
        exec = exec or ExecPolicy()
        vb, vc = self._range(view_begin, view_count)
        if out is None:
            out = self.new_stack(vc)
        r = roi._c() if roi is not None else None
        N.check(N.lib().cvpb_project_siddon(self._h, int(k_per_edge),
                                            C.byref(r) if r is not None else None,
                                            C.byref(exec._c()), self._vol(vol), self._stk(out, vc), vb,
                                            vc, _stream(stream)))
        return out

    def backproject_siddon(self, proj, k_per_edge: int, out=None, exec: ExecPolicy = None,
                           view_begin=0, view_count=None, accumulate=False, stream=None):
        exec = exec or ExecPolicy()
        vb, vc = self._range(view_begin, view_count)
        if out is None:
            out = self.new_volume()
        N.check(N.lib().cvpb_backproject_siddon(self._h, int(k_per_edge), C.byref(exec._c()),
                                                self._stk(proj, vc), self._vol(out), vb, vc,
                                                int(bool(accumulate)), _stream(stream)))
        return out

    def project_siddon_host(self, vol64: np.ndarray, k_per_edge: int, out64: np.ndarray = None,
                            roi: PixelRoi = None, exec: ExecPolicy = None):
        """Reference-facing Siddon-K: float64 host buffers, float64 on the
        device end to end (the reference's ground-truth projector)."""
        exec = exec or ExecPolicy()
        vol64 = _host64(vol64, self.vol_geom.voxel_count())
        if out64 is None:
            out64 = np.zeros(self.det.pixel_count() * self.n_views)
        _check_host_out(out64, self.det.pixel_count() * self.n_views)
        r = roi._c() if roi is not None else None
        N.check(N.lib().cvpb_project_siddon_host(self._h, int(k_per_edge),
                                                 C.byref(r) if r is not None else None,
                                                 C.byref(exec._c()), C.c_void_p(vol64.ctypes.data),
                                                 C.c_void_p(out64.ctypes.data)))
        return out64

    def backproject_siddon_host(self, proj64: np.ndarray, k_per_edge: int, out64: np.ndarray = None,
                                exec: ExecPolicy = None):
        exec = exec or ExecPolicy()
        proj64 = _host64(proj64, self.det.pixel_count() * self.n_views)
        if out64 is None:
            out64 = np.zeros(self.vol_geom.voxel_count())
        _check_host_out(out64, self.vol_geom.voxel_count())
        N.check(N.lib().cvpb_backproject_siddon_host(self._h, int(k_per_edge), C.byref(exec._c()),
                                                     C.c_void_p(proj64.ctypes.data),
                                                     C.c_void_p(out64.ctypes.data)))
        return out64

    # ---- TT --------------------------------------------------------------------
    def project_tt(self, vol, out=None, opts: TTOptions = None, view_begin=0, view_count=None,
                   stream=None):
        opts = opts or TTOptions()
        vb, vc = self._range(view_begin, view_count)
        if out is None:
            out = self.new_stack(vc)
        N.check(N.lib().cvpb_project_tt(self._h, C.byref(opts._c()), self._vol(vol),
                                        self._stk(out, vc), vb, vc,
                                        _stream(stream)))
        return out

    def backproject_tt(self, proj, out=None, opts: TTOptions = None, view_begin=0,
                       view_count=None, accumulate=False, stream=None):
        opts = opts or TTOptions()
        vb, vc = self._range(view_begin, view_count)
        if out is None:
            out = self.new_volume()
        N.check(N.lib().cvpb_backproject_tt(self._h, C.byref(opts._c()), self._stk(proj, vc),
                                            self._vol(out),
                                            vb, vc, int(bool(accumulate)), _stream(stream)))
        return out

    # ---- vector ops / CGLS --------------------------------------------------------
    def dot(self, a, b, stream=None) -> float:
        out = C.c_double()
        N.check(N.lib().cvpb_vec_dot(self._h, _ptr(a), _ptr(b), a.numel(), C.byref(out),
                                     _stream(stream)))
        return out.value

    def axpy(self, alpha, x, y, stream=None):
        N.check(N.lib().cvpb_vec_axpy(self._h, float(alpha), _ptr(x), _ptr(y), x.numel(),
                                      _stream(stream)))
        return y

    def xpby(self, s, beta, p, stream=None):
        N.check(N.lib().cvpb_vec_xpby(self._h, _ptr(s), float(beta), _ptr(p), s.numel(),
                                      _stream(stream)))
        return p

    def all_finite(self, x, stream=None) -> bool:
        out = C.c_int()
        N.check(N.lib().cvpb_vec_all_finite(self._h, _ptr(x), x.numel(), C.byref(out),
                                            _stream(stream)))
        return bool(out.value)

    def cgls(self, b, iterations: int, projector: str = "cvp", opts: CvpOptions = None,
             k_per_edge: int = 1, x=None, stream=None, tt_opts: "TTOptions" = None,
             exec: ExecPolicy = None):
        """Device-resident CGLS (solver.cpp:55-106); returns (x, residual_norms).
        Every operator call uses the given options and ExecPolicy (the same
        operator the pair's own forward/adjoint apply)."""
        pid = {"cvp": 0, "siddon": 1, "tt": 2}[projector]
        opts = opts or CvpOptions()
        tt_opts = tt_opts or TTOptions()
        exec = exec or ExecPolicy()
        if x is None:
            x = self.new_volume()
        res = (C.c_double * (iterations + 1))()
        N.check(N.lib().cvpb_cgls(self._h, pid, C.byref(opts._c()), C.byref(tt_opts._c()),
                                  C.byref(exec._c()), int(k_per_edge), self._stk(b, self.n_views),
                                  self._vol(x), int(iterations), res, _stream(stream)))
        return x, list(res)


class GroupScene:
    """One scene over several GPUs in this process (libcvpb200 cvpb_group,
    include/cvpb200.h "multi-device scenes"): views sharded in contiguous
    ranges, the volume in contiguous z-slabs, the backprojection's partial
    volumes reduce-scattered over peer memory. ``devices`` may repeat a GPU
    (``[0, 0]``: two members on one device — the same code path, used to test
    it on a single-GPU box); None = every visible GPU. Host (float64 numpy)
    entry points, the reference's call shapes."""

    def __init__(self, vol_geom: VolumeGeometry, det: DetectorGeometry,
                 views: Sequence[ViewGeometry], devices: Optional[Sequence[int]] = None):
        L = N.lib()
        self.vol_geom, self.det = vol_geom, det
        self.views = list(views)
        h = C.c_void_p()
        if devices:
            arr = (C.c_int * len(devices))(*[int(d) for d in devices])
            N.check(L.cvpb_group_create(arr, len(devices), C.byref(h)))
        else:
            N.check(L.cvpb_group_create(None, 0, C.byref(h)))
        self._h = h
        varr = (N.cvpb_view * max(len(self.views), 1))()
        for i, v in enumerate(self.views):
            C.memmove(C.byref(varr[i]), C.byref(v._v), C.sizeof(N.cvpb_view))
        N.check(L.cvpb_group_set_geometry(h, C.byref(vol_geom._c()), C.byref(det._c()),
                                          len(self.views), varr))

    def close(self):
        if getattr(self, "_h", None):
            N.lib().cvpb_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_views(self):
        return len(self.views)

    @property
    def size(self) -> int:
        n = C.c_int()
        N.check(N.lib().cvpb_group_size(self._h, C.byref(n)))
        return n.value

    def member(self, m: int) -> dict:
        """device, view shard and volume slab (elements) of member m"""
        d, vb, vc = C.c_int(), C.c_int(), C.c_int()
        sb, sn = C.c_size_t(), C.c_size_t()
        N.check(N.lib().cvpb_group_member(self._h, m, C.byref(d), C.byref(vb), C.byref(vc),
                                          C.byref(sb), C.byref(sn)))
        return {"device": d.value, "view_begin": vb.value, "view_count": vc.value,
                "slab_begin": sb.value, "slab_count": sn.value}

    def project_cvp_host(self, vol64, out64=None, opts: CvpOptions = None,
                         exec: ExecPolicy = None, view_seconds=None):
        opts = opts or CvpOptions()
        exec = exec or ExecPolicy()
        npx = self.det.pixel_count() * self.n_views
        vol64 = _host64(vol64, self.vol_geom.voxel_count())
        out64 = np.zeros(npx) if out64 is None else out64
        _check_host_out(out64, npx)
        vs = np.zeros(self.n_views) if view_seconds is not None else None
        N.check(N.lib().cvpb_group_project_cvp_host(
            self._h, C.byref(opts._c()), C.byref(exec._c()), C.c_void_p(vol64.ctypes.data),
            C.c_void_p(out64.ctypes.data), C.c_void_p(vs.ctypes.data) if vs is not None else None))
        if view_seconds is not None:
            view_seconds[:] = list(vs)
        return out64

    def backproject_cvp_host(self, proj64, out64=None, opts: CvpOptions = None,
                             exec: ExecPolicy = None, view_seconds=None):
        opts = opts or CvpOptions()
        exec = exec or ExecPolicy()
        nv = self.vol_geom.voxel_count()
        proj64 = _host64(proj64, self.det.pixel_count() * self.n_views)
        out64 = np.zeros(nv) if out64 is None else out64
        _check_host_out(out64, nv)
        vs = np.zeros(self.n_views) if view_seconds is not None else None
        N.check(N.lib().cvpb_group_backproject_cvp_host(
            self._h, C.byref(opts._c()), C.byref(exec._c()), C.c_void_p(proj64.ctypes.data),
            C.c_void_p(out64.ctypes.data), C.c_void_p(vs.ctypes.data) if vs is not None else None))
        if view_seconds is not None:
            view_seconds[:] = list(vs)
        return out64

    def project_tt_host(self, vol64, out64=None, opts: TTOptions = None):
        opts = opts or TTOptions()
        npx = self.det.pixel_count() * self.n_views
        vol64 = _host64(vol64, self.vol_geom.voxel_count())
        out64 = np.zeros(npx) if out64 is None else out64
        _check_host_out(out64, npx)
        N.check(N.lib().cvpb_group_project_tt_host(self._h, C.byref(opts._c()),
                                                   C.c_void_p(vol64.ctypes.data),
                                                   C.c_void_p(out64.ctypes.data)))
        return out64

    def backproject_tt_host(self, proj64, out64=None, opts: TTOptions = None):
        opts = opts or TTOptions()
        nv = self.vol_geom.voxel_count()
        proj64 = _host64(proj64, self.det.pixel_count() * self.n_views)
        out64 = np.zeros(nv) if out64 is None else out64
        _check_host_out(out64, nv)
        N.check(N.lib().cvpb_group_backproject_tt_host(self._h, C.byref(opts._c()),
                                                       C.c_void_p(proj64.ctypes.data),
                                                       C.c_void_p(out64.ctypes.data)))
        return out64

    def cgls_host(self, b64, iterations: int, projector: str = "cvp", opts: CvpOptions = None,
                  tt: TTOptions = None, exec: ExecPolicy = None, k_per_edge: int = 1):
        """cgls (solver.cpp:55-106) device-resident across the members; returns
        (x float64, residual norms)."""
        kind = {"cvp": 0, "siddon": 1, "tt": 2}[projector]
        opts = opts or CvpOptions()
        tt = tt or TTOptions()
        exec = exec or ExecPolicy()
        b64 = _host64(b64, self.det.pixel_count() * self.n_views)
        x = np.zeros(self.vol_geom.voxel_count())
        hist = np.zeros(int(iterations) + 1)
        N.check(N.lib().cvpb_group_cgls_host(
            self._h, kind, C.byref(opts._c()), C.byref(tt._c()), C.byref(exec._c()),
            int(k_per_edge), C.c_void_p(b64.ctypes.data), C.c_void_p(x.ctypes.data),
            int(iterations), hist.ctypes.data_as(C.POINTER(C.c_double))))
        return x, hist


def _host64(a, n):
    a = np.ascontiguousarray(a, dtype=np.float64).ravel()
    if a.size != n:
        raise InvalidArgument("host buffer size does not match the scene")
    return a


def _check_host_out(a, n):
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
            and a.size == n):
        raise InvalidArgument("output must be a contiguous float64 array of the scene's size")


# ---------------------------------------------------------------------------
# Reference-shaped free functions with a small scene cache.
_SCENES: "OrderedDict[tuple, DeviceScene]" = OrderedDict()


def scene_for(vol_geom: VolumeGeometry, det: DetectorGeometry, views: Sequence[ViewGeometry],
              device: int = 0) -> DeviceScene:
    key = (device, vol_geom, det, views_to_array(views).tobytes())
    sc = _SCENES.get(key)
    if sc is None:
        sc = DeviceScene(vol_geom, det, views, device)
        _SCENES[key] = sc
        while len(_SCENES) > 4:
            _SCENES.popitem(last=False)[1].close()
    else:
        _SCENES.move_to_end(key)
    return sc


def _is_torch(x):
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:
        return False


def _device_of(t):
    return t.device.index if t.device.index is not None else 0


def project_cvp_into(vol: AttenuationVolume, views: Sequence[ViewGeometry], det: DetectorGeometry,
                     opts: CvpOptions, exec: ExecPolicy, out: ProjectionStack, view_seconds=None):
    """cvp.cpp:615-626."""
    if out.det != det or out.n_views != len(views):
        raise InvalidArgument("output stack does not match detector/views")
    if _is_torch(vol.values):
        sc = scene_for(vol.geom, det, views, _device_of(vol.values))
        sc.project_cvp(vol.values, out.values, opts, exec)
    else:
        sc = scene_for(vol.geom, det, views)
        sc.project_cvp_host(vol.values, out.values, opts, exec, view_seconds)


def project_cvp(vol: AttenuationVolume, views, det, opts: CvpOptions = None,
                exec: ExecPolicy = None) -> ProjectionStack:
    device = _device_of(vol.values) if _is_torch(vol.values) else None
    out = ProjectionStack.zeros(det, len(views), device=device)
    project_cvp_into(vol, views, det, opts or CvpOptions(), exec or ExecPolicy(), out)
    return out


def backproject_cvp_into(proj: ProjectionStack, views, vol_geom: VolumeGeometry, opts: CvpOptions,
                         exec: ExecPolicy, out: AttenuationVolume, view_seconds=None):
    """cvp.cpp:636-650."""
    if out.geom != vol_geom:
        raise InvalidArgument("output volume does not match geometry")
    if proj.n_views != len(views):
        raise InvalidArgument("projection stack does not match views")
    if _is_torch(proj.values):
        sc = scene_for(vol_geom, proj.det, views, _device_of(proj.values))
        sc.backproject_cvp(proj.values, out.values, opts, exec)
    else:
        sc = scene_for(vol_geom, proj.det, views)
        sc.backproject_cvp_host(proj.values, out.values, opts, exec, view_seconds)


def backproject_cvp(proj: ProjectionStack, views, vol_geom: VolumeGeometry,
                    opts: CvpOptions = None, exec: ExecPolicy = None) -> AttenuationVolume:
    device = _device_of(proj.values) if _is_torch(proj.values) else None
    out = AttenuationVolume.zeros(vol_geom, device=device)
    backproject_cvp_into(proj, views, vol_geom, opts or CvpOptions(), exec or ExecPolicy(), out)
    return out


def _to_device(values, shape, device):
    import torch
    if _is_torch(values):
        return values.reshape(shape).to(device=device, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.asarray(values, dtype=np.float32).reshape(shape)).to(device)


def project_siddon_k_into(vol: AttenuationVolume, views, det: DetectorGeometry, k_per_edge: int,
                          exec: ExecPolicy, out: ProjectionStack, roi: PixelRoi = None,
                          view_seconds=None):
    """siddon.cpp:166-249."""
    if out.det != det or out.n_views != len(views):
        raise InvalidArgument("output stack does not match detector/views")
    if _is_torch(out.values):
        device = _device_of(out.values)
        sc = scene_for(vol.geom, det, views, device)
        sc.project_siddon(_to_device(vol.values, vol.geom.shape(), f"cuda:{device}"), k_per_edge,
                          out.values, roi, exec)
    else:  # reference buffers: the float64 host path
        sc = scene_for(vol.geom, det, views)
        x = vol.values.double().cpu().numpy() if _is_torch(vol.values) else vol.values
        sc.project_siddon_host(x, k_per_edge, out.values, roi, exec)


def project_siddon_k(vol: AttenuationVolume, views, det, k_per_edge: int,
                     exec: ExecPolicy = None) -> ProjectionStack:
    device = _device_of(vol.values) if _is_torch(vol.values) else None
    out = ProjectionStack.zeros(det, len(views), device=device)
    project_siddon_k_into(vol, views, det, k_per_edge, exec or ExecPolicy(), out)
    return out


def backproject_siddon_k_into(proj: ProjectionStack, views, vol_geom: VolumeGeometry,
                              k_per_edge: int, exec: ExecPolicy, out: AttenuationVolume,
                              view_seconds=None):
    """siddon.cpp:259-313."""
    if out.geom != vol_geom:
        raise InvalidArgument("output volume does not match geometry")
    if proj.n_views != len(views):
        raise InvalidArgument("projection stack does not match views")
    if _is_torch(out.values):
        device = _device_of(out.values)
        sc = scene_for(vol_geom, proj.det, views, device)
        sc.backproject_siddon(_to_device(proj.values, (proj.n_views, proj.det.rows, proj.det.cols),
                                         f"cuda:{device}"), k_per_edge, out.values, exec)
    else:  # reference buffers: the float64 host path
        sc = scene_for(vol_geom, proj.det, views)
        b = proj.values.double().cpu().numpy() if _is_torch(proj.values) else proj.values
        sc.backproject_siddon_host(b, k_per_edge, out.values, exec)


def backproject_siddon_k(proj: ProjectionStack, views, vol_geom, k_per_edge: int,
                         exec: ExecPolicy = None) -> AttenuationVolume:
    device = _device_of(proj.values) if _is_torch(proj.values) else None
    out = AttenuationVolume.zeros(vol_geom, device=device)
    backproject_siddon_k_into(proj, views, vol_geom, k_per_edge, exec or ExecPolicy(), out)
    return out


def collect_cut_records(vol_geom: VolumeGeometry, view: ViewGeometry, det: DetectorGeometry,
                        opts: CvpOptions, i: int, j: int, k: int) -> List[CutVolumeRecord]:
    """cvp.cpp:652-689, evaluated by the device kernel's geometry code."""
    if not (0 <= i < vol_geom.counts[0] and 0 <= j < vol_geom.counts[1] and
            0 <= k < vol_geom.counts[2]):
        raise N.OutOfRange("voxel index outside lattice")
    sc = scene_for(vol_geom, det, [view])
    return sc.collect_cut_records(opts, 0, i, j, k, clamp=False)


def pixel_scale_cos(view: ViewGeometry, det: DetectorGeometry, m: int, n: int) -> float:
    out = C.c_double()
    N.check(N.lib().cvpb_pixel_scale(C.byref(view._v), C.byref(det._c()), 0, m, n, C.byref(out)))
    return out.value


def pixel_scale_exact(view: ViewGeometry, det: DetectorGeometry, m: int, n: int) -> float:
    out = C.c_double()
    N.check(N.lib().cvpb_pixel_scale(C.byref(view._v), C.byref(det._c()), 1, m, n, C.byref(out)))
    return out.value
