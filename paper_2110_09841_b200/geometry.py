"""Geometry and data model — Python mirror of the reference's
include/cbct/geometry.hpp and volume.hpp.

All numerics that define a view (frame validation and snapping, camera rows,
trajectory angles, 3x4 factorisation) run in libcvpb200's C++ host code
(paper_2110_09841_b200/csrc/api.cpp), so Python, the C-ABI and the device
kernels share bit-identical view parameters.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from . import _native as N
from ._native import InvalidArgument


@dataclass(frozen=True)
class VolumeGeometry:
    """N1 x N2 x N3 voxels of a1 x a2 x a3 mm centred at the origin
    (geometry.hpp:15-39)."""
    counts: Tuple[int, int, int]
    voxel_size: Tuple[float, float, float]

    @staticmethod
    def make(counts, voxel_size) -> "VolumeGeometry":
        counts = tuple(int(c) for c in counts)
        voxel_size = tuple(float(a) for a in voxel_size)
        if len(counts) != 3 or len(voxel_size) != 3:
            raise InvalidArgument("volume geometry needs three counts and three sizes")
        if any(c <= 0 for c in counts):
            raise InvalidArgument("voxel counts must be positive")
        for a in voxel_size:
            if not np.isfinite(a):
                raise InvalidArgument("voxel size is not finite")
            if a <= 0.0:
                raise InvalidArgument("voxel sizes must be positive")
        return VolumeGeometry(counts, voxel_size)

    def extent(self):
        return tuple(c * a for c, a in zip(self.counts, self.voxel_size))

    def min_corner(self):
        return tuple(e * -0.5 for e in self.extent())

    def voxel_center(self, i, j, k):
        """Centre of voxel (i,j,k) (geometry.cpp:33-40)."""
        if not (0 <= i < self.counts[0] and 0 <= j < self.counts[1] and 0 <= k < self.counts[2]):
            raise N.OutOfRange("voxel index outside lattice")
        ext = self.extent()
        a = self.voxel_size
        return tuple((a[d] - ext[d]) * 0.5 + idx * a[d] for d, idx in enumerate((i, j, k)))

    def voxel_count(self) -> int:
        return self.counts[0] * self.counts[1] * self.counts[2]

    def linear_index(self, i, j, k) -> int:
        """i fastest, k slowest (geometry.hpp:34-36)."""
        return (k * self.counts[1] + j) * self.counts[0] + i

    def shape(self):
        """numpy/torch shape of the volume array: (N3, N2, N1)."""
        return (self.counts[2], self.counts[1], self.counts[0])

    def _c(self):
        return N.cvpb_volume_geometry((C.c_int * 3)(*self.counts),
                                      (C.c_double * 3)(*self.voxel_size))


@dataclass(frozen=True)
class DetectorGeometry:
    """rows x cols pixels of b1 x b2 mm; pixel (m, n) centred at (chi1, chi2) =
    (n, m) (geometry.hpp:43-56)."""
    rows: int
    cols: int
    pixel_width: float = 1.0
    pixel_height: float = 1.0

    @staticmethod
    def make(rows, cols, pixel_width, pixel_height) -> "DetectorGeometry":
        if rows <= 0 or cols <= 0:
            raise InvalidArgument("detector counts must be positive")
        for b in (pixel_width, pixel_height):
            if not np.isfinite(b):
                raise InvalidArgument("pixel size is not finite")
            if b <= 0.0:
                raise InvalidArgument("pixel sizes must be positive")
        return DetectorGeometry(int(rows), int(cols), float(pixel_width), float(pixel_height))

    def pixel_area(self):
        return self.pixel_width * self.pixel_height

    def pixel_size(self):
        return (self.pixel_width, self.pixel_height)

    def pixel_count(self):
        return self.rows * self.cols

    def _c(self):
        return N.cvpb_detector_geometry(self.rows, self.cols, self.pixel_width, self.pixel_height)


class ViewGeometry:
    """One source/detector pose (geometry.hpp:70-123). Construct through
    :meth:`make`, :meth:`from_standard_matrix` or
    :func:`make_circular_trajectory`."""

    __slots__ = ("_v",)

    def __init__(self, cview: N.cvpb_view):
        self._v = cview

    @staticmethod
    def make(source, frame, focal_length, principal_point, pixel_size) -> "ViewGeometry":
        out = N.cvpb_view()
        s = (C.c_double * 3)(*[float(x) for x in source])
        fr = (C.c_double * 9)(*[float(x) for x in np.asarray(frame, dtype=float).ravel()])
        pp = (C.c_double * 2)(*[float(x) for x in principal_point])
        b = (C.c_double * 2)(*[float(x) for x in pixel_size])
        N.check(N.lib().cvpb_view_make(s, fr, float(focal_length), pp, b, C.byref(out)))
        return ViewGeometry(out)

    @staticmethod
    def from_standard_matrix(P, pixel_size) -> "ViewGeometry":
        out = N.cvpb_view()
        Pa = (C.c_double * 12)(*[float(x) for x in np.asarray(P, dtype=float).ravel()])
        b = (C.c_double * 2)(*[float(x) for x in pixel_size])
        N.check(N.lib().cvpb_view_from_standard_matrix(Pa, b, C.byref(out)))
        return ViewGeometry(out)

    @staticmethod
    def from_array(a17) -> "ViewGeometry":
        a = np.asarray(a17, dtype=np.float64).ravel()
        return ViewGeometry.make(a[0:3], a[3:12], a[12], a[13:15], a[15:17])

    def to_array(self) -> np.ndarray:
        v = self._v
        return np.array(list(v.source) + list(v.frame) + [v.focal_length] +
                        list(v.principal_point) + list(v.pixel_size), dtype=np.float64)

    def source(self):
        return tuple(self._v.source)

    def frame(self):
        return np.array(self._v.frame, dtype=np.float64).reshape(3, 3)

    def focal_length(self):
        return self._v.focal_length

    def principal_point(self):
        return tuple(self._v.principal_point)

    def pixel_size(self):
        return tuple(self._v.pixel_size)

    def camera_matrix(self):
        P = self.standard_matrix()
        return P[:, :3].copy()

    def standard_matrix(self) -> np.ndarray:
        P = (C.c_double * 12)()
        N.check(N.lib().cvpb_view_standard_matrix(C.byref(self._v), P))
        return np.array(P, dtype=np.float64).reshape(3, 4)

    def project_point(self, x):
        chi = (C.c_double * 2)()
        N.check(N.lib().cvpb_view_project_point(C.byref(self._v),
                                                (C.c_double * 3)(*[float(t) for t in x]), chi))
        return (chi[0], chi[1])

    def depth(self, x):
        ew = self.frame()[2]
        return float(np.dot(ew, np.asarray(x, dtype=float) - np.asarray(self.source())))

    def detector_point(self, chi):
        """World position of detector coordinate chi (geometry.cpp:115-118)."""
        local = np.array([(chi[0] - self._v.principal_point[0]) * self._v.pixel_size[0],
                          (chi[1] - self._v.principal_point[1]) * self._v.pixel_size[1],
                          self._v.focal_length])
        return tuple(np.asarray(self.source()) + self.frame().T @ local)

    def elevation_angle(self, chi):
        u = (chi[0] - self._v.principal_point[0]) * self._v.pixel_size[0]
        v = (chi[1] - self._v.principal_point[1]) * self._v.pixel_size[1]
        return float(np.arctan2(abs(v), np.hypot(u, self._v.focal_length)))

    def __eq__(self, other):
        return isinstance(other, ViewGeometry) and np.array_equal(self.to_array(), other.to_array())

    def __repr__(self):
        return f"ViewGeometry(source={self.source()}, f={self.focal_length()})"


def make_circular_trajectory(sid, sdd, n_views, arc_deg, det: DetectorGeometry) -> List[ViewGeometry]:
    """Circular trajectory around x3 (geometry.cpp:182-210)."""
    if n_views <= 0:
        raise InvalidArgument("need at least one view")
    arr = (N.cvpb_view * n_views)()
    N.check(N.lib().cvpb_make_circular_trajectory(float(sid), float(sdd), int(n_views),
                                                  float(arc_deg), C.byref(det._c()), arr))
    out = []
    for i in range(n_views):
        v = N.cvpb_view()
        C.memmove(C.byref(v), C.byref(arr[i]), C.sizeof(N.cvpb_view))
        out.append(ViewGeometry(v))
    return out


def views_to_array(views: Sequence[ViewGeometry]) -> np.ndarray:
    """(V, 17) float64 array in the cvpb_view layout."""
    return np.stack([v.to_array() for v in views]) if len(views) else np.zeros((0, 17))


def write_camera_matrices(path, views: Sequence[ViewGeometry]):
    """One row-major 3x4 matrix per line, 17 significant digits
    (geometry.cpp:212-222)."""
    with open(path, "w") as f:
        for v in views:
            P = v.standard_matrix().ravel()
            f.write(" ".join(f"{x:.17g}" for x in P) + "\n")


def read_camera_matrices(path, pixel_size) -> List[ViewGeometry]:
    """Inverse of write_camera_matrices; '#' lines skipped (geometry.cpp:224-249)."""
    if not os.path.exists(path):
        raise N.CvpbRuntimeError(f"cannot open {path}")
    views = []
    with open(path) as f:
        for lineno, line in enumerate(f, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            parts = s.split()
            if len(parts) != 12:
                raise N.CvpbRuntimeError(f"{path}:{lineno}: expected 12 numbers per line")
            try:
                P = [float(x) for x in parts]
            except ValueError:
                raise N.CvpbRuntimeError(f"{path}:{lineno}: expected 12 numbers per line")
            views.append(ViewGeometry.from_standard_matrix(P, pixel_size))
    if not views:
        raise N.CvpbRuntimeError(f"{path}: no matrices found")
    return views


@dataclass
class AttenuationVolume:
    """Per-voxel attenuation (volume.hpp:11-21). ``values`` is a float64
    numpy array (host, reference layout) or a float32 CUDA tensor of shape
    (N3, N2, N1) (device-resident)."""
    geom: VolumeGeometry
    values: object = None

    @staticmethod
    def zeros(g: VolumeGeometry, device=None):
        if device is None:
            return AttenuationVolume(g, np.zeros(g.voxel_count(), dtype=np.float64))
        import torch
        return AttenuationVolume(g, torch.zeros(g.shape(), dtype=torch.float32, device=device))


@dataclass
class ProjectionStack:
    """Per-view extinction images, view-major (volume.hpp:25-47). ``values``
    is a float64 numpy array or a float32 CUDA tensor of shape (V, rows, cols)."""
    det: DetectorGeometry
    n_views: int
    values: object = None

    @staticmethod
    def zeros(d: DetectorGeometry, n_views: int, device=None):
        if device is None:
            return ProjectionStack(d, n_views, np.zeros(d.pixel_count() * n_views, dtype=np.float64))
        import torch
        return ProjectionStack(d, n_views, torch.zeros((n_views, d.rows, d.cols),
                                                       dtype=torch.float32, device=device))

    def view_size(self):
        return self.det.pixel_count()
