"""DEN volume / projection-stack files — Python restatement of the reference's
den.hpp / den.cpp, plus a zero-conversion device loader.

Format (den.hpp:11-23): three little-endian uint16 (dim_y, dim_x, dim_z) and
dim_z frames of row-major (y, x) float32. A volume maps to (N2, N1, N3), a
stack to (rows, cols, views) — the DEN payload order is exactly the device
layout of libcvpb200 ([N3][N2][N1] / [V][R][C], float32), so
:func:`den_read_device` streams the payload into pinned memory and straight
onto the GPU without a conversion pass.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from ._native import CvpbRuntimeError
from .geometry import AttenuationVolume, DetectorGeometry, ProjectionStack, VolumeGeometry

_DIM_CAP = 65535


def _check_dims(y, x, z, what):
    if y == 0 or x == 0 or z == 0:
        raise CvpbRuntimeError(f"{what}: DEN dimensions must be at least 1")
    if y > _DIM_CAP or x > _DIM_CAP or z > _DIM_CAP:
        raise CvpbRuntimeError(f"{what}: dimension exceeds the DEN 16-bit limit of 65535")


@dataclass
class DenFile:
    dim_y: int = 0
    dim_x: int = 0
    dim_z: int = 0
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.float32))

    def value_count(self) -> int:
        return int(self.dim_y) * int(self.dim_x) * int(self.dim_z)


def _read_header(path):
    if not os.path.exists(path):
        raise CvpbRuntimeError(f"cannot open {path}")
    with open(path, "rb") as f:
        head = f.read(6)
    if len(head) < 6:
        raise CvpbRuntimeError(f"{path}: truncated DEN header")
    y, x, z = (int(v) for v in np.frombuffer(head, dtype="<u2"))
    _check_dims(y, x, z, str(path))
    expected = 6 + 4 * y * x * z
    size = os.path.getsize(path)
    if size != expected:
        raise CvpbRuntimeError(f"{path}: file size {size} does not match header "
                               f"(expected {expected} bytes)")
    return y, x, z


def den_read(path) -> DenFile:
    """den.cpp:27-54."""
    y, x, z = _read_header(path)
    vals = np.fromfile(path, dtype="<f4", offset=6, count=y * x * z)
    if vals.size != y * x * z:
        raise CvpbRuntimeError(f"{path}: truncated DEN payload")
    return DenFile(y, x, z, vals.astype(np.float32, copy=False))


def den_write(path, den: DenFile):
    """den.cpp:56-68."""
    _check_dims(den.dim_y, den.dim_x, den.dim_z, str(path))
    vals = np.ascontiguousarray(den.values, dtype="<f4").ravel()
    if vals.size != den.value_count():
        raise CvpbRuntimeError(f"{path}: DEN payload size does not match dimensions")
    try:
        with open(path, "wb") as f:
            f.write(np.array([den.dim_y, den.dim_x, den.dim_z], dtype="<u2").tobytes())
            f.write(vals.tobytes())
    except OSError as e:
        raise CvpbRuntimeError(f"cannot open {path} for writing") from e


def to_den(obj) -> DenFile:
    """den.cpp:70-89: volumes as (N2, N1, N3), stacks as (rows, cols, views)."""
    if isinstance(obj, AttenuationVolume):
        n1, n2, n3 = obj.geom.counts
        _check_dims(n2, n1, n3, "volume")
        return DenFile(n2, n1, n3, _as_f32(obj.values))
    if isinstance(obj, ProjectionStack):
        _check_dims(obj.det.rows, obj.det.cols, obj.n_views, "projection stack")
        return DenFile(obj.det.rows, obj.det.cols, obj.n_views, _as_f32(obj.values))
    raise TypeError("to_den expects an AttenuationVolume or a ProjectionStack")


def _as_f32(values):
    try:
        import torch
        if isinstance(values, torch.Tensor):
            return values.detach().float().cpu().numpy().ravel()
    except ImportError:
        pass
    return np.asarray(values, dtype=np.float32).ravel()


def volume_from_den(den: DenFile, voxel_size) -> AttenuationVolume:
    """den.cpp:91-95 (float64 host values, reference convention)."""
    g = VolumeGeometry.make((den.dim_x, den.dim_y, den.dim_z), voxel_size)
    return AttenuationVolume(g, np.asarray(den.values, dtype=np.float64).ravel().copy())


def stack_from_den(den: DenFile, pixel_width, pixel_height) -> ProjectionStack:
    """den.cpp:97-100."""
    d = DetectorGeometry.make(den.dim_y, den.dim_x, pixel_width, pixel_height)
    return ProjectionStack(d, den.dim_z, np.asarray(den.values, dtype=np.float64).ravel().copy())


def den_read_device(path, device="cuda"):
    """Read a DEN payload into pinned host memory and copy it to `device` as a
    float32 tensor of shape (dim_z, dim_y, dim_x) — the device layout of a
    volume (N3, N2, N1) or a stack (V, R, C). No format conversion pass."""
    import torch
    y, x, z = _read_header(path)
    host = torch.empty((z, y, x), dtype=torch.float32).pin_memory()
    with open(path, "rb") as f:
        f.seek(6)
        n = f.readinto(memoryview(host.numpy()).cast("B"))
    if n != 4 * y * x * z:
        raise CvpbRuntimeError(f"{path}: truncated DEN payload")
    return host.to(device, non_blocking=True)


def den_write_device(path, tensor):
    """Write a (dim_z, dim_y, dim_x) float32 tensor (device or host) as DEN."""
    t = tensor.detach()
    if t.dim() != 3:
        raise CvpbRuntimeError(f"{path}: expected a 3-D tensor")
    z, y, x = t.shape
    den_write(path, DenFile(y, x, z, t.float().cpu().numpy().ravel()))
