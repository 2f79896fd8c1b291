"""Operator plug + Krylov solver — Python mirror of include/cbct/solver.hpp.

``LinearOperatorPair`` keeps the reference's shape (solver.hpp:14-23).
``cvp_pair`` / ``siddon_pair`` / ``tt_pair`` build device-backed pairs; ``cgls``
runs the CGLS recurrence of solver.cpp:55-106 with libcvpb200's device vector
kernels (compensated float64 dots of float32 vectors), and hands a pair that
carries a :class:`DeviceScene` to the fully device-resident C++ driver
(cvpb_cgls).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _native as N
from ._native import InvalidArgument
from .geometry import AttenuationVolume, DetectorGeometry, ProjectionStack, VolumeGeometry
from .operators import CvpOptions, DeviceScene, ExecPolicy, TTOptions, _ptr, _stream


@dataclass
class LinearOperatorPair:
    forward: Callable[[AttenuationVolume, ProjectionStack], None]
    adjoint: Callable[[ProjectionStack, AttenuationVolume], None]
    vol_geom: VolumeGeometry
    det: DetectorGeometry
    n_views: int
    scene: Optional[DeviceScene] = None
    projector: str = ""
    cvp_opts: Optional[CvpOptions] = None
    k_per_edge: int = 1
    tt_opts: Optional[TTOptions] = None
    exec: Optional[ExecPolicy] = None

    def domain_size(self):
        return self.vol_geom.voxel_count()

    def range_size(self):
        return self.det.pixel_count() * self.n_views


def cvp_pair(scene: DeviceScene, opts: CvpOptions = None, exec: ExecPolicy = None) -> LinearOperatorPair:
    opts = opts or CvpOptions()
    exec = exec or ExecPolicy()
    return LinearOperatorPair(
        forward=lambda x, out: scene.project_cvp(x.values, out.values, opts, exec),
        adjoint=lambda b, out: scene.backproject_cvp(b.values, out.values, opts, exec),
        vol_geom=scene.vol_geom, det=scene.det, n_views=scene.n_views, scene=scene,
        projector="cvp", cvp_opts=opts, exec=exec)


def siddon_pair(scene: DeviceScene, k_per_edge: int, exec: ExecPolicy = None) -> LinearOperatorPair:
    exec = exec or ExecPolicy()
    return LinearOperatorPair(
        forward=lambda x, out: scene.project_siddon(x.values, k_per_edge, out.values, None, exec),
        adjoint=lambda b, out: scene.backproject_siddon(b.values, k_per_edge, out.values, exec),
        vol_geom=scene.vol_geom, det=scene.det, n_views=scene.n_views, scene=scene,
        projector="siddon", k_per_edge=k_per_edge, exec=exec)


def tt_pair(scene: DeviceScene, opts: TTOptions = None) -> LinearOperatorPair:
    opts = opts or TTOptions()
    return LinearOperatorPair(
        forward=lambda x, out: scene.project_tt(x.values, out.values, opts),
        adjoint=lambda b, out: scene.backproject_tt(b.values, out.values, opts),
        vol_geom=scene.vol_geom, det=scene.det, n_views=scene.n_views, scene=scene,
        projector="tt", tt_opts=opts)


def fill_uniform01(n: int, seed: int) -> np.ndarray:
    """mt19937_64 stream, (x >> 11) * 2^-53 (solver.cpp:30-33)."""
    out = np.zeros(int(n), dtype=np.float64)
    N.check(N.lib().cvpb_fill_uniform01(out.ctypes.data_as(C.POINTER(C.c_double)), out.size,
                                        C.c_uint64(seed)))
    return out


def relative_projector_error(view, view_ref) -> float:
    """100 * ||P - P_ref||_F / ||P_ref||_F (solver.cpp:108-119)."""
    a = np.asarray(view, dtype=np.float64).ravel()
    b = np.asarray(view_ref, dtype=np.float64).ravel()
    if a.size != b.size:
        raise InvalidArgument("view dimensions do not match")
    den = float(np.dot(b, b))
    if den == 0.0:
        raise N.DomainError("reference view has zero norm")
    d = a - b
    return 100.0 * math.sqrt(float(np.dot(d, d)) / den)


def extinction_from_intensity(I0: float, I: float) -> float:
    if not (I0 > 0.0) or not (I > 0.0):
        raise N.DomainError("intensities must be positive")
    return math.log(I0) - math.log(I)


class _VecCtx:
    """A geometry-less libcvpb200 context for the vector kernels."""
    _h = {}

    @classmethod
    def get(cls, device):
        h = cls._h.get(device)
        if h is None:
            h = C.c_void_p()
            N.check(N.lib().cvpb_context_create(device, C.byref(h)))
            cls._h[device] = h
        return h


def _dot(device, a, b):
    out = C.c_double()
    N.check(N.lib().cvpb_vec_dot(_VecCtx.get(device), _ptr(a), _ptr(b), a.numel(), C.byref(out),
                                 _stream(None)))
    return out.value


def _device_pair_buffers(pair: LinearOperatorPair, device):
    import torch
    dev = torch.device("cuda", device)
    vol = lambda: AttenuationVolume(pair.vol_geom, torch.zeros(pair.vol_geom.shape(),
                                                               dtype=torch.float32, device=dev))
    stk = lambda: ProjectionStack(pair.det, pair.n_views,
                                  torch.zeros((pair.n_views, pair.det.rows, pair.det.cols),
                                              dtype=torch.float32, device=dev))
    return vol, stk


def adjoint_test(pair: LinearOperatorPair, seed: int, device: int = 0) -> float:
    """|b.(Ax) - x.(A'b)| / max(|b.(Ax)|, |x.(A'b)|) with x then b drawn from
    one mt19937_64 stream (solver.cpp:35-53); dots in compensated float64."""
    import torch
    n, m = pair.domain_size(), pair.range_size()
    draws = fill_uniform01(n + m, seed)
    dev = torch.device("cuda", device)
    vol, stk = _device_pair_buffers(pair, device)
    x = AttenuationVolume(pair.vol_geom, torch.from_numpy(draws[:n].astype(np.float32))
                          .reshape(pair.vol_geom.shape()).to(dev))
    b = ProjectionStack(pair.det, pair.n_views, torch.from_numpy(draws[n:].astype(np.float32))
                        .reshape(pair.n_views, pair.det.rows, pair.det.cols).to(dev))
    ax, atb = stk(), vol()
    pair.forward(x, ax)
    pair.adjoint(b, atb)
    lhs = _dot(device, b.values, ax.values)
    rhs = _dot(device, x.values, atb.values)
    den = max(abs(lhs), abs(rhs))
    if den == 0.0:
        return float("nan")
    return abs(lhs - rhs) / den


@dataclass
class CglsResult:
    x: AttenuationVolume
    residual_norms: List[float] = field(default_factory=list)


def cgls(pair: LinearOperatorPair, b: ProjectionStack, iterations: int, device: int = 0) -> CglsResult:
    """Classical CGLS from x0 = 0 (solver.cpp:55-106)."""
    import torch
    if iterations < 1:
        raise InvalidArgument("cgls needs at least one iteration")
    if b.det != pair.det or b.n_views != pair.n_views:
        raise InvalidArgument("cgls data does not match the operator range")
    dev = torch.device("cuda", device)
    bt = b.values
    if not isinstance(bt, torch.Tensor):
        bt = torch.from_numpy(np.asarray(bt, dtype=np.float32))
    bt = bt.reshape(pair.n_views, pair.det.rows, pair.det.cols).to(dev, torch.float32).contiguous()
    if pair.scene is not None and pair.projector in ("cvp", "siddon", "tt"):
        x, res = pair.scene.cgls(bt, iterations, pair.projector, pair.cvp_opts, pair.k_per_edge,
                                 tt_opts=pair.tt_opts, exec=pair.exec)
        return CglsResult(AttenuationVolume(pair.vol_geom, x), res)
    # generic pair: same recurrence with the device vector kernels
    h = _VecCtx.get(device)
    L = N.lib()
    st = _stream(None)
    vol, stk = _device_pair_buffers(pair, device)
    x = vol()
    r = ProjectionStack(pair.det, pair.n_views, bt.clone())
    res = [math.sqrt(_dot(device, r.values, r.values))]
    s = vol()
    pair.adjoint(r, s)
    p = AttenuationVolume(pair.vol_geom, s.values.clone())
    q = stk()
    gamma = _dot(device, s.values, s.values)
    for it in range(1, iterations + 1):
        if gamma == 0.0:
            res.append(res[-1])
            continue
        pair.forward(p, q)
        qq = _dot(device, q.values, q.values)
        if qq == 0.0:
            raise N.CvpbRuntimeError(f"CGLS breakdown (A p = 0) at iteration {it}")
        alpha = gamma / qq
        N.check(L.cvpb_vec_axpy(h, alpha, _ptr(p.values), _ptr(x.values), p.values.numel(), st))
        N.check(L.cvpb_vec_axpy(h, -alpha, _ptr(q.values), _ptr(r.values), q.values.numel(), st))
        pair.adjoint(r, s)
        gamma_new = _dot(device, s.values, s.values)
        beta = gamma_new / gamma
        N.check(L.cvpb_vec_xpby(h, _ptr(s.values), beta, _ptr(p.values), s.values.numel(), st))
        gamma = gamma_new
        for vec in (x.values, r.values):
            ok = C.c_int()
            N.check(L.cvpb_vec_all_finite(h, _ptr(vec), vec.numel(), C.byref(ok), st))
            if not ok.value:
                raise N.CvpbRuntimeError(f"CGLS diverged (non-finite iterate) at iteration {it}")
        res.append(math.sqrt(_dot(device, r.values, r.values)))
    return CglsResult(x, res)


@dataclass
class SartResult:
    x: object
    residual_norms: List[float] = field(default_factory=list)


def os_sart(scene: DeviceScene, b, iterations: int, n_subsets: int = 1, lam: float = 1.0,
            nonneg: bool = False, projector: str = "cvp", opts: CvpOptions = None,
            k_per_edge: int = 1, track_residual: bool = True) -> SartResult:
    """Ordered-subset SART (Andersen & Kak 1984; Kak & Slaney ch. 7) with the
    device projector pair — the reconstruction loop the paper's KCT uses
    (SURVEY §8 row f4).

    Subsets interleave views (subset s = views s, s+S, s+2S, ...); internally
    the views are reordered so each subset is a contiguous view range of one
    resident scene. Per sub-iteration:
        r = (b_S - A_S x) / (A_S 1),   x += lam * (A_S^T r) / (A_S^T 1)
    with the two vector steps as fused device kernels (cvpb_vec_sart_*)."""
    import torch
    if iterations < 1:
        raise InvalidArgument("sart needs at least one iteration")
    V = scene.n_views
    S = max(1, min(int(n_subsets), V))
    order = [v for s in range(S) for v in range(s, V, S)]
    bounds = []
    pos = 0
    for s in range(S):
        cnt = len(range(s, V, S))
        bounds.append((pos, cnt))
        pos += cnt
    sc = scene if order == list(range(V)) else DeviceScene(
        scene.vol_geom, scene.det, [scene.views[i] for i in order], scene.device)
    opts = opts or CvpOptions()
    bt = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.asarray(b, dtype=np.float32))
    bt = bt.reshape(V, scene.det.rows, scene.det.cols).to(sc._torch_device(), torch.float32)
    bp = bt[torch.as_tensor(order, device=bt.device)].contiguous()

    def P(x, out, vb, vc):
        if projector == "cvp":
            return sc.project_cvp(x, out, opts, view_begin=vb, view_count=vc)
        if projector == "siddon":
            return sc.project_siddon(x, k_per_edge, out, view_begin=vb, view_count=vc)
        return sc.project_tt(x, out, view_begin=vb, view_count=vc)

    def BP(p, out, vb, vc):
        if projector == "cvp":
            return sc.backproject_cvp(p, out, opts, view_begin=vb, view_count=vc)
        if projector == "siddon":
            return sc.backproject_siddon(p, k_per_edge, out, view_begin=vb, view_count=vc)
        return sc.backproject_tt(p, out, view_begin=vb, view_count=vc)

    ones_v = torch.ones(scene.vol_geom.shape(), device=bt.device)
    rowsum = sc.new_stack()
    colsum = []
    for vb, vc in bounds:
        P(ones_v, rowsum[vb:vb + vc], vb, vc)
        cs = sc.new_volume()
        BP(torch.ones_like(rowsum[vb:vb + vc]), cs, vb, vc)
        colsum.append(cs)
    x = sc.new_volume()
    ax = sc.new_stack()
    r = sc.new_stack()
    corr = sc.new_volume()
    L = N.lib()
    st = _stream(None)
    res = []
    for _ in range(iterations):
        for (vb, vc), cs in zip(bounds, colsum):
            axs, rs, bs, ws = ax[vb:vb + vc], r[vb:vb + vc], bp[vb:vb + vc], rowsum[vb:vb + vc]
            P(x, axs, vb, vc)
            N.check(L.cvpb_vec_sart_residual(sc._h, _ptr(bs), _ptr(axs), _ptr(ws), _ptr(rs),
                                             rs.numel(), st))
            BP(rs, corr, vb, vc)
            N.check(L.cvpb_vec_sart_update(sc._h, _ptr(x), _ptr(corr), _ptr(cs), float(lam),
                                           int(bool(nonneg)), x.numel(), st))
        if track_residual:
            P(x, ax, 0, V)
            r.copy_(bp).sub_(ax)
            res.append(math.sqrt(sc.dot(r, r)))
    return SartResult(x, res)
