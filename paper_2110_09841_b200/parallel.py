"""Multi-GPU partitioning of the projector pair.

One process per GPU (torch.distributed; NCCL on the box, gloo in CPU tests).
Views are sharded contiguously across ranks:

* forward projection is embarrassingly parallel per view — each rank holds the
  whole volume and writes only its own views; no exchange;
* backprojection has one real exchange: every rank backprojects its views into
  a full-size partial volume, and a reduce-scatter sums the partials while
  handing each rank one contiguous z-slab (the volume is k-slowest,
  geometry.hpp:34-36, so slabs are contiguous);
* device-resident CGLS keeps x, s, p as slabs and r, q as view shards; it
  all-gathers p before each forward projection and all-reduces the float64
  dot-product scalars (solver.cpp:55-106 recurrence).

The per-rank compute is injected (``forward_local`` / ``adjoint_local`` and a
``vec`` object), so the same orchestration runs over libcvpb200 on GPUs and
over a CPU stand-in in the gloo tests.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Optional

import torch
import torch.distributed as dist

from ._native import InvalidArgument


def view_shard(n_views: int, world: int, rank: int):
    """Contiguous view range [begin, begin + count) owned by `rank`."""
    b = rank * n_views // world
    e = (rank + 1) * n_views // world
    return b, e - b


def slab_elems(n_vox: int, world: int) -> int:
    """Elements per z-slab after padding the flat volume to a multiple of world."""
    return (n_vox + world - 1) // world


class DistributedOperator:
    """Sharded projector pair over a process group.

    forward_local(x_full, out_local)  projects the full volume into this rank's views
    adjoint_local(b_local, out_full)  backprojects this rank's views into a
                                      full-size partial volume (overwrites out)
    """

    def __init__(self, forward_local: Callable, adjoint_local: Callable, n_vox: int,
                 local_stack_shape, device, group=None):
        self.forward_local = forward_local
        self.adjoint_local = adjoint_local
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n_vox = int(n_vox)
        self.slab = slab_elems(self.n_vox, self.world)
        self.device = device
        self.local_stack_shape = tuple(local_stack_shape)
        self._full = torch.zeros(self.slab * self.world, dtype=torch.float32, device=device)

    # ---- layout helpers -------------------------------------------------
    def slab_range(self, rank=None):
        r = self.rank if rank is None else rank
        b = min(r * self.slab, self.n_vox)
        return b, min(b + self.slab, self.n_vox)

    def new_slab(self):
        return torch.zeros(self.slab, dtype=torch.float32, device=self.device)

    def new_local_stack(self):
        return torch.zeros(self.local_stack_shape, dtype=torch.float32, device=self.device)

    # ---- collectives -------------------------------------------------------
    def reduce_scatter(self, partial_full: torch.Tensor, out_slab: torch.Tensor):
        """Sum the ranks' full-size partial volumes; keep this rank's z-slab."""
        flat = partial_full.reshape(-1)
        if flat.numel() != self.slab * self.world:
            buf = self._full
            buf.zero_()
            buf[: flat.numel()].copy_(flat)
            flat = buf
        if self.world == 1:
            out_slab.copy_(flat[: self.slab])
        else:
            dist.reduce_scatter_tensor(out_slab, flat, group=self.group)
        return out_slab

    def all_gather(self, slab: torch.Tensor) -> torch.Tensor:
        """Reassemble the full volume (flat, unpadded) from the z-slabs."""
        if self.world == 1:
            self._full[: self.slab].copy_(slab)
        else:
            dist.all_gather_into_tensor(self._full, slab.contiguous(), group=self.group)
        return self._full[: self.n_vox]

    def all_reduce_scalar(self, v: float) -> float:
        if self.world == 1:
            return float(v)
        t = torch.tensor([v], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, group=self.group)
        return float(t.item())

    # ---- operators -------------------------------------------------------------
    def project(self, x_full: torch.Tensor, out_local: torch.Tensor = None):
        if out_local is None:
            out_local = self.new_local_stack()
        self.forward_local(x_full, out_local)
        return out_local

    def backproject(self, b_local: torch.Tensor, out_slab: torch.Tensor = None,
                    partial: torch.Tensor = None):
        if out_slab is None:
            out_slab = self.new_slab()
        if partial is None:
            partial = torch.zeros(self.n_vox, dtype=torch.float32, device=self.device)
        self.adjoint_local(b_local, partial)
        return self.reduce_scatter(partial, out_slab)


class TorchVec:
    """Vector ops on torch tensors (any device) with float64 dots."""

    def dot(self, a, b):
        return float(torch.dot(a.reshape(-1).double(), b.reshape(-1).double()).item())

    def axpy(self, alpha, x, y):
        y.add_(x, alpha=alpha)

    def xpby(self, s, beta, p):
        p.mul_(beta).add_(s)

    def all_finite(self, x):
        return bool(torch.isfinite(x).all().item())


class SceneVec:
    """libcvpb200 device vector kernels (compensated float64 dots)."""

    def __init__(self, scene):
        self.scene = scene

    def dot(self, a, b):
        return self.scene.dot(a.reshape(-1), b.reshape(-1))

    def axpy(self, alpha, x, y):
        self.scene.axpy(alpha, x.reshape(-1), y.reshape(-1))

    def xpby(self, s, beta, p):
        self.scene.xpby(s.reshape(-1), beta, p.reshape(-1))

    def all_finite(self, x):
        return self.scene.all_finite(x.reshape(-1))


@dataclass
class DistributedCglsResult:
    x_slab: torch.Tensor
    residual_norms: List[float]


def distributed_cgls(op: DistributedOperator, b_local: torch.Tensor, iterations: int,
                     vec=None) -> DistributedCglsResult:
    """CGLS from x0 = 0 (solver.cpp:55-106) with slab-resident x, s, p and
    view-sharded r, q. Every rank returns its own slab of x."""
    if iterations < 1:
        raise InvalidArgument("cgls needs at least one iteration")
    vec = vec or TorchVec()
    r = b_local.clone()
    x = op.new_slab()
    s = op.new_slab()
    q = op.new_local_stack()
    partial = torch.zeros(op.n_vox, dtype=torch.float32, device=op.device)
    res = [math.sqrt(op.all_reduce_scalar(vec.dot(r, r)))]
    op.backproject(r, s, partial)
    p = s.clone()
    gamma = op.all_reduce_scalar(vec.dot(s, s))
    for it in range(1, iterations + 1):
        if gamma == 0.0:
            res.append(res[-1])
            continue
        p_full = op.all_gather(p)
        op.project(p_full, q)
        qq = op.all_reduce_scalar(vec.dot(q, q))
        if qq == 0.0:
            raise RuntimeError(f"CGLS breakdown (A p = 0) at iteration {it}")
        alpha = gamma / qq
        vec.axpy(alpha, p, x)
        vec.axpy(-alpha, q, r)
        op.backproject(r, s, partial)
        gamma_new = op.all_reduce_scalar(vec.dot(s, s))
        beta = gamma_new / gamma
        vec.xpby(s, beta, p)
        gamma = gamma_new
        ok = op.all_reduce_scalar(float(vec.all_finite(x) and vec.all_finite(r)))
        if ok < op.world:
            raise RuntimeError(f"CGLS diverged (non-finite iterate) at iteration {it}")
        res.append(math.sqrt(op.all_reduce_scalar(vec.dot(r, r))))
    return DistributedCglsResult(x, res)


def scene_operator(scene, opts=None, projector: str = "cvp", k_per_edge: int = 1,
                   group=None) -> DistributedOperator:
    """DistributedOperator over a DeviceScene: this rank's view shard."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    vb, vc = view_shard(scene.n_views, world, rank)
    shape3 = scene.vol_geom.shape()

    def fwd(x_full, out_local):
        x = x_full.reshape(shape3)
        if projector == "cvp":
            scene.project_cvp(x, out_local, opts, view_begin=vb, view_count=vc)
        elif projector == "siddon":
            scene.project_siddon(x, k_per_edge, out_local, view_begin=vb, view_count=vc)
        else:
            scene.project_tt(x, out_local, view_begin=vb, view_count=vc)

    def adj(b_local, out_full):
        out = out_full.reshape(shape3)
        if projector == "cvp":
            scene.backproject_cvp(b_local, out, opts, view_begin=vb, view_count=vc)
        elif projector == "siddon":
            scene.backproject_siddon(b_local, k_per_edge, out, view_begin=vb, view_count=vc)
        else:
            scene.backproject_tt(b_local, out, view_begin=vb, view_count=vc)

    return DistributedOperator(fwd, adj, scene.vol_geom.voxel_count(),
                               (vc, scene.det.rows, scene.det.cols),
                               torch.device("cuda", scene.device), group)
