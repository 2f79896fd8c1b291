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

For CVP the backprojection and its reduce-scatter are one kernel plus a
local sum (:class:`PeerSlabs`): every rank's receive buffer is mapped into
every other rank's process with CUDA IPC, each rank's bricks store their
voxels straight into the owning rank's region for that source over NVLink as
they finish (cvpb_backproject_cvp_scatter, store mode), and each owner sums
its regions in rank order (cvpb_sum_slabs) — no partial volume crosses the
network after the kernel, no NCCL reduce-scatter; two 1-element NCCL
all-reduces order the ranks' streams (regions free before anyone stores, all
stores landed before anyone sums). NCCL's reduce_scatter_tensor remains the
path for TT / Siddon and volumes whose plane count the world size does not
divide (``CVPB_FUSED_RS=0`` forces it).

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
                 local_stack_shape, device, group=None, adjoint_scatter: Callable = None):
        self.forward_local = forward_local
        self.adjoint_local = adjoint_local
        # adjoint_scatter(b_local) -> this rank's summed slab (fused
        # backprojection + reduce-scatter, PeerSlabs); None: partial + NCCL
        self.adjoint_scatter = adjoint_scatter
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
        if self.adjoint_scatter is not None:
            own = self.adjoint_scatter(b_local)
            out_slab[: own.numel()].copy_(own)
            return out_slab
        if partial is None:
            partial = torch.zeros(self.n_vox, dtype=torch.float32, device=self.device)
        self.adjoint_local(b_local, partial)
        return self.reduce_scatter(partial, out_slab)


class _CudaBuffer:
    """__cuda_array_interface__ view of a raw float32 device buffer (so torch
    can wrap library-allocated IPC memory without a copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


class PeerSlabs:
    """The receive buffers of all ranks, each mapped into every rank's process
    (CUDA IPC), for the fused backprojection + reduce-scatter of CVP.

    Rank r owns planes [r * N3 / world, (r + 1) * N3 / world) (N3 divisible by
    the world size, so the slabs are the same contiguous element ranges the
    NCCL path uses) and a receive buffer of world slab-sized regions, one per
    source rank. :meth:`backproject` stores this rank's voxels of every slab
    straight into the owners' regions for this rank (plain stores over NVLink,
    as each brick finishes; cvpb_backproject_cvp_scatter in store mode), then
    sums its own regions in rank order (cvpb_sum_slabs): the own slab summed
    over all ranks' views, bit-reproducible."""

    def __init__(self, scene, group=None):
        import ctypes as C
        from . import _native as N
        self.scene, self.group = scene, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        n1, n2, n3 = scene.vol_geom.counts
        if n3 % self.world:
            raise InvalidArgument("PeerSlabs needs a plane count divisible by the world size")
        planes = n3 // self.world
        self.elems = planes * n1 * n2
        self.bounds = [r * planes for r in range(self.world + 1)]
        L = N.lib()
        own = C.c_void_p()
        handle = (C.c_char * 64)()
        # every step is agreed on by all ranks (a rank that fails alone must
        # not leave the others waiting in a collective): on any failure every
        # rank releases what it mapped and raises, and callers fall back to
        # the NCCL reduce-scatter
        ok = L.cvpb_ipc_alloc(scene._h, self.elems * 4 * self.world, C.byref(own),
                              C.cast(handle, C.c_void_p)) == 0
        self._own_ptr = own.value if ok else None
        self._opened = []
        msgs = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(msgs, (ok, bytes(handle)), group=group)
        else:
            msgs = [(ok, bytes(handle))]
        recv = []
        if all(m[0] for m in msgs):
            for r in range(self.world):
                if r == self.rank:
                    recv.append(self._own_ptr)
                    continue
                hb = (C.c_char * 64).from_buffer_copy(msgs[r][1])
                p = C.c_void_p()
                if L.cvpb_ipc_open(scene._h, C.cast(hb, C.c_void_p), C.byref(p)) != 0:
                    ok = False
                    break
                self._opened.append(p.value)
                recv.append(p.value)
        else:
            ok = False
        flags = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(flags, ok, group=group)
        else:
            flags = [ok]
        if not all(flags):
            self.own = None
            self._release()
            raise RuntimeError("CUDA IPC slab mapping failed on at least one rank")
        # owner r's region for this rank (source) and this rank's own regions
        self.ptrs = [recv[r] + self.rank * self.elems * 4 for r in range(self.world)]
        self.sources = [self._own_ptr + h * self.elems * 4 for h in range(self.world)]
        self.own = torch.zeros(self.elems, dtype=torch.float32, device=torch.device("cuda", scene.device))
        # device-side barrier: a 1-element NCCL all-reduce completes on every
        # rank's stream only after all ranks' earlier stream work (gloo, in
        # tests: synchronize + host barrier)
        self._nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"
        self._one = torch.zeros(1, dtype=torch.float32, device=self.own.device)

    def _barrier(self):
        if self.world == 1:
            return
        if self._nccl:
            dist.all_reduce(self._one, group=self.group)
        else:
            torch.cuda.synchronize(self.own.device)
            dist.barrier(group=self.group)

    def scatter(self, b_local, opts, view_begin, view_count, stream=None):
        """This rank's views into every owner's receive region for this rank
        (after a barrier: the regions' previous contents have been summed)."""
        self._barrier()
        self.scene.backproject_cvp_scatter(b_local, self.ptrs, self.bounds, opts,
                                           view_begin=view_begin, view_count=view_count,
                                           stream=stream, store=True)

    def finish(self, stream=None):
        """Barrier (every rank's stores have landed), then the own slab = the
        own regions summed in rank order."""
        self._barrier()
        self.scene.sum_slabs(self.sources, self.elems, self.own, stream=stream)
        return self.own

    def backproject(self, b_local, opts, view_begin, view_count, stream=None):
        """This rank's views backprojected and reduce-scattered; returns the
        own slab (flat float32)."""
        self.scatter(b_local, opts, view_begin, view_count, stream)
        return self.finish(stream)

    def _release(self):
        from . import _native as N
        L = N.lib()
        for p in self._opened:
            L.cvpb_ipc_close(self.scene._h, p)
        self._opened = []
        if self._own_ptr:
            L.cvpb_ipc_free(self.scene._h, self._own_ptr)
            self._own_ptr = None

    def close(self):
        if self.own is not None:
            torch.cuda.synchronize(self.own.device)
        self.own = None
        self._release()


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


def fused_reduce_scatter_ok(scene, projector: str = "cvp", exec=None, group=None) -> bool:
    """Whether the CVP backprojection can run fused with the reduce-scatter
    (PeerSlabs): CVP, several ranks, N3 divisible by the world size, not
    disabled by CVPB_FUSED_RS=0 (store mode + fixed-order sums: deterministic
    too)."""
    import os
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    return (projector == "cvp" and world > 1 and scene.vol_geom.counts[2] % world == 0
            and os.environ.get("CVPB_FUSED_RS", "1") != "0")


def scene_operator(scene, opts=None, projector: str = "cvp", k_per_edge: int = 1,
                   group=None) -> DistributedOperator:
    """DistributedOperator over a DeviceScene: this rank's view shard (CVP:
    the backprojection fused with the reduce-scatter when possible)."""
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

    scatter = None
    if fused_reduce_scatter_ok(scene, projector, group=group):
        try:
            peers = PeerSlabs(scene, group)
        except RuntimeError:  # (raised on every rank alike) -> NCCL reduce-scatter
            peers = None
        if peers is not None:
            def scatter(b_local):
                return peers.backproject(b_local, opts, vb, vc)
            scatter.peers = peers
    return DistributedOperator(fwd, adj, scene.vol_geom.voxel_count(),
                               (vc, scene.det.rows, scene.det.cols),
                               torch.device("cuda", scene.device), group, adjoint_scatter=scatter)
