"""Worker for test_parallel_gloo.py: one rank of a world-size-2 gloo group.

The per-rank compute is the CPU checker (oracle restatement) — test
infrastructure standing in for the device kernels — so this exercises the
multi-GPU orchestration (view sharding, reduce-scatter over z-slabs,
all-gather, distributed CGLS) without a GPU.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    from oracle.pyoracle import Restatement, Scene
    from paper_2110_09841_b200.parallel import (DistributedOperator, TorchVec, distributed_cgls,
                                                view_shard)

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    orc = Restatement()
    counts, voxel, R, C, nv = (16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 8
    views = orc.circular_trajectory(40.0, 70.0, nv, 360.0, R, C, 1.0, 1.0)
    vb, vc = view_shard(nv, world, rank)
    local = Scene(counts, voxel, R, C, 1.0, 1.0, views[vb:vb + vc])
    n_vox = int(np.prod(counts))

    def fwd(x_full, out_local):
        p = orc.project_cvp(local, x_full.double().numpy())
        out_local.copy_(torch.from_numpy(p).float())

    def adj(b_local, out_full):
        v = orc.backproject_cvp(local, b_local.double().numpy())
        out_full.copy_(torch.from_numpy(v.ravel()).float())

    op = DistributedOperator(fwd, adj, n_vox, (vc, R, C), torch.device("cpu"))
    x = torch.from_numpy(orc.fill_uniform01(n_vox, 7)).float()
    b_all = torch.from_numpy(orc.fill_uniform01(R * C * nv, 8)).float().reshape(nv, R, C)
    p_local = op.project(x)
    slab = op.backproject(b_all[vb:vb + vc].contiguous())
    full = op.all_gather(slab).clone()
    res = distributed_cgls(op, b_all[vb:vb + vc].contiguous(), 4, TorchVec())
    xg = op.all_gather(res.x_slab).clone()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), p_local=p_local.numpy(), vb=vb, vc=vc,
             slab=slab.numpy(), full=full.numpy(), cgls_res=np.array(res.residual_norms),
             cgls_x=xg.numpy(), slab_range=np.array(op.slab_range()))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
