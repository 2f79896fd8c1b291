"""Worker for test_parallel_ipc_gpu.py: one rank of a world-size-2 group on
ONE GPU (both processes use cuda:0; gloo carries the host-side barriers and
the IPC-handle exchange). The CVP backprojection of this rank's view shard is
fused with the reduce-scatter: it adds straight into both ranks' z-slabs,
mapped into both processes with CUDA IPC (parallel.PeerSlabs)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    import paper_2110_09841_b200 as cb
    from paper_2110_09841_b200 import parallel as par

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    det = cb.DetectorGeometry.make(64, 72, 0.8, 0.8)
    geom = cb.VolumeGeometry.make((40, 36, 32), (0.7, 0.7, 0.7))
    views = cb.make_circular_trajectory(120.0, 200.0, 10, 360.0, det)
    scene = cb.DeviceScene(geom, det, views, device=0)
    vb, vc = par.view_shard(len(views), world, rank)
    b_all = cb.fill_uniform01(det.pixel_count() * len(views), 8).astype(np.float32)
    b_local = torch.from_numpy(b_all[vb * det.pixel_count():(vb + vc) * det.pixel_count()]).reshape(
        vc, det.rows, det.cols).cuda()
    op = par.scene_operator(scene, cb.CvpOptions())
    assert op.adjoint_scatter is not None  # the fused path is the one under test
    slab = op.backproject(b_local)
    again = op.backproject(b_local)  # slabs re-zeroed between calls
    torch.cuda.synchronize()
    b0, b1 = op.slab_range()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), slab=slab.cpu().numpy(),
             again=again.cpu().numpy(), slab_range=np.array([b0, b1]))
    op.adjoint_scatter.peers.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
