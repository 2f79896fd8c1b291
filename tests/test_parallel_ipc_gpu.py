"""The one-process-per-GPU path's fused backprojection + reduce-scatter
(parallel.PeerSlabs over CUDA IPC, cvpb_backproject_cvp_scatter) with two
ranks sharing the one B200: each rank's slab equals the single-process
backprojection of all views over that slab's planes."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_fused_reduce_scatter_over_ipc(tmp_path):
    import torch
    import paper_2110_09841_b200 as cb
    port = _free_port()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_ipc_worker.py"), str(r), "2",
                               str(port), str(tmp_path)]) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(2)]
    det = cb.DetectorGeometry.make(64, 72, 0.8, 0.8)
    geom = cb.VolumeGeometry.make((40, 36, 32), (0.7, 0.7, 0.7))
    views = cb.make_circular_trajectory(120.0, 200.0, 10, 360.0, det)
    scene = cb.DeviceScene(geom, det, views)
    b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * len(views), 8).astype(np.float32)).reshape(
        len(views), det.rows, det.cols).cuda()
    full = scene.backproject_cvp(b).reshape(-1).double().cpu().numpy()
    ranges = [tuple(int(t) for t in r["slab_range"]) for r in res]
    assert ranges == [(0, full.size // 2), (full.size // 2, full.size)]
    for r, (b0, b1) in zip(res, ranges):
        assert rel_l2(r["slab"][: b1 - b0], full[b0:b1]) < 1e-6
        assert rel_l2(r["again"][: b1 - b0], full[b0:b1]) < 1e-6
    scene.close()
