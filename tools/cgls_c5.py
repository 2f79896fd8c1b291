"""BASELINE configs[4] on one B200: CGLS on the 1024^3 / 1024x768 / 720-view
scene (device-resident cvpb_cgls, U[0,1) data, seed 1 as in the reference's
bench), seconds per iteration over `--iterations` after a warm-up iteration.
The 8-GPU run shards the views (parallel.distributed_cgls)."""
import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iterations", type=int, default=3)
a = ap.parse_args()
det = cb.DetectorGeometry.make(768, 1024, 1.0, 1.0)
geom = cb.VolumeGeometry.make((1024, 1024, 1024), (0.4, 0.4, 0.4))
views = cb.make_circular_trajectory(541.0, 949.0, 720, 360.0, det)
scene = cb.DeviceScene(geom, det, views)
b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * 720, 1).astype(np.float32)).reshape(720, 768, 1024).cuda()
scene.cgls(b, 1)
torch.cuda.synchronize()
t0 = time.perf_counter()
_, r1 = scene.cgls(b, 1)
torch.cuda.synchronize()
t1 = time.perf_counter()
_, rn = scene.cgls(b, 1 + a.iterations)
torch.cuda.synchronize()
t2 = time.perf_counter()
per = ((t2 - t1) - (t1 - t0)) / a.iterations
print(f"c5 CGLS on 1 B200: {per:.2f} s/iteration ({1024**3 * 720 / 1e9 / (per / 2):.1f} Gvox-view/s per "
      f"direction); residual {rn[0]:.4e} -> {rn[-1]:.4e} after {1 + a.iterations} iterations")
