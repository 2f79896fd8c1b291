"""c3 end-to-end timing through the float64 host C ABI (project_cvp_host +
backproject_cvp_host, pinned host buffers), for A/B of host-path variants."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_09841_b200 as cb

det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
geom = cb.VolumeGeometry.make((512,) * 3, (0.09,) * 3)
views = cb.make_circular_trajectory(749.0, 1198.0, 496, 360.0, det)
sc = cb.DeviceScene(geom, det, views)
x = torch.from_numpy(cb.fill_uniform01(geom.voxel_count(), 7)).pin_memory().numpy()
b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * 496, 8)).pin_memory().numpy()
p = torch.empty(det.pixel_count() * 496, dtype=torch.float64).pin_memory().numpy()
o = torch.empty(geom.voxel_count(), dtype=torch.float64).pin_memory().numpy()
for it in range(4):
    t0 = time.perf_counter()
    sc.project_cvp_host(x, p)
    t1 = time.perf_counter()
    sc.backproject_cvp_host(b, o)
    t2 = time.perf_counter()
    if it:
        w = geom.voxel_count() * 496 / 1e9
        print(f"e2e P {w / (t1 - t0):.1f} BP {w / (t2 - t1):.1f} pair {w / (t2 - t0):.1f} Gvox-view/s")
