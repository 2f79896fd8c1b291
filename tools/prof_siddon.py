"""Profiling driver for the Siddon-K pair (c2 geometry, 16 views, K=1 and
K=8 forward, K=1 backward) under ncu."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb
det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
geom = cb.VolumeGeometry.make((256,) * 3, (0.18,) * 3)
views = cb.make_circular_trajectory(749.0, 1198.0, 16, 200.0, det)
sc = cb.DeviceScene(geom, det, views)
x = torch.rand(geom.shape(), device="cuda")
b = torch.rand((16, 480, 616), device="cuda")
p1 = sc.project_siddon(x, k_per_edge=1)
v1 = sc.backproject_siddon(b, k_per_edge=1)
p8 = sc.project_siddon(x, k_per_edge=8)
torch.cuda.synchronize()
