"""Profiling driver for the TT pair (c3 geometry, 16 views) under ncu."""
import sys, torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb
det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
geom = cb.VolumeGeometry.make((512,)*3, (0.09,)*3)
views = cb.make_circular_trajectory(749.0, 1198.0, 16, 360.0, det)
sc = cb.DeviceScene(geom, det, views)
x = torch.rand(geom.shape(), device="cuda"); b = torch.rand((16, 480, 616), device="cuda")
p = sc.project_tt(x); v = sc.backproject_tt(b); torch.cuda.synchronize()
