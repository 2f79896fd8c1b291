"""Diagnostic: forward projection of all 496 c3 views in one launch vs the
same views projected one at a time (multi-view state carried across views
in a brick must not change a view's result)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb
N, V = 512, 496
det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
geom = cb.VolumeGeometry.make((N, N, N), (0.09,) * 3)
views = cb.make_circular_trajectory(749.0, 1198.0, V, 360.0, det)
scene = cb.DeviceScene(geom, det, views)
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.rand(geom.shape(), device="cuda", generator=g)
ax = scene.project_cvp(x)
out = []
for v in (0, 61, 62, 93, 124, 248):
    axv = scene.project_cvp(x, view_begin=v, view_count=1)
    out.append("%d:%.1e" % (v, float((axv[0] - ax[v]).norm() / ax[v].norm())))
print(" ".join(out))
