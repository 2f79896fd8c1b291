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
y = torch.rand((V, 480, 616), device="cuda", generator=g)
ax = scene.project_cvp(x)
aty = scene.backproject_cvp(y)
# per-view
bad = []
tot_l = tot_r = 0.0
for v in list(range(0, V, 31)) + [1, 2, 3, 62, 124, 186, 248]:
    axv = scene.project_cvp(x, view_begin=v, view_count=1)
    atv = scene.backproject_cvp(y[v:v+1].contiguous(), view_begin=v, view_count=1)
    l = float(torch.dot(axv.reshape(-1).double(), y[v].reshape(-1).double()))
    r = float(torch.dot(x.reshape(-1).double(), atv.reshape(-1).double()))
    d_full = float((axv[0] - ax[v]).norm() / ax[v].norm())
    print(v, "adj %.3e" % ((l - r) / r), "P(single) vs P(all) %.3e" % d_full, flush=True)
lhs = float(torch.dot(ax.reshape(-1).double(), y.reshape(-1).double()))
rhs = float(torch.dot(x.reshape(-1).double(), aty.reshape(-1).double()))
print("all", lhs, rhs, (lhs - rhs) / rhs)
# BP sum over single views vs all
acc = torch.zeros_like(aty)
for v in range(0, V, 62):
    acc += scene.backproject_cvp(y[v:v+62].contiguous(), view_begin=v, view_count=62)
print("BP chunks-of-62 vs all: %.3e" % float((acc - aty).norm() / aty.norm()))
