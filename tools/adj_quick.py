"""Diagnostic: projection of all views in one launch vs the same views one at
a time, and the full-launch adjointness <Ax, y> vs <x, A^T y> (multi-view
state carried across views in a brick, and the cut-table view chunks, must
not change a view's result).

    python tools/adj_quick.py [c3|c5]
"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
N, a, R, C, px, sid, sdd, V = {"c3": (512, 0.09, 480, 616, 0.154, 749.0, 1198.0, 496),
                               "c5": (1024, 0.4, 768, 1024, 1.0, 541.0, 949.0, 720)}[cfg]
det = cb.DetectorGeometry.make(R, C, px, px)
geom = cb.VolumeGeometry.make((N, N, N), (a,) * 3)
views = cb.make_circular_trajectory(sid, sdd, V, 360.0, det)
scene = cb.DeviceScene(geom, det, views)
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.rand(geom.shape(), device="cuda", generator=g)
ax = scene.project_cvp(x)
out = []
for v in (0, V // 8 - 1, V // 8, V // 4, V // 2, V - 1):
    axv = scene.project_cvp(x, view_begin=v, view_count=1)
    out.append("%d:%.1e" % (v, float((axv[0] - ax[v]).norm() / ax[v].norm())))
print(cfg, "single-view vs full launch:", " ".join(out))
y = torch.rand((V, R, C), device="cuda", generator=g)
aty = scene.backproject_cvp(y)
lhs = float(torch.dot(ax.reshape(-1).double(), y.reshape(-1).double()))
rhs = float(torch.dot(x.reshape(-1).double(), aty.reshape(-1).double()))
print(cfg, "adjointness %.2e" % (abs(lhs - rhs) / max(abs(lhs), abs(rhs))))
