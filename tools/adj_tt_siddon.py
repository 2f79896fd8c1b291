"""Diagnostic: full-size (c3) adjointness and single-view vs full-launch
consistency of the TT and Siddon-1 pairs."""
import sys, torch
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
for name, P, B in (("tt", lambda: scene.project_tt(x), lambda: scene.backproject_tt(y)),
                   ("siddon1", lambda: scene.project_siddon(x, 1), lambda: scene.backproject_siddon(y, 1))):
    ax, aty = P(), B()
    lhs = float(torch.dot(ax.reshape(-1).double(), y.reshape(-1).double()))
    rhs = float(torch.dot(x.reshape(-1).double(), aty.reshape(-1).double()))
    out = []
    for v in (0, 61, 124, 248):
        axv = scene.project_tt(x, view_begin=v, view_count=1) if name == "tt" else scene.project_siddon(x, 1, view_begin=v, view_count=1)
        out.append("%d:%.1e" % (v, float((axv[0] - ax[v]).norm() / ax[v].norm())))
    print(name, "adjointness %.2e" % (abs(lhs - rhs) / max(abs(lhs), abs(rhs))), " ".join(out), flush=True)
