"""Small CVP / TT / Siddon P+BP case for compute-sanitizer (memcheck,
racecheck, synccheck): one brick walks several views (deterministic mode) so
the shared tile, the named barrier and the flush re-zeroing are exercised."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb

det = cb.DetectorGeometry.make(40, 36, 1.0, 1.0)
geom = cb.VolumeGeometry.make((24, 20, 70), (1.0, 1.0, 1.0))
views = cb.make_circular_trajectory(70.0, 110.0, 5, 360.0, det)
scene = cb.DeviceScene(geom, det, views)
x = torch.rand(geom.shape(), device="cuda")
ex = cb.ExecPolicy(deterministic=True)
for prec in (cb.CvpPrecision.Double, cb.CvpPrecision.Single):
    o = cb.CvpOptions(precision=prec)
    p = scene.project_cvp(x, opts=o, exec=ex)
    b = scene.backproject_cvp(p, opts=o, exec=ex)
p = scene.project_tt(x)
b = scene.backproject_tt(p)
p = scene.project_siddon(x, 2)
b = scene.backproject_siddon(p, 2)
torch.cuda.synchronize()
print("sanitize case ok")

# round 2: the default (non-deterministic) forward — float-atomic flush,
# virtual tile rows for bricks crossing the detector's top / bottom edge (the
# volume is taller than the detector's field of view) — and a two-member
# multi-device group on one GPU (peer all-gather and peer-load reduction)
for prec in (cb.CvpPrecision.Double, cb.CvpPrecision.Single):
    o = cb.CvpOptions(precision=prec)
    p = scene.project_cvp(x, opts=o)
    b = scene.backproject_cvp(p, opts=o)
import numpy as np
grp = cb.GroupScene(geom, det, views, devices=[0, 0])
x64 = x.double().cpu().numpy().ravel()
pg = grp.project_cvp_host(x64)
bg = grp.backproject_cvp_host(pg)
grp.close()
torch.cuda.synchronize()
print("sanitize case (round 2 paths) ok")
