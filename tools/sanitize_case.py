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
