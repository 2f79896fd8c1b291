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

# round 2 (later): relaxed precision on a scene whose bricks take the
# per-voxel-cut radius (small voxels far from the source), the three-boundary
# fast walk (voxels ~2-3 rows tall), and the scatter backprojection in store
# and atomic mode
det2 = cb.DetectorGeometry.make(64, 48, 0.1, 0.1)
geom2 = cb.VolumeGeometry.make((16, 16, 64), (0.05, 0.05, 0.05))
views2 = cb.make_circular_trajectory(700.0, 1100.0, 6, 360.0, det2)
sc2 = cb.DeviceScene(geom2, det2, views2)
x2 = torch.rand(geom2.shape(), device="cuda")
rel = cb.CvpOptions(precision=cb.CvpPrecision.Single)
p2 = sc2.project_cvp(x2, opts=rel)
b2 = sc2.backproject_cvp(p2, opts=rel)
det3 = cb.DetectorGeometry.make(96, 80, 0.1, 0.1)
geom3 = cb.VolumeGeometry.make((24, 20, 64), (0.15, 0.15, 0.15))
views3 = cb.make_circular_trajectory(300.0, 500.0, 5, 360.0, det3)
sc3 = cb.DeviceScene(geom3, det3, views3)
x3 = torch.rand(geom3.shape(), device="cuda")
p3 = sc3.project_cvp(x3)
b3 = sc3.backproject_cvp(p3)
n1, n2, n3 = geom3.counts
bounds = [0, 20, 20, n3]
slabs = [torch.zeros((bounds[t + 1] - bounds[t], n2, n1), device="cuda") for t in range(3)]
sc3.backproject_cvp_scatter(p3, slabs, bounds, store=True)
sc3.backproject_cvp_scatter(p3, slabs, bounds)
out = torch.empty(n1 * n2 * (bounds[1] - bounds[0]), dtype=torch.float64, device="cuda")
sc3.sum_slabs([slabs[0].reshape(-1), slabs[0].reshape(-1)], out.numel(), out)
torch.cuda.synchronize()
print("sanitize case (relaxed radius, three-boundary walk, scatter) ok")
