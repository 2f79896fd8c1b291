"""GPU-vs-reference parity table (rel-L2 and max|d|/max|ref|) for the CVP
pair over the parity scenes; exact and relaxed device modes against the
reference's Double and Single paths. Prints markdown."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import paper_2110_09841_b200 as cb
from paper_2110_09841_b200.phantom import shepp_logan_3d
from oracle.pyoracle import Reference, Restatement, Scene, reference_available

chk = Reference() if reference_available() else Restatement()
SCENES = [
    ("c1 64^3 SL, 64x64 @1mm, 36v", (64,)*3, (0.5,)*3, 64, 64, 1.0, 541., 949., 36, "sl"),
    ("desk 64^3, 128^2 @1mm, 12v", (64,)*3, (0.5,)*3, 128, 128, 1.0, 541., 949., 12, "u"),
    ("C-arm 64^3 @0.72, 480x616 @0.154, 6v", (64,)*3, (0.72,)*3, 480, 616, 0.154, 749., 1198., 6, "u"),
    ("c2-geom 96^3 @0.18, 480x616 @0.154, 4v", (96,)*3, (0.18,)*3, 480, 616, 0.154, 749., 1198., 4, "u"),
    ("c4-geom 64^3 @0.5, 256^2 @1mm SID300, 6v", (64,)*3, (0.5,)*3, 256, 256, 1.0, 300., 500., 6, "u"),
]
rel = lambda a, b: float(np.linalg.norm(a.ravel() - b.ravel()) / np.linalg.norm(b.ravel()))
mx = lambda a, b: float(np.abs(a.ravel() - b.ravel()).max() / np.abs(b.ravel()).max())
print("| scene | op | GPU exact vs ref Double (rel-L2 / max) | GPU relaxed vs ref Double | ref Single vs ref Double |")
print("|---|---|---|---|---|")
for name, counts, vox, R, C, px, sid, sdd, nv, kind in SCENES:
    det = cb.DetectorGeometry.make(R, C, px, px)
    geom = cb.VolumeGeometry.make(counts, vox)
    views = cb.make_circular_trajectory(sid, sdd, nv, 360.0, det)
    sc = Scene(counts, vox, R, C, px, px, cb.views_to_array(views))
    x = shepp_logan_3d(geom) if kind == "sl" else cb.fill_uniform01(geom.voxel_count(), 7)
    x = x.astype(np.float32).astype(np.float64)
    b = cb.fill_uniform01(R * C * nv, 8).astype(np.float32).astype(np.float64)
    scene = cb.DeviceScene(geom, det, views)
    xt = torch.from_numpy(x.astype(np.float32)).reshape(geom.shape()).cuda()
    bt = torch.from_numpy(b.astype(np.float32)).reshape(nv, R, C).cuda()
    res = {}
    for prec, p in (("exact", cb.CvpPrecision.Double), ("relaxed", cb.CvpPrecision.Single)):
        o = cb.CvpOptions(precision=p)
        res[prec] = (scene.project_cvp(xt, opts=o).double().cpu().numpy(),
                     scene.backproject_cvp(bt, opts=o).double().cpu().numpy())
    pd = chk.project_cvp(sc, x, (1, 1, 0, 1)); bd = chk.backproject_cvp(sc, b, (1, 1, 0, 1))
    ps = chk.project_cvp(sc, x, (1, 1, 1, 1)); bs = chk.backproject_cvp(sc, b, (1, 1, 1, 1))
    for op, ref, refs, i in (("P", pd, ps, 0), ("BP", bd, bs, 1)):
        e, r = res["exact"][i].reshape(ref.shape), res["relaxed"][i].reshape(ref.shape)
        print(f"| {name} | {op} | {rel(e, ref):.2e} / {mx(e, ref):.2e} | {rel(r, ref):.2e} / {mx(r, ref):.2e} | {rel(refs, ref):.2e} / {mx(refs, ref):.2e} |")
    sys.stdout.flush()
