"""Dump TT P/BP outputs on three scenes (small, C-arm, large cone) for
tools/tt_cmp.py; CVPB_LIB selects the library build."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb
out = {}
cases = {"small": ((24, 20, 40), 0.7, 40, 44, 1.0, 60., 100., 6),
         "c3ish": ((96, 96, 96), 0.09 * 512 / 96 / 2, 480, 616, 0.154, 749., 1198., 4),
         "cone": ((64, 64, 70), 0.5, 256, 256, 1.0, 300., 500., 5)}
for name, (cnt, a, R, C, px, sid, sdd, V) in cases.items():
    det = cb.DetectorGeometry.make(R, C, px, px)
    geom = cb.VolumeGeometry.make(cnt, (a,) * 3)
    views = cb.make_circular_trajectory(sid, sdd, V, 360.0, det)
    sc = cb.DeviceScene(geom, det, views)
    x = torch.from_numpy(cb.fill_uniform01(geom.voxel_count(), 3).astype(np.float32)).reshape(geom.shape()).cuda()
    b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * V, 4).astype(np.float32)).reshape(V, R, C).cuda()
    for amp in (0, 1):
        o = cb.TTOptions(amp)
        out[f"{name}_p{amp}"] = sc.project_tt(x, opts=o).cpu().numpy()
        out[f"{name}_b{amp}"] = sc.backproject_tt(b, opts=o).cpu().numpy()
np.savez(sys.argv[1], **out)
