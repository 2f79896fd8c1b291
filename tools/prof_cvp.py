"""Profiling driver: c3 geometry with a reduced view count; one P and one BP
launch per precision (used under ncu)."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_09841_b200 as cb

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=16)
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--precision", default="exact")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--config", default="c3")
a = ap.parse_args()
cfgs = {"c3": ((a.n,)*3, (0.09*512/a.n,)*3, 480, 616, 0.154, 749., 1198.),
        "c4": ((a.n,)*3, (0.5*512/a.n,)*3, 1024, 1024, 1.0, 300., 500.),
        "c2": ((256,)*3, (0.18,)*3, 480, 616, 0.154, 749., 1198.),
        "c5": ((a.n,)*3, (0.4*1024/a.n,)*3, 768, 1024, 1.0, 541., 949.)}
counts, vox, R, Cc, px, sid, sdd = cfgs[a.config]
det = cb.DetectorGeometry.make(R, Cc, px, px)
geom = cb.VolumeGeometry.make(counts, vox)
views = cb.make_circular_trajectory(sid, sdd, a.views, 360.0, det)
sc = cb.DeviceScene(geom, det, views)
opts = cb.CvpOptions(precision=cb.CvpPrecision.Double if a.precision == "exact" else cb.CvpPrecision.Single)
x = torch.rand(geom.shape(), device="cuda")
b = torch.rand((a.views, R, Cc), device="cuda")
p = sc.new_stack(); v = sc.new_volume()
for _ in range(a.reps):
    sc.project_cvp(x, p, opts)
    sc.backproject_cvp(b, v, opts)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record(); sc.project_cvp(x, p, opts); e[1].record(); sc.backproject_cvp(b, v, opts); e[2].record()
torch.cuda.synchronize()
w = np.prod(counts) * a.views / 1e9
print(f"{a.config} {a.precision} views={a.views}: P {e[0].elapsed_time(e[1]):.2f} ms ({w/e[0].elapsed_time(e[1])*1e3:.1f} Gvox/s)  BP {e[1].elapsed_time(e[2]):.2f} ms ({w/e[1].elapsed_time(e[2])*1e3:.1f} Gvox/s)")
