import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb
det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
geom = cb.VolumeGeometry.make((512,)*3, (0.09,)*3)
views = cb.make_circular_trajectory(749.0, 1198.0, 496, 360.0, det)
scene = cb.DeviceScene(geom, det, views)
x = torch.rand(geom.shape(), device="cuda")
bt = scene.project_cvp(x); scene.backproject_cvp(bt); torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); scene.cgls(bt, 1); torch.cuda.synchronize(); t1 = time.perf_counter()
    scene.cgls(bt, 3); torch.cuda.synchronize(); t2 = time.perf_counter()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); scene.project_cvp(x, bt); e[1].record(); scene.backproject_cvp(bt); e[2].record(); torch.cuda.synchronize()
    print("cgls ms/iter %.1f   P %.1f BP %.1f" % (((t2 - t1) - (t1 - t0)) / 2 * 1e3, e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])), flush=True)
