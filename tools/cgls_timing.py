"""CGLS ms/iteration on the c3 scene (device-resident cvpb_cgls), before and
after a host-path call: (T(3) - T(1)) / 2 after a warm-up call."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb
det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
geom = cb.VolumeGeometry.make((512,)*3, (0.09,)*3)
views = cb.make_circular_trajectory(749.0, 1198.0, 496, 360.0, det)
scene = cb.DeviceScene(geom, det, views)
x = torch.rand(geom.shape(), device="cuda")
bt = scene.project_cvp(x); scene.backproject_cvp(bt); torch.cuda.synchronize()
def cg(tag):
    scene.cgls(bt, 1); torch.cuda.synchronize()
    t0 = time.perf_counter(); scene.cgls(bt, 1); torch.cuda.synchronize(); t1 = time.perf_counter()
    scene.cgls(bt, 3); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(tag, "cgls ms/iter %.1f" % (((t2 - t1) - (t1 - t0)) / 2 * 1e3), flush=True)
cg("before host path")
x64 = torch.from_numpy(cb.fill_uniform01(geom.voxel_count(), 7)).pin_memory()
p64 = torch.empty(det.pixel_count() * 496, dtype=torch.float64).pin_memory()
v64 = torch.empty(geom.voxel_count(), dtype=torch.float64).pin_memory()
scene.project_cvp_host(x64.numpy(), p64.numpy()); scene.backproject_cvp_host(p64.numpy(), v64.numpy())
cg("after host path")
