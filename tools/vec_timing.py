"""Timing of the CGLS vector kernels (dot, axpy, xpby, all_finite) on a
c3-sized stack."""
import sys, time, torch
sys.path.insert(0, ".")
import paper_2110_09841_b200 as cb
det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
geom = cb.VolumeGeometry.make((512,)*3, (0.09,)*3)
views = cb.make_circular_trajectory(749.0, 1198.0, 496, 360.0, det)
sc = cb.DeviceScene(geom, det, views)
a = torch.rand(496*480*616, device="cuda"); b = torch.rand_like(a)
for name, fn in (("dot", lambda: sc.dot(a, b)), ("axpy", lambda: sc.axpy(0.5, a, b)), ("xpby", lambda: sc.xpby(a, 0.5, b)), ("all_finite", lambda: sc.all_finite(a))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize()
    print(name, "%.2f ms" % ((time.perf_counter() - t0) / 10 * 1e3))
