"""ExecPolicy::deterministic (exec.hpp:6-15): the reference's deterministic
policy makes every run bit-identical. On the device:

* backward: one view group per brick (fixed accumulation order, no atomics);
* forward: each brick's records sum in its int32 fixed-point tile (integer
  adds commute) and the bricks merge into an int64 fixed-point stack at a
  launch-wide power-of-two quantum (2^61 / bound, bound >= any pixel's sum),
  so the float atomics' order dependence is gone.

Runs must be bit-identical, and within float32 reassociation of the default
(atomic) path and within the north-star bar of the reference."""
import os

import numpy as np
import pytest

from conftest import make_case, max_rel, rel_l2

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


@pytest.mark.parametrize("case", [
    ((64, 64, 64), (0.72, 0.72, 0.72), 480, 616, 0.154, 0.154, 749.0, 1198.0, 12),
    ((40, 48, 56), (1.0, 0.9, 0.8), 72, 80, 1.0, 1.0, 90.0, 160.0, 9),
])
def test_deterministic_forward_is_bit_reproducible(case, reference):
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, sc = make_case(*case)
    scene = cb.DeviceScene(geom, det, views)
    x64 = cb.fill_uniform01(geom.voxel_count(), 7)
    x = torch.from_numpy(x64.astype(np.float32)).reshape(geom.shape()).cuda()
    ex = cb.ExecPolicy(deterministic=True)
    runs = [scene.project_cvp(x, exec=ex).cpu().numpy() for _ in range(3)]
    assert all(np.array_equal(runs[0], r) for r in runs[1:])
    loose = scene.project_cvp(x).cpu().numpy()
    assert rel_l2(runs[0], loose) < 1e-6
    p_ref = reference.project_cvp(sc, x64.astype(np.float32).astype(np.float64), (1, 1, 0, 1),
                                  threads=THREADS)
    assert rel_l2(runs[0], p_ref) <= 1e-5 and max_rel(runs[0], p_ref) <= 1e-4
    # the host path (float64 volume read in place) takes the same merge
    h = [scene.project_cvp_host(x64.astype(np.float32).astype(np.float64), exec=ex) for _ in range(2)]
    assert np.array_equal(h[0], h[1])
    assert rel_l2(h[0], p_ref) <= 1e-5


def test_deterministic_backward_is_bit_reproducible():
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((32, 32, 32), (1.0, 1.0, 1.0), 48, 48, 1.0, 1.0, 60.0, 100.0,
                                    40)
    scene = cb.DeviceScene(geom, det, views)
    b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * 40, 8).astype(np.float32)).reshape(
        40, 48, 48).cuda()
    ex = cb.ExecPolicy(deterministic=True)
    a = scene.backproject_cvp(b, exec=ex).cpu().numpy()
    c = scene.backproject_cvp(b, exec=ex).cpu().numpy()
    assert np.array_equal(a, c)


def test_deterministic_forward_nonfinite_falls_back():
    """A NaN voxel has no fixed-point image: the launch takes the float
    atomics (NaN propagates like the reference's double sum)."""
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((32, 32, 32), (1.0, 1.0, 1.0), 48, 48, 1.0, 1.0, 60.0, 100.0, 6)
    scene = cb.DeviceScene(geom, det, views)
    x = torch.rand(geom.shape(), device="cuda")
    x[16, 16, 16] = float("nan")
    p = scene.project_cvp(x, exec=cb.ExecPolicy(deterministic=True))
    assert torch.isnan(p).any()
    zero = scene.project_cvp(torch.zeros_like(x), exec=cb.ExecPolicy(deterministic=True))
    assert float(zero.abs().max()) == 0.0
