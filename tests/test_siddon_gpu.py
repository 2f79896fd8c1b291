"""GPU parity of the Siddon-K pair (siddon.cpp) against the CPU checker.

Tolerance: the device traverses in float64 exactly like the reference and
only the attenuation inputs / outputs are float32, so results agree to float32
rounding: max|d|/max|ref| <= 1e-6."""
import numpy as np
import pytest

from conftest import make_case, max_rel, rel_l2

pytestmark = pytest.mark.gpu


def _t(a, shape):
    import torch
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).reshape(shape).cuda()


@pytest.mark.parametrize("K", [1, 2, 4])
def test_siddon_pair_matches_reference(checker, K):
    import paper_2110_09841_b200 as cb
    geom, det, views, sc = make_case((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, 40.0, 70.0, 6)
    x = cb.fill_uniform01(geom.voxel_count(), 3).astype(np.float32).astype(np.float64)
    b = cb.fill_uniform01(det.pixel_count() * 6, 5).astype(np.float32).astype(np.float64)
    scene = cb.DeviceScene(geom, det, views)
    p = scene.project_siddon(_t(x, geom.shape()), K).double().cpu().numpy()
    bp = scene.backproject_siddon(_t(b, (6, 32, 32)), K).double().cpu().numpy()
    p_ref = checker.project_siddon(sc, x, K)
    bp_ref = checker.backproject_siddon(sc, b, K).reshape(bp.shape)
    assert max_rel(p, p_ref) <= 1e-6
    assert max_rel(bp, bp_ref) <= 1e-6


def test_siddon_roi_and_sparse_volume(checker):
    """PixelRoi (siddon.hpp:28-33) and the tight nonzero sub-box (siddon.cpp:182-211)."""
    import paper_2110_09841_b200 as cb
    geom, det, views, sc = make_case((24, 24, 24), (0.5, 0.5, 0.5), 48, 40, 0.8, 0.8, 60.0, 100.0, 3)
    x = np.zeros(geom.voxel_count())
    x3 = x.reshape(geom.shape())
    x3[5:9, 10:20, 3:7] = 1.5
    scene = cb.DeviceScene(geom, det, views)
    roi = cb.PixelRoi(10, 30, 5, 25)
    p = scene.project_siddon(_t(x, geom.shape()), 2, roi=roi).double().cpu().numpy()
    p_ref = checker.project_siddon(sc, x, 2, roi=(10, 30, 5, 25))
    assert max_rel(p, p_ref) <= 1e-6
    assert np.count_nonzero(p[:, :10]) == 0 and np.count_nonzero(p[:, :, 25:]) == 0


def test_siddon_expensive_k_gate():
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((8, 8, 8), (1.0, 1.0, 1.0), 8, 8, 1.0, 1.0, 40.0, 70.0, 1)
    scene = cb.DeviceScene(geom, det, views)
    x = scene.new_volume()
    with pytest.raises(cb.InvalidArgument):
        scene.project_siddon(x, 128)
    with pytest.raises(cb.InvalidArgument):
        scene.project_siddon(x, 0)
    scene.project_siddon(x, 128, exec=cb.ExecPolicy(allow_expensive=True))


def test_siddon_adjointness_device():
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((24, 24, 24), (1.0, 1.0, 1.0), 40, 40, 1.0, 1.0, 60.0, 100.0, 6)
    scene = cb.DeviceScene(geom, det, views)
    for K in (1, 2):
        assert cb.adjoint_test(cb.siddon_pair(scene, K), 1) < 1e-5


def test_siddon_homogeneous_volume_gives_box_chords():
    """test_siddon.cpp:154-172: a constant volume projects to c * chord length
    through the box; the central pixel sees the full box depth."""
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((16, 16, 16), (1.0, 1.0, 1.0), 33, 33, 1.0, 1.0, 40.0, 70.0, 1)
    scene = cb.DeviceScene(geom, det, views)
    import torch
    x = torch.full(geom.shape(), 2.0, device="cuda")
    p = scene.project_siddon(x, 1).double().cpu().numpy()
    assert p[0, 16, 16] == pytest.approx(2.0 * 16.0, rel=1e-6)
