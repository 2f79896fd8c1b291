"""GPU parity of the CVP pair on edge-case geometries against the reference:
non-cubic / odd / anisotropic lattices, off-centre principal points from 3x4
matrices, short-scan arcs, volumes wider than the field of view (detector
clamping), many columns per voxel (the cut-cache overflow path), sparse
phantoms (zero-column skipping) and partial view ranges. Tolerance as in
test_cvp_gpu.py: rel-L2 <= 1e-5, max|d|/max|ref| <= 1e-4."""
import numpy as np
import pytest

from conftest import max_rel, rel_l2

pytestmark = pytest.mark.gpu


def _case(checker, counts, voxel, rows, cols, pw, ph, views, opts4=(1, 1, 0, 1), x64=None,
          exec=None):
    import torch
    import paper_2110_09841_b200 as cb
    from oracle.pyoracle import Scene
    det = cb.DetectorGeometry.make(rows, cols, pw, ph)
    geom = cb.VolumeGeometry.make(counts, voxel)
    sc = Scene(tuple(counts), tuple(voxel), rows, cols, pw, ph, cb.views_to_array(views))
    if x64 is None:
        x64 = cb.fill_uniform01(geom.voxel_count(), 5)
    x64 = np.asarray(x64, dtype=np.float32).astype(np.float64)
    b64 = cb.fill_uniform01(det.pixel_count() * len(views), 6).astype(np.float32).astype(np.float64)
    scene = cb.DeviceScene(geom, det, views)
    o = cb.CvpOptions(cb.PixelScaling(opts4[0]), bool(opts4[1]), cb.CvpPrecision(opts4[2]),
                      cb.RadiusEstimate(opts4[3]))
    xt = torch.from_numpy(x64.astype(np.float32)).reshape(geom.shape()).cuda()
    bt = torch.from_numpy(b64.astype(np.float32)).reshape(len(views), rows, cols).cuda()
    p = scene.project_cvp(xt, opts=o, exec=exec).double().cpu().numpy()
    bp = scene.backproject_cvp(bt, opts=o, exec=exec).double().cpu().numpy().ravel()
    p_ref = checker.project_cvp(sc, x64, opts4)
    bp_ref = checker.backproject_cvp(sc, b64, opts4).ravel()
    return p, p_ref, bp, bp_ref


def _assert_close(p, p_ref, bp, bp_ref):
    assert rel_l2(p, p_ref) <= 1e-5 and max_rel(p, p_ref) <= 1e-4, (rel_l2(p, p_ref), max_rel(p, p_ref))
    assert rel_l2(bp, bp_ref) <= 1e-5 and max_rel(bp, bp_ref) <= 1e-4, (rel_l2(bp, bp_ref),
                                                                      max_rel(bp, bp_ref))


def test_odd_anisotropic_lattice_short_scan(checker):
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(50, 70, 0.9, 1.1)
    views = cb.make_circular_trajectory(120.0, 200.0, 7, 200.0, det)
    _assert_close(*_case(checker, (37, 23, 19), (0.7, 0.5, 1.3), 50, 70, 0.9, 1.1, views))


def test_matrices_with_offset_principal_point(checker):
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(40, 56, 1.0, 1.0)
    base = cb.make_circular_trajectory(90.0, 150.0, 5, 360.0, det)
    views = []
    for k, v in enumerate(base):
        shifted = cb.ViewGeometry.make(v.source(), v.frame(), v.focal_length(),
                                       (v.principal_point()[0] + 3.25 * (k - 2),
                                        v.principal_point()[1] - 1.75 * k), v.pixel_size())
        views.append(cb.ViewGeometry.from_standard_matrix(shifted.standard_matrix(),
                                                          det.pixel_size()))
    _assert_close(*_case(checker, (24, 24, 24), (1.0, 1.0, 1.0), 40, 56, 1.0, 1.0, views))


def test_volume_wider_than_detector_clamps(checker):
    """Columns and rows outside the detector are dropped (cvp.cpp:144-147,
    197-200); the tile / global fallback must agree."""
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(24, 20, 1.0, 1.0)
    views = cb.make_circular_trajectory(60.0, 100.0, 6, 360.0, det)
    _assert_close(*_case(checker, (32, 32, 32), (1.0, 1.0, 1.0), 24, 20, 1.0, 1.0, views))


def test_views_walked_by_one_brick_with_columns_off_the_detector(checker):
    """Deterministic mode keeps every view in one CTA (no view groups), as
    large volumes do: a column whose cuts all fall off the detector in one
    view must still be projected in the next ones (regression: the per-view
    cut count once overwrote the forward's nonzero-column flag)."""
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(24, 20, 1.0, 1.0)
    views = cb.make_circular_trajectory(60.0, 100.0, 12, 360.0, det)
    _assert_close(*_case(checker, (32, 32, 32), (1.0, 1.0, 1.0), 24, 20, 1.0, 1.0, views,
                         exec=cb.ExecPolicy(deterministic=True)))


@pytest.mark.parametrize("opts4", [(1, 1, 0, 1), (0, 0, 0, 0)])
def test_many_columns_per_voxel_overflow_path(checker, opts4):
    """2 mm voxels on 0.154 mm pixels: ~20 columns per voxel, far beyond the
    4 cached cuts; the extra cuts are recomputed in the V-phase."""
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(96, 160, 0.154, 0.154)
    views = cb.make_circular_trajectory(749.0, 1198.0, 4, 360.0, det)
    _assert_close(*_case(checker, (5, 5, 4), (2.0, 2.0, 2.0), 96, 160, 0.154, 0.154, views, opts4))


def test_sparse_phantom_zero_columns(checker):
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(48, 48, 1.0, 1.0)
    views = cb.make_circular_trajectory(70.0, 120.0, 5, 360.0, det)
    x = np.zeros((20, 33, 40))
    x[3:9, 5:12, 30:37] = 1.0
    x[15, 20, 2] = 4.0
    _assert_close(*_case(checker, (40, 33, 20), (1.0, 1.0, 1.0), 48, 48, 1.0, 1.0, views,
                         x64=x.ravel()))


def test_view_subrange_equals_slice(checker):
    import torch
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(32, 32, 1.0, 1.0)
    views = cb.make_circular_trajectory(50.0, 90.0, 9, 360.0, det)
    geom = cb.VolumeGeometry.make((20, 20, 20), (1.0, 1.0, 1.0))
    scene = cb.DeviceScene(geom, det, views)
    x = torch.rand(geom.shape(), device="cuda")
    full = scene.project_cvp(x)
    part = scene.project_cvp(x, view_begin=4, view_count=3)
    assert float((part - full[4:7]).norm() / full[4:7].norm()) < 1e-6
    empty = scene.project_cvp(x, view_begin=2, view_count=0)
    assert empty.shape[0] == 0


@pytest.mark.parametrize("shape", ["0", "1", "2"])
def test_every_brick_shape_matches_reference(checker, monkeypatch, shape):
    """The library carries three brick shapes (8x16x64 at three CTAs per SM,
    8x8x64 at four, 8x24x64 with 384 threads at two) and times them on a
    scene's first launches; each must match the reference on its own
    (CVPB_CVP_SHAPE forces one)."""
    import paper_2110_09841_b200 as cb
    monkeypatch.setenv("CVPB_CVP_SHAPE", shape)
    det = cb.DetectorGeometry.make(40, 52, 1.0, 1.0)
    views = cb.make_circular_trajectory(70.0, 120.0, 9, 360.0, det)
    _assert_close(*_case(checker, (30, 36, 70), (0.8, 0.8, 0.8), 40, 52, 1.0, 1.0, views,
                         exec=cb.ExecPolicy(deterministic=True)))
    det = cb.DetectorGeometry.make(96, 128, 0.154, 0.154)
    views = cb.make_circular_trajectory(749.0, 1198.0, 8, 360.0, det)
    _assert_close(*_case(checker, (40, 40, 40), (0.09, 0.09, 0.09), 96, 128, 0.154, 0.154, views,
                         opts4=(0, 1, 0, 0)))
