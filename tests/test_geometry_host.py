"""CPU: host-side geometry of libcvpb200 (csrc/api.cpp) — the reference's
geometry unit tests (test_geometry.cpp) restated, plus bit-identity of view
parameters against the reference (golden vectors)."""
import math
import os

import numpy as np
import pytest

import paper_2110_09841_b200 as cb

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cvp_golden.npz")


def test_trajectory_bitwise_equal_to_reference():
    g = np.load(GOLD)
    det = cb.DetectorGeometry.make(32, 32, 1.0, 1.0)
    assert np.array_equal(cb.views_to_array(cb.make_circular_trajectory(40.0, 70.0, 4, 360.0, det)),
                          g["small_views"])
    det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
    assert np.array_equal(cb.views_to_array(cb.make_circular_trajectory(749.0, 1198.0, 36, 200.0,
                                                                        det)), g["carm_views"])


def test_voxel_centers_and_validation():
    g = cb.VolumeGeometry.make((512, 512, 512), (0.5, 0.5, 0.5))
    assert g.voxel_center(0, 0, 0) == (-127.75, -127.75, -127.75)
    with pytest.raises(cb.OutOfRange):
        g.voxel_center(512, 0, 0)
    with pytest.raises(cb.InvalidArgument):
        cb.VolumeGeometry.make((0, 1, 1), (1, 1, 1))
    with pytest.raises(cb.InvalidArgument):
        cb.VolumeGeometry.make((1, 1, 1), (0.0, 1, 1))
    with pytest.raises(cb.InvalidArgument):
        cb.DetectorGeometry.make(0, 4, 1, 1)
    with pytest.raises(cb.InvalidArgument):
        cb.DetectorGeometry.make(4, 4, -1, 1)


def test_circular_trajectory_spacing():
    det = cb.DetectorGeometry.make(128, 128, 1.0, 1.0)
    views = cb.make_circular_trajectory(541.0, 949.0, 720, 360.0, det)
    s = views[1].source()
    assert s[0] == pytest.approx(541.0 * math.cos(0.5 * math.pi / 180.0), rel=1e-14)
    assert s[1] == pytest.approx(541.0 * math.sin(0.5 * math.pi / 180.0), rel=1e-14)
    assert s[2] == 0.0
    views = cb.make_circular_trajectory(750.0, 1000.0, 100, 198.0, det)
    last = math.degrees(math.atan2(views[99].source()[1], views[99].source()[0]))
    assert last == pytest.approx(198.0 - 360.0, rel=1e-12)
    for v in cb.make_circular_trajectory(541.0, 949.0, 8, 360.0, det):
        ew = v.frame()[2]
        want = -np.asarray(v.source()) / np.linalg.norm(v.source())
        assert float(ew @ want) == pytest.approx(1.0, rel=1e-14)
        assert v.frame()[1][2] == -1.0
        assert v.focal_length() == 949.0
    for args in ((541, 949, 0, 360), (541, 949, 4, 0.0), (-1, 949, 4, 360)):
        with pytest.raises(cb.InvalidArgument):
            cb.make_circular_trajectory(*args, det)


def test_view_frame_validation():
    s, b = (541, 0, 0), (1.0, 1.0)
    cb.ViewGeometry.make(s, [[0, 1, 0], [0, 0, -1], [-1, 0, 0]], 949.0, (63.5, 63.5), b)
    for bad in ([[0, -1, 0], [0, 0, 1], [-1, 0, 0]],      # chi2 up
                [[0, -1, 0], [0, 0, -1], [-1, 0, 0]],     # left-handed
                [[0, 1, 1e-6], [0, 0, -1], [-1, 0, 0]]):  # skew
        with pytest.raises(cb.InvalidArgument):
            cb.ViewGeometry.make(s, bad, 949.0, (63.5, 63.5), b)


def _project_3x4(P, x):
    h = P @ np.append(x, 1.0)
    return h[0] / h[2], h[1] / h[2]


def test_projection_matches_the_standard_matrix():
    det = cb.DetectorGeometry.make(128, 128, 1.0, 1.0)
    v = cb.make_circular_trajectory(541.0, 949.0, 5, 360.0, det)[0]
    P = v.standard_matrix()
    rng = np.random.default_rng(5)
    for _ in range(200):
        x = (rng.random(3) - 0.5) * np.array([200.0, 200.0, 100.0])
        chi = v.project_point(x)
        ref = _project_3x4(P, x)
        assert chi[0] == pytest.approx(ref[0], rel=1e-12)
        assert chi[1] == pytest.approx(ref[1], rel=1e-12)
    c = v.project_point((0, 0, 0))
    assert c == pytest.approx((63.5, 63.5), rel=1e-13)
    with pytest.raises(cb.DomainError):
        v.project_point((1000.0, 0.0, 0.0))
    assert v.depth((0, 0, 0)) == pytest.approx(541.0)


def test_standard_matrix_factorization_roundtrip():
    det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
    views = cb.make_circular_trajectory(749.0, 1198.0, 12, 360.0, det)
    rng = np.random.default_rng(9)
    for v in views:
        back = cb.ViewGeometry.from_standard_matrix(v.standard_matrix(), det.pixel_size())
        assert np.linalg.norm(np.subtract(back.source(), v.source())) < 1e-9
        assert back.focal_length() == pytest.approx(v.focal_length(), rel=1e-12)
        assert back.principal_point() == pytest.approx(v.principal_point(), rel=1e-10)
        for _ in range(20):
            x = (rng.random(3) - 0.5) * 100.0
            assert back.project_point(x) == pytest.approx(v.project_point(x), rel=1e-10)
    P = views[3].standard_matrix() * -7.25
    back = cb.ViewGeometry.from_standard_matrix(P, det.pixel_size())
    assert np.linalg.norm(np.subtract(back.source(), views[3].source())) < 1e-9
    assert back.focal_length() == pytest.approx(views[3].focal_length(), rel=1e-12)


def test_camera_matrix_text_roundtrip(tmp_path):
    det = cb.DetectorGeometry.make(128, 128, 1.0, 1.0)
    views = cb.make_circular_trajectory(541.0, 949.0, 36, 360.0, det)
    path = str(tmp_path / "m.txt")
    cb.write_camera_matrices(path, views)
    back = cb.read_camera_matrices(path, det.pixel_size())
    assert len(back) == len(views)
    for a, b in zip(back, views):
        assert np.linalg.norm(np.subtract(a.source(), b.source())) < 1e-9
        assert a.focal_length() == pytest.approx(b.focal_length(), rel=1e-12)
    with open(path, "a") as f:
        f.write("# trailing comment\n")
    assert len(cb.read_camera_matrices(path, det.pixel_size())) == len(views)
    with open(path, "a") as f:
        f.write("1 2 3\n")
    with pytest.raises(cb.CvpbRuntimeError):
        cb.read_camera_matrices(path, det.pixel_size())


def test_pixel_scale_cos_known_answers():
    """test_cvp.cpp:251-279"""
    det = cb.DetectorGeometry.make(127, 127, 1.0, 1.0)
    v = cb.make_circular_trajectory(541.0, 949.0, 1, 360.0, det)[0]
    assert cb.pixel_scale_cos(v, det, 63, 63) == pytest.approx(949.0 ** 2, rel=1e-12)
    det5 = cb.DetectorGeometry.make(5, 5, 1.0, 1.0)
    v5 = cb.ViewGeometry.make((10.0, 0.0, 0.0), [[0, 1, 0], [0, 0, -1], [-1, 0, 0]],
                              2.0 / math.sqrt(3.0), (2.0, 2.0), (1.0, 1.0))
    assert (cb.pixel_scale_cos(v5, det5, 2, 4) / cb.pixel_scale_cos(v5, det5, 2, 2)
            == pytest.approx(8.0, rel=1e-12))
    detc = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
    vc = cb.make_circular_trajectory(749.0, 1198.0, 1, 360.0, detc)[0]
    corner = np.subtract(vc.detector_point((0.0, 0.0)), vc.source())
    axis = np.subtract(vc.detector_point(vc.principal_point()), vc.source())
    cos_t = corner @ axis / (np.linalg.norm(corner) * np.linalg.norm(axis))
    want = vc.focal_length() ** 2 / (detc.pixel_area() * cos_t ** 3)
    assert cb.pixel_scale_cos(vc, detc, 0, 0) == pytest.approx(want, rel=1e-12)
    with pytest.raises(cb.OutOfRange):
        cb.pixel_scale_cos(vc, detc, 480, 0)


def test_pixel_scale_exact_against_reference_and_cos():
    """test_cvp.cpp:298-317 + the reference's own values (golden)."""
    g = np.load(GOLD)
    det = cb.DetectorGeometry.make(480, 616, 0.154, 0.154)
    v = cb.ViewGeometry.from_array(g["carm_views"][3])
    for (m, n), ex, co in zip(g["carm_scale_px"], g["carm_scale_exact"], g["carm_scale_cos"]):
        assert cb.pixel_scale_exact(v, det, int(m), int(n)) == pytest.approx(ex, rel=1e-6)
        assert cb.pixel_scale_cos(v, det, int(m), int(n)) == pytest.approx(co, rel=1e-13)
    for m, n in ((240, 308), (0, 0)):
        c, e = cb.pixel_scale_cos(v, det, m, n), cb.pixel_scale_exact(v, det, m, n)
        assert abs(c / e - 1.0) < 1e-3


def test_fill_uniform01_matches_reference_stream():
    g = np.load(GOLD)
    assert np.array_equal(cb.fill_uniform01(16, 7), g["rng_seed7_first16"])


def test_shepp_logan_phantom_is_deterministic():
    from paper_2110_09841_b200.phantom import shepp_logan_3d
    geom = cb.VolumeGeometry.make((32, 32, 32), (1.0, 1.0, 1.0))
    a, b = shepp_logan_3d(geom), shepp_logan_3d(geom)
    assert np.array_equal(a, b)
    assert a.max() == pytest.approx(1.0) and a.min() >= -1e-12
    assert 0.1 < float((a > 0).mean()) < 0.7
