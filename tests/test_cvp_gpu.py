"""GPU parity of the CVP pair against the CPU checker (the reference compiled
from /root/reference when available, else the C restatement).

Tolerances (north star, stated here): exact AND relaxed mode vs reference
Double — rel-L2 <= 1e-5 and max|d|/max|ref| <= 1e-4 on float32 outputs (the
reference's own Single-vs-Double bound, per-view rel-Frobenius <= 1e-3 of
test_cvp.cpp:434-458, is far looser).
"""
import numpy as np
import pytest

from conftest import make_case, max_rel, rel_l2

pytestmark = pytest.mark.gpu

EXACT_L2, EXACT_MAX = 1e-5, 1e-4


def _torch_vol(x64, geom):
    import torch
    return torch.from_numpy(np.asarray(x64, dtype=np.float32)).reshape(geom.shape()).cuda()


def _torch_stack(p64, n_views, det):
    import torch
    return torch.from_numpy(np.asarray(p64, dtype=np.float32)).reshape(n_views, det.rows,
                                                                      det.cols).cuda()


def _np(t):
    return t.double().cpu().numpy()


def _opts(scaling, elev, precision, rest):
    import paper_2110_09841_b200 as cb
    return cb.CvpOptions(cb.PixelScaling(scaling), bool(elev), cb.CvpPrecision(precision),
                         cb.RadiusEstimate(rest))


def _run_pair(checker, counts, voxel, rows, cols, pw, ph, sid, sdd, nv, opts4, x64=None, b64=None,
              arc=360.0, threads=0):
    import paper_2110_09841_b200 as cb
    geom, det, views, sc = make_case(counts, voxel, rows, cols, pw, ph, sid, sdd, nv, arc)
    if x64 is None:
        x64 = cb.fill_uniform01(geom.voxel_count(), 7)
    if b64 is None:
        b64 = cb.fill_uniform01(det.pixel_count() * nv, 8)
    # the device computes on float32 inputs: give the checker the same values
    x32 = np.asarray(x64, dtype=np.float32).astype(np.float64)
    b32 = np.asarray(b64, dtype=np.float32).astype(np.float64)
    scene = cb.DeviceScene(geom, det, views)
    opts = _opts(*opts4)
    p = _np(scene.project_cvp(_torch_vol(x32, geom), opts=opts))
    bp = _np(scene.backproject_cvp(_torch_stack(b32, nv, det), opts=opts))
    p_ref = checker.project_cvp(sc, x32, opts4, threads=threads)
    bp_ref = checker.backproject_cvp(sc, b32, opts4, threads=threads)
    return p, p_ref, bp.reshape(bp_ref.shape), bp_ref, scene


ALL_COMBOS = [(s, e, 0, r) for s in (0, 1) for e in (0, 1) for r in (0, 1)]


@pytest.mark.parametrize("opts4", ALL_COMBOS)
def test_exact_all_option_combos(checker, opts4):
    """Scene of test_cvp.cpp:349-373 (16^3, 32^2, 8 views, SID 40 / SDD 70)."""
    p, p_ref, bp, bp_ref, _ = _run_pair(checker, (16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0,
                                        40.0, 70.0, 8, opts4)
    assert rel_l2(p, p_ref) <= EXACT_L2 and max_rel(p, p_ref) <= EXACT_MAX, (
        rel_l2(p, p_ref), max_rel(p, p_ref))
    assert rel_l2(bp, bp_ref) <= EXACT_L2 and max_rel(bp, bp_ref) <= EXACT_MAX, (
        rel_l2(bp, bp_ref), max_rel(bp, bp_ref))


def test_c1_shepp_logan_exact(checker):
    """configs[0]: exact CVP P+BP, 64^3 Shepp-Logan, 64x64 detector, 36 views."""
    import paper_2110_09841_b200 as cb
    from paper_2110_09841_b200.phantom import shepp_logan_3d
    geom = cb.VolumeGeometry.make((64, 64, 64), (0.5, 0.5, 0.5))
    x64 = shepp_logan_3d(geom)
    p, p_ref, bp, bp_ref, _ = _run_pair(checker, (64, 64, 64), (0.5, 0.5, 0.5), 64, 64, 1.0, 1.0,
                                        541.0, 949.0, 36, (1, 1, 0, 1), x64=x64)
    assert rel_l2(p, p_ref) <= EXACT_L2, rel_l2(p, p_ref)
    assert max_rel(p, p_ref) <= EXACT_MAX, max_rel(p, p_ref)
    assert rel_l2(bp, bp_ref) <= EXACT_L2, rel_l2(bp, bp_ref)
    assert max_rel(bp, bp_ref) <= EXACT_MAX, max_rel(bp, bp_ref)


def test_carm_fine_pixels_exact_beats_reference_single(checker):
    """at 0.72 mm voxels / 0.154 mm pixels the reference's own float
    path misses 1e-5 rel-L2 (6e-5). The exact device path must hold 1e-5."""
    p, p_ref, bp, bp_ref, _ = _run_pair(checker, (64, 64, 64), (0.72, 0.72, 0.72), 480, 616, 0.154,
                                        0.154, 749.0, 1198.0, 6, (1, 1, 0, 1))
    assert rel_l2(p, p_ref) <= EXACT_L2, rel_l2(p, p_ref)
    assert max_rel(p, p_ref) <= EXACT_MAX, max_rel(p, p_ref)
    assert rel_l2(bp, bp_ref) <= EXACT_L2, rel_l2(bp, bp_ref)
    assert max_rel(bp, bp_ref) <= EXACT_MAX, max_rel(bp, bp_ref)


def test_c2_geometry_tall_voxels_exact(checker):
    """configs[1] geometry (0.18 mm voxels, 0.154 mm C-arm pixels, SID 749 /
    SDD 1198): voxels ~1.9 detector rows tall, so the launch takes the
    three-straight-line-row walk; exact parity with the reference Double."""
    p, p_ref, bp, bp_ref, scene = _run_pair(checker, (96, 96, 96), (0.18, 0.18, 0.18), 480, 616,
                                            0.154, 0.154, 749.0, 1198.0, 4, (1, 1, 0, 1), arc=200.0)
    assert rel_l2(p, p_ref) <= EXACT_L2 and max_rel(p, p_ref) <= EXACT_MAX, (
        rel_l2(p, p_ref), max_rel(p, p_ref))
    assert rel_l2(bp, bp_ref) <= EXACT_L2 and max_rel(bp, bp_ref) <= EXACT_MAX, (
        rel_l2(bp, bp_ref), max_rel(bp, bp_ref))


def test_large_cone_angle_exact(checker):
    """configs[3]-style short SID/SDD (300/500), 1 mm pixels, 0.5 mm voxels."""
    p, p_ref, bp, bp_ref, _ = _run_pair(checker, (48, 48, 48), (0.5, 0.5, 0.5), 128, 128, 1.0, 1.0,
                                        300.0, 500.0, 6, (1, 1, 0, 1))
    assert rel_l2(p, p_ref) <= EXACT_L2 and max_rel(p, p_ref) <= EXACT_MAX
    assert rel_l2(bp, bp_ref) <= EXACT_L2 and max_rel(bp, bp_ref) <= EXACT_MAX


@pytest.mark.parametrize("opts4", [(1, 1, 1, 1), (0, 0, 1, 0), (1, 0, 1, 1), (0, 1, 1, 0)])
def test_relaxed_meets_the_exact_bar(checker, opts4):
    """Relaxed (Single) device results against the reference DOUBLE at the
    north-star bar (rel-L2 <= 1e-5, max <= 1e-4) — the device's float32 path is
    offset-stable, so it does not inherit the reference Single's ~5e-5 gap
    (that gap is reported, not gated: profiles/parity_*.md)."""
    exact4 = (opts4[0], opts4[1], 0, opts4[3])
    for case in (((64, 64, 64), (0.5, 0.5, 0.5), 128, 128, 1.0, 1.0, 541.0, 949.0, 6),
                 ((64, 64, 64), (0.72, 0.72, 0.72), 480, 616, 0.154, 0.154, 749.0, 1198.0, 4)):
        p, _, bp, _, _ = _run_pair(checker, *case, opts4)
        _, p_ref, _, bp_ref, _ = _run_pair(checker, *case, exact4)
        assert rel_l2(p, p_ref) <= EXACT_L2 and max_rel(p, p_ref) <= EXACT_MAX, (
            case, rel_l2(p, p_ref), max_rel(p, p_ref))
        assert rel_l2(bp, bp_ref) <= EXACT_L2 and max_rel(bp, bp_ref) <= EXACT_MAX, (
            case, rel_l2(bp, bp_ref), max_rel(bp, bp_ref))
        for v in range(p.shape[0]):  # and per view (test_cvp.cpp:434-458 shape)
            assert rel_l2(p[v], p_ref[v]) <= 1e-4


def test_adjoint_identity_device():
    """<A x, y> vs <x, A^T y> on the device (compensated float64 dots)."""
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((32, 32, 32), (1.0, 1.0, 1.0), 48, 48, 1.0, 1.0, 60.0, 100.0,
                                    12)
    scene = cb.DeviceScene(geom, det, views)
    for prec in (cb.CvpPrecision.Double, cb.CvpPrecision.Single):
        pair = cb.cvp_pair(scene, cb.CvpOptions(precision=prec))
        for seed in (1, 2, 3):
            d = cb.adjoint_test(pair, seed)
            assert d < 1e-5, (prec, seed, d)


def test_cut_records_match_reference(reference):
    """Device geometry code vs collect_cut_records (cvp.cpp:652-689)."""
    import paper_2110_09841_b200 as cb
    geom, det, views, sc = make_case((64, 64, 64), (0.5, 0.5, 0.5), 128, 128, 1.0, 1.0, 541.0,
                                     949.0, 36)
    scene = cb.DeviceScene(geom, det, views)
    rng = np.random.default_rng(17)
    for trial in range(40):
        i, j, k = (int(t) for t in rng.integers(0, 64, 3))
        v = int(rng.integers(0, 36))
        for opts4 in ((1, 1, 0, 1), (1, 0, 0, 1), (1, 1, 0, 0)):
            recs = scene.collect_cut_records(_opts(*opts4), v, i, j, k, clamp=False)
            rr, rc, rv, ri = reference.collect_cut_records(sc, sc.views[v], opts4, i, j, k)
            got = {(r.row, r.column): (r.volume, r.inv_r2) for r in recs}
            ref = {(int(a), int(b)): (c, d) for a, b, c, d in zip(rr, rc, rv, ri)}
            # records below 1e-6 of the voxel volume may appear/disappear on rounding
            big = {key for key, (vol, _) in ref.items() if vol > 1e-6 * 0.125}
            assert big <= set(got), (trial, opts4, big - set(got))
            for key in big:
                assert abs(got[key][0] - ref[key][0]) <= 1e-6 * 0.125
                assert abs(got[key][1] / ref[key][1] - 1.0) <= 1e-6
            assert abs(sum(x[0] for x in got.values()) - 0.125) <= 1e-7


def test_zero_volume_gives_zero_projection():
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, 40.0, 70.0, 4)
    scene = cb.DeviceScene(geom, det, views)
    p = scene.project_cvp(scene.new_volume())
    assert torch.count_nonzero(p).item() == 0


def test_linearity():
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, 40.0, 70.0, 4)
    scene = cb.DeviceScene(geom, det, views)
    x = _torch_vol(cb.fill_uniform01(geom.voxel_count(), 3), geom)
    p1 = scene.project_cvp(x)
    p2 = scene.project_cvp(2 * x)
    assert rel_l2(_np(p2), 2 * _np(p1)) < 1e-6


def test_rejects_unsupported_configurations():
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(32, 32, 1.0, 1.0)
    geom = cb.VolumeGeometry.make((16, 16, 16), (1.0, 1.0, 1.0))
    inside = cb.make_circular_trajectory(4.0, 70.0, 1, 360.0, det)
    scene = cb.DeviceScene(geom, det, inside)
    with pytest.raises(cb.CvpbRuntimeError):
        scene.project_cvp(scene.new_volume())
    other = cb.DetectorGeometry.make(32, 32, 0.5, 1.0)
    views = cb.make_circular_trajectory(40.0, 70.0, 1, 360.0, det)
    scene2 = cb.DeviceScene(geom, other, views)
    with pytest.raises(cb.InvalidArgument):
        scene2.project_cvp(scene2.new_volume())


def test_host_path_matches_device_path():
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((32, 32, 32), (1.0, 1.0, 1.0), 48, 48, 1.0, 1.0, 60.0, 100.0, 5)
    x64 = cb.fill_uniform01(geom.voxel_count(), 11)
    vol = cb.AttenuationVolume(geom, x64)
    p_host = cb.project_cvp(vol, views, det)
    scene = cb.scene_for(geom, det, views)
    p_dev = _np(scene.project_cvp(_torch_vol(x64, geom)))
    assert rel_l2(p_host.values, p_dev) < 1e-6
    b_host = cb.backproject_cvp(p_host, views, geom)
    b_dev = _np(scene.backproject_cvp(scene.project_cvp(_torch_vol(x64, geom))))
    assert rel_l2(b_host.values, b_dev) < 1e-6


def test_host_path_view_chunks_match_device_path():
    # >= 32 views: the host path pipelines its stack transfers over view
    # chunks (copy stream) and backprojects the chunks with accumulation
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((24, 20, 28), (1.0, 1.0, 1.0), 40, 36, 1.0, 1.0, 60.0, 100.0, 37)
    x64 = cb.fill_uniform01(geom.voxel_count(), 12)
    vol = cb.AttenuationVolume(geom, x64)
    p_host = cb.project_cvp(vol, views, det)
    scene = cb.scene_for(geom, det, views)
    p_dev = _np(scene.project_cvp(_torch_vol(x64, geom)))
    assert rel_l2(p_host.values, p_dev) < 1e-6
    b_host = cb.backproject_cvp(p_host, views, geom)
    b_dev = _np(scene.backproject_cvp(scene.project_cvp(_torch_vol(x64, geom))))
    assert rel_l2(b_host.values, b_dev) < 1e-6


@pytest.mark.parametrize("n_views", [5, 37])
def test_host_path_pinned_buffers_match_pageable(n_views):
    # pinned float64 host buffers take the zero-copy route (the forward
    # stages bricks straight from the host volume, the backward's last view
    # chunk writes the float64 result in place); same results up to the
    # float atomic merge order of view groups (small scenes)
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((24, 20, 28), (1.0, 1.0, 1.0), 40, 36, 1.0, 1.0, 60.0, 100.0,
                                    n_views)
    scene = cb.DeviceScene(geom, det, views)
    x64 = cb.fill_uniform01(geom.voxel_count(), 13)
    b64 = cb.fill_uniform01(det.pixel_count() * n_views, 14)
    xp = torch.from_numpy(x64).pin_memory()
    bp = torch.from_numpy(b64).pin_memory()
    pp = torch.zeros(det.pixel_count() * n_views, dtype=torch.float64).pin_memory()
    vp = torch.zeros(geom.voxel_count(), dtype=torch.float64).pin_memory()
    for _ in range(2):  # the second pass reuses the context's host-path buffers
        scene.project_cvp_host(xp.numpy(), pp.numpy())
        scene.backproject_cvp_host(bp.numpy(), vp.numpy())
        p_ref = scene.project_cvp_host(np.array(x64))
        v_ref = scene.backproject_cvp_host(np.array(b64))
        assert rel_l2(pp.numpy(), p_ref) < 1e-6
        assert rel_l2(vp.numpy(), v_ref) < 1e-6


def test_scale_images_match_reference(reference):
    import paper_2110_09841_b200 as cb
    geom, det, views, sc = make_case((8, 8, 8), (1.0, 1.0, 1.0), 480, 616, 0.154, 0.154, 749.0,
                                     1198.0, 2)
    scene = cb.DeviceScene(geom, det, views)
    for exact in (0, 1):
        img = scene.scale_image(1, exact=bool(exact))
        for m, n in ((0, 0), (240, 308), (479, 615), (100, 500)):
            want = reference.pixel_scale(sc, sc.views[1], exact, m, n)
            assert abs(img[m, n] / want - 1.0) < 1e-7


def test_view_chunks_and_accumulate_compose():
    """Backprojection of view chunks with accumulate=1 equals one launch."""
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((32, 32, 32), (1.0, 1.0, 1.0), 48, 48, 1.0, 1.0, 60.0, 100.0, 10)
    scene = cb.DeviceScene(geom, det, views)
    b = _torch_stack(cb.fill_uniform01(det.pixel_count() * 10, 5), 10, det)
    full = scene.backproject_cvp(b)
    part = scene.backproject_cvp(b[:4].contiguous(), view_begin=0, view_count=4)
    scene.backproject_cvp(b[4:].contiguous(), out=part, view_begin=4, view_count=6, accumulate=True)
    assert rel_l2(_np(part), _np(full)) < 1e-6
    p_full = scene.project_cvp(full)
    p_part = scene.project_cvp(full, view_begin=3, view_count=5)
    assert rel_l2(_np(p_part), _np(p_full)[3:8]) < 1e-6


def test_cut_table_view_chunks_match_single_chunk(checker, monkeypatch):
    """A cut table too small for the launch splits it into view chunks (c5
    at full size takes two); chunked P / BP match the reference and the
    single-chunk launch."""
    import paper_2110_09841_b200 as cb
    counts, nv = (24, 20, 28), 37
    per_view = counts[0] * counts[1] * 144
    p1, p_ref, b1, b_ref, _ = _run_pair(checker, counts, (1.0, 1.0, 1.0), 40, 36, 1.0, 1.0, 60.0,
                                        100.0, nv, (1, 1, 0, 1))
    monkeypatch.setenv("CVPB_CUT_TABLE_MAX_BYTES", str(5 * per_view))  # 8 chunks of <= 5 views
    p8, _, b8, _, _ = _run_pair(checker, counts, (1.0, 1.0, 1.0), 40, 36, 1.0, 1.0, 60.0, 100.0,
                                nv, (1, 1, 0, 1))
    for got in (p1, p8):
        assert rel_l2(got, p_ref) <= EXACT_L2 and max_rel(got, p_ref) <= EXACT_MAX
    for got in (b1, b8):
        assert rel_l2(got, b_ref) <= EXACT_L2 and max_rel(got, b_ref) <= EXACT_MAX
    assert rel_l2(p8, p1) < 1e-6 and rel_l2(b8, b1) < 1e-6


def test_cut_table_reuse_follows_options_views_and_streams():
    """The context keeps the cut table of its last single-chunk launch and
    reuses it for the same views and options (the P and BP of a CGLS
    iteration). Switching options or views must recompute it, and launches on
    different streams are ordered on the shared table."""
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((24, 20, 40), (1.0, 1.0, 1.0), 40, 36, 1.0, 1.0, 60.0, 100.0, 9)
    x = torch.rand(geom.shape(), device="cuda")
    y = torch.rand((9, 36, 40), device="cuda")
    combos = [cb.CvpOptions(), cb.CvpOptions(precision=cb.CvpPrecision.Single),
              cb.CvpOptions(elevation_correction=False), cb.CvpOptions()]
    fresh = []
    for o in combos:
        sc = cb.DeviceScene(geom, det, views)
        fresh.append((sc.project_cvp(x, opts=o), sc.backproject_cvp(y, opts=o),
                      sc.project_cvp(x, opts=o, view_begin=3, view_count=4)))
    scene = cb.DeviceScene(geom, det, views)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for o, (p_ref, b_ref, ps_ref) in zip(combos, fresh):
        with torch.cuda.stream(s1):
            p = scene.project_cvp(x, opts=o, stream=s1)
        with torch.cuda.stream(s2):
            b = scene.backproject_cvp(y, opts=o, stream=s2)
        ps = scene.project_cvp(x, opts=o, view_begin=3, view_count=4)
        torch.cuda.synchronize()
        assert rel_l2(p.cpu().numpy(), p_ref.cpu().numpy()) < 1e-6
        assert rel_l2(b.cpu().numpy(), b_ref.cpu().numpy()) < 1e-6
        assert rel_l2(ps.cpu().numpy(), ps_ref.cpu().numpy()) < 1e-6
