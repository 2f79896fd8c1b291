"""GPU: the TT (SF-TT, Long et al. 2010) pair. The reference has no TT code
(SPEC.md:8); parity is pinned against the float64 restatement of the
published algorithm in oracle/tt_oracle.c (itself checked against the paper's
known answers in tests/test_tt_oracle.py) at the north-star bar — rel-L2
<= 1e-5 and max|d|/max|ref| <= 1e-4 — plus self-tests: adjointness,
linearity, footprint mass vs Siddon, accuracy vs high-K Siddon."""
import numpy as np
import pytest

from conftest import make_case

pytestmark = pytest.mark.gpu


def _scene(counts=(24, 24, 24), vox=(1.0, 1.0, 1.0), R=40, C=40, px=1.0, sid=60.0, sdd=100.0, nv=6):
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case(counts, vox, R, C, px, px, sid, sdd, nv)
    return cb, geom, det, views, cb.DeviceScene(geom, det, views)


TT_CASES = {
    # configs[0]: 64^3 Shepp-Logan box, 64x64 @1 mm, SID 541 / SDD 949
    "c1": ((64, 64, 64), (0.5, 0.5, 0.5), 64, 64, 1.0, 541.0, 949.0, 12),
    # configs[1] geometry: C-arm pixels (0.154 mm), 0.18 mm voxels, SID 749 / SDD 1198
    "c2": ((96, 96, 96), (0.18, 0.18, 0.18), 480, 616, 0.154, 749.0, 1198.0, 4),
    # configs[3] geometry: large cone angle, SID 300 / SDD 500, 1 mm pixels
    "c4": ((48, 48, 48), (0.5, 0.5, 0.5), 128, 128, 1.0, 300.0, 500.0, 6),
}


@pytest.mark.parametrize("case", sorted(TT_CASES))
@pytest.mark.parametrize("amplitude", [0, 1])
def test_tt_matches_the_sf_tt_oracle(case, amplitude, restatement):
    import torch
    from conftest import max_rel, rel_l2
    from oracle.pyoracle import Scene
    counts, vox, R, C, px, sid, sdd, nv = TT_CASES[case]
    cb, geom, det, views, scene = _scene(counts, vox, R, C, px, sid, sdd, nv)
    sc = Scene(counts, vox, R, C, px, px, cb.views_to_array(views))
    x = cb.fill_uniform01(geom.voxel_count(), 7).astype(np.float32)
    b = cb.fill_uniform01(det.pixel_count() * nv, 8).astype(np.float32)
    opts = cb.TTOptions(amplitude)
    p = scene.project_tt(torch.from_numpy(x).reshape(geom.shape()).cuda(), opts=opts)
    bp = scene.backproject_tt(torch.from_numpy(b).reshape(nv, R, C).cuda(), opts=opts)
    p_ref = restatement.project_tt(sc, x.astype(np.float64), amplitude)
    bp_ref = restatement.backproject_tt(sc, b.astype(np.float64), amplitude)
    got_p, got_bp = p.double().cpu().numpy(), bp.double().cpu().numpy()
    assert rel_l2(got_p, p_ref) <= 1e-5 and max_rel(got_p, p_ref) <= 1e-4, (
        rel_l2(got_p, p_ref), max_rel(got_p, p_ref))
    assert rel_l2(got_bp, bp_ref) <= 1e-5 and max_rel(got_bp, bp_ref) <= 1e-4, (
        rel_l2(got_bp, bp_ref), max_rel(got_bp, bp_ref))


@pytest.mark.parametrize("amplitude", [0, 1])
def test_tt_adjointness(amplitude):
    cb, geom, det, views, scene = _scene()
    pair = cb.tt_pair(scene, cb.TTOptions(amplitude))
    for seed in (1, 2):
        assert cb.adjoint_test(pair, seed) < 1e-5


def test_tt_linearity_and_zero():
    import torch
    cb, geom, det, views, scene = _scene()
    assert torch.count_nonzero(scene.project_tt(scene.new_volume())).item() == 0
    x = torch.from_numpy(cb.fill_uniform01(geom.voxel_count(), 3).astype(np.float32)).reshape(
        geom.shape()).cuda()
    p1 = scene.project_tt(x)
    p2 = scene.project_tt(3 * x)
    assert float((p2 - 3 * p1).norm() / p2.norm()) < 1e-6


def test_tt_footprint_mass_matches_siddon():
    """Sum over the detector of one voxel's line integrals (pixel units) equals
    vol * magnification^2 / pixel area for any exact projector; compare with
    Siddon K=16."""
    import torch
    cb, geom, det, views, scene = _scene((9, 9, 9), (1.0, 1.0, 1.0), 64, 64, 0.5, 60.0, 100.0, 4)
    x = scene.new_volume()
    x[4, 6, 3] = 1.0
    tt = scene.project_tt(x).double().sum(dim=(1, 2)).cpu().numpy()
    sid = scene.project_siddon(x, 16).double().sum(dim=(1, 2)).cpu().numpy()
    np.testing.assert_allclose(tt, sid, rtol=0.02)


def test_tt_accuracy_vs_high_k_siddon_large_cone():
    """configs[3]-style large cone angle: per-view error of TT and CVP against
    Siddon K=64 on a uniform block; both small, CVP at least as good."""
    import torch
    cb, geom, det, views, scene = _scene((16, 16, 16), (0.5, 0.5, 0.5), 96, 96, 1.0, 30.0, 50.0, 4)
    x = torch.ones(geom.shape(), device="cuda")
    ref = scene.project_siddon(x, 64, exec=cb.ExecPolicy(allow_expensive=True)).double().cpu().numpy()
    tt = scene.project_tt(x).double().cpu().numpy()
    cvp = scene.project_cvp(x).double().cpu().numpy()
    e_tt = [cb.relative_projector_error(tt[v], ref[v]) for v in range(4)]
    e_cvp = [cb.relative_projector_error(cvp[v], ref[v]) for v in range(4)]
    assert max(e_tt) < 5.0 and max(e_cvp) < 5.0
    assert np.mean(e_cvp) <= np.mean(e_tt) * 1.5
