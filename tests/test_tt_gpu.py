"""GPU: the TT (SF-TT, Long et al. 2010) pair. No reference code exists
(SPEC.md:8), so parity is unpinned; the operator is pinned by self-tests:
adjointness, linearity, footprint mass vs Siddon, accuracy vs high-K Siddon."""
import numpy as np
import pytest

from conftest import make_case

pytestmark = pytest.mark.gpu


def _scene(counts=(24, 24, 24), vox=(1.0, 1.0, 1.0), R=40, C=40, px=1.0, sid=60.0, sdd=100.0, nv=6):
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case(counts, vox, R, C, px, px, sid, sdd, nv)
    return cb, geom, det, views, cb.DeviceScene(geom, det, views)


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
