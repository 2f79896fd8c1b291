"""GPU: device-resident CGLS (solver.cpp:55-106) and the operator plug."""
import numpy as np
import pytest

from conftest import make_case

pytestmark = pytest.mark.gpu


def test_cgls_matches_reference_history(reference):
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, sc = make_case((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, 40.0, 70.0, 8)
    b = cb.fill_uniform01(det.pixel_count() * 8, 8).astype(np.float32).astype(np.float64)
    scene = cb.DeviceScene(geom, det, views)
    x, res = scene.cgls(torch.from_numpy(b.astype(np.float32)).reshape(8, 32, 32).cuda(), 6)
    x_ref, res_ref = reference.cgls(sc, b, 6)
    np.testing.assert_allclose(res, res_ref, rtol=1e-5)
    xr = x.double().cpu().numpy().ravel()
    assert np.linalg.norm(xr - x_ref.ravel()) <= 1e-4 * np.linalg.norm(x_ref)


def test_cgls_consistent_system_converges_monotonically():
    """test_solver.cpp:120-141: Gaussian blob, 60 views; residual monotone
    (float32 iterates: within 1e-6 of ||b||) and below 1e-3 ||b|| in 40 iterations."""
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, 40.0, 70.0, 60)
    scene = cb.DeviceScene(geom, det, views)
    k, j, i = np.meshgrid(np.arange(16), np.arange(16), np.arange(16), indexing="ij")
    blob = np.exp(-((i - 7.5) ** 2 + (j - 7.5) ** 2 + (k - 7.5) ** 2) / 18.0)
    xt = torch.from_numpy(blob.astype(np.float32)).cuda()
    b = scene.project_cvp(xt)
    for r in (cb.cgls(cb.cvp_pair(scene), cb.ProjectionStack(det, 60, b), 40),
              cb.CglsResult(None, scene.cgls(b, 40)[1])):
        res = np.array(r.residual_norms)
        assert np.all(np.diff(res) <= 1e-6 * res[0])
        assert res[-1] < 1e-3 * res[0]


def test_generic_pair_cgls_zero_data_and_breakdown():
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((8, 8, 8), (1.0, 1.0, 1.0), 16, 16, 1.0, 1.0, 40.0, 70.0, 2)
    # identity-like scalar pair through the generic (callable) path
    pair = cb.LinearOperatorPair(
        forward=lambda x, out: out.values.view(-1)[: x.values.numel()].copy_(x.values.view(-1) * 3.0),
        adjoint=lambda b, out: out.values.view(-1).copy_(b.values.view(-1)[: out.values.numel()] * 3.0),
        vol_geom=geom, det=det, n_views=2)
    zero = cb.ProjectionStack(det, 2, torch.zeros((2, 16, 16), device="cuda"))
    r = cb.cgls(pair, zero, 3)
    assert r.residual_norms == [0.0, 0.0, 0.0, 0.0]
    dead = cb.LinearOperatorPair(forward=lambda x, out: out.values.zero_(),
                                 adjoint=lambda b, out: out.values.fill_(1.0),
                                 vol_geom=geom, det=det, n_views=2)
    one = cb.ProjectionStack(det, 2, torch.ones((2, 16, 16), device="cuda"))
    with pytest.raises(cb.CvpbRuntimeError):
        cb.cgls(dead, one, 2)


def test_vector_ops_against_float64():
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((8, 8, 8), (1.0, 1.0, 1.0), 16, 16, 1.0, 1.0, 40.0, 70.0, 2)
    scene = cb.DeviceScene(geom, det, views)
    g = torch.Generator().manual_seed(3)
    a = torch.rand(1_000_003, generator=g).cuda()
    b = torch.rand(1_000_003, generator=g).cuda()
    want = float(torch.dot(a.double(), b.double()))
    assert scene.dot(a, b) == pytest.approx(want, rel=1e-13)
    y = b.clone()
    scene.axpy(0.25, a, y)
    assert torch.allclose(y, b + 0.25 * a)
    p = b.clone()
    scene.xpby(a, 0.5, p)
    assert torch.allclose(p, a + 0.5 * b)
    assert scene.all_finite(a)
    a[17] = float("nan")
    assert not scene.all_finite(a)


def test_multi_view_group_backprojection_matches_single_group():
    """Small volumes split views across CTA groups (atomic volume merge); the
    deterministic policy keeps one group — both agree to float32 rounding."""
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((32, 32, 32), (1.0, 1.0, 1.0), 48, 48, 1.0, 1.0, 60.0, 100.0, 24)
    scene = cb.DeviceScene(geom, det, views)
    b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * 24, 2).astype(np.float32)).reshape(
        24, 48, 48).cuda()
    a = scene.backproject_cvp(b)
    d = scene.backproject_cvp(b, exec=cb.ExecPolicy(deterministic=True))
    d2 = scene.backproject_cvp(b, exec=cb.ExecPolicy(deterministic=True))
    assert torch.equal(d, d2)
    assert float((a - d).norm() / d.norm()) < 1e-6


def test_os_sart_reconstructs_the_blob():
    """OS-SART with 1 and 6 subsets: the error to the true
    volume falls monotonically in the first iterations and ordered subsets
    converge faster per iteration."""
    import torch
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((16, 16, 16), (1.0, 1.0, 1.0), 32, 32, 1.0, 1.0, 40.0, 70.0, 60)
    scene = cb.DeviceScene(geom, det, views)
    k, j, i = np.meshgrid(np.arange(16), np.arange(16), np.arange(16), indexing="ij")
    blob = torch.from_numpy(np.exp(-((i - 7.5) ** 2 + (j - 7.5) ** 2 + (k - 7.5) ** 2) / 18.0)
                            .astype(np.float32)).cuda()
    b = scene.project_cvp(blob)
    r1 = cb.os_sart(scene, b, 5, n_subsets=1)
    r6 = cb.os_sart(scene, b, 5, n_subsets=6)
    assert all(a >= c for a, c in zip(r1.residual_norms, r1.residual_norms[1:]))
    assert r6.residual_norms[0] < r1.residual_norms[0]
    err6 = float((r6.x - blob).norm() / blob.norm())
    assert err6 < 0.2
    rn = cb.os_sart(scene, b, 2, n_subsets=4, nonneg=True)
    assert float(rn.x.min()) >= 0.0


def test_scene_operator_distributed_cgls_single_rank_matches_device_cgls():
    """parallel.scene_operator + distributed_cgls (the bench's N > 1 CGLS path)
    on one rank, over the device scene and its vector kernels: same residual
    history as the device-resident cvpb_cgls."""
    import torch
    import paper_2110_09841_b200 as cb
    from paper_2110_09841_b200 import parallel as par
    geom, det, views, _ = make_case((16, 12, 20), (1.0, 1.0, 1.0), 32, 28, 1.0, 1.0, 40.0, 70.0, 9)
    scene = cb.DeviceScene(geom, det, views)
    b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * 9, 5).astype(np.float32)).reshape(
        9, 28, 32).cuda()
    op = par.scene_operator(scene)
    r = par.distributed_cgls(op, b, 5, par.SceneVec(scene))
    x, res = scene.cgls(b, 5)
    np.testing.assert_allclose(r.residual_norms, res, rtol=1e-5)
    xs = r.x_slab[: geom.voxel_count()].double().cpu().numpy()
    xd = x.double().cpu().numpy().ravel()
    assert np.linalg.norm(xs - xd) <= 1e-4 * np.linalg.norm(xd)
