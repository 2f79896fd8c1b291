"""GPU regression tests for boundary semantics: cut-table reuse after a
reallocation, CGLS running the pair's own operator (TT amplitude, ExecPolicy),
buffer size / device validation, and the device CGLS's early exits."""
import numpy as np
import pytest

from conftest import make_case, rel_l2

pytestmark = pytest.mark.gpu


def _scene(nv=64, n=24):
    import paper_2110_09841_b200 as cb
    geom, det, views, _ = make_case((n, n, n), (1.0, 1.0, 1.0), 40, 40, 1.0, 1.0, 60.0, 100.0, nv)
    return cb, geom, det, views, cb.DeviceScene(geom, det, views)


def test_cut_table_reallocation_invalidates_its_key(monkeypatch):
    """A device launch on views [0, 16) leaves a table keyed to them; a host
    call over all 64 views that forces the table to be re-allocated (and not
    to fit in one piece) must not trust the old key for its first chunk."""
    import torch
    cb, geom, det, views, scene = _scene()
    x = torch.from_numpy(cb.fill_uniform01(geom.voxel_count(), 3).astype(np.float32)).reshape(
        geom.shape()).cuda()
    full = scene.project_cvp(x).double().cpu().numpy()
    scene.project_cvp(x, view_begin=0, view_count=16)
    per_view = geom.counts[0] * geom.counts[1] * 144
    monkeypatch.setenv("CVPB_CUT_TABLE_MAX_BYTES", str(per_view * 20))
    out = scene.project_cvp_host(x.double().cpu().numpy().ravel())
    assert rel_l2(out.reshape(full.shape), full) < 1e-6


def test_tt_cgls_uses_the_pairs_amplitude():
    """Device CGLS of tt_pair(scene, TTOptions(amplitude=0)) equals the generic
    recurrence over the same pair's forward/adjoint."""
    import torch
    cb, geom, det, views, scene = _scene(nv=12, n=16)
    x = torch.from_numpy(cb.fill_uniform01(geom.voxel_count(), 4).astype(np.float32)).reshape(
        geom.shape()).cuda()
    for amp in (0, 1):
        pair = cb.tt_pair(scene, cb.TTOptions(amplitude=amp))
        b = scene.project_tt(x, opts=cb.TTOptions(amplitude=amp))
        dev = cb.cgls(pair, cb.ProjectionStack(det, len(views), b), 5)
        generic = cb.LinearOperatorPair(pair.forward, pair.adjoint, geom, det, len(views))
        ref = cb.cgls(generic, cb.ProjectionStack(det, len(views), b), 5)
        assert np.allclose(dev.residual_norms, ref.residual_norms, rtol=1e-4), (
            amp, dev.residual_norms, ref.residual_norms)
    # and the two amplitudes are different operators
    r0 = cb.cgls(cb.tt_pair(scene, cb.TTOptions(amplitude=0)), cb.ProjectionStack(det, 12, b), 3)
    r1 = cb.cgls(cb.tt_pair(scene, cb.TTOptions(amplitude=1)), cb.ProjectionStack(det, 12, b), 3)
    assert r0.residual_norms[-1] != r1.residual_norms[-1]


def test_siddon_cgls_honours_allow_expensive():
    import torch
    cb, geom, det, views, scene = _scene(nv=4, n=8)
    b = scene.new_stack()
    with pytest.raises(cb.InvalidArgument):
        scene.cgls(b, 1, projector="siddon", k_per_edge=128)
    b += 1.0
    _, res = scene.cgls(b, 1, projector="siddon", k_per_edge=128,
                        exec=cb.ExecPolicy(allow_expensive=True))
    assert res[1] < res[0]


def test_device_buffers_are_validated():
    import torch
    cb, geom, det, views, scene = _scene(nv=8, n=16)
    short = torch.zeros(geom.voxel_count() - 1, device="cuda")
    with pytest.raises(cb.InvalidArgument):
        scene.project_cvp(short)
    with pytest.raises(cb.InvalidArgument):
        scene.project_cvp(scene.new_volume(), out=scene.new_stack(7))
    with pytest.raises(cb.InvalidArgument):
        scene.backproject_cvp(scene.new_stack(7))
    with pytest.raises(cb.InvalidArgument):
        scene.backproject_tt(scene.new_stack(), out=torch.zeros(10, device="cuda"))
    with pytest.raises(cb.InvalidArgument):
        scene.project_siddon(scene.new_volume().double(), 1)
    # a stack covering more than the launch's range is fine (it is the
    # caller's slice starting at view_begin)
    scene.project_cvp(scene.new_volume(), out=scene.new_stack(8), view_begin=2, view_count=4)


def test_device_cgls_flat_history_and_breakdown():
    import torch
    cb, geom, det, views, scene = _scene(nv=8, n=8)
    zero = scene.new_stack()
    x, res = scene.cgls(zero, 4)
    assert res == [0.0] * 5 and float(x.abs().max()) == 0.0
    # data the operator cannot see: A^T b = 0 for a stack that is nonzero only
    # on pixels no voxel projects to -> gamma = 0 -> flat history
    b = scene.new_stack()
    b[:, 0, 0] = 1.0  # detector corner: outside every footprint of this scene
    x, res = scene.cgls(b, 3)
    assert res[1:] == [res[0]] * 3


def test_view_seconds_attribute_the_call_time_by_view_work():
    """view_seconds (cvp.cpp:469-477): the device runs a launch's views at
    once, so the call's time is split by each view's cut count. The 45 deg
    views cut the voxel-column bases into more detector-column pieces than
    the axis-aligned ones: the weights must differ and sum to one, and both
    host calls must split their time by them."""
    import paper_2110_09841_b200 as cb
    det = cb.DetectorGeometry.make(64, 96, 1.0, 1.0)
    geom = cb.VolumeGeometry.make((48, 8, 16), (1.0, 1.0, 1.0))
    views = cb.make_circular_trajectory(120.0, 200.0, 8, 360.0, det)
    sc = cb.DeviceScene(geom, det, views)
    opts = cb.CvpOptions()
    w = sc.cvp_view_weights(opts)
    assert w.shape == (8,) and np.all(w > 0) and abs(w.sum() - 1.0) < 1e-12
    # every column has at least one cut; oblique views cut each column base
    # into more detector-column pieces than the axis-aligned ones
    assert w.max() / w.min() > 1.2
    assert min(w[1], w[3], w[5], w[7]) > max(w[0], w[2], w[4], w[6])
    x = cb.fill_uniform01(geom.voxel_count(), 3)
    vs = [0.0] * 8
    sc.project_cvp_host(x, opts=opts, view_seconds=vs)
    vs = np.array(vs)
    assert np.all(vs > 0)
    np.testing.assert_allclose(vs / vs.sum(), w, rtol=1e-9)
    vb = [0.0] * 8
    sc.backproject_cvp_host(sc.project_cvp_host(x, opts=opts), opts=opts, view_seconds=vb)
    np.testing.assert_allclose(np.array(vb) / sum(vb), w, rtol=1e-9)
    # sub-range weights are the range's own shares
    w2 = sc.cvp_view_weights(opts, view_begin=2, view_count=3)
    np.testing.assert_allclose(w2, w[2:5] / w[2:5].sum(), rtol=1e-12)
    sc.close()


def test_sync_reports_no_error_after_clean_device_calls():
    """cvpb_sync: device-path calls are asynchronous; a clean sequence
    reports nothing (and the context's own stream is accepted)."""
    import torch
    import paper_2110_09841_b200 as cb
    _, geom, _, _, sc = _scene(nv=8, n=16)
    x = torch.rand(geom.shape(), device="cuda")
    p = sc.project_cvp(x)
    sc.backproject_cvp(p)
    sc.synchronize()
    from paper_2110_09841_b200 import _native as N
    N.check(N.lib().cvpb_sync(sc._h, None))
    sc.close()
