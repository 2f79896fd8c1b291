"""GPU: randomized parity against the reference — random lattices, voxel and
pixel aspect ratios, detector sizes, source distances, arcs, view counts,
options, execution modes and brick shapes (tools/random_parity.py runs the
same generator at larger counts; profiles/random_parity_r01.md)."""
import numpy as np
import pytest

from conftest import max_rel, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(12))
def test_random_geometry_exact_parity(checker, monkeypatch, seed):
    import torch
    import paper_2110_09841_b200 as cb
    from oracle.pyoracle import Scene
    rng = np.random.default_rng(1000 + seed)
    counts = tuple(int(x) for x in rng.integers(5, 48, 3))
    vox = tuple(float(x) for x in rng.uniform(0.2, 1.5, 3))
    rows, cols = (int(x) for x in rng.integers(16, 120, 2))
    pw, ph = (float(x) for x in rng.uniform(0.3, 1.6, 2))
    ext = float(np.linalg.norm(np.array(counts) * np.array(vox)))
    sid = float(rng.uniform(0.6, 3.0) * ext + 5.0)
    sdd = float(sid * rng.uniform(1.2, 2.5))
    nv = int(rng.integers(1, 24))
    arc = float(rng.choice([360.0, 200.0, 90.0]))
    opts4 = (int(rng.integers(0, 2)), int(rng.integers(0, 2)), 0, int(rng.integers(0, 2)))
    ex = cb.ExecPolicy(deterministic=bool(rng.integers(0, 2)))
    monkeypatch.setenv("CVPB_CVP_SHAPE", str(int(rng.integers(0, 3))))
    det = cb.DetectorGeometry.make(rows, cols, pw, ph)
    geom = cb.VolumeGeometry.make(counts, vox)
    views = cb.make_circular_trajectory(sid, sdd, nv, arc, det)
    sc = Scene(counts, vox, rows, cols, pw, ph, cb.views_to_array(views))
    x = cb.fill_uniform01(geom.voxel_count(), 100 + seed).astype(np.float32).astype(np.float64)
    if seed % 3 == 0:
        x[rng.random(x.size) < 0.9] = 0.0
    b = cb.fill_uniform01(det.pixel_count() * nv, 200 + seed).astype(np.float32).astype(np.float64)
    scene = cb.DeviceScene(geom, det, views)
    o = cb.CvpOptions(cb.PixelScaling(opts4[0]), bool(opts4[1]), cb.CvpPrecision(0),
                      cb.RadiusEstimate(opts4[3]))
    p = scene.project_cvp(torch.from_numpy(x.astype(np.float32)).reshape(geom.shape()).cuda(), opts=o,
                          exec=ex).double().cpu().numpy()
    bp = scene.backproject_cvp(torch.from_numpy(b.astype(np.float32)).reshape(nv, rows, cols).cuda(),
                               opts=o, exec=ex).double().cpu().numpy()
    p_ref = checker.project_cvp(sc, x, opts4)
    bp_ref = checker.backproject_cvp(sc, b, opts4)
    if np.abs(p_ref).max() > 0:
        assert rel_l2(p, p_ref) <= 1e-5 and max_rel(p, p_ref) <= 1e-4, (rel_l2(p, p_ref), max_rel(p, p_ref))
    else:
        assert np.abs(p).max() == 0
    assert rel_l2(bp, bp_ref) <= 1e-5 and max_rel(bp, bp_ref) <= 1e-4, (rel_l2(bp, bp_ref), max_rel(bp, bp_ref))


def _random_scene(rng, max_n=40, odd=False):
    import paper_2110_09841_b200 as cb
    from oracle.pyoracle import Scene
    counts = tuple(int(x) for x in rng.integers(4, max_n, 3))
    if odd:  # no voxel-boundary plane through the rotation axis / central plane
        counts = tuple(c | 1 for c in counts)
    vox = tuple(float(x) for x in rng.uniform(0.3, 1.5, 3))
    rows, cols = (int(x) for x in rng.integers(12, 64, 2))
    pw, ph = (float(x) for x in rng.uniform(0.4, 1.6, 2))
    ext = float(np.linalg.norm(np.array(counts) * np.array(vox)))
    sid = float(rng.uniform(0.6, 3.0) * ext + 5.0)
    sdd = float(sid * rng.uniform(1.2, 2.5))
    nv = int(rng.integers(1, 10))
    arc = float(rng.choice([360.0, 200.0, 90.0]))
    det = cb.DetectorGeometry.make(rows, cols, pw, ph)
    geom = cb.VolumeGeometry.make(counts, vox)
    views = cb.make_circular_trajectory(sid, sdd, nv, arc, det)
    return cb, geom, det, views, Scene(counts, vox, rows, cols, pw, ph, cb.views_to_array(views))


@pytest.mark.parametrize("seed", range(6))
def test_random_geometry_siddon_parity(checker, seed):
    """Siddon-K (siddon.cpp:166-313) on random scenes: the reference's
    float64 traversal, so the bar is 1e-6 (float32 outputs). Lattices are odd
    so no sub-ray runs exactly inside a voxel-boundary plane: the circular
    trajectory's sources sit on the axes, and a ray in a boundary plane takes
    either neighbour depending on the last bit of its direction (the reference
    and its own C restatement then differ by up to 5% on that pixel)."""
    import torch
    rng = np.random.default_rng(2000 + seed)
    cb, geom, det, views, sc = _random_scene(rng, odd=True)
    K = int(rng.integers(1, 4))
    nv = len(views)
    x = cb.fill_uniform01(geom.voxel_count(), 300 + seed).astype(np.float32).astype(np.float64)
    b = cb.fill_uniform01(det.pixel_count() * nv, 400 + seed).astype(np.float32).astype(np.float64)
    scene = cb.DeviceScene(geom, det, views)
    p = scene.project_siddon(torch.from_numpy(x.astype(np.float32)).reshape(geom.shape()).cuda(), K)
    bp = scene.backproject_siddon(torch.from_numpy(b.astype(np.float32)).reshape(nv, det.rows, det.cols).cuda(), K)
    p_ref = checker.project_siddon(sc, x, K)
    bp_ref = checker.backproject_siddon(sc, b, K)
    if np.abs(p_ref).max() > 0:
        assert max_rel(p.double().cpu().numpy(), p_ref) <= 1e-6
    if np.abs(bp_ref).max() > 0:
        assert max_rel(bp.double().cpu().numpy().ravel(), bp_ref.ravel()) <= 1e-6


@pytest.mark.parametrize("seed", range(6))
def test_random_geometry_tt_adjoint(seed):
    """TT has no reference code (parity unpinned): on random scenes the pair
    stays adjoint (compensated float64 dots) and linear."""
    import torch
    rng = np.random.default_rng(3000 + seed)
    cb, geom, det, views, _ = _random_scene(rng)
    scene = cb.DeviceScene(geom, det, views)
    pair = cb.tt_pair(scene, cb.TTOptions(int(rng.integers(0, 2))))
    assert cb.adjoint_test(pair, seed) < 1e-5
