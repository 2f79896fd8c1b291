"""Randomized parity sweep: random lattices, voxel sizes, detectors, source
distances, arcs, view counts, options and execution modes, device CVP pair vs
the reference (oracle/_ref) — exact mode at rel-L2 <= 1e-5 and
max|d|/max|ref| <= 1e-4.

    python tools/random_parity.py [n_cases] [seed]
"""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2110_09841_b200 as cb  # noqa: E402
from oracle.pyoracle import Reference, Restatement, Scene, reference_available  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
chk = Reference() if reference_available() else Restatement()
rel = lambda a, b: float(np.linalg.norm(a.ravel() - b.ravel()) / np.linalg.norm(b.ravel()))
mx = lambda a, b: float(np.abs(a.ravel() - b.ravel()).max() / np.abs(b.ravel()).max())
worst = 0.0
fails = 0
for t in range(n_cases):
    counts = tuple(int(x) for x in rng.integers(5, 72, 3))
    vox = tuple(float(x) for x in rng.uniform(0.2, 1.5, 3))
    rows, cols = (int(x) for x in rng.integers(16, 160, 2))
    pw, ph = (float(x) for x in rng.uniform(0.3, 1.6, 2))
    ext = float(np.linalg.norm(np.array(counts) * np.array(vox)))
    sid = float(rng.uniform(0.6, 3.0) * ext + 5.0)
    sdd = float(sid * rng.uniform(1.2, 2.5))
    nv = int(rng.integers(1, 40))
    arc = float(rng.choice([360.0, 200.0, 90.0]))
    opts4 = (int(rng.integers(0, 2)), int(rng.integers(0, 2)), 0, int(rng.integers(0, 2)))
    det_mode = bool(rng.integers(0, 2))
    shape = str(int(rng.integers(0, 3)))
    import os
    os.environ["CVPB_CVP_SHAPE"] = shape
    det = cb.DetectorGeometry.make(rows, cols, pw, ph)
    geom = cb.VolumeGeometry.make(counts, vox)
    views = cb.make_circular_trajectory(sid, sdd, nv, arc, det)
    sc = Scene(counts, vox, rows, cols, pw, ph, cb.views_to_array(views))
    x = cb.fill_uniform01(geom.voxel_count(), 100 + t).astype(np.float32).astype(np.float64)
    if rng.integers(0, 3) == 0:  # sparse phantom
        x[rng.random(x.size) < 0.9] = 0.0
    b = cb.fill_uniform01(det.pixel_count() * nv, 200 + t).astype(np.float32).astype(np.float64)
    scene = cb.DeviceScene(geom, det, views)
    o = cb.CvpOptions(cb.PixelScaling(opts4[0]), bool(opts4[1]), cb.CvpPrecision(0), cb.RadiusEstimate(opts4[3]))
    ex = cb.ExecPolicy(deterministic=det_mode)
    p = scene.project_cvp(torch.from_numpy(x.astype(np.float32)).reshape(geom.shape()).cuda(), opts=o, exec=ex)
    bp = scene.backproject_cvp(torch.from_numpy(b.astype(np.float32)).reshape(nv, rows, cols).cuda(), opts=o, exec=ex)
    p_ref = chk.project_cvp(sc, x, opts4)
    bp_ref = chk.backproject_cvp(sc, b, opts4)
    pv, bv = p.double().cpu().numpy(), bp.double().cpu().numpy()
    if np.abs(p_ref).max() == 0:
        ok_p, e_p = np.abs(pv).max() == 0, (0.0, 0.0)
    else:
        e_p = (rel(pv, p_ref), mx(pv, p_ref))
        ok_p = e_p[0] <= 1e-5 and e_p[1] <= 1e-4
    e_b = (rel(bv, bp_ref), mx(bv, bp_ref))
    ok_b = e_b[0] <= 1e-5 and e_b[1] <= 1e-4
    worst = max(worst, e_p[0], e_b[0])
    fails += not (ok_p and ok_b)
    print(f"case {t:2d} {'ok  ' if ok_p and ok_b else 'FAIL'} counts={counts} vox=({vox[0]:.2f},{vox[1]:.2f},{vox[2]:.2f}) "
          f"det={rows}x{cols}@({pw:.2f},{ph:.2f}) sid={sid:.0f} sdd={sdd:.0f} v={nv} arc={arc:.0f} "
          f"opts={opts4} det={int(det_mode)} shape={shape}  P {e_p[0]:.1e}/{e_p[1]:.1e}  BP {e_b[0]:.1e}/{e_b[1]:.1e}",
          flush=True)
print(f"{n_cases - fails}/{n_cases} cases within the exact bar; worst rel-L2 {worst:.2e}")
