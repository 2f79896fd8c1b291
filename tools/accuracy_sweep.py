"""Large-cone-angle accuracy sweep (BASELINE configs[3]: 512^3 @0.5 mm,
1024x1024 @1 mm, SID 300 / SDD 500): per-view relative projector error
(solver.cpp:108-119, percent) of CVP (exact, relaxed), TT (A1, A2) and
Siddon-K against Siddon-512 ground truth over the footprint ROI
(acceptance.cpp:100-147), for single voxels at increasing cone / fan angles.
The paper's claim: CVP stays accurate where TT degrades.

    python tools/accuracy_sweep.py [--views 36] > profiles/accuracy_c4_r01.md
"""
import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2110_09841_b200 as cb  # noqa: E402


def roi_of(view, det, lo, hi, pad=3):
    c1, c2 = [], []
    for q in range(8):
        p = (hi[0] if q & 1 else lo[0], hi[1] if q & 2 else lo[1], hi[2] if q & 4 else lo[2])
        chi = view.project_point(p)
        c1.append(chi[0])
        c2.append(chi[1])
    cl = lambda v, a, b: max(a, min(b, v))
    return cb.PixelRoi(cl(int(math.floor(min(c2) + 0.5)) - pad, 0, det.rows),
                       cl(int(math.floor(max(c2) + 0.5)) + 1 + pad, 0, det.rows),
                       cl(int(math.floor(min(c1) + 0.5)) - pad, 0, det.cols),
                       cl(int(math.floor(max(c1) + 0.5)) + 1 + pad, 0, det.cols))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=36)
    ap.add_argument("--n", type=int, default=512)
    a = ap.parse_args()
    n, vox = a.n, 0.5 * 512 / a.n
    det = cb.DetectorGeometry.make(1024, 1024, 1.0, 1.0)
    geom = cb.VolumeGeometry.make((n, n, n), (vox, vox, vox))
    views = cb.make_circular_trajectory(300.0, 500.0, a.views, 360.0, det)
    scene = cb.DeviceScene(geom, det, views)
    ex = cb.ExecPolicy(allow_expensive=True)
    mc = geom.min_corner()
    # voxel index offsets from the centre: on axis, in-plane off-axis, high
    # elevation, both (the cone-angle corner of the FOV)
    off = n // 4
    cases = [("centre", (0, 0, 0)), ("off-axis x", (off, 0, 0)), ("elevation z", (0, 0, off)),
             ("off-axis + elevation", (off, off, off))]
    print(f"# Accuracy sweep, configs[3] geometry ({n}^3 @{vox:g} mm, 1024x1024 @1 mm, "
          f"SID 300 / SDD 500, {a.views} views)\n")
    print("Per-view relative projector error in percent (solver.cpp:108-119) against "
          "Siddon-512 over the footprint ROI (acceptance.cpp:100-147); median / max over views. "
          "`tools/accuracy_sweep.py`.\n")
    print("| voxel | cone angle | CVP exact | CVP relaxed | TT A1 | TT A2 | Siddon-8 | Siddon-32 |")
    print("|---|---|---|---|---|---|---|---|")
    for name, (di, dj, dk) in cases:
        i, j, k = n // 2 + di, n // 2 + dj, n // 2 + dk
        x = scene.new_volume()
        x[k, j, i] = 1.0
        lo = (mc[0] + i * vox, mc[1] + j * vox, mc[2] + k * vox)
        hi = (lo[0] + vox, lo[1] + vox, lo[2] + vox)
        zc = lo[2] + 0.5 * vox
        cone = math.degrees(math.atan2(abs(zc), 300.0 - math.hypot(lo[0], lo[1])))

        def siddon(K):
            out = np.zeros((len(views), det.rows, det.cols))
            for v in range(len(views)):
                p = scene.project_siddon(x, K, roi=roi_of(views[v], det, lo, hi), exec=ex,
                                         view_begin=v, view_count=1)
                out[v] = p[0].double().cpu().numpy()
            return out

        ref = siddon(512)
        errs = {}
        errs["cvp"] = scene.project_cvp(x).double().cpu().numpy()
        errs["cvpr"] = scene.project_cvp(x, opts=cb.CvpOptions(precision=cb.CvpPrecision.Single)).double().cpu().numpy()
        errs["tt1"] = scene.project_tt(x, opts=cb.TTOptions(0)).double().cpu().numpy()
        errs["tt2"] = scene.project_tt(x, opts=cb.TTOptions(1)).double().cpu().numpy()
        errs["s8"] = siddon(8)
        errs["s32"] = siddon(32)
        cells = []
        for key in ("cvp", "cvpr", "tt1", "tt2", "s8", "s32"):
            e = np.array([cb.relative_projector_error(errs[key][v], ref[v]) for v in range(len(views))])
            cells.append(f"{np.median(e):.3f} / {e.max():.3f}")
        print(f"| {name} ({i},{j},{k}) | {cone:.1f} deg | " + " | ".join(cells) + " |", flush=True)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
