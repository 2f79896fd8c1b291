"""cbctproj-compatible command line over the B200 path.

    python -m paper_2110_09841_b200 <subcommand> [options]

Subcommands, flags, CSV formats, presets and exit codes follow the
reference's tools/commands.cpp:472-585:
  project | backproject | recon | compare | bench | adjoint-test.
All operators run on the GPU (DEN payloads stream straight to the device);
`--projector` additionally accepts `tt`.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

PRESETS = {
    # tools/commands.cpp:141-152 — volume counts, voxel, det rows, cols, pixel, sid, sdd, arc, views
    "desk": ((64, 64, 64), (0.5, 0.5, 0.5), 128, 128, 1.0, 1.0, 541.0, 949.0, 360.0, 36),
    "long2010": ((512, 512, 128), (0.5, 0.5, 0.5), 512, 512, 1.0, 1.0, 541.0, 949.0, 360.0, 720),
    "pfeiffer2021": ((256, 256, 256), (0.5, 0.5, 0.5), 960, 1280, 0.25, 0.25, 750.0, 1000.0, 198.0,
                     100),
}


class ExitWith(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _add_projector_flags(p):
    p.add_argument("--projector", choices=["cvp", "siddon", "tt"], default="cvp")
    p.add_argument("--siddon-k", type=int, default=8)
    g = p.add_mutually_exclusive_group()
    g.add_argument("--cos-scaling", action="store_true")
    g.add_argument("--exact-scaling", action="store_true")
    e = p.add_mutually_exclusive_group()
    e.add_argument("--elevation-correction", action="store_true")
    e.add_argument("--no-elevation-correction", action="store_true")
    p.add_argument("--relaxed", action="store_true")
    p.add_argument("--threads", type=int, default=0, help="ignored on the device")
    p.add_argument("--deterministic", action="store_true")


def _add_trajectory_flags(p):
    g = p.add_mutually_exclusive_group()
    g.add_argument("--matrices")
    g.add_argument("--circular", type=float, nargs=4, metavar=("SID", "SDD", "N_VIEWS", "ARC_DEG"))
    p.add_argument("--pixel-width", type=float, default=1.0)
    p.add_argument("--pixel-height", type=float, default=1.0)


def _cvp_opts(a):
    import paper_2110_09841_b200 as cb
    return cb.CvpOptions(cb.PixelScaling.Cos if a.cos_scaling else cb.PixelScaling.Exact,
                         not a.no_elevation_correction,
                         cb.CvpPrecision.Single if a.relaxed else cb.CvpPrecision.Double)


def _exec(a):
    import paper_2110_09841_b200 as cb
    # a user typing --siddon-k 512 is deliberate (commands.cpp:56-59)
    return cb.ExecPolicy(a.threads, a.deterministic, True)


def _load_views(a, det):
    import paper_2110_09841_b200 as cb
    if a.matrices:
        return cb.read_camera_matrices(a.matrices, det.pixel_size())
    if a.circular:
        sid, sdd, n, arc = a.circular
        if n < 1 or int(n) != n:
            raise cb.InvalidArgument("--circular N_VIEWS must be a positive integer")
        return cb.make_circular_trajectory(sid, sdd, int(n), arc, det)
    raise ExitWith(1, "either --matrices or --circular is required")


def _voxel(v):
    if not v:
        return (1.0, 1.0, 1.0)
    if len(v) == 1:
        return (v[0],) * 3
    if len(v) == 3:
        return tuple(v)
    import paper_2110_09841_b200 as cb
    raise cb.InvalidArgument("--voxel-size takes one or three values")


def view_angle_deg(v, n_views, arc):
    step = arc / n_views if abs(arc - 360.0) < 1e-9 else (arc / (n_views - 1) if n_views > 1 else 0.0)
    return v * step


class TimedPair:
    """Operator pair on device tensors with per-application timers
    (OpTimers, commands.cpp:156-204)."""

    def __init__(self, a, scene):
        import paper_2110_09841_b200 as cb
        self.a, self.scene = a, scene
        self.opts, self.exec = _cvp_opts(a), _exec(a)
        self.fwd_s = self.bwd_s = 0.0
        self.fwd_n = self.bwd_n = 0
        self.pair = cb.LinearOperatorPair(self.forward, self.adjoint, scene.vol_geom, scene.det,
                                          scene.n_views)

    def _sync(self):
        import torch
        torch.cuda.synchronize()

    def forward(self, x, out):
        self._sync()
        t = time.perf_counter()
        s, a = self.scene, self.a
        if a.projector == "cvp":
            s.project_cvp(x.values, out.values, self.opts, self.exec)
        elif a.projector == "siddon":
            s.project_siddon(x.values, a.siddon_k, out.values, exec=self.exec)
        else:
            s.project_tt(x.values, out.values)
        self._sync()
        self.fwd_s += time.perf_counter() - t
        self.fwd_n += 1

    def adjoint(self, b, out):
        self._sync()
        t = time.perf_counter()
        s, a = self.scene, self.a
        if a.projector == "cvp":
            s.backproject_cvp(b.values, out.values, self.opts, self.exec)
        elif a.projector == "siddon":
            s.backproject_siddon(b.values, a.siddon_k, out.values, exec=self.exec)
        else:
            s.backproject_tt(b.values, out.values)
        self._sync()
        self.bwd_s += time.perf_counter() - t
        self.bwd_n += 1


def run_project(a):
    import paper_2110_09841_b200 as cb
    from . import den
    det = cb.DetectorGeometry.make(a.det_rows, a.det_cols, a.pixel_width, a.pixel_height)
    views = _load_views(a, det)
    hdr = den.den_read(a.volume)
    geom = cb.VolumeGeometry.make((hdr.dim_x, hdr.dim_y, hdr.dim_z), _voxel(a.voxel_size))
    x = den.den_read_device(a.volume)
    scene = cb.DeviceScene(geom, det, views)
    tp = TimedPair(a, scene)
    out = scene.new_stack()
    tp.forward(cb.AttenuationVolume(geom, x), cb.ProjectionStack(det, len(views), out))
    den.den_write_device(a.output, out)
    print(f"wrote {a.output} ({det.rows} x {det.cols} x {len(views)})")
    return 0


def run_backproject(a):
    import paper_2110_09841_b200 as cb
    from . import den
    hdr = den.den_read(a.projections)
    det = cb.DetectorGeometry.make(hdr.dim_y, hdr.dim_x, a.pixel_width, a.pixel_height)
    views = _load_views(a, det)
    if len(views) != hdr.dim_z:
        raise cb.CvpbRuntimeError(f"trajectory has {len(views)} views but projection stack has "
                                  f"{hdr.dim_z}")
    geom = cb.VolumeGeometry.make(tuple(a.vol_dims), _voxel(a.voxel_size))
    b = den.den_read_device(a.projections)
    scene = cb.DeviceScene(geom, det, views)
    tp = TimedPair(a, scene)
    out = scene.new_volume()
    tp.adjoint(cb.ProjectionStack(det, len(views), b), cb.AttenuationVolume(geom, out))
    den.den_write_device(a.output, out)
    print(f"wrote {a.output} ({geom.counts[0]} x {geom.counts[1]} x {geom.counts[2]} voxels)")
    return 0


def run_recon(a):
    import paper_2110_09841_b200 as cb
    from . import den
    hdr = den.den_read(a.projections)
    det = cb.DetectorGeometry.make(hdr.dim_y, hdr.dim_x, a.pixel_width, a.pixel_height)
    views = _load_views(a, det)
    if len(views) != hdr.dim_z:
        raise cb.CvpbRuntimeError("trajectory/projection view count mismatch")
    geom = cb.VolumeGeometry.make(tuple(a.vol_dims), _voxel(a.voxel_size))
    b = den.den_read_device(a.projections)
    scene = cb.DeviceScene(geom, det, views)
    tp = TimedPair(a, scene)
    res = cb.cgls(tp.pair, cb.ProjectionStack(det, len(views), b), a.iterations)
    bn = res.residual_norms[0]
    rel = res.residual_norms[-1] / bn if bn > 0 else res.residual_norms[-1]
    print(f"CGLS {len(res.residual_norms) - 1} iterations, relative residual {rel:.6e}")
    if a.residuals:
        with open(a.residuals, "w") as f:
            f.write("iteration,residual_norm,relative_residual\n")
            for i, r in enumerate(res.residual_norms):
                f.write(f"{i},{r:.17g},{(r / bn if bn > 0 else 0.0):.17g}\n")
    den.den_write_device(a.output, res.x.values)
    print(f"wrote {a.output} ({geom.counts[0]} x {geom.counts[1]} x {geom.counts[2]} voxels)")
    return 0


def run_compare(a):
    """Per-view relative error of B against A (commands.cpp:322-371); CPU only."""
    from . import den
    A, B = den.den_read(a.a), den.den_read(a.b)
    if (A.dim_x, A.dim_y, A.dim_z) != (B.dim_x, B.dim_y, B.dim_z):
        raise RuntimeError(f"dimension mismatch: {a.a} vs {a.b}")
    fa = A.values.reshape(A.dim_z, -1).astype(np.float64)
    fb = B.values.reshape(B.dim_z, -1).astype(np.float64)
    ref2 = (fa * fa).sum(1)
    diff2 = ((fb - fa) ** 2).sum(1)
    with np.errstate(divide="ignore", invalid="ignore"):
        err = np.where(ref2 > 0, 100.0 * np.sqrt(diff2 / np.where(ref2 > 0, ref2, 1)),
                       np.where(diff2 > 0, np.inf, 0.0))
    if a.report:
        with open(a.report, "w") as f:
            f.write("view,angle_deg,error_percent\n")
            for v, e in enumerate(err):
                f.write(f"{v},{view_angle_deg(v, A.dim_z, a.arc):.6f},{e:.9g}\n")
    mean, worst = float(err.mean()) if err.size else 0.0, float(err.max()) if err.size else 0.0
    print(f"views {A.dim_z}, mean error {mean:.6g}%, max error {worst:.6g}%")
    if a.tol is not None and a.tol >= 0 and not (worst <= a.tol):
        print(f"max error {worst:.6g}% exceeds tolerance {a.tol:.6g}%", file=sys.stderr)
        return 1
    return 0


def run_bench(a):
    """CGLS benchmark on seeded U[0,1) data (commands.cpp:382-429) — the
    paper's timing protocol (mean P / BP time within CGLS)."""
    import torch
    import paper_2110_09841_b200 as cb
    counts, vox, R, C, pw, ph, sid, sdd, arc, V = PRESETS[a.preset]
    det = cb.DetectorGeometry.make(R, C, pw, ph)
    geom = cb.VolumeGeometry.make(counts, vox)
    need = 4 * (3 * geom.voxel_count() + 2 * det.pixel_count() * V)
    free, _ = torch.cuda.mem_get_info()
    if not a.force and need > free:
        raise ExitWith(2, f"estimated peak device memory {need / 2**30:.2f} GiB exceeds free "
                          f"{free / 2**30:.2f} GiB; use --preset desk or pass --force")
    views = cb.make_circular_trajectory(sid, sdd, V, arc, det)
    if a.save_matrices:
        cb.write_camera_matrices(a.save_matrices, views)
    scene = cb.DeviceScene(geom, det, views)
    tp = TimedPair(a, scene)
    b = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * V, a.seed).astype(np.float32))
    b = b.reshape(V, R, C).cuda()
    print(f"bench {a.preset}: volume {counts[0]}x{counts[1]}x{counts[2]}, detector {R}x{C}, "
          f"{V} views, {a.iterations} CGLS iterations ({a.projector})")
    res = cb.cgls(tp.pair, cb.ProjectionStack(det, V, b), a.iterations)
    fm = tp.fwd_s / tp.fwd_n if tp.fwd_n else 0.0
    bm = tp.bwd_s / tp.bwd_n if tp.bwd_n else 0.0
    path = a.csv or f"bench_{a.preset}.csv"
    with open(path, "w") as f:
        f.write("record,index,angle_deg,value\n")
        # device launches cover all views at once: per-view time is the mean
        for v in range(V):
            f.write(f"project_view_s,{v},{view_angle_deg(v, V, arc):.6f},{fm / V:.9f}\n")
        f.write(f"project_applications,,,{tp.fwd_n}\n")
        f.write(f"backproject_applications,,,{tp.bwd_n}\n")
        f.write(f"project_mean_s,,,{fm:.9f}\n")
        f.write(f"backproject_mean_s,,,{bm:.9f}\n")
        for i, r in enumerate(res.residual_norms):
            f.write(f"cgls_residual,{i},,{r:.17g}\n")
    bn = res.residual_norms[0]
    print(f"mean projector time {fm:.3f} s, mean backprojector time {bm:.3f} s")
    print(f"relative residual after {a.iterations} iterations: "
          f"{(res.residual_norms[-1] / bn if bn > 0 else 0.0):.6e}")
    print(f"wrote {path}")
    return 0


def run_adjoint_test(a):
    """Randomized dot-product test (commands.cpp:439-468). Device outputs are
    float32, so the threshold is 1e-5 (the reference: 1e-12 double, 1e-4
    relaxed)."""
    import paper_2110_09841_b200 as cb
    counts, vox, R, C, pw, ph, sid, sdd, arc, V = PRESETS[a.preset]
    det = cb.DetectorGeometry.make(R, C, pw, ph)
    geom = cb.VolumeGeometry.make(counts, vox)
    scene = cb.DeviceScene(geom, det, cb.make_circular_trajectory(sid, sdd, V, arc, det))
    if a.mismatched_pair:
        # negative control: forward with 1 ray per pixel, adjoint with 4
        f, b = cb.siddon_pair(scene, 1), cb.siddon_pair(scene, 2)
        pair = cb.LinearOperatorPair(f.forward, b.adjoint, geom, det, V)
    else:
        pair = TimedPair(a, scene).pair
    thr = 1e-5
    worst = 0.0
    for i in range(a.seeds):
        d = cb.adjoint_test(pair, a.seed + i)
        print(f"seed {a.seed + i}: discrepancy {d:.6e}")
        worst = max(worst, d)
    ok = worst < thr
    print(f"max discrepancy {worst:.6e}, threshold {thr:.0e} -> {'PASS' if ok else 'FAIL'}")
    return 0 if ok else 1


def build_parser():
    ap = argparse.ArgumentParser(prog="cbctproj-b200",
                                 description="Cone-beam CT projection/backprojection toolkit (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("project", help="Forward project a volume to extinction images")
    p.add_argument("--volume", required=True)
    p.add_argument("--output", required=True)
    p.add_argument("--det-rows", type=int, required=True)
    p.add_argument("--det-cols", type=int, required=True)
    p.add_argument("--voxel-size", type=float, nargs="+")
    _add_trajectory_flags(p)
    _add_projector_flags(p)
    p.set_defaults(fn=run_project)
    for name, fn, hlp in (("backproject", run_backproject, "Apply the adjoint operator"),
                          ("recon", run_recon, "CGLS reconstruction from projections")):
        q = sub.add_parser(name, help=hlp)
        q.add_argument("--projections", required=True)
        q.add_argument("--output", required=True)
        q.add_argument("--vol-dims", type=int, nargs=3, required=True)
        q.add_argument("--voxel-size", type=float, nargs="+")
        if name == "recon":
            q.add_argument("--iterations", type=int, default=30)
            q.add_argument("--residuals")
        _add_trajectory_flags(q)
        _add_projector_flags(q)
        q.set_defaults(fn=fn)
    c = sub.add_parser("compare", help="Per-view relative error of B against A")
    c.add_argument("a")
    c.add_argument("b")
    c.add_argument("--report")
    c.add_argument("--arc", type=float, default=360.0)
    c.add_argument("--tol", type=float)
    c.set_defaults(fn=run_compare)
    b = sub.add_parser("bench", help="CGLS benchmark on seeded random data")
    b.add_argument("--preset", choices=list(PRESETS), default="desk")
    b.add_argument("--iterations", type=int, default=2)
    b.add_argument("--csv")
    b.add_argument("--save-matrices")
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--force", action="store_true")
    _add_projector_flags(b)
    b.set_defaults(fn=run_bench)
    t = sub.add_parser("adjoint-test", help="Randomized dot-product test of the pair")
    t.add_argument("--preset", choices=list(PRESETS), default="desk")
    t.add_argument("--seed", type=int, default=1)
    t.add_argument("--seeds", type=int, default=1)
    t.add_argument("--mismatched-pair", action="store_true", help=argparse.SUPPRESS)
    _add_projector_flags(t)
    t.set_defaults(fn=run_adjoint_test)
    return ap


def main(argv=None):
    ap = build_parser()
    a = ap.parse_args(argv)
    try:
        return a.fn(a)
    except ExitWith as e:
        print(f"error: {e}", file=sys.stderr)
        return e.code
    except Exception as e:  # reference prints and exits 1 (commands.cpp:578-584)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
