"""Per-config throughput table (BASELINE.json configs c1..c5) for every
projector on one GPU. Views are subsampled for the slow comparison
projectors; throughput is Gvoxel-views/s = N^3 * V / t / 1e9 (1e9 voxel-view
updates per second), each timing the mean of `reps` launches after a warm-up."""
import argparse, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_09841_b200 as cb

CFG = {
    "c1": dict(n=64, a=0.5, R=64, C=64, px=1.0, sid=541., sdd=949., V=36, arc=360.),
    "c2": dict(n=256, a=0.18, R=480, C=616, px=0.154, sid=749., sdd=1198., V=248, arc=200.),
    "c3": dict(n=512, a=0.09, R=480, C=616, px=0.154, sid=749., sdd=1198., V=496, arc=360.),
    "c4": dict(n=512, a=0.5, R=1024, C=1024, px=1.0, sid=300., sdd=500., V=360, arc=360.),
    "c5": dict(n=1024, a=0.4, R=768, C=1024, px=1.0, sid=541., sdd=949., V=720, arc=360.),
}


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    rows = []
    for name in a.configs.split(","):
        c = CFG[name]
        det = cb.DetectorGeometry.make(c["R"], c["C"], c["px"], c["px"])
        geom = cb.VolumeGeometry.make((c["n"],) * 3, (c["a"],) * 3)
        views = cb.make_circular_trajectory(c["sid"], c["sdd"], c["V"], c["arc"], det)
        scene = cb.DeviceScene(geom, det, views)
        x = torch.rand(geom.shape(), device="cuda")
        nv = lambda v: geom.voxel_count() * v / 1e9
        res = {"config": name}
        for label, prec in (("cvp_exact", cb.CvpPrecision.Double), ("cvp_relaxed", cb.CvpPrecision.Single)):
            o = cb.CvpOptions(precision=prec)
            p = scene.new_stack()
            b = torch.rand_like(p)
            v = scene.new_volume()
            tp = timeit(lambda: scene.project_cvp(x, p, o), a.reps)
            tb = timeit(lambda: scene.backproject_cvp(b, v, o), a.reps)
            res[label] = (nv(c["V"]) / tp, nv(c["V"]) / tb, tp, tb)
            del p, b
        # comparison projectors on a view subset (same geometry)
        vs = max(1, min(c["V"], 16))
        p = scene.new_stack(vs)
        b = torch.rand_like(p)
        v = scene.new_volume()
        tp = timeit(lambda: scene.project_tt(x, p, view_count=vs), a.reps)
        tb = timeit(lambda: scene.backproject_tt(b, v, view_count=vs), a.reps)
        res["tt"] = (nv(vs) / tp, nv(vs) / tb, tp * c["V"] / vs, tb * c["V"] / vs)
        for K in (1, 8):
            vk = vs if K == 1 else max(1, vs // 8)
            tp = timeit(lambda: scene.project_siddon(x, K, p[:vk], view_count=vk), 1)
            tb = timeit(lambda: scene.backproject_siddon(b[:vk].contiguous(), K, v, view_count=vk), 1)
            res[f"siddon{K}"] = (nv(vk) / tp, nv(vk) / tb, tp * c["V"] / vk, tb * c["V"] / vk)
        rows.append(res)
        print(json.dumps(res), flush=True)
        del scene, x, p, b, v
        torch.cuda.empty_cache()
    print("\n| config | projector | P Gvox-view/s | BP Gvox-view/s | P s (all views) | BP s (all views) |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        for k in ("cvp_exact", "cvp_relaxed", "tt", "siddon1", "siddon8"):
            p, b, tp, tb = r[k]
            print(f"| {r['config']} | {k} | {p:.2f} | {b:.2f} | {tp:.3f} | {tb:.3f} |")


if __name__ == "__main__":
    main()
