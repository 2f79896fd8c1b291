"""Headline benchmark: exact CVP project + backproject, 512^3 x 496 views on a
616x480 detector (BASELINE.json configs[2]; SURVEY §8d pinned geometry).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision exact|relaxed]
  python bench.py --impl reference ...      # the reference's CPU path (oracle/_ref)

One step = one forward projection of the whole volume into all views + one
backprojection of a whole stack (the two halves of a CGLS iteration). The
metric counts voxel-view pairs: value = N1*N2*N3*V / (t_P + t_BP) / 1e9,
whole job over all ranks. Multi-GPU (torchrun): views are sharded across
ranks; P needs no exchange, BP partial volumes are summed with an NCCL
reduce-scatter over z-slabs (the path's one real exchange step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = dict(counts=(512, 512, 512), voxel=(0.09, 0.09, 0.09), rows=480, cols=616, pw=0.154,
              ph=0.154, sid=749.0, sdd=1198.0, n_views=496, arc=360.0)
METRIC = "CVP project+backproject Gvoxel-views/s at 512^3 x 496 views"
UNIT = "Gvoxel-views/s"
WORKLOAD = ("c3: CVP P+BP, 512^3 @0.09 mm, 616x480 @0.154 mm, SID 749 / SDD 1198, "
            "496 views / 360 deg, dense U[0,1] volume (seed 7) and stack (seed 8)")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu_index=0):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")
        self.gpu = gpu_index

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = max(mx, float(parts[2]))
                except ValueError:
                    continue
                for name, val in zip(names, parts[5:9]):
                    if val.lower() == "active":
                        reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline_sample(precision, n_sample_views=2, threads=None):
    """Reference CPU path (oracle/_ref = the reference compiled from its own
    sources; falls back to the C restatement) on a bounded sample of the same
    workload: `n_sample_views` evenly spaced views of the 496, P + BP."""
    from oracle import pyoracle
    import paper_2110_09841_b200 as cb
    threads = threads or os.cpu_count()
    if pyoracle.reference_available():
        chk, kind = pyoracle.Reference(), "reference"
    else:
        chk, kind = pyoracle.Restatement(), "port"
        threads = 1
    c = CONFIG
    det = cb.DetectorGeometry.make(c["rows"], c["cols"], c["pw"], c["ph"])
    views = cb.make_circular_trajectory(c["sid"], c["sdd"], c["n_views"], c["arc"], det)
    idx = np.linspace(0, c["n_views"] - 1, n_sample_views).round().astype(int)
    arr = cb.views_to_array(views)[idx]
    sc = pyoracle.Scene(c["counts"], c["voxel"], c["rows"], c["cols"], c["pw"], c["ph"], arr)
    nvox = int(np.prod(c["counts"]))
    x = np.asarray(cb.fill_uniform01(nvox, 7), dtype=np.float32).astype(np.float64)
    b = np.asarray(cb.fill_uniform01(c["rows"] * c["cols"] * n_sample_views, 8),
                   dtype=np.float32).astype(np.float64)
    opts = (1, 1, 0 if precision == "exact" else 1, 1)
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    t0 = time.perf_counter()
    chk.project_cvp(sc, x, opts, threads=threads)
    t1 = time.perf_counter()
    chk.backproject_cvp(sc, b, opts, threads=threads)
    t2 = time.perf_counter()
    work = nvox * n_sample_views / 1e9
    return {"value": work / ((t1 - t0) + (t2 - t1)), "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{n_sample_views} evenly spaced views of the 496 at full 512^3 / 616x480 "
                      f"({precision} CVP, P {t1 - t0:.2f} s + BP {t2 - t1:.2f} s, "
                      f"{threads} threads)",
            "p_gvps": work / (t1 - t0), "bp_gvps": work / (t2 - t1)}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = []
    last = None
    for s in range(args.warmup + args.steps):
        r = cpu_baseline_sample(args.precision, n_sample_views=args.ref_views)
        if s >= args.warmup:
            steps.append(r["value"])
            last = r
    val = statistics.mean(steps)
    c = CONFIG
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": float(np.prod(c["counts"])) * c["n_views"] / 1e9 / val * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64" if args.precision == "exact" else "f32", "data": "synthetic",
           "config": {"workload": WORKLOAD, "precision": args.precision,
                      "sample_per_step": last["sample"]},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": last["cores"],
                            "kind": last["kind"], "sample": last["sample"]},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precision", choices=["exact", "relaxed"], default="exact")
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--ref-views", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cgls-iters", type=int, default=2,
                    help="device-resident CGLS iterations timed for cgls_ms_per_iter (0 = skip)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist
    import paper_2110_09841_b200 as cb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    c = CONFIG
    det = cb.DetectorGeometry.make(c["rows"], c["cols"], c["pw"], c["ph"])
    geom = cb.VolumeGeometry.make(c["counts"], c["voxel"])
    views = cb.make_circular_trajectory(c["sid"], c["sdd"], c["n_views"], c["arc"], det)
    V = len(views)
    # shard views: rank r owns [v0, v1)
    v0 = rank * V // world
    v1 = (rank + 1) * V // world
    scene = cb.DeviceScene(geom, det, views, device=local)
    opts = cb.CvpOptions(precision=cb.CvpPrecision.Double if args.precision == "exact"
                         else cb.CvpPrecision.Single)
    nvox = geom.voxel_count()
    x = torch.from_numpy(cb.fill_uniform01(nvox, 7).astype(np.float32)).reshape(geom.shape()).cuda()
    b_all = cb.fill_uniform01(det.pixel_count() * V, 8).astype(np.float32)
    b = torch.from_numpy(b_all[v0 * det.pixel_count():v1 * det.pixel_count()]).reshape(
        v1 - v0, det.rows, det.cols).cuda()
    del b_all
    p = scene.new_stack(v1 - v0)
    bp = scene.new_volume()
    slab = torch.empty(nvox // world if world > 1 else 1, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        scene.project_cvp(x, p, opts, view_begin=v0, view_count=v1 - v0)
        if ev:
            ev[1].record(stream)
        scene.backproject_cvp(b, bp, opts, view_begin=v0, view_count=v1 - v0)
        if ev:
            ev[2].record(stream)
        if world > 1:
            dist.reduce_scatter_tensor(slab, bp.view(-1))
        if ev:
            ev[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for s in range(args.steps):
        step(evs[s])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    p_ms = [e[0].elapsed_time(e[1]) for e in evs]
    bp_ms = [e[1].elapsed_time(e[2]) for e in evs]
    rs_ms = [e[2].elapsed_time(e[3]) for e in evs]
    if world > 1:
        t = torch.tensor([total_ms, statistics.mean(p_ms), statistics.mean(bp_ms),
                          statistics.mean(rs_ms)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, pm, bm, rm = t.tolist()
    else:
        pm, bm, rm = statistics.mean(p_ms), statistics.mean(bp_ms), statistics.mean(rs_ms)
    ms_per_step = total_ms / args.steps
    work = nvox * V / 1e9  # Gvoxel-views per application, whole job
    value = work / (ms_per_step * 1e-3)

    # ---- e2e through the reference-facing C-ABI host path (rank 0 / N=1) ---
    e2e = None
    if not args.no_e2e and world == 1:
        x64 = torch.from_numpy(cb.fill_uniform01(nvox, 7)).pin_memory()
        b64 = torch.from_numpy(cb.fill_uniform01(det.pixel_count() * V, 8)).pin_memory()
        p64 = torch.empty(det.pixel_count() * V, dtype=torch.float64).pin_memory()
        v64 = torch.empty(nvox, dtype=torch.float64).pin_memory()
        x64n, b64n, p64n, v64n = x64.numpy(), b64.numpy(), p64.numpy(), v64.numpy()
        e2e_steps = max(1, min(args.steps, 3))
        scene.project_cvp_host(x64n, p64n, opts)
        scene.backproject_cvp_host(b64n, v64n, opts)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            scene.project_cvp_host(x64n, p64n, opts)
            scene.backproject_cvp_host(b64n, v64n, opts)
        t1 = time.perf_counter()
        e2e = {"value": work / ((t1 - t0) / e2e_steps), "unit": UNIT,
               "h2d_bytes_per_step": int(x64.numel() * 8 + b64.numel() * 8),
               "d2h_bytes_per_step": int(p64.numel() * 8 + v64.numel() * 8),
               "path": "cvpb_project_cvp_host + cvpb_backproject_cvp_host (float64 pinned host "
                       "buffers, conversions and copies inside the timed region)",
               "steps": e2e_steps}
    elif not args.no_e2e:
        # N > 1: each rank moves its own inputs (float64 pinned host: the full
        # volume for P, its view shard for BP) and its outputs (its projection
        # shard, its z-slab of the reduce-scattered volume) through the public
        # API (DeviceScene + reduce-scatter); max over ranks of the wall time.
        npx = det.pixel_count()
        x64 = torch.from_numpy(cb.fill_uniform01(nvox, 7)).pin_memory()
        b64 = torch.from_numpy(cb.fill_uniform01(npx * V, 8)[v0 * npx:v1 * npx].copy()).pin_memory()
        p64 = torch.empty((v1 - v0) * npx, dtype=torch.float64).pin_memory()
        s64 = torch.empty(slab.numel(), dtype=torch.float64).pin_memory()
        e2e_steps = max(1, min(args.steps, 3))

        def e2e_step():
            xd = x64.to("cuda", non_blocking=True).float().reshape(geom.shape())
            bd = b64.to("cuda", non_blocking=True).float().reshape(v1 - v0, det.rows, det.cols)
            scene.project_cvp(xd, p, opts, view_begin=v0, view_count=v1 - v0)
            scene.backproject_cvp(bd, bp, opts, view_begin=v0, view_count=v1 - v0)
            dist.reduce_scatter_tensor(slab, bp.view(-1))
            p64.copy_(p.view(-1).double(), non_blocking=True)
            s64.copy_(slab.double(), non_blocking=True)
            torch.cuda.synchronize()

        e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        dt = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": work / float(dt.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(x64.numel() * 8 + b64.numel() * 8),
               "d2h_bytes_per_step": int(p64.numel() * 8 + s64.numel() * 8),
               "path": "per rank: pinned float64 -> device, DeviceScene P/BP on its view shard, "
                       "NCCL reduce-scatter, its projections + z-slab back to pinned float64 "
                       "(bytes per rank)",
               "steps": e2e_steps}

    # ---- CGLS ms/iter (BASELINE metric, second half) ---------------------------
    cgls = None
    if args.cgls_iters > 0 and world == 1:
        bt = scene.project_cvp(x, opts=opts)
        scene.cgls(bt, 1, opts=opts)  # warm-up: allocates the context's CGLS vectors
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, res0 = scene.cgls(bt, 1, opts=opts)          # 1 BP + 1 iteration
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        _, res = scene.cgls(bt, 1 + args.cgls_iters, opts=opts)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        cgls = {"ms_per_iter": ((t2 - t1) - (t1 - t0)) / args.cgls_iters * 1e3,
                "iterations_timed": args.cgls_iters,
                "residual_ratio": res[-1] / res[0],
                "how": "device-resident cvpb_cgls on the c3 scene (1 P + 1 BP + float64-accumulated "
                       "vector ops per iteration); ms/iter = (T(1+n) - T(1)) / n, wall clock "
                       "around synchronized calls"}
    elif args.cgls_iters > 0:
        # N > 1: view-sharded CGLS (parallel.distributed_cgls): x, s, p as
        # z-slabs, r, q as view shards; all-gather of p before each P,
        # reduce-scatter of the BP partials, all-reduced float64 scalars
        from paper_2110_09841_b200 import parallel as par
        op = par.scene_operator(scene, opts)
        bt = op.project(x.reshape(-1))
        vec = par.SceneVec(scene)

        def run(n):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            r = par.distributed_cgls(op, bt, n, vec)
            torch.cuda.synchronize()
            dist.barrier()
            return time.perf_counter() - t0, r

        run(1)  # warm-up
        ta, _ = run(1)
        tb, r = run(1 + args.cgls_iters)
        dt = torch.tensor([(tb - ta) / args.cgls_iters], device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        cgls = {"ms_per_iter": float(dt.item()) * 1e3, "iterations_timed": args.cgls_iters,
                "residual_ratio": r.residual_norms[-1] / r.residual_norms[0],
                "how": f"view-sharded CGLS over {world} ranks on the c3 scene (parallel."
                       "distributed_cgls: slab-resident x/s/p, NCCL all-gather + reduce-scatter "
                       "per iteration); ms/iter = (T(1+n) - T(1)) / n, max over ranks"}

    # ---- roofline of the dominant kernel -----------------------------------
    hbm, peak_src = _peaks()
    dom_ms = max(pm, bm)
    dom = "cvp_brick_kernel<EXACT,FWD>" if pm >= bm else "cvp_brick_kernel<EXACT,BWD>"
    views_here = v1 - v0
    alg_bytes = 4.0 * nvox * views_here  # 4 B per voxel-view
    achieved = alg_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_r01.json")
    if os.path.exists(tp) and world == 1:
        with open(tp) as f:
            t = json.load(f).get(dom)
        if t:
            traffic = t["dram_read"] + t["dram_write"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic,
                "traffic_source": "profiles/traffic_r01.json (ncu dram bytes, same launch)",
                "kernel": dom, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes,
                "note": "4 B/voxel-view (SURVEY 8d); the kernel is issue-bound, see DESIGN.md"}
    # the bound that binds: instruction issue (ncu smsp__issue_active of the
    # same kernel, committed capture)
    issue = None
    sp = os.path.join(ROOT, "profiles", "ncu_r01_fwd_summary.txt" if pm >= bm else "ncu_r01_bwd_summary.txt")
    if os.path.exists(sp):
        with open(sp) as f:
            for line in f:
                if "smsp__issue_active.avg.pct_of_peak_sustained_active" in line:
                    issue = float(line.split()[-1]) / 100.0
    if issue is not None:
        roofline["issue"] = {"bound": "issue", "frac": issue, "metric": "smsp__issue_active",
                             "source": os.path.relpath(sp, ROOT) + " (ncu --set full, 16-view launch)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(args.precision)
        except Exception as e:  # the checker library may be absent on a fresh box
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "unavailable",
                   "sample": str(e)[:200]}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f32 (f64 cut geometry + anchors)" if args.precision == "exact" else "f32",
               "data": "synthetic",
               "config": {"workload": WORKLOAD, "precision": args.precision,
                          "global_views": V, "volume": list(c["counts"]),
                          "detector": [c["rows"], c["cols"]],
                          "parallelism": f"view-sharded x{world}",
                          "l2": "inputs larger than L2 (512 MiB volume, 587 MB stack)"},
               "p_ms": pm, "bp_ms": bm, "cgls": cgls, "reduce_scatter_ms": rm if world > 1 else 0.0,
               "p_gvps": work / (pm * 1e-3) if world == 1 else None,
               "bp_gvps": work / (bm * 1e-3) if world == 1 else None,
               # per step: cvp_brick_kernel<FWD> + apply_scale_kernel, cvp_brick_kernel<BWD>
               # (profiles/launches_r01.csv); the cut table was built (and the brick
               # shape timed) in the warm-up and is reused; the stack memset is a
               # cudaMemsetAsync
               "gpu_launches": 3 * args.steps,
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk}
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
