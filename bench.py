"""Headline benchmark: exact CVP project + backproject, 512^3 x 496 views on a
616x480 detector (BASELINE.json configs[2]; SURVEY §8d pinned geometry).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision exact|relaxed]
  python bench.py --impl reference ...      # the reference's CPU path (oracle/_ref)

One step = one forward projection of the whole volume into all views + one
backprojection of a whole stack (the two halves of a CGLS iteration). The
metric counts voxel-view pairs: value = N1*N2*N3*V / (t_P + t_BP) / 1e9,
whole job over all ranks. Multi-GPU: one process per GPU (``--gpus N``
re-launches itself under torch.distributed.run when WORLD_SIZE is unset);
views are sharded across ranks, P needs no exchange, BP partial volumes are
summed with an NCCL reduce-scatter over z-slabs (the path's one real exchange
step). The total job is fixed: "scaling": "strong".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
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
REF_SAMPLE_VIEWS = 16  # evenly spaced angles the reference arm cycles through


def config_dict(args, world):
    """The `config` of both arms (identical keys and values)."""
    c = CONFIG
    return {"workload": WORKLOAD, "precision": args.precision, "global_views": c["n_views"],
            "volume": list(c["counts"]), "detector": [c["rows"], c["cols"]],
            "parallelism": f"view-sharded x{world}",
            "l2": "inputs larger than L2 (512 MiB volume, 587 MB stack)"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _profile_file(*names):
    """Newest committed profile summary of the given names (r02 before r01)."""
    for n in names:
        p = os.path.join(ROOT, "profiles", n)
        if os.path.exists(p):
            return p
    return None


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


# ---------------------------------------------------------------------------
# the reference's CPU path (test infrastructure: oracle/_ref is the reference
# compiled from its own sources; oracle/ C restatement if it is absent)

def _checker():
    from oracle import pyoracle
    if pyoracle.reference_available():
        return pyoracle.Reference(), "reference"
    return pyoracle.Restatement(), "port"


class RefSample:
    """The c3 workload through the reference's own API on the host cores: the
    geometry and data come from the reference library itself
    (make_circular_trajectory, fill_uniform01), nothing from this package."""

    def __init__(self, precision, threads):
        from oracle import pyoracle
        c = CONFIG
        self.chk, self.kind = _checker()
        self.threads = threads if self.kind == "reference" else 1
        self.views = self.chk.circular_trajectory(c["sid"], c["sdd"], c["n_views"], c["arc"],
                                                  c["rows"], c["cols"], c["pw"], c["ph"])
        self.nvox = int(np.prod(c["counts"]))
        # the GPU arm computes on float32 copies of the same draws
        self.x = self.chk.fill_uniform01(self.nvox, 7).astype(np.float32).astype(np.float64)
        self.npx = c["rows"] * c["cols"]
        self.opts = (1, 1, 0 if precision == "exact" else 1, 1)
        self.Scene = pyoracle.Scene
        # 16 evenly spaced angles (every 31st view of 496); steps cycle through them
        self.angles = [int(round(i * c["n_views"] / REF_SAMPLE_VIEWS))
                       for i in range(REF_SAMPLE_VIEWS)]
        os.environ.setdefault("OMP_NUM_THREADS", str(self.threads))

    def step(self, s, per_step):
        """P + BP of `per_step` sample views (step s takes the next ones of the
        16-angle cycle, interleaved so every step spans the circle)."""
        c = CONFIG
        stride = max(1, REF_SAMPLE_VIEWS // per_step)
        idx = [self.angles[(s + j * stride) % REF_SAMPLE_VIEWS] for j in range(per_step)]
        sc = self.Scene(c["counts"], c["voxel"], c["rows"], c["cols"], c["pw"], c["ph"],
                        self.views[idx])
        b = self.chk.fill_uniform01(self.npx * per_step, 8 + s).astype(np.float32).astype(np.float64)
        t0 = time.perf_counter()
        self.chk.project_cvp(sc, self.x, self.opts, threads=self.threads)
        t1 = time.perf_counter()
        self.chk.backproject_cvp(sc, b, self.opts, threads=self.threads)
        t2 = time.perf_counter()
        return idx, t1 - t0, t2 - t1


def cpu_baseline_sample(precision, per_step=2, steps=1):
    """`steps` reference steps (P + BP of `per_step` views each) on the host
    cores; Gvoxel-views/s over the timed sample."""
    rs = RefSample(precision, os.cpu_count() or 1)
    rs.step(0, 1)  # the first OpenMP call is several times slower
    tp = tb = 0.0
    seen = []
    for s in range(steps):
        idx, a, b = rs.step(s, per_step)
        tp, tb = tp + a, tb + b
        seen += idx
    work = rs.nvox * per_step * steps / 1e9
    return {"value": work / (tp + tb), "unit": UNIT, "cores": rs.threads, "kind": rs.kind,
            "cpu_model": cpu_model(),
            "sample": f"{per_step * steps} of the 496 views ({sorted(set(seen))}) at full 512^3 / "
                      f"616x480, {precision} CVP, P {tp:.2f} s + BP {tb:.2f} s on {rs.threads} "
                      f"threads of {cpu_model()}",
            "p_gvps": work / tp, "bp_gvps": work / tb}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    rs = RefSample(args.precision, os.cpu_count() or 1)
    per = args.ref_views
    times, seen = [], []
    for s in range(args.warmup + args.steps):
        idx, tp, tb = rs.step(s, per)
        if s >= args.warmup:
            times.append((tp, tb))
        seen += idx
    step_s = [a + b for a, b in times]
    work = rs.nvox * per / 1e9  # Gvoxel-views per reference step
    val = work / statistics.mean(step_s)
    c = CONFIG
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": statistics.mean(step_s) * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64" if args.precision == "exact" else "f32", "data": "synthetic",
           "config": config_dict(args, world),
           "step_definition": f"P + BP of {per} of the 496 views (bounded sample of the c3 job; "
                              f"steps cycle through {REF_SAMPLE_VIEWS} evenly spaced angles)",
           "full_job_ms_extrapolated": float(np.prod(c["counts"])) * c["n_views"] / 1e9 / val * 1e3,
           "views_timed": sorted(set(seen)),
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": rs.threads, "kind": rs.kind,
                            "cpu_model": cpu_model(),
                            "sample": f"{per} views per step, {args.steps} timed steps, "
                                      f"{len(set(seen))} distinct angles"},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    sys.stdout.flush()
    return 0


# ---------------------------------------------------------------------------
# multi-process launch: one process per GPU

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(n, argv):
    """Re-run this script as n ranks under torch.distributed.run (rank 0
    prints the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + argv
    return subprocess.run(cmd).returncode


def selftest_spawn():
    """CPU check of the launch plumbing (tests/test_bench_spawn.py): every rank
    joins a gloo group, rank 0 prints how many ranks it saw."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if dist.get_rank() == 0:
        print(json.dumps({"n_gpus": dist.get_world_size(), "ranks_seen": int(t.item())}))
    dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# the product arm

def run_native(args):
    import torch
    import torch.distributed as dist
    import paper_2110_09841_b200 as cb
    from paper_2110_09841_b200 import _native as N
    import ctypes as C

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CVPB_BENCH_SHARE_GPU=1 (code-path check on a one-GPU box, never a
    # measurement): every rank on cuda:0 over gloo
    share = os.environ.get("CVPB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coll_dev = "cpu" if share else "cuda"  # device of the small timing all-reduces

    def reduce_scatter(out, full):
        # NCCL reduce-scatter; gloo (the shared-GPU code-path check) has no
        # CUDA reduce-scatter, so it all-reduces a host copy and slices
        if not share:
            dist.reduce_scatter_tensor(out, full)
            return
        h = full.cpu()
        dist.all_reduce(h)
        out.copy_(h[rank * out.numel():(rank + 1) * out.numel()])

    c = CONFIG
    det = cb.DetectorGeometry.make(c["rows"], c["cols"], c["pw"], c["ph"])
    geom = cb.VolumeGeometry.make(c["counts"], c["voxel"])
    views = cb.make_circular_trajectory(c["sid"], c["sdd"], c["n_views"], c["arc"], det)
    V = len(views)
    v0 = rank * V // world  # rank r owns views [v0, v1)
    v1 = (rank + 1) * V // world
    nvox = geom.voxel_count()
    npx = det.pixel_count()
    scene = cb.DeviceScene(geom, det, views, device=local)
    opts = cb.CvpOptions(precision=cb.CvpPrecision.Double if args.precision == "exact"
                         else cb.CvpPrecision.Single)
    x = torch.from_numpy(cb.fill_uniform01(nvox, 7).astype(np.float32)).reshape(geom.shape()).cuda()
    b_all = cb.fill_uniform01(npx * V, 8)
    b = torch.from_numpy(b_all[v0 * npx:v1 * npx].astype(np.float32)).reshape(
        v1 - v0, det.rows, det.cols).cuda()
    p = scene.new_stack(v1 - v0)
    bp = scene.new_volume()
    slab = torch.empty(nvox // world if world > 1 else 1, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    # N > 1: the backprojection fused with its reduce-scatter — every rank's
    # bricks add into the owning rank's z-slab over CUDA IPC / NVLink
    # (parallel.PeerSlabs); NCCL reduce_scatter_tensor when that is off
    peers = None
    if world > 1:
        from paper_2110_09841_b200 import parallel as par
        if par.fused_reduce_scatter_ok(scene, "cvp"):
            try:
                peers = par.PeerSlabs(scene)
            except RuntimeError:  # (every rank alike) -> NCCL reduce-scatter
                peers = None

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        scene.project_cvp(x, p, opts, view_begin=v0, view_count=v1 - v0)
        if ev:
            ev[1].record(stream)
        if peers is not None:
            peers.scatter(b, opts, v0, v1 - v0)  # (barrier: receive regions free)
        else:
            scene.backproject_cvp(b, bp, opts, view_begin=v0, view_count=v1 - v0)
        if ev:
            ev[2].record(stream)
        if peers is not None:
            peers.finish()  # barrier: every rank's stores landed; own slab = ordered sum
        elif world > 1:
            reduce_scatter(slab, bp.view(-1))
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
                          statistics.mean(rs_ms)], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, pm, bm, rm = t.tolist()
    else:
        pm, bm, rm = statistics.mean(p_ms), statistics.mean(bp_ms), statistics.mean(rs_ms)
    ms_per_step = total_ms / args.steps
    work = nvox * V / 1e9  # Gvoxel-views per application, whole job
    value = work / (ms_per_step * 1e-3)
    del b_all

    # the other precision of the same P + BP (BASELINE configs[2] names exact
    # and relaxed): device-timed like the headline, 2 warm + 3 timed steps,
    # reported beside it (N = 1 only; the headline stays args.precision)
    other = None
    if world == 1 and not args.no_other_precision:
        oprec = "relaxed" if args.precision == "exact" else "exact"
        oopts = cb.CvpOptions(precision=cb.CvpPrecision.Double if oprec == "exact"
                              else cb.CvpPrecision.Single)
        oe = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        pms, bms = [], []
        for it in range(5):
            oe[0].record(stream)
            scene.project_cvp(x, p, oopts, view_begin=v0, view_count=v1 - v0)
            oe[1].record(stream)
            scene.backproject_cvp(b, bp, oopts, view_begin=v0, view_count=v1 - v0)
            oe[2].record(stream)
            torch.cuda.synchronize()
            if it >= 2:
                pms.append(oe[0].elapsed_time(oe[1]))
                bms.append(oe[1].elapsed_time(oe[2]))
        opm, obm = statistics.mean(pms), statistics.mean(bms)
        other = {"precision": oprec, "value": work / ((opm + obm) * 1e-3), "unit": UNIT,
                 "p_gvps": work / (opm * 1e-3), "bp_gvps": work / (obm * 1e-3), "steps": 3,
                 "how": "same P + BP, device-timed with CUDA events after 2 warm-up steps"}

    # ---- e2e through the reference-facing C-ABI host path ------------------
    # N = 1: cvpb_project_cvp_host + cvpb_backproject_cvp_host (project_cvp_into /
    # backproject_cvp_into with float64 host buffers). N > 1, per rank, on a
    # context holding its own views: cvpb_project_cvp_host (full volume in, its
    # projections out) + cvpb_backproject_cvp_host_partial (its stack shard in,
    # partial volume on the device) + NCCL reduce-scatter + cvpb_vec_to_host64
    # of its z-slab. Inputs in pinned float64 host memory, copies and
    # conversions inside the timed region; max over ranks of the wall time.
    e2e = None
    if not args.no_e2e:
        x64 = torch.from_numpy(cb.fill_uniform01(nvox, 7)).pin_memory()
        b64 = torch.from_numpy(cb.fill_uniform01(npx * V, 8)[v0 * npx:v1 * npx].copy()).pin_memory()
        p64 = torch.empty((v1 - v0) * npx, dtype=torch.float64).pin_memory()
        out_n = nvox // world if world > 1 else nvox
        o64 = torch.empty(out_n, dtype=torch.float64).pin_memory()
        x64n, b64n, p64n, o64n = x64.numpy(), b64.numpy(), p64.numpy(), o64.numpy()
        e2e_steps = max(1, min(args.steps, 3))
        if world == 1:
            shard = scene

            def e2e_step():
                shard.project_cvp_host(x64n, p64n, opts)
                shard.backproject_cvp_host(b64n, o64n, opts)
        else:
            shard = cb.DeviceScene(geom, det, views[v0:v1], device=local)
            L = N.lib()
            ex = cb.ExecPolicy()
            st = C.c_void_p(stream.cuda_stream)

            def e2e_step():
                shard.project_cvp_host(x64n, p64n, opts)
                N.check(L.cvpb_backproject_cvp_host_partial(
                    shard._h, C.byref(opts._c()), C.byref(ex._c()), C.c_void_p(b64n.ctypes.data),
                    C.c_void_p(bp.data_ptr()), st))
                reduce_scatter(slab, bp.view(-1))
                N.check(L.cvpb_vec_to_host64(shard._h, C.c_void_p(slab.data_ptr()),
                                             C.c_void_p(o64n.ctypes.data), slab.numel(), st))

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            d = torch.tensor([dt], device=coll_dev)
            dist.all_reduce(d, op=dist.ReduceOp.MAX)
            dt = float(d.item())
        e2e = {"value": work / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(x64.numel() * 8 + b64.numel() * 8),
               "d2h_bytes_per_step": int(p64.numel() * 8 + o64.numel() * 8),
               "path": ("cvpb_project_cvp_host + cvpb_backproject_cvp_host" if world == 1 else
                        "per rank: cvpb_project_cvp_host + cvpb_backproject_cvp_host_partial + "
                        "NCCL reduce-scatter + cvpb_vec_to_host64 (bytes per rank)") +
                       " (float64 pinned host buffers, conversions and copies inside the timed "
                       "region)",
               "steps": e2e_steps}
        if shard is not scene:
            shard.close()
        del x64, b64, p64, o64

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
                "how": "device-resident cvpb_cgls on the c3 scene (1 P + 1 BP + fused "
                       "float64-accumulated vector kernels per iteration, scalars on the device); "
                       "ms/iter = (T(1+n) - T(1)) / n, wall clock around synchronized calls"}
        del bt
    elif args.cgls_iters > 0:
        # view-sharded CGLS (parallel.distributed_cgls): x, s, p as z-slabs,
        # r, q as view shards; all-gather of p before each P, reduce-scatter
        # of the BP partials, all-reduced float64 scalars
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
        dt = torch.tensor([(tb - ta) / args.cgls_iters], device=coll_dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        cgls = {"ms_per_iter": float(dt.item()) * 1e3, "iterations_timed": args.cgls_iters,
                "residual_ratio": r.residual_norms[-1] / r.residual_norms[0],
                "how": f"view-sharded CGLS over {world} ranks on the c3 scene (parallel."
                       "distributed_cgls: slab-resident x/s/p, all-gather of p + "
                       + ("backprojection fused with the reduce-scatter (CUDA IPC slabs) "
                          if op.adjoint_scatter is not None else "NCCL reduce-scatter ")
                       + "per iteration); ms/iter = (T(1+n) - T(1)) / n, max over ranks"}

    # ---- roofline of the dominant kernel -----------------------------------
    hbm, peak_src = _peaks()
    dom_ms = max(pm, bm)
    fwd_dom = pm >= bm
    dom = "cvp_brick_kernel<EXACT,FWD>" if fwd_dom else "cvp_brick_kernel<EXACT,BWD>"
    views_here = v1 - v0
    alg_bytes = 4.0 * nvox * views_here  # 4 B per voxel-view
    achieved = alg_bytes / (dom_ms * 1e-3) / 1e9
    traffic, traffic_src = None, None
    tp = _profile_file("traffic_r02.json", "traffic_r01.json")
    if tp and world == 1:
        with open(tp) as f:
            t = json.load(f).get(dom)
        if t:
            traffic = t["dram_read"] + t["dram_write"]
            traffic_src = os.path.relpath(tp, ROOT) + " (ncu dram bytes of the same 496-view launch)"
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": dom, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes,
                "note": "4 B/voxel-view (SURVEY 8d); the kernel is issue-bound, see DESIGN.md"}
    # secondary roof: shared-memory int32 atomic updates of the
    # forward's detector tile, U = 4.22 updates per voxel-view at c3 (the
    # reference's collect_cut_records over 20,000 random voxel-views), against
    # the microbenchmarked red.shared.add.s32 peak (tools/smem_atomic_peak.cu)
    ap = _profile_file("smem_atomic_peak_r02.json")
    if ap:
        with open(ap) as f:
            peak_ups = json.load(f)["results"][0]["updates_per_s"]
        ups = work / world / (pm * 1e-3) * 1e9 * 4.22
        roofline["smem_atomic"] = {"bound": "shared atomics", "achieved": ups, "peak": peak_ups,
                                   "unit": "updates/s", "frac": ups / peak_ups,
                                   "U_per_voxel_view": 4.22,
                                   "source": os.path.relpath(ap, ROOT)}
    sp = (_profile_file("ncu_r02_fwd_summary.txt", "ncu_r01_fwd_summary.txt") if fwd_dom else
          _profile_file("ncu_r02_bwd_summary.txt", "ncu_r01_bwd_summary.txt"))
    if sp:
        # the summary may list several kernels: take the dominant direction's
        # block (FWD: template flag 1, BWD: 0) and only a finite value
        issue, want, in_block = None, ("<1, 1," if fwd_dom else "<1, 0,"), False
        with open(sp) as f:
            for line in f:
                if line.startswith("=="):
                    in_block = want in line
                elif in_block and "smsp__issue_active.avg.pct_of_peak_sustained_active" in line:
                    try:
                        val = float(line.split()[-1]) / 100.0
                    except ValueError:
                        continue
                    if math.isfinite(val) and issue is None:
                        issue = val
        if issue is not None:
            roofline["issue"] = {"bound": "issue", "frac": issue, "metric": "smsp__issue_active",
                                 "source": os.path.relpath(sp, ROOT) + " (ncu --set full)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_sample(args.precision, per_step=2, steps=2)
            # the reference's other precision (report Double and
            # Single), a smaller sample: one step of 2 views
            oc = cpu_baseline_sample("relaxed" if args.precision == "exact" else "exact",
                                     per_step=2, steps=1)
            cpu["other_precision"] = {k: oc[k] for k in ("value", "p_gvps", "bp_gvps", "sample")}
        except Exception as e:  # the checker library may be absent on a fresh box
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "unavailable",
                   "sample": str(e)[:200]}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f32 (f64 cut geometry + anchors)" if args.precision == "exact" else "f32",
               "data": "synthetic",
               "config": config_dict(args, world),
               "p_ms": pm, "bp_ms": bm, "cgls": cgls, "reduce_scatter_ms": rm if world > 1 else 0.0,
               "exchange": ("none" if world == 1 else "fused backprojection + reduce-scatter (stores into CUDA IPC receive regions over NVLink, ordered local sums)" if peers is not None else "NCCL reduce_scatter_tensor"),
               "p_gvps": work / world / (pm * 1e-3), "bp_gvps": work / world / (bm * 1e-3),
               # per step: cvp_brick_kernel<FWD> + apply_scale_kernel, cvp_brick_kernel<BWD>
               # (profiles/launches_r0*.csv); the cut table was built (and the brick
               # shape timed) in the warm-up and is reused; the stack memset is a
               # cudaMemsetAsync
               "gpu_launches": 3 * args.steps,
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
               "other_precision": other}
        print(json.dumps(out))
        sys.stdout.flush()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precision", choices=["exact", "relaxed"], default="exact")
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--ref-views", type=int, default=2,
                    help="reference arm: sample views per step (P + BP each)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other-precision", action="store_true")
    ap.add_argument("--cgls-iters", type=int, default=10,
                    help="device-resident CGLS iterations timed for cgls.ms_per_iter (0 = skip)")
    ap.add_argument("--selftest-spawn", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch as args.gpus ranks
        return spawn_ranks(args.gpus, sys.argv[1:])
    if args.selftest_spawn:
        return selftest_spawn()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
