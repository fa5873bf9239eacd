#!/usr/bin/env python
"""Benchmark: forward + backward(pose gradient) pose-estimation iterations/s on
a 1M-Gaussian, 1008x756 synthetic scene (BASELINE.json config C3), one
process per GPU, views sharded across ranks with no data-path collective.

One step = one pose_descent iteration (render -> L1+SSIM loss -> backward with
the SE(3) pose gradient -> pose step; pipelines.cpp:66-90) for each of the
rank's views, all inputs resident in HBM. `value` = iterations/s over all
ranks (max-over-ranks device time). `e2e` = the same metric through the public
C-ABI call a user makes (gsb_estimate_pose) starting from host FP64 images,
host<->device copies inside the timed region. `--impl reference` times the
reference algorithm on the host CPU (oracle port) on the same
workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_GAUSS = 1_000_000
WIDTH, HEIGHT = 1008, 756
TOTAL_VIEWS = 64            # C3: 64 independent views
VIEWS_PER_GPU = int(os.environ.get("GSB_BENCH_VIEWS_PER_GPU", "8"))  # weak scaling: 8 per rank (64 at 8 GPUs)
SCENE_SEED = 3
NOISE_SEED = 1002
SH_DEGREE = 3
METRIC = "fwd+bwd(pose grad) iters/sec @1M Gaussians 1008x756"


def log_scale_offset(n):
    """log_scales += ln(500/N)/3 keeps the reference's 500-Gaussian footprint density."""
    return math.log(500.0 / n) / 3.0 if n > 500 else 0.0


# Plumbing check on a box with fewer GPUs than ranks (GSB_BENCH_SHARE_GPU=1):
# every rank uses GPU 0, torch.distributed runs over gloo and the NCCL joint
# leg is skipped. Only for exercising the multi-rank code path; the numbers
# of such a run are not a measurement of N GPUs.
SHARE_GPU = os.environ.get("GSB_BENCH_SHARE_GPU", "0") == "1"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, 0 if SHARE_GPU else local


def _reduce_max(dist, v, local):
    """max over ranks of a host float (device tensor for NCCL, host for gloo)."""
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if SHARE_GPU else f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------- scene
def all_views():
    """GT poses (forward-facing, synth.cpp:86-90) and perturbed inits
    (perturb_pose 15 deg / 0.15, eval.cpp:130-146, Rng(1002)) for all 64 views."""
    from paper_2410_08743_b200 import gsb
    gt = gsb.synth_poses(SCENE_SEED, N_GAUSS, SH_DEGREE, 1, TOTAL_VIEWS)
    rng = gsb.PoseRng(NOISE_SEED)
    init = np.stack([rng.perturb_pose(p, 15.0, 0.15) for p in gt])
    return gt, init


def my_views(rank, ws):
    return [(rank * VIEWS_PER_GPU + k) % TOTAL_VIEWS for k in range(VIEWS_PER_GPU)]


def fp32_peak_tflops(sm_count, clock_mhz):
    return sm_count * 128 * 2 * clock_mhz * 1e6 / 1e12


# ------------------------------------------------------------ our arm
def run_ours(args, ws, rank, local):
    from paper_2410_08743_b200 import gsb
    dist = None
    if ws > 1:
        import torch
        import torch.distributed as td
        if SHARE_GPU:
            td.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            td.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = td
    ctx = gsb.Context(local)
    fp32 = gsb.measure_fp32_peaks(local)  # FFMA / MUFU microbenchmarks: the FP32 roofline denominators
    cloud = gsb.Cloud(ctx, N_GAUSS, SH_DEGREE)
    cloud.synth(SCENE_SEED, log_scale_offset(N_GAUSS))
    gt, init = all_views()
    intr = gsb.synth_intrinsics(WIDTH, HEIGHT)
    views = my_views(rank, ws)
    host_targets, images = {}, {}
    for v in views:
        cam = gsb.Camera.from_pose12(*intr, WIDTH, HEIGHT, gt[v])
        host_targets[v] = gsb.render(ctx, cloud, cam).image
        images[v] = gsb.Image(ctx, host_targets[v])
    budget = max(100, args.warmup + 2 * args.steps + 4)
    cfg = gsb.PoseConfig.default(budget=budget, pose_converged_eps=0.0)
    sessions = [gsb.PoseSession(ctx, cloud, images[v], intr, init[v], cfg) for v in views]
    batch = gsb.PoseBatch(ctx, sessions)

    def step():
        batch.step_async(1)  # one CUDA-graph replay advances every view one iteration; no host round trip

    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    batch.sync()  # re-runs any iteration discarded for entry-capacity growth
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launch_count()
    discarded0 = batch.discarded()
    ctx.timer_start()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dev_ms = ctx.timer_stop()
    wall_s = time.perf_counter() - t0
    launches = ctx.launch_count() - launches0
    clk = clocks.stop()
    batch.sync()
    discarded = batch.discarded() - discarded0
    if discarded:
        raise RuntimeError(f"{discarded} iteration(s) discarded for entry-capacity growth inside the timed region")
    # Attribution (untimed, after the timed region): per-stage CUDA event
    # nodes (1) inside every branch of the same batch graph ("live": branch
    # wall time, queueing behind the other branches included) and (2) around
    # every stage of each session's own graph run one at a time ("solo": the
    # kernel durations the roofline uses).
    ctx.set_profiling(True)
    batch.step_async(1)  # recaptures the batch graph with event nodes (untimed)
    batch.sync()
    live_tot, solo_tot = {}, {}
    ctx.timer_start()
    for _ in range(args.steps):
        batch.step_async(1)
        for s in sessions:
            for k, v in s.stage_times().items():
                live_tot[k] = live_tot.get(k, 0.0) + v
    live_ms = ctx.timer_stop()
    batch.sync()
    if batch.discarded() - discarded0:
        raise RuntimeError("iterations discarded during the attribution pass")
    batch.close()
    for s in sessions:
        s.step_async(1)  # own graphs, with event nodes (untimed)
    ctx.synchronize()
    ctx.timer_start()
    for _ in range(args.steps):
        for s in sessions:
            s.step_async(1)
            for k, v in s.stage_times().items():
                solo_tot[k] = solo_tot.get(k, 0.0) + v
    solo_ms = ctx.timer_stop()
    ctx.set_profiling(False)
    if dist:
        dev_ms = _reduce_max(dist, dev_ms, local)
    iters = VIEWS_PER_GPU * ws * args.steps
    value = iters / (dev_ms / 1e3)
    for s in sessions:
        s.read()
    fi = sessions[0].frame_info()
    res = sessions[0].read()
    # ---- e2e: gsb_estimate_poses from host FP64 images (the user-facing call
    # for C3's independent views: one call per GPU over its views)
    e2e_iters = args.e2e_iters
    e2e_cfg = gsb.PoseConfig.default(budget=e2e_iters, pose_converged_eps=0.0)
    # one untimed warm-up call (first-call allocations, graph instantiation)
    warm = [gsb.Image(ctx, host_targets[v]) for v in views]
    gsb.estimate_poses(ctx, cloud, warm, intr, init[views], gsb.PoseConfig.default(budget=4, pose_converged_eps=0.0))
    del warm
    if dist:
        dist.barrier()
    ctx.synchronize()
    t0 = time.perf_counter()
    h2d = d2h = 0
    imgs = []
    for v in views:
        imgs.append(gsb.Image(ctx, host_targets[v]))          # H2D of the view's frame
        h2d += host_targets[v].size * 4 + 12 * 8            # FP32 planes uploaded + pose
        d2h += 12 * 8 + 8 + 4                                 # pose, loss, steps
    out = gsb.estimate_poses(ctx, cloud, imgs, intr, init[views], e2e_cfg)
    assert all(int(k) == e2e_iters for k in out["steps"])
    del imgs
    ctx.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist:
        e2e_s = _reduce_max(dist, e2e_s, local)
    e2e_value = VIEWS_PER_GPU * ws * e2e_iters / e2e_s

    joint = None if (args.no_joint or (SHARE_GPU and ws > 1)) else run_joint(args, ws, rank, local, dist)
    single = None if args.no_joint else run_single_view(args, ws, rank, local)
    kernel_only = None if args.no_joint else run_kernel_only(args, ws, rank, local)
    c3_job = None if args.no_c3_job else run_c3_job(args, ws, rank, local, ctx, cloud, gt, init, intr)
    out = None
    if rank == 0:
        # roofline for the dominant stage, from the solo kernel durations
        per_iter_stage_ms = {k: v / (VIEWS_PER_GPU * args.steps) for k, v in solo_tot.items()}
        live_stage_ms = {k: v / (VIEWS_PER_GPU * args.steps) for k, v in live_tot.items()}
        dom = max(per_iter_stage_ms, key=per_iter_stage_ms.get)
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        cpu = None
        work = None
        if not args.no_cpu_baseline and ws == 1:
            cpu = cpu_baseline(args, gt, init, views, intr)
        if not args.no_work_counts:
            work = work_counts([(gt[v], init[v]) for v in views], intr)
        roof = roofline(dom, per_iter_stage_ms[dom], fi, work, peaks, clk, fp32)
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dev_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32 (fp64 geometry, pose step and loss accumulation)",
            "data": "synthetic (synth.cpp draw sequence, seed 3; targets rendered at GT poses)",
            "config": common_config(ws),
            "e2e": {"value": round(e2e_value, 3), "unit": "iters/s", "h2d_bytes_per_step": int(h2d * ws / e2e_iters),
                    "d2h_bytes_per_step": int(d2h * ws / e2e_iters),
                    "how": f"gsb_estimate_poses over the GPU's views from host FP64 HWC images, {e2e_iters} "
                           "iterations; bytes per iteration-of-all-views"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "roofline": roof,
            "stages_ms_per_iter": {k: round(v, 4) for k, v in per_iter_stage_ms.items()},
            # the metric's second half: pose-estimation views completed per second
            # (C3's fixed budget of 100 pose_descent iterations per view, early exits off)
            "pose_est_views_per_s": {"value": round(value / 100.0, 3), "e2e": round(e2e_value / 100.0, 3),
                                     "iterations_per_view": 100},
            "scene": {"n_splats": int(fi.n_splats), "n_entries": int(fi.n_entries)},
            "wall_s": round(wall_s, 3),
            "attribution": {
                "how": "stages_ms_per_iter / roofline: CUDA event nodes around every stage of each session's own "
                       f"graph, sessions one at a time ({args.steps} iterations each, same process, same "
                       "buffers); live: event nodes inside every branch of the timed pose-batch graph "
                       "(the shared multi-view preprocess charged once per replay)",
                "live_ms_per_step": round(live_ms / args.steps, 4),
                "solo_ms_per_step": round(solo_ms / args.steps, 4),
                "live_stages_ms_per_iter (branch wall time incl. queueing)": {
                    k: round(v, 4) for k, v in live_stage_ms.items()}},
            "discarded_in_timed_region": int(discarded),
            "build_id": gsb.build_id()[:16],
            "pose_check": {"view": int(views[0]), "final_loss": res["final_loss"], "steps": res["steps"]},
        }
        if joint is not None:
            out["joint_c4"] = joint
        if single is not None:
            out["single_view_c2"] = single
        if kernel_only is not None:
            out["kernel_only_c3"] = kernel_only
        if c3_job is not None:
            out["c3_job_1gpu"] = c3_job
        out["fp32_peaks_measured"] = {k: round(v, 2) for k, v in fp32.items()}
        if cpu is not None:
            out["cpu_baseline"] = cpu
        if work is not None:
            out["work_counts"] = work
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


# ------------------------------------------------ C4: joint DP (secondary)
C4_N, C4_VIEWS, C4_SEED = 300_000, 20, 4
C2_N, C2_SEED = 300_000, 2


def run_single_view(args, ws, rank, local):
    """Secondary line, config C2: one view's pose_descent on a
    300k-Gaussian forward-facing scene at 1008x756 (seed 2, perturb 15 deg /
    0.15 from Rng(1002)) through one session — the single-view latency path
    (one CUDA-graph replay per iteration, no other views to overlap with).
    Rank 0 only (a replica per GPU would measure the same thing)."""
    if rank != 0:
        return None
    from paper_2410_08743_b200 import gsb
    ctx = gsb.Context(local)
    cloud = gsb.Cloud(ctx, C2_N, SH_DEGREE)
    cloud.synth(C2_SEED, log_scale_offset(C2_N))
    gt = gsb.synth_poses(C2_SEED, C2_N, SH_DEGREE, 1, 1)
    init = gsb.PoseRng(NOISE_SEED).perturb_pose(gt[0], 15.0, 0.15)
    intr = gsb.synth_intrinsics(WIDTH, HEIGHT)
    img = gsb.Image(ctx, gsb.render(ctx, cloud, gsb.Camera.from_pose12(*intr, WIDTH, HEIGHT, gt[0])).image)
    steps = max(args.steps, 10)
    s = gsb.PoseSession(ctx, cloud, img, intr, init,
                        gsb.PoseConfig.default(budget=args.warmup + steps + 4, pose_converged_eps=0.0))
    s.step(args.warmup)
    ctx.timer_start()
    s.step_async(steps)  # graph replays back to back, no host round trip
    ms = ctx.timer_stop()
    res = s.read()  # (re-runs any iteration discarded for capacity growth)
    assert res["steps"] == args.warmup + steps, res["steps"]
    return {"workload": f"C2 single-view pose estimation: {C2_N} Gaussians SH3, {WIDTH}x{HEIGHT}, forward-facing, "
                        "perturb 15deg/0.15, one session", "iters_per_s": round(steps / (ms / 1e3), 2),
            "ms_per_iter": round(ms / steps, 4), "steps": steps}


def run_kernel_only(args, ws, rank, local):
    """SURVEY §8d metric (1), kernel-only variant: render -> render_backward
    (pose-only) through the reference-API calls with a fixed random d_image
    already on the device (tests/gradcheck.hpp:204-208 reuses one d_image),
    C3's scene at view 0's initial pose; no loss, no pose step. Host-driven:
    two C-ABI calls per iteration (the backward returns d_pose to the host),
    so this includes the per-call launch and synchronisation a drop-in caller
    pays, unlike the graph-replayed sessions. Rank 0 only."""
    if rank != 0:
        return None
    from paper_2410_08743_b200 import gsb
    ctx = gsb.Context(local)
    cloud = gsb.Cloud(ctx, N_GAUSS, SH_DEGREE)
    cloud.synth(SCENE_SEED, log_scale_offset(N_GAUSS))
    _, init = all_views()
    intr = gsb.synth_intrinsics(WIDTH, HEIGHT)
    cam = gsb.Camera.from_pose12(*intr, WIDTH, HEIGHT, init[0])
    d_img = gsb.Image(ctx, np.random.default_rng(7).uniform(-1e-6, 1e-6, (HEIGHT, WIDTH, 3)))
    frame = gsb.Frame(ctx)

    def iteration():
        out = gsb.render(ctx, cloud, cam, frame=frame, want_image=False)
        return gsb.render_backward(ctx, cloud, cam, out, d_img, pose_only=True)[1]

    for _ in range(max(args.warmup, 3)):
        iteration()
    steps = max(args.steps, 10)
    ctx.synchronize()
    launches0 = ctx.launch_count()
    t0 = time.perf_counter()
    ctx.timer_start()
    for _ in range(steps):
        dp = iteration()
    ms = ctx.timer_stop()
    wall = time.perf_counter() - t0
    assert np.all(np.isfinite(dp)) and np.any(dp != 0.0)
    return {"workload": f"render + render_backward(pose-only), fixed random d_image on the device, C3 scene "
                        f"({N_GAUSS} Gaussians SH{SH_DEGREE}, {WIDTH}x{HEIGHT}) at view 0's initial pose, "
                        "one C-ABI call each (gsb_render, gsb_render_backward_image)",
            "iters_per_s": round(steps / (ms / 1e3), 2), "ms_per_iter": round(ms / steps, 4),
            "wall_ms_per_iter": round(wall * 1e3 / steps, 4), "steps": steps,
            "launches_per_iter": round((ctx.launch_count() - launches0) / steps, 1)}


def run_joint(args, ws, rank, local, dist):
    """Config C4: joint reconstruction + pose refinement on 20 LLFF-shaped
    views (300k Gaussians SH3, 1008x756), data parallel: one view per GPU per
    step, NCCL all-reduce of the gradient planes inside the step graph.
    Returns steps/s and views/s (whole job, max-over-ranks device time)."""
    from paper_2410_08743_b200 import gsb
    ctx = gsb.Context(local)
    comm = None
    if ws > 1:
        uid = [gsb.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = gsb.Comm(ctx, uid[0], rank, ws)
    gt_cloud = gsb.Cloud(ctx, C4_N, SH_DEGREE)
    gt_cloud.synth(C4_SEED, log_scale_offset(C4_N))
    gt = gsb.synth_poses(C4_SEED, C4_N, SH_DEGREE, 1, C4_VIEWS)
    intr = gsb.synth_intrinsics(WIDTH, HEIGHT)
    targets = [gsb.Image(ctx, gsb.render(ctx, gt_cloud, gsb.Camera.from_pose12(*intr, WIDTH, HEIGHT, p)).image)
               for p in gt]
    noise = gsb.PoseRng(55)
    init = np.stack([gsb.perturb_pose_tangent(p, 0.05, noise) for p in gt])
    cloud = gsb.Cloud(ctx, C4_N, SH_DEGREE)
    cloud.synth(C4_SEED, log_scale_offset(C4_N))
    cloud.jitter(700, 0.05, 0.3)  # tests/test_trainer.cpp:598-601
    iters = args.warmup + args.steps
    cfg = gsb.JointConfig.default(iterations=max(iters, 1000), sh_degree=SH_DEGREE, sh_degree_interval=0,
                                  densify_interval=0)
    j = gsb.JointOptimizer(ctx, cloud, targets, intr, init, cfg, 800, local_views=1, comm=comm)
    j.step(args.warmup)
    if dist:
        dist.barrier()
    ctx.timer_start()
    j.step(args.steps)
    ms = ctx.timer_stop()
    if dist:
        ms = _reduce_max(dist, ms, local)
    res = j.read()
    j.close()
    if comm:
        comm.close()
    return {"workload": f"C4 joint reconstruction + pose refinement: {C4_N} Gaussians SH3, {C4_VIEWS} views "
                        f"{WIDTH}x{HEIGHT}, 1 view/GPU/step, densify off",
            "steps_per_s": round(args.steps / (ms / 1e3), 3), "views_per_s": round(ws * args.steps / (ms / 1e3), 3),
            "ms_per_step": round(ms / args.steps, 4),
            "parallelism": f"data parallel over {ws} GPU(s): NCCL all-reduce of {(11 + 48 + 2)} FP32 gradient "
                           "planes per step" if ws > 1 else "1 GPU (no collective)",
            "final_total_loss": float(res["trace_total"][-1]) if len(res["trace_total"]) else None}


def ncu_traffic(stage):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the stage's
    kernel from the committed ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(stage, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def roofline(stage, ms, fi, work, peaks, clk, fp32):
    """Dominant-stage roofline (SURVEY §8d units). FP32-bound stages are
    measured against the FFMA microbenchmark of this run (gsb_measure_fp32_peaks)."""
    V, K = fi.n_splats, fi.n_entries
    P = fi.width * fi.height
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback 6.65 TB/s"
    bytes_per = {
        "preprocess": 12 * N_GAUSS + 224 * V + 52 * V,
        "sort": 8 * V + 16 * V + 12 * K + 24 * K + 8 * K + 8 * fi.tiles_x * fi.tiles_y,
        "loss": 24 * P + 12 * P,
        "bwd_geom": 36 * K + 288 * V + 8 * V,
    }
    if stage in ("composite", "bwd_raster") and work is not None:
        hf, cf, hb, cb = work["H_f"], work["C_f"], work["H_b"], work["C_b"]
        flops = 26 * hf + 12 * cf if stage == "composite" else 64 * hb + 12 * cb
        peak = fp32["ffma_tflops"]
        nominal = fp32_peak_tflops(148, peaks.get("sm_max_mhz", 1965.0))
        achieved = flops / (ms / 1e3) / 1e12
        return {"stage": stage, "bound": "fp32", "achieved": round(achieved, 3), "peak": round(peak, 2),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": ncu_traffic(stage),
                "traffic_unit": "DRAM bytes per launch (ncu, profiles/ncu_traffic.json)",
                "peak_source": "FFMA microbenchmark measured in this run (gsb_measure_fp32_peaks); "
                               f"nominal 148 SM x 128 x 2 x sm_max = {nominal:.2f}",
                "frac_of_nominal": round(achieved / nominal, 4),
                "algorithmic": f"{flops} FLOP per launch = 64 H_b + 12 C_b (SURVEY §8d), view-averaged",
                "ms_per_launch": round(ms, 4)}
    if stage in bytes_per:
        b = bytes_per[stage]
        achieved = b / (ms / 1e3) / 1e9
        return {"stage": stage, "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": ncu_traffic(stage), "peak_source": hbm_src,
                "algorithmic": f"{b} bytes per launch (SURVEY §8d)", "ms_per_launch": round(ms, 4)}
    return {"stage": stage, "bound": "fp32", "achieved": None, "peak": None, "unit": "TFLOP/s", "frac": None,
            "traffic": None, "note": "work counts unavailable", "ms_per_launch": round(ms, 4)}


# ------------------------------------------------- CPU (reference build)
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_scene():
    """The same FP32-representable cloud the GPU arm generates (synth.cpp draw
    sequence, seed 3, + ln(500/N)/3 log-scale offset), as FP64 host arrays."""
    from oracle import oracle as O
    rng = O.make_rng(SCENE_SEED)
    hc = O.synth_cloud(N_GAUSS, SH_DEGREE, rng)
    hc.log_scales += log_scale_offset(N_GAUSS)
    return O, hc.as_float32_exact()


def oracle_views():
    """GT poses and perturbed inits for all 64 views from the oracle's Rng
    (identical draw sequence to gsb.synth_poses / PoseRng; no product code)."""
    from oracle import oracle as O
    rng = O.make_rng(SCENE_SEED)
    O.synth_cloud(N_GAUSS, SH_DEGREE, rng)  # the poses are drawn after the cloud (synth.cpp:45-95)
    gt = O.synth_poses(1, TOTAL_VIEWS, rng)
    noise = O.make_rng(NOISE_SEED)
    init = np.stack([O.perturb_pose(p, 15.0, 0.15, noise) for p in gt])
    return gt, init


class RefCpu:
    """The reference's own render / rgb_loss / render_backward / pose_step
    (oracle/_ref: /root/reference/proj sources built by oracle/build_ref.py,
    thread pool = all host cores, core.cpp:21-22) when present, else the FP64
    restatement (oracle/gsopt_oracle.c)."""

    def __init__(self):
        from oracle import oracle as O
        self.O = O
        self.kind = "reference" if O.ref_available() else "port"
        self.O_scene = _oracle_scene()[1]
        self.intr = (0.75 * WIDTH, 0.75 * WIDTH, 0.5 * (WIDTH - 1), 0.5 * (HEIGHT - 1))
        self.targets = {}

    def _ctx(self):
        import contextlib
        return self.O.reference_backend() if self.kind == "reference" else contextlib.nullcontext()

    def cores(self):
        return int(self.O.ref_lib().ref_thread_count()) if self.kind == "reference" else self.O.num_threads()

    def target(self, v, gt12):
        if v not in self.targets:
            O = self.O
            with self._ctx():
                cam = O.make_camera(*self.intr, WIDTH, HEIGHT, *O.pose_split(gt12))
                self.targets[v] = O.render(self.O_scene, cam).image
        return self.targets[v]

    def iteration(self, v, gt12, init12):
        """One pose_descent iteration (render, rgb_loss, render_backward,
        pose_step; pipelines.cpp:66-90) of view v from its init pose."""
        O = self.O
        tgt = self.target(v, gt12)
        if self.kind == "reference":
            r = O.ref_estimate_pose(self.O_scene, tgt, *self.intr, init12, budget=1, pose_converged_eps=0.0)
        else:
            r = O.estimate_pose(self.O_scene, tgt, *self.intr, init12, budget=1, pose_converged_eps=0.0)
        return r["steps"]


def cpu_baseline(args, gt, init, views, intr, seconds=None):
    """cpu_baseline: the reference on the host cores, bounded sample of the
    same workload (one pose_descent iteration per view of the GPU's views,
    round robin, until ~`seconds` of CPU work)."""
    seconds = args.cpu_seconds if seconds is None else seconds
    ref = RefCpu()
    for v in views:
        ref.target(v, gt[v])
    ref.iteration(views[0], gt[views[0]], init[views[0]])  # warm-up (acceptance.cpp:472)
    n, t0 = 0, time.perf_counter()
    while True:
        v = views[n % len(views)]
        n += ref.iteration(v, gt[v], init[v])
        dt = time.perf_counter() - t0
        if dt >= seconds and n >= 3:
            break
    return {"value": round(n / dt, 5), "unit": "iters/s", "cores": ref.cores(), "kind": ref.kind,
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "sample": f"{n} pose_descent iterations (render+rgb_loss+render_backward+pose_step, FP64) of the "
                      f"GPU's {len(views)} views round robin at full size ({N_GAUSS} Gaussians, {WIDTH}x{HEIGHT}), "
                      f"{dt:.1f} s, " + ("the reference's own sources (oracle/_ref)" if ref.kind == "reference"
                                         else "oracle port")}


def work_counts(view_poses, intr):
    """H_f/C_f/H_b/C_b averaged over the GPU's views at their init
    poses, counted by the oracle from contrib_count / tile lists / the upstream
    gradient of the same scene."""
    O, hc = _oracle_scene()
    acc = np.zeros(4)
    for gt12, init12 in view_poses:
        cam_gt = O.make_camera(*intr, WIDTH, HEIGHT, *O.pose_split(gt12))
        target = O.render(hc, cam_gt).image
        cam0 = O.make_camera(*intr, WIDTH, HEIGHT, *O.pose_split(init12))
        rr = O.render(hc, cam0, keep_handle=True)
        _, d_img = O.rgb_loss(rr.image, target, 0.2)
        acc += np.array(O.count_work(rr, d_img), np.float64)
        rr.free()
    acc /= len(view_poses)
    return {"H_f": int(acc[0]), "C_f": int(acc[1]), "H_b": int(acc[2]), "C_b": int(acc[3]),
            "source": f"oracle count_work, mean over the GPU's {len(view_poses)} views at their init poses"}


def run_c3_job(args, ws, rank, local, ctx, cloud, gt, init, intr):
    """C3's whole 64-view job on ONE GPU (rank 0 only): gsb_estimate_poses over
    all 64 views, 100 pose_descent iterations each (early exits off), from
    device-resident targets; views/s of the completed job."""
    if rank != 0 or ws != 1:
        return None
    from paper_2410_08743_b200 import gsb
    imgs = [gsb.Image(ctx, gsb.render(ctx, cloud, gsb.Camera.from_pose12(*intr, WIDTH, HEIGHT, gt[v])).image)
            for v in range(TOTAL_VIEWS)]
    cfg = gsb.PoseConfig.default(budget=100, pose_converged_eps=0.0)
    gsb.estimate_poses(ctx, cloud, imgs[:VIEWS_PER_GPU], intr, init[:VIEWS_PER_GPU],
                       gsb.PoseConfig.default(budget=2, pose_converged_eps=0.0))  # warm-up
    ctx.synchronize()
    ctx.timer_start()
    out = gsb.estimate_poses(ctx, cloud, imgs, intr, init[:TOTAL_VIEWS], cfg)
    ms = ctx.timer_stop()
    assert all(int(k) == 100 for k in out["steps"])
    rot = [gsb_abs_err(out["pose"][v], gt[v]) for v in range(TOTAL_VIEWS)]
    return {"workload": f"C3 complete job: {TOTAL_VIEWS} views x 100 iterations, {N_GAUSS} Gaussians, one GPU, "
                        "one gsb_estimate_poses call (views advanced in pose batches of 8)",
            "views_per_s": round(TOTAL_VIEWS / (ms / 1e3), 3), "iters_per_s": round(TOTAL_VIEWS * 100 / (ms / 1e3), 2),
            "job_s": round(ms / 1e3, 3),
            "recovered_views": int(sum(1 for r, t in rot if r < 0.1 and t < 1e-3)),
            "converged_views_acceptance": int(sum(1 for r, t in rot if r < 5.0 and t < 0.05)),
            "note": "pose_descent's own convergence at C3's 100-iteration budget from 15 deg / 0.15 (the reference "
                    "algorithm; the C2 parity test shows the reference CPU build no closer to GT)",
            "median_rot_err_deg": float(np.median([r for r, _ in rot])),
            "median_trans_err": float(np.median([t for _, t in rot]))}


def gsb_abs_err(p12, g12):
    """(rotation error in degrees, translation error) between two world->camera poses."""
    P, G = np.asarray(p12).reshape(3, 4), np.asarray(g12).reshape(3, 4)
    Rr = P[:, :3] @ G[:, :3].T
    ang = math.degrees(math.acos(max(-1.0, min(1.0, (np.trace(Rr) - 1) / 2))))
    cp = -P[:, :3].T @ P[:, 3]
    cg = -G[:, :3].T @ G[:, 3]
    return ang, float(np.linalg.norm(cp - cg))


def common_config(ws):
    return {"workload": f"C3 pose estimation: {N_GAUSS} Gaussians SH3, {WIDTH}x{HEIGHT}, "
                        f"{VIEWS_PER_GPU} views/GPU ({TOTAL_VIEWS} at 8 GPUs), forward-facing, perturb 15deg/0.15",
            "views_per_gpu": VIEWS_PER_GPU, "n_gaussians": N_GAUSS, "width": WIDTH, "height": HEIGHT,
            "l2": "inputs larger than L2 (236 MB cloud + per-view state > 126 MB L2)",
            "parallelism": f"views sharded over {ws} GPU(s), no collective"}


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    all host threads) on this arm's config; one step = one pose_descent
    iteration of one of the rank-0 GPU's views (round robin). No product code."""
    if rank != 0:
        return None
    gt, init = oracle_views()
    views = my_views(0, ws)
    ref = RefCpu()
    for v in views:
        ref.target(v, gt[v])
    for k in range(max(args.warmup, 1)):
        v = views[k % len(views)]
        ref.iteration(v, gt[v], init[v])
    times = []
    for k in range(args.steps):
        v = views[k % len(views)]
        t0 = time.perf_counter()
        ref.iteration(v, gt[v], init[v])
        times.append(time.perf_counter() - t0)
    dt = sum(times)
    value = args.steps / dt
    cfg = common_config(ws)
    return {"metric": METRIC, "value": round(value, 5), "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * dt / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp64",
            "data": "synthetic (same scene, views and inits as the GPU arm)", "impl": "reference",
            "config": cfg,
            "cpu_baseline": {"value": round(value, 5), "unit": "iters/s", "cores": ref.cores(), "kind": ref.kind,
                             "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                             "sample": f"{args.steps} timed pose_descent iterations, one per step, over the rank-0 "
                                       f"GPU's {len(views)} views round robin, at full size"},
            "e2e": {"value": round(value, 5), "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def spawn_ranks(n):
    """--gpus N without a torchrun environment: relaunch this script under
    torch.distributed.run, one process per GPU (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-iters", type=int, default=100)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded CPU-baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-work-counts", action="store_true")
    ap.add_argument("--no-c3-job", action="store_true", help="skip the 64-view one-GPU job measurement")
    ap.add_argument("--no-joint", action="store_true", help="skip the secondary C4 joint-DP measurement")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if rank == 0 and os.environ.get("OMP_NUM_THREADS") == "1" and ws > 1:
        # torchrun pins every rank to one OpenMP thread; rank 0's host-side
        # oracle work (FLOP counts) gets the host's cores back
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if ws != args.gpus and args.gpus != 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        out = run_reference(args, ws, rank)
    else:
        out = run_ours(args, ws, rank, local)
    if out is not None and rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
