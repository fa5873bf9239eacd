"""C5-shaped joint reconstruction on ONE GPU (BASELINE configs[4] is quoted at
8xB200): 3M Gaussians SH-3, 200 random-walk views at 1920x1080 (synth.cpp
draw sequence, seed 5), init = the GT cloud jittered as tests/test_trainer.cpp
598-601, joint_optimize with densify_and_prune every 100 steps (from step 100
so that the run sees several events; n_target = 3M). Prints one JSON line:
device-timed steps/s over each 100-step segment, population and densify
reports. Usage: python tools/run_c5.py [steps]"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2410_08743_b200 import gsb  # noqa: E402

N, W, H, VIEWS, SEED = 3_000_000, 1920, 1080, 200, 5
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
ctx = gsb.Context(0)
off = math.log(500.0 / N) / 3.0
gt_cloud = gsb.Cloud(ctx, N, 3)
gt_cloud.synth(SEED, off)
gt = gsb.synth_poses(SEED, N, 3, 2, VIEWS)  # kind 2 = random walk (synth.cpp:91-95)
intr = gsb.synth_intrinsics(W, H)
t0 = time.perf_counter()
targets = [gsb.Image(ctx, gsb.render(ctx, gt_cloud, gsb.Camera.from_pose12(*intr, W, H, p)).image) for p in gt]
t_targets = time.perf_counter() - t0
del gt_cloud
noise = gsb.PoseRng(55)
init = np.stack([gsb.perturb_pose_tangent(p, 0.05, noise) for p in gt])
cloud = gsb.Cloud(ctx, N, 3)
cloud.synth(SEED, off)
cloud.jitter(700, 0.05, 0.3)
cfg = gsb.JointConfig.default(iterations=steps + 8, sh_degree=3, sh_degree_interval=0, densify_interval=100,
                              densify_start=100, densify_stop=steps + 8, n_target=N)
j = gsb.JointOptimizer(ctx, cloud, targets, intr, init, cfg, 800)
j.step(4)  # warm-up (graph capture, first-use allocations)
segs = []
done = 4
while done < steps:
    k = min(100, steps - done)
    ctx.timer_start()
    j.step(k)
    ms = ctx.timer_stop()
    done += k
    r = j.read()
    segs.append({"steps": k, "ms_per_step": round(ms / k, 4), "steps_per_s": round(1e3 * k / ms, 2),
                 "n_gaussians": r["n_gaussians"], "densify_events": r["densify_events"],
                 "last_report": r["densify_report"], "total_loss": float(r["trace_total"][-1])})
r = j.read()
print(json.dumps({"workload": f"C5 shape on 1 GPU: {N} Gaussians SH3, {VIEWS} random-walk views {W}x{H}, joint "
                              "optimize + pose refinement, densify every 100 steps from step 100 (n_target 3M)",
                  "target_render_s": round(t_targets, 2), "segments": segs, "steps": r["steps"],
                  "first_loss": float(r["trace_total"][0]), "final_loss": float(r["trace_total"][-1])}))
