"""Fixed vs per-iteration cost of gsb_estimate_poses (8 views of the bench
scene): budgets 25 / 100 / 200, 3 reps each."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_08743_b200 import gsb  # noqa: E402

ctx = gsb.Context(0)
cloud = gsb.Cloud(ctx, bench.N_GAUSS, bench.SH_DEGREE)
cloud.synth(bench.SCENE_SEED, bench.log_scale_offset(bench.N_GAUSS))
gt, init = bench.all_views()
intr = gsb.synth_intrinsics(bench.WIDTH, bench.HEIGHT)
views = list(range(8))
imgs = [gsb.Image(ctx, gsb.render(ctx, cloud, gsb.Camera.from_pose12(*intr, bench.WIDTH, bench.HEIGHT, gt[v])).image)
        for v in views]
gsb.estimate_poses(ctx, cloud, imgs, intr, init[views], gsb.PoseConfig.default(budget=4, pose_converged_eps=0.0))
for budget in (25, 100, 200):
    for rep in range(3):
        cfg = gsb.PoseConfig.default(budget=budget, pose_converged_eps=0.0)
        ctx.synchronize()
        t0 = time.perf_counter()
        gsb.estimate_poses(ctx, cloud, imgs, intr, init[views], cfg)
        ctx.synchronize()
        dt = time.perf_counter() - t0
        print(f"budget {budget}: {1e3 * dt:.1f} ms = {1e3 * dt / budget:.3f} ms/iter", flush=True)
