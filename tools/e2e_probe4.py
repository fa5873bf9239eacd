"""Per-iteration rate of a pose batch stepped three ways in one process:
100 x step_async(1) (wall clock and device timer) and batch.step(100)."""
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
imgs = [gsb.Image(ctx, gsb.render(ctx, cloud, gsb.Camera.from_pose12(*intr, bench.WIDTH, bench.HEIGHT, gt[v])).image) for v in views]
cfg = gsb.PoseConfig.default(budget=1000, pose_converged_eps=0.0)
sessions = [gsb.PoseSession(ctx, cloud, imgs[k], intr, init[v], cfg) for k, v in enumerate(views)]
batch = gsb.PoseBatch(ctx, sessions)
batch.step_async(3); batch.sync()
for rep in range(2):
    ctx.synchronize(); t0 = time.perf_counter()
    for _ in range(100): batch.step_async(1)
    ctx.synchronize(); dt = time.perf_counter() - t0
    print(f"100 x step_async(1): {1e3*dt/100:.3f} ms/iter", flush=True)
    ctx.timer_start()
    for _ in range(100): batch.step_async(1)
    ms = ctx.timer_stop()
    print(f"  device timer: {ms/100:.3f} ms/iter", flush=True)
    ctx.synchronize(); t0 = time.perf_counter()
    batch.step(100)
    ctx.synchronize(); dt = time.perf_counter() - t0
    print(f"batch.step(100): {1e3*dt/100:.3f} ms/iter", flush=True)
