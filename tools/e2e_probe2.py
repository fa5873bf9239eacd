"""Phases of the e2e measurement (bench.py's e2e leg) on the bench scene."""
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
hosts = [gsb.render(ctx, cloud, gsb.Camera.from_pose12(*intr, bench.WIDTH, bench.HEIGHT, gt[v])).image for v in views]
cfg = gsb.PoseConfig.default(budget=100, pose_converged_eps=0.0)
for rep in range(5):
    ctx.synchronize()
    t0 = time.perf_counter()
    imgs = [gsb.Image(ctx, h) for h in hosts]
    ctx.synchronize()
    t1 = time.perf_counter()
    out = gsb.estimate_poses(ctx, cloud, imgs, intr, init[views], cfg)
    ctx.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: uploads {1e3*(t1-t0):.1f} ms, estimate_poses {1e3*(t2-t1):.1f} ms "
          f"({800/(t2-t0):.0f} iters/s e2e)", flush=True)
    del imgs
