"""Profiling driver: the bench scene (1M Gaussians, 1008x756, view 0), a few
pose_descent iterations through a session. Used under ncu (one GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_08743_b200 import gsb  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = gsb.Context(0)
cloud = gsb.Cloud(ctx, bench.N_GAUSS, bench.SH_DEGREE)
cloud.synth(bench.SCENE_SEED, bench.log_scale_offset(bench.N_GAUSS))
gt, init = bench.all_views()
intr = gsb.synth_intrinsics(bench.WIDTH, bench.HEIGHT)
cam = gsb.Camera.from_pose12(*intr, bench.WIDTH, bench.HEIGHT, gt[0])
img = gsb.Image(ctx, gsb.render(ctx, cloud, cam).image)
s = gsb.PoseSession(ctx, cloud, img, intr, init[0], gsb.PoseConfig.default(budget=100, pose_converged_eps=0.0))
for _ in range(iters):
    s.step(1)
ctx.synchronize()
print("done", s.read()["final_loss"])
