"""Profiling driver: the bench's pose batch (8 views of the 1M-Gaussian
scene, one graph replay per iteration). Used under ncu (one GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_08743_b200 import gsb  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = gsb.Context(0)
cloud = gsb.Cloud(ctx, bench.N_GAUSS, bench.SH_DEGREE)
cloud.synth(bench.SCENE_SEED, bench.log_scale_offset(bench.N_GAUSS))
gt, init = bench.all_views()
intr = gsb.synth_intrinsics(bench.WIDTH, bench.HEIGHT)
views = bench.my_views(0, 1)
imgs = [gsb.Image(ctx, gsb.render(ctx, cloud, gsb.Camera.from_pose12(*intr, bench.WIDTH, bench.HEIGHT, gt[v])).image)
        for v in views]
cfg = gsb.PoseConfig.default(budget=100, pose_converged_eps=0.0)
sessions = [gsb.PoseSession(ctx, cloud, imgs[k], intr, init[v], cfg) for k, v in enumerate(views)]
batch = gsb.PoseBatch(ctx, sessions)
batch.step_async(iters)
batch.sync()
print("done")
