"""Profiling driver: the bench's C4 joint step (300k Gaussians, 20 views at
1008x756, full backward + Adam + pose step). Used under ncu (one GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2410_08743_b200 import gsb  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = gsb.Context(0)
N, V = bench.C4_N, bench.C4_VIEWS
gt_cloud = gsb.Cloud(ctx, N, bench.SH_DEGREE)
gt_cloud.synth(bench.C4_SEED, bench.log_scale_offset(N))
gt = gsb.synth_poses(bench.C4_SEED, N, bench.SH_DEGREE, 1, V)
intr = gsb.synth_intrinsics(bench.WIDTH, bench.HEIGHT)
targets = [gsb.Image(ctx, gsb.render(ctx, gt_cloud, gsb.Camera.from_pose12(*intr, bench.WIDTH, bench.HEIGHT, p)).image)
           for p in gt]
noise = gsb.PoseRng(55)
init = np.stack([gsb.perturb_pose_tangent(p, 0.05, noise) for p in gt])
cloud = gsb.Cloud(ctx, N, bench.SH_DEGREE)
cloud.synth(bench.C4_SEED, bench.log_scale_offset(N))
cloud.jitter(700, 0.05, 0.3)
cfg = gsb.JointConfig.default(iterations=1000, sh_degree=bench.SH_DEGREE, sh_degree_interval=0)
j = gsb.JointOptimizer(ctx, cloud, targets, intr, init, cfg, 800)
j.step(steps)
print("done", j.read()["trace_total"][-1])
