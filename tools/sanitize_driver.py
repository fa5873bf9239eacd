"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the hot path on C1-sized inputs — render
(tile-local and global binning), loss, full and pose-only backward, pose
batch of 2 sessions (graph replays, capacity-growth replay), a 2-slot joint
run with densification, expected depth. Usage: python tools/sanitize_driver.py"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2410_08743_b200 import gsb  # noqa: E402

ctx = gsb.Context(0)
n, w, h = 4000, 128, 96
cloud = gsb.Cloud(ctx, n, 3)
cloud.synth(99, math.log(500 / n) / 3)
poses = gsb.synth_poses(99, n, 3, 0, 4)
intr = gsb.synth_intrinsics(w, h)
cams = [gsb.Camera.from_pose12(*intr, w, h, p) for p in poses]
imgs = []
for binning in (gsb.Context.BINNING_TILE_LOCAL, gsb.Context.BINNING_GLOBAL):
    ctx.set_binning(binning)
    out = gsb.render(ctx, cloud, cams[0])
    loss, d = gsb.rgb_loss(ctx, out.image, np.clip(out.image + 0.05, 0, 1), 0.2)
    gsb.render_backward(ctx, cloud, cams[0], out, d)
    gsb.render_backward(ctx, cloud, cams[0], out, d, pose_only=True)
ctx.set_binning(gsb.Context.BINNING_TILE_LOCAL)
targets = [gsb.Image(ctx, gsb.render(ctx, cloud, c).image) for c in cams]
rng = gsb.PoseRng(1002)
init = np.stack([rng.perturb_pose(p, 5.0, 0.05) for p in poses])
cfg = gsb.PoseConfig.default(budget=4, pose_converged_eps=0.0)
sessions = [gsb.PoseSession(ctx, cloud, targets[k], intr, init[k], cfg) for k in range(2)]
batch = gsb.PoseBatch(ctx, sessions)
batch.step(3)
batch.close()
gsb.render_expected_depth(ctx, cloud, cams[1])
jc = gsb.JointConfig.default(iterations=4, sh_degree=3, sh_degree_interval=0, densify_interval=2, densify_start=2,
                             n_target=n + 200, grad_threshold=1e-5)
jcloud = gsb.Cloud(ctx, n, 3)
jcloud.synth(99, math.log(500 / n) / 3)
jcloud.jitter(7, 0.02, 0.1)
j = gsb.JointOptimizer(ctx, jcloud, targets, intr, init, jc, 5, local_views=2)
j.step(4)
print("sanitize driver done:", j.read()["steps"], "joint steps")
j.close()
