"""Breaks the e2e (gsb_estimate_pose from a host image) time into phases on
the bench scene: image upload, session create, graph capture + first chunk,
steady chunks, read-back. Run on one GPU."""
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
hosts = []
for v in range(3):
    cam = gsb.Camera.from_pose12(*intr, bench.WIDTH, bench.HEIGHT, gt[v])
    hosts.append(gsb.render(ctx, cloud, cam).image)
cfg = gsb.PoseConfig.default(budget=100, pose_converged_eps=0.0)
for v in range(3):
    ctx.synchronize()
    t0 = time.perf_counter()
    img = gsb.Image(ctx, hosts[v])
    ctx.synchronize()
    t1 = time.perf_counter()
    s = gsb.PoseSession(ctx, cloud, img, intr, init[v], cfg)
    t2 = time.perf_counter()
    s.step(1)
    t3 = time.perf_counter()
    s.step(15)
    t4 = time.perf_counter()
    s.step(84)
    t5 = time.perf_counter()
    r = s.read()
    t6 = time.perf_counter()
    print(f"view {v}: upload {1e3*(t1-t0):.2f} ms, create {1e3*(t2-t1):.2f}, first iter {1e3*(t3-t2):.2f}, "
          f"15 iters {1e3*(t4-t3):.2f}, 84 iters {1e3*(t5-t4):.2f}, read {1e3*(t6-t5):.2f}, steps {r['steps']}",
          flush=True)
    del s, img
for v in range(3):
    ctx.synchronize()
    t0 = time.perf_counter()
    img = gsb.Image(ctx, hosts[v])
    out = gsb.estimate_pose(ctx, cloud, img, intr, init[v], cfg)
    ctx.synchronize()
    print(f"estimate_pose view {v}: {1e3*(time.perf_counter()-t0):.2f} ms, steps {out['steps']}", flush=True)
