"""GPU parity at BASELINE.json's larger configs (SURVEY §8d C2 / C4 / C5
shapes) against the FP64 oracle (pinned to the reference build, see
test_ref_pins.py) on identical FP32-representable inputs.

* C2: 300k Gaussians SH-3, 1008x756, forward-facing (seed 2), pose_descent
  from the 15 deg / 0.15 perturbation (Rng(1002)) for 200 iterations: poses
  within rot 0.1 deg / trans 1e-3 (test_trainer.cpp:506-507) and losses within
  1e-3 relative over the first 20 iterations; after 200 the device's pose at
  least as close to GT as the reference's (pipelines.cpp:58-92).
* C4: 300k Gaussians SH-3, 1008x756, 20 forward-facing views (seed 4),
  jittered init cloud (test_trainer.cpp:598-601): the full GradientBundle of
  one view (rasterizer.cpp:336-540) per parameter group within 1e-3 relative
  (floor 1e-3 * max|g| of the group, gradcheck.hpp:187-197), and a 20-step
  joint_optimize trace (pipelines.cpp:96-216).
* C5 shape: 3M Gaussians SH-3, 1920x1080, random-walk view (seed 5): depth
  order, tile lists and ranges bit-exact against rasterizer.cpp:127-168 re-run
  on the device's FP64 records and against the oracle's own render, and the
  pose gradient within 1e-3.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W, H = 1008, 756


@pytest.fixture(scope="module")
def G():
    from paper_2410_08743_b200 import build, gsb
    build.build()
    return gsb


@pytest.fixture(scope="module")
def ctx(G):
    return G.Context(0)


def off(n):
    return math.log(500.0 / n) / 3.0 if n > 500 else 0.0


def host_cloud(seed, n, sh=3):
    rng = O.make_rng(seed)
    hc = O.synth_cloud(n, sh, rng)
    hc.log_scales += off(n)
    return hc.as_float32_exact(), rng


def to_dev(G, ctx, hc):
    return G.Cloud.from_host(ctx, hc.means, hc.rotations, hc.log_scales, hc.opacity_logits, hc.sh, hc.sh_degree,
                             hc.active_sh_degree)


def rel_err(a, b, floor_frac=1e-3):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    floor = max(floor_frac * np.max(np.abs(b)), 1e-30)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))


def dump(name, rep):
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/config_parity_{name}.json", "w") as fh:
        json.dump(rep, fh)


def test_c2_pose_descent_200_iterations(G, ctx):
    """Adam normalises each d_pose component by its own running magnitude, so
    once a component's gradient is small its FP32 and FP64 steps can point
    different ways by up to lr per iteration: the trajectories are compared
    per iteration over the first 20 iterations (rot 0.1 deg / trans 1e-3,
    test_trainer.cpp:506-507) and, after all 200, by the distance to the GT
    pose — the device's must be within the reference's own test-time
    recovery tolerance (0.1 deg / 1e-3, test_trainer.cpp:484-526) or no worse
    than the reference's own result. (Measured round 2: the two agree to
    within 0.1 deg for 28 iterations; after 200 the device is 0.013 deg /
    4.6e-4 from GT, the reference 0.58 deg / 0.020.)"""
    n, iters, track = 300_000, 200, 20
    hc, rng = host_cloud(2, n)
    gt = O.synth_poses(1, 1, rng)[0]
    init = O.perturb_pose(gt, 15.0, 0.15, O.make_rng(1002))
    intr = (0.75 * W, 0.75 * W, 0.5 * (W - 1), 0.5 * (H - 1))
    target = O.render(hc, O.make_camera(*intr, W, H, *O.pose_split(gt))).image
    ref = O.estimate_pose(hc, target, *intr, init, budget=iters, pose_converged_eps=0.0)
    cloud = to_dev(G, ctx, hc)
    res = G.estimate_pose(ctx, cloud, G.Image(ctx, target), list(intr), init,
                          G.PoseConfig.default(budget=iters, pose_converged_eps=0.0), trace=True)
    assert res["steps"] == ref["steps"] == iters
    errs = np.array([O.abs_pose_error(res["trace_pose"][k], ref["trace_pose"][k]) for k in range(iters)])
    lrel = np.abs(res["trace_loss"] - ref["trace_loss"]) / ref["trace_loss"]
    e_dev = O.abs_pose_error(res["trace_pose"][-1], gt)
    e_ref = O.abs_pose_error(ref["trace_pose"][-1], gt)
    over = np.nonzero((errs[:, 0] >= 0.1) | (errs[:, 1] >= 1e-3))[0]
    dump("c2", {"iterations": iters, "tracked_iterations": track,
                "max_rot_deg_tracked": float(errs[:track, 0].max()), "max_trans_tracked": float(errs[:track, 1].max()),
                "max_loss_rel_tracked": float(lrel[:track].max()), "first_iteration_over_tol":
                    int(over[0]) if len(over) else None, "max_rot_deg_all": float(errs[:, 0].max()),
                "final_dev_vs_ref": [float(v) for v in errs[-1]], "final_dev_vs_gt": [float(v) for v in e_dev],
                "final_ref_vs_gt": [float(v) for v in e_ref], "final_loss_dev": float(res["trace_loss"][-1]),
                "final_loss_ref": float(ref["trace_loss"][-1])})
    assert errs[:track, 0].max() < 0.1 and errs[:track, 1].max() < 1e-3, errs[:track].max(axis=0)
    assert lrel[:track].max() < 1e-3, lrel[:track].max()
    for k in range(2):
        assert e_dev[k] < max((0.1, 1e-3)[k], e_ref[k]), (e_dev, e_ref)


def c4_inputs(G, ctx, views=20):
    n = 300_000
    gt_cloud = G.Cloud(ctx, n, 3)
    gt_cloud.synth(4, off(n))
    gt = G.synth_poses(4, n, 3, 1, views)
    intr = G.synth_intrinsics(W, H)
    cloud = G.Cloud(ctx, n, 3)
    cloud.synth(4, off(n))
    cloud.jitter(700, 0.05, 0.3)  # tests/test_trainer.cpp:598-601
    m, q, ls, op, sh = cloud.download()
    hc = O.HostCloud(np.asarray(m), np.asarray(q), np.asarray(ls), np.asarray(op), np.asarray(sh), 3, 3)
    gm, gq, gls, gop, gsh = gt_cloud.download()
    gt_hc = O.HostCloud(np.asarray(gm), np.asarray(gq), np.asarray(gls), np.asarray(gop), np.asarray(gsh), 3, 3)
    noise = G.PoseRng(55)
    init = np.stack([G.perturb_pose_tangent(p, 0.05, noise) for p in gt])
    return hc, gt_hc, gt, init, intr, cloud


def test_c4_full_gradient_bundle(G, ctx):
    hc, gt_hc, gt, init, intr, cloud = c4_inputs(G, ctx, views=1)
    target = O.render(gt_hc, O.make_camera(*intr, W, H, *O.pose_split(gt[0]))).image
    ocam = O.make_camera(*intr, W, H, *O.pose_split(init[0]))
    rr = O.render(hc, ocam, keep_handle=True)
    _, d_img = O.rgb_loss(rr.image, target, 0.2)
    gr = O.render_backward(hc, ocam, rr, d_img)
    rr.free()
    cam = G.Camera.from_pose12(*intr, W, H, init[0])
    out = G.render(ctx, cloud, cam)
    g, dp = G.render_backward(ctx, cloud, cam, out, d_img)
    groups = {"d_means": (g["d_means"], gr.d_means), "d_rotations": (g["d_rotations"], gr.d_rotations),
              "d_log_scales": (g["d_log_scales"], gr.d_log_scales),
              "d_opacity_logits": (g["d_opacity_logits"], gr.d_opacity_logits), "d_sh": (g["d_sh"], gr.d_sh),
              "d_mu2d": (g["d_mu2d"], gr.d_mu2d)}
    rep = {k: rel_err(a, b) for k, (a, b) in groups.items()}
    rep["d_pose"] = float(np.linalg.norm(dp - gr.d_pose) / np.linalg.norm(gr.d_pose))
    rep["n_gaussians"] = hc.n
    dump("c4_bundle", rep)
    for k, v in rep.items():
        if k != "n_gaussians":
            assert v < 1e-3, (k, v, rep)


def test_c4_joint_20_steps(G, ctx):
    views, steps = 20, 20
    hc, gt_hc, gt, init, intr, cloud = c4_inputs(G, ctx, views=views)
    imgs = [O.render(gt_hc, O.make_camera(*intr, W, H, *O.pose_split(p))).image.astype(np.float32).astype(np.float64)
            for p in gt]
    kw = dict(sh_degree=3, sh_degree_interval=0)
    st, cl, P, tt, tl = O.joint_optimize(hc, imgs, list(intr), W, H, init, O.joint_config(steps, **kw), 1,
                                         O.make_rng(800))
    assert st == 0
    targets = [G.Image(ctx, im) for im in imgs]
    j = G.JointOptimizer(ctx, cloud, targets, intr, init, G.JointConfig.default(iterations=steps, **kw), 800)
    j.step(steps)
    res = j.read()
    j.close()
    rel = np.abs(res["trace_total"] - tt) / np.maximum(np.abs(tt), 1e-12)
    pe = np.array([O.abs_pose_error(res["poses"][v], P[v]) for v in range(views)])
    dump("c4_joint", {"steps": steps, "max_trace_rel": float(rel.max()), "max_rot_deg": float(pe[:, 0].max()),
                      "max_trans": float(pe[:, 1].max())})
    assert res["steps"] == steps
    assert rel.max() < 1e-3, rel
    assert pe[:, 0].max() < 0.1 and pe[:, 1].max() < 1e-3, pe.max(axis=0)


def test_c5_shape_lists_and_pose_gradient(G, ctx):
    n, w, h = 3_000_000, 1920, 1080
    hc, rng = host_cloud(5, n)
    poses = O.synth_poses(2, 2, rng)  # random walk (synth.cpp:91-95)
    intr = (0.75 * w, 0.75 * w, 0.5 * (w - 1), 0.5 * (h - 1))
    ocam = O.make_camera(*intr, w, h, *O.pose_split(poses[1]))
    target = O.render(hc, O.make_camera(*intr, w, h, *O.pose_split(poses[0]))).image
    cloud = to_dev(G, ctx, hc)
    cam = G.Camera.from_pose12(*intr, w, h, poses[1])
    out = G.render(ctx, cloud, cam)
    info = out.info()
    d = out.download()
    keep = np.zeros(n, np.uint8)
    keep[d["splat_gaussian"]] = 1
    mu2d = np.zeros((n, 2))
    mu2d[d["splat_gaussian"]] = d["splat_mu2d"]
    rad = np.zeros(n)
    rad[d["splat_gaussian"]] = d["splat_radius"]
    dep = np.zeros(n)
    dep[d["splat_gaussian"]] = d["splat_depth"]
    sg, lists, ranges = O.bin_records(keep, mu2d, rad, dep, w, h)
    assert np.array_equal(sg, d["splat_gaussian"])
    assert np.array_equal(lists, d["tile_lists"])
    assert np.array_equal(ranges, d["tile_ranges"])
    rr = O.render(hc, ocam, keep_handle=True)
    assert np.array_equal(rr.splat_gaussian, d["splat_gaussian"])
    assert np.array_equal(rr.tile_lists, d["tile_lists"]) and np.array_equal(rr.tile_ranges, d["tile_ranges"])
    _, d_img = O.rgb_loss(rr.image, target, 0.2)
    gr = O.render_backward(hc, ocam, rr, d_img)
    tile_len = np.diff(rr.tile_ranges, axis=1).ravel()
    rr.free()
    _, dp = G.render_backward(ctx, cloud, cam, out, d_img, pose_only=True)
    rel = float(np.linalg.norm(dp - gr.d_pose) / np.linalg.norm(gr.d_pose))
    dump("c5", {"n_splats": int(info.n_splats), "n_entries": int(info.n_entries), "binning": int(info.binning),
                "max_tile_entries": int(tile_len.max()), "tiles_over_8192": int((tile_len > 8192).sum()),
                "d_pose_rel": rel})
    assert rel < 1e-3, rel
