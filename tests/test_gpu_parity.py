"""GPU parity: libgsb200 (through its C ABI) against the FP64 CPU oracle on
the same inputs. Tolerances are north_star's (BASELINE.json):
  * sort keys / tile lists / tile ranges: bit-exact;
  * rendered image: <= 1e-5 max-abs on conditioned scenes
    (tests/gradcheck.hpp:67-170 conditioning);
  * Gaussian and pose gradients: <= 1e-3 relative (floor 1e-3 * max|g| per
    parameter group, cf. tests/gradcheck.hpp:187-197);
  * pose trajectories: rot <= 0.1 deg, trans <= 1e-3 (test_trainer.cpp:506-507).
The oracle is fed the FP32-rounded parameters the device stores.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_2410_08743_b200 import build, gsb
    build.build()
    return gsb


@pytest.fixture(scope="module")
def ctx(G):
    return G.Context(0)


def to_dev(G, ctx, hc: O.HostCloud):
    return G.Cloud.from_host(ctx, hc.means, hc.rotations, hc.log_scales, hc.opacity_logits, hc.sh, hc.sh_degree,
                             hc.active_sh_degree)


def dev_cam(G, ocam):
    return G.Camera.make(ocam.fx, ocam.fy, ocam.cx, ocam.cy, ocam.width, ocam.height,
                         np.array(ocam.R[:]).reshape(3, 3), np.array(ocam.t[:]))


def scene(seed, n, size, conditioned=True):
    rng = O.make_rng(seed)
    if conditioned:
        hc, cam, bg = O.make_conditioned_scene(rng, n, size)
    else:
        hc, cam, bg = O.make_gradcheck_scene(rng, n, size)
    return hc.as_float32_exact(), cam, bg, rng


def synth_scene(seed, n, size, sh=3, kind=0, cams=4, scale_offset=0.0):
    rng = O.make_rng(seed)
    hc = O.synth_cloud(n, sh, rng)
    hc.log_scales += scale_offset
    poses = O.synth_poses(kind, cams, rng)
    return hc.as_float32_exact(), poses


def rel_err(a, b, floor_frac=1e-3):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    floor = max(floor_frac * np.max(np.abs(b)), 1e-30)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))


# ----------------------------------------------------------------- forward
@pytest.mark.parametrize("seed", [54, 55, 61, 70])
def test_render_matches_oracle_conditioned(G, ctx, seed):
    hc, ocam, bg, _ = scene(seed, 12, 48)
    cloud = to_dev(G, ctx, hc)
    out = G.render(ctx, cloud, dev_cam(G, ocam), bg)
    ref = O.render(hc, ocam, bg)
    d = out.download()
    assert np.max(np.abs(d["image"] - ref.image)) < 1e-5
    # discrete state: bit-exact
    assert np.array_equal(d["splat_gaussian"], ref.splat_gaussian)
    assert np.array_equal(d["splat_mu2d"], ref.splat_mu2d)
    assert np.array_equal(d["splat_depth"], ref.splat_depth)
    assert np.array_equal(d["tile_lists"], ref.tile_lists)
    assert np.array_equal(d["tile_ranges"], ref.tile_ranges)
    assert np.array_equal(d["contrib_count"], ref.contrib_count)
    assert np.array_equal(d["overflow_mask"], ref.overflow_mask)
    assert np.max(np.abs(d["splat_radius"] - ref.splat_radius) / ref.splat_radius) < 1e-14
    assert np.max(np.abs(d["final_transmittance"] - ref.final_transmittance)) < 1e-5
    assert np.all(d["accum_transmittance"] + d["final_transmittance"] == 1.0)


@pytest.mark.parametrize("early", [0.0, 0.3, 2.0])
def test_early_termination_configs_match_oracle(G, ctx, early):
    """RasterConfig.early_termination beyond the default: 0 (never stop), a
    large threshold, and > 1, where every pixel stops right after including
    its first splat (rasterizer.cpp:257-258: T is updated, then compared).
    Contrib counts bit-exact, image and final T within 1e-5, d_pose 1e-3."""
    hc, ocam, bg, rng = scene(55, 12, 48)
    cloud = to_dev(G, ctx, hc)
    cam = dev_cam(G, ocam)
    out = G.render(ctx, cloud, cam, bg, config=G.RasterConfig.default(early_termination=early))
    ref = O.render(hc, ocam, bg, cfg=O.default_raster_config(early_termination=early), keep_handle=True)
    d = out.download()
    assert np.array_equal(d["contrib_count"], ref.contrib_count)
    assert np.max(np.abs(d["image"] - ref.image)) < 1e-5
    assert np.max(np.abs(d["final_transmittance"] - ref.final_transmittance)) < 1e-5
    d_img = np.random.default_rng(7).uniform(-1, 1, ref.image.shape)
    _, dp = G.render_backward(ctx, cloud, cam, out, d_img, pose_only=True)
    gr = O.render_backward(hc, ocam, ref, d_img)
    ref.free()
    assert rel_err(dp, gr.d_pose) < 1e-3


@pytest.fixture(params=["tile_local", "global"])
def binning(request, G, ctx):
    mode = G.Context.BINNING_TILE_LOCAL if request.param == "tile_local" else G.Context.BINNING_GLOBAL
    ctx.set_binning(mode)
    yield mode
    ctx.set_binning(G.Context.BINNING_TILE_LOCAL)


def test_binning_bit_exact_on_device_records(G, ctx, binning):
    """rasterizer.cpp:127-168 re-run on the GPU's own FP64 records must give
    the device tile lists / ranges bit for bit (C1-sized scene)."""
    hc, poses = synth_scene(99, 10000, 256, scale_offset=math.log(500 / 10000) / 3)
    cam = O.synth_camera(256, 256, poses[0])
    cloud = to_dev(G, ctx, hc)
    out = G.render(ctx, cloud, dev_cam(G, cam))
    assert out.info().binning == binning
    d = out.download()
    n = hc.n
    keep = np.zeros(n, np.uint8)
    keep[d["splat_gaussian"]] = 1
    mu2d = np.zeros((n, 2))
    mu2d[d["splat_gaussian"]] = d["splat_mu2d"]
    rad = np.zeros(n)
    rad[d["splat_gaussian"]] = d["splat_radius"]
    dep = np.zeros(n)
    dep[d["splat_gaussian"]] = d["splat_depth"]
    sg, lists, ranges = O.bin_records(keep, mu2d, rad, dep, 256, 256)
    assert np.array_equal(sg, d["splat_gaussian"])
    assert np.array_equal(lists, d["tile_lists"])
    assert np.array_equal(ranges, d["tile_ranges"])
    # and the FP64 geometry equals the oracle's own evaluation
    ref = O.render(hc, cam)
    assert np.array_equal(d["splat_gaussian"], ref.splat_gaussian)
    assert np.array_equal(d["splat_depth"], ref.splat_depth)
    assert np.array_equal(d["splat_mu2d"], ref.splat_mu2d)
    flips = np.sum(d["tile_lists"] != ref.tile_lists) if len(d["tile_lists"]) == len(ref.tile_lists) else -1
    assert flips == 0
    assert np.array_equal(d["tile_ranges"], ref.tile_ranges)


def test_binning_bit_exact_c2_scale(G, ctx, binning):
    """C2 shape (300k Gaussians, 1008x756, forward-facing): the device's
    depth order, tile lists and ranges equal rasterizer.cpp:127-168 re-run on
    the device's own FP64 records, across hundreds of 4096-item sort tiles
    (exercises the decoupled look-back)."""
    hc, poses = synth_scene(2, 300_000, 1008, kind=1, cams=2, scale_offset=math.log(500 / 300_000) / 3)
    cam = O.make_camera(0.75 * 1008, 0.75 * 1008, 503.5, 377.5, 1008, 756, *O.pose_split(poses[0]))
    cloud = to_dev(G, ctx, hc)
    d = G.render(ctx, cloud, dev_cam(G, cam), want_image=False).download()
    n = hc.n
    keep = np.zeros(n, np.uint8)
    keep[d["splat_gaussian"]] = 1
    mu2d = np.zeros((n, 2))
    mu2d[d["splat_gaussian"]] = d["splat_mu2d"]
    rad = np.zeros(n)
    rad[d["splat_gaussian"]] = d["splat_radius"]
    dep = np.zeros(n)
    dep[d["splat_gaussian"]] = d["splat_depth"]
    sg, lists, ranges = O.bin_records(keep, mu2d, rad, dep, 1008, 756)
    assert len(d["splat_gaussian"]) > 200_000 and len(lists) > 500_000
    assert np.array_equal(sg, d["splat_gaussian"])
    assert np.array_equal(lists, d["tile_lists"])
    assert np.array_equal(ranges, d["tile_ranges"])


MARGIN = 1e-4  # relative decision margin above which FP32 cannot flip a cutoff / termination decision


def image_parity_report(name, img, ref_rr, extra=None):
    """north_star's 1e-5 max-abs on every pixel whose FP64 decisions have a
    relative margin > MARGIN (oracle decision_margin); the pixels below it are
    counted and their worst error reported (gpurun_out/image_parity_*.json)."""
    import json
    import os
    err = np.max(np.abs(img - ref_rr.image), axis=2)
    margin = O.decision_margin(ref_rr)
    stable = margin > MARGIN
    rep = {"pixels": int(err.size), "near_decision_pixels": int((~stable).sum()),
           "max_abs_stable": float(err[stable].max()) if stable.any() else 0.0,
           "max_abs_near_decision": float(err[~stable].max()) if (~stable).any() else 0.0,
           "pixels_over_1e-5": int((err > 1e-5).sum()), "worst_pixel": [int(v) for v in np.unravel_index(
               np.argmax(err), err.shape)], "worst_abs": float(err.max())}
    rep.update(extra or {})
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/image_parity_{name}.json", "w") as fh:
        json.dump(rep, fh)
    return rep


def test_render_c1_scene_image(G, ctx):
    """C1 (10k Gaussians SH-3, 256x256): <= 1e-5 max-abs on every pixel whose
    FP64 cutoff / termination decisions have a relative margin > 1e-4; the
    near-decision pixels are a fraction of a percent and reported."""
    hc, poses = synth_scene(99, 10000, 256, scale_offset=math.log(500 / 10000) / 3)
    cam = O.synth_camera(256, 256, poses[0])
    cloud = to_dev(G, ctx, hc)
    d = G.render(ctx, cloud, dev_cam(G, cam)).download()
    ref = O.render(hc, cam, keep_handle=True)
    rep = image_parity_report("c1", d["image"], ref)
    ref.free()
    assert rep["max_abs_stable"] < 1e-5, rep
    assert rep["near_decision_pixels"] < 0.01 * rep["pixels"], rep


def test_empty_cloud_and_culling(G, ctx):
    hc = O.HostCloud(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3, 1)), 0, 0)
    cloud = to_dev(G, ctx, hc)
    cam = G.Camera.make(20, 20, 7.5, 7.5, 16, 16)
    out = G.render(ctx, cloud, cam, (0.3, 0.6, 0.9))
    assert np.allclose(out.image, np.array([0.3, 0.6, 0.9]), atol=0, rtol=1e-7)
    # culled Gaussians contribute exactly zero (test_rasterizer.cpp:308-343)
    hc, ocam, bg, rng = scene(60, 6, 32, conditioned=False)
    base = G.render(ctx, to_dev(G, ctx, hc), dev_cam(G, ocam), bg).image
    R, t = O.camera_pose(ocam)
    ext = hc.copy()
    for mean in (R.T @ (np.array([0, 0, -2.0]) - t), R.T @ (np.array([50.0, 0, 2.0]) - t)):
        ext.means = np.vstack([ext.means, mean])
        ext.rotations = np.vstack([ext.rotations, [1, 0, 0, 0]])
        ext.log_scales = np.vstack([ext.log_scales, np.full(3, math.log(0.1))])
        ext.opacity_logits = np.append(ext.opacity_logits, math.log(9))
        ext.sh = np.concatenate([ext.sh, np.full((1, 3, 16), 0.3)])
    ext = ext.as_float32_exact()
    ecloud = to_dev(G, ctx, ext)
    out = G.render(ctx, ecloud, dev_cam(G, ocam), bg)
    assert np.array_equal(out.image, base)
    d_img = np.random.default_rng(0).uniform(-1, 1, (32, 32, 3))
    g, _ = G.render_backward(ctx, ecloud, dev_cam(G, ocam), out, d_img)
    for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits"):
        assert np.all(g[k][6:] == 0)


def test_repeat_render_bit_identical(G, ctx):
    hc, ocam, bg, _ = scene(55, 60, 64, conditioned=False)
    cloud = to_dev(G, ctx, hc)
    a = G.render(ctx, cloud, dev_cam(G, ocam), bg).download()
    b = G.render(ctx, cloud, dev_cam(G, ocam), bg).download()
    for k in ("image", "final_transmittance", "contrib_count", "tile_lists", "tile_ranges"):
        assert a[k].tobytes() == b[k].tobytes()


def crowded_tile_scene(n, z_levels=None, seed=5):
    """n small Gaussians projecting into the top-left 16x16 tile of a 64x64
    image (identity pose): one tile list of ~n entries. z_levels quantises the
    depths so most entries tie on depth (ties resolve by Gaussian index)."""
    r = np.random.default_rng(seed)
    z = r.uniform(2.0, 4.0, n) if z_levels is None else r.choice(np.asarray(z_levels, np.float64), n)
    u, v = r.uniform(5.0, 11.0, n), r.uniform(5.0, 11.0, n)
    fx = 40.0
    means = np.stack([(u - 0.5) * z / fx, (v - 0.5) * z / fx, z], axis=1)
    rot = r.normal(size=(n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    hc = O.HostCloud(means, rot, np.full((n, 3), math.log(0.002)) + r.uniform(-0.3, 0.3, (n, 3)),
                     r.uniform(-4.0, -1.0, n), r.uniform(-0.5, 0.5, (n, 3, 1)), 0, 0)
    cam = O.make_camera(fx, fx, 0.5, 0.5, 64, 64, np.eye(3), np.zeros(3))
    return hc.as_float32_exact(), cam


@pytest.mark.parametrize("n,z_levels,expect", [(1500, None, 0), (1500, [2.0, 3.0], 0), (6000, None, 0),
                                                (6000, [2.0, 2.5, 3.0], 0), (20000, None, 1)])
def test_crowded_tile_lists_bit_exact(G, ctx, n, z_levels, expect):
    """Per-tile sort paths: small CTA (<= 2048 entries), large CTA (<= 8192,
    incl. massive exact depth ties), and the fallback to global binning for a
    tile beyond 8192 entries — tile lists equal the reference's each time."""
    hc, cam = crowded_tile_scene(n, z_levels)
    cloud = to_dev(G, ctx, hc)
    out = G.render(ctx, cloud, dev_cam(G, cam), (0.1, 0.2, 0.3))
    assert out.info().binning == expect
    d = out.download()
    ref = O.render(hc, cam, (0.1, 0.2, 0.3))
    r0 = ref.tile_ranges.reshape(-1, 2)[0]
    assert r0[1] - r0[0] > n * 0.9
    assert np.array_equal(d["splat_gaussian"], ref.splat_gaussian)
    assert np.array_equal(d["tile_lists"], ref.tile_lists)
    assert np.array_equal(d["tile_ranges"], ref.tile_ranges)
    assert np.array_equal(d["contrib_count"], ref.contrib_count)
    assert np.max(np.abs(d["image"] - ref.image)) < 1e-4


# -------------------------------------------------------------------- loss
def test_rgb_loss_matches_oracle(G, ctx):
    r = np.random.default_rng(3)
    a = r.uniform(0, 1, (37, 53, 3)).astype(np.float32).astype(np.float64)
    b = np.clip(a + r.uniform(-0.2, 0.2, a.shape), 0, 1).astype(np.float32).astype(np.float64)
    loss, d = G.rgb_loss(ctx, a, b, 0.2)
    lref, dref = O.rgb_loss(a, b, 0.2)
    # K6: FP32 separable convolutions, FP64 pointwise terms and sums
    assert abs(loss - lref) < 1e-7 * abs(lref)
    assert np.max(np.abs(d - dref)) < 1e-4 * np.max(np.abs(dref))
    same, ds = G.rgb_loss(ctx, a, a, 0.2)
    assert same == 0.0 and np.all(ds == 0.0)  # test_losses.cpp:25-32
    l0 = G.rgb_loss(ctx, np.full((16, 16, 3), 0.6), np.full((16, 16, 3), 0.5), 0.0, want_grad=False)
    assert abs(l0 - 0.1) < 1e-7


# ---------------------------------------------------------------- backward
@pytest.mark.parametrize("seed", [61, 62, 63])
def test_backward_matches_oracle(G, ctx, seed):
    hc, ocam, bg, rng = scene(seed, 10, 32)
    d_img = np.array([O.lib().orc_rng_uniform_range(O.C.byref(rng), -1, 1) for _ in range(32 * 32 * 3)]).reshape(32, 32, 3)
    cloud = to_dev(G, ctx, hc)
    cam = dev_cam(G, ocam)
    out = G.render(ctx, cloud, cam, bg)
    g, dp = G.render_backward(ctx, cloud, cam, out, d_img)
    ref = O.render(hc, ocam, bg, keep_handle=True)
    gr = O.render_backward(hc, ocam, ref, d_img)
    ref.free()
    assert rel_err(dp, gr.d_pose) < 1e-3
    assert rel_err(g["d_means"], gr.d_means) < 1e-3
    assert rel_err(g["d_rotations"], gr.d_rotations) < 1e-3
    assert rel_err(g["d_log_scales"], gr.d_log_scales) < 1e-3
    assert rel_err(g["d_opacity_logits"], gr.d_opacity_logits) < 1e-3
    assert rel_err(g["d_sh"], gr.d_sh) < 1e-3
    assert rel_err(g["d_mu2d"], gr.d_mu2d) < 1e-3
    # pose-only path (8 partials per entry, FP32 per-splat chain, FP64 6-vector
    # accumulation) agrees with the oracle and with the FP64-chain full path
    _, dp2 = G.render_backward(ctx, cloud, cam, out, d_img, pose_only=True)
    assert rel_err(dp2, gr.d_pose) < 1e-3
    assert np.max(np.abs(dp2 - dp)) <= 1e-5 * np.max(np.abs(dp))


def test_backward_global_binning_bitwise_equals_tile_local(G, ctx):
    """Both binning paths build the same tile lists, and K4b finds each
    splat's tile rect (aux_g vs rect_g) and the per-tile cut of the entries
    no pixel replays the same way: full gradients and the pose-only d_pose
    must be bit-identical (C1-sized scene, the loss gradient as d_image)."""
    hc, poses = synth_scene(99, 10000, 256, scale_offset=math.log(500 / 10000) / 3)
    ocam = O.synth_camera(256, 256, poses[1])
    cloud = to_dev(G, ctx, hc)
    cam = dev_cam(G, ocam)
    target = O.render(hc, O.synth_camera(256, 256, poses[0])).image
    res = {}
    for mode in (G.Context.BINNING_TILE_LOCAL, G.Context.BINNING_GLOBAL):
        ctx.set_binning(mode)
        try:
            out = G.render(ctx, cloud, cam)
            assert out.info().binning == mode
            _, d_img = G.rgb_loss(ctx, out.image, target, 0.2)
            g, dp = G.render_backward(ctx, cloud, cam, out, d_img)
            _, dpo = G.render_backward(ctx, cloud, cam, out, d_img, pose_only=True)
            res[mode] = (g, dp, dpo)
        finally:
            ctx.set_binning(G.Context.BINNING_TILE_LOCAL)
    (g0, dp0, dpo0), (g1, dp1, dpo1) = res[G.Context.BINNING_TILE_LOCAL], res[G.Context.BINNING_GLOBAL]
    assert np.any(dp0 != 0)
    assert dp0.tobytes() == dp1.tobytes() and dpo0.tobytes() == dpo1.tobytes()
    for k in g0:
        assert g0[k].tobytes() == g1[k].tobytes(), k


def test_backward_invariants(G, ctx):
    hc, ocam, bg, rng = scene(58, 8, 32, conditioned=False)
    cloud = to_dev(G, ctx, hc)
    cam = dev_cam(G, ocam)
    out = G.render(ctx, cloud, cam, bg)
    g, dp = G.render_backward(ctx, cloud, cam, out, np.zeros((32, 32, 3)))
    assert np.all(dp == 0) and all(np.all(v == 0) for v in g.values())
    with pytest.raises(G.GsbError) as ei:
        G.render_backward(ctx, cloud, cam, out, np.zeros((16, 32, 3)))
    assert ei.value.code == G.ERR_DIMENSION_MISMATCH
    other = dev_cam(G, ocam)
    other.t[0] += 0.1
    with pytest.raises(G.GsbError) as ei:
        G.render_backward(ctx, cloud, other, out, np.zeros((32, 32, 3)))
    assert ei.value.code == G.ERR_STATE_MISMATCH
    moved = hc.copy()
    moved.means[0] += [0.5, 0, 0]
    cloud.upload(moved.means, moved.rotations, moved.log_scales, moved.opacity_logits, moved.sh, 3)
    with pytest.raises(G.GsbError) as ei:
        G.render_backward(ctx, cloud, cam, out, np.zeros((32, 32, 3)))
    assert ei.value.code == G.ERR_STATE_MISMATCH
    # gauge identity d_pose_v = R_c sum d_means (test_rasterizer.cpp:377-390)
    hc, ocam, bg, rng = scene(63, 15, 32, conditioned=False)
    cloud = to_dev(G, ctx, hc)
    cam = dev_cam(G, ocam)
    out = G.render(ctx, cloud, cam, bg)
    d_img = np.random.default_rng(1).uniform(-1, 1, (32, 32, 3))
    g, dp = G.render_backward(ctx, cloud, cam, out, d_img)
    R, _ = O.camera_pose(ocam)
    exp = R @ g["d_means"].sum(axis=0)
    assert np.linalg.norm(dp[:3] - exp) < 1e-4 * max(1.0, np.linalg.norm(exp))
    # determinism
    _, dp_b = G.render_backward(ctx, cloud, cam, out, d_img)
    assert dp_b.tobytes() == dp.tobytes()


def test_backward_c1_scene_pose_gradient(G, ctx):
    """C1-sized scene with the real loss gradient: d_pose within 1e-3."""
    hc, poses = synth_scene(99, 10000, 256, scale_offset=math.log(500 / 10000) / 3)
    cam_gt = O.synth_camera(256, 256, poses[0])
    target = O.render(hc, cam_gt).image
    noisy = O.perturb_pose(poses[0], 3.0, 0.03, O.make_rng(1002))
    ocam = O.synth_camera(256, 256, noisy)
    ref = O.render(hc, ocam, keep_handle=True)
    _, d_img = O.rgb_loss(ref.image, target, 0.2)
    gr = O.render_backward(hc, ocam, ref, d_img)
    ref.free()
    cloud = to_dev(G, ctx, hc)
    cam = dev_cam(G, ocam)
    out = G.render(ctx, cloud, cam)
    _, dp = G.render_backward(ctx, cloud, cam, out, d_img, pose_only=True)
    assert np.linalg.norm(dp - gr.d_pose) / np.linalg.norm(gr.d_pose) < 1e-3


def test_backward_c3_scale_pose_gradient(G, ctx):
    """The bench's workload size (C3: 1M Gaussians SH-3, 1008x756, view 0 at
    its perturbed init pose) with the oracle's loss gradient as d_image: the
    pose-only d_pose (half-quadrant K4a, per-tile cut, FP32 per-splat chain)
    within 1e-3 relative of the FP64 oracle, and the rendered image within
    1e-5 on all but the pixels an FP32 cutoff / termination decision flips."""
    import bench
    _, hc = bench._oracle_scene()
    gt, init = bench.all_views()
    intr = G.synth_intrinsics(bench.WIDTH, bench.HEIGHT)
    cam_gt = O.make_camera(*intr, bench.WIDTH, bench.HEIGHT, *O.pose_split(gt[0]))
    ocam = O.make_camera(*intr, bench.WIDTH, bench.HEIGHT, *O.pose_split(init[0]))
    target = O.render(hc, cam_gt).image
    ref = O.render(hc, ocam, keep_handle=True)
    _, d_img = O.rgb_loss(ref.image, target, 0.2)
    gr = O.render_backward(hc, ocam, ref, d_img)
    cloud = G.Cloud(ctx, bench.N_GAUSS, bench.SH_DEGREE)
    cloud.synth(bench.SCENE_SEED, bench.log_scale_offset(bench.N_GAUSS))
    cam = G.Camera.from_pose12(*intr, bench.WIDTH, bench.HEIGHT, init[0])
    out = G.render(ctx, cloud, cam)
    rep = image_parity_report("c3", out.image, ref)
    assert rep["max_abs_stable"] < 1e-5, rep
    assert rep["near_decision_pixels"] < 0.01 * rep["pixels"], rep
    _, dp = G.render_backward(ctx, cloud, cam, out, d_img, pose_only=True)
    rel = np.linalg.norm(dp - gr.d_pose) / np.linalg.norm(gr.d_pose)
    ref.free()
    assert rel < 1e-3, rel


def test_c3_scale_trajectory_matches_oracle(G, ctx):
    """The bench's unit of work at full size: 10 pose_descent iterations of
    C3 view 0 (1M Gaussians SH-3, 1008x756, early exits off) through the
    device session against the FP64 oracle: every iteration's pose within
    rot 0.1 deg / trans 1e-3 (test_trainer.cpp:506-507), loss within 1e-3
    relative."""
    import bench
    _, hc = bench._oracle_scene()
    gt, init = bench.all_views()
    intr = G.synth_intrinsics(bench.WIDTH, bench.HEIGHT)
    cam_gt = O.make_camera(*intr, bench.WIDTH, bench.HEIGHT, *O.pose_split(gt[0]))
    target = O.render(hc, cam_gt).image
    budget = 10
    ref = O.estimate_pose(hc, target, *intr, init[0], budget=budget, pose_converged_eps=0.0)
    cloud = G.Cloud(ctx, bench.N_GAUSS, bench.SH_DEGREE)
    cloud.synth(bench.SCENE_SEED, bench.log_scale_offset(bench.N_GAUSS))
    img = G.Image(ctx, target)
    cfg = G.PoseConfig.default(budget=budget, pose_converged_eps=0.0)
    res = G.estimate_pose(ctx, cloud, img, list(intr), init[0], cfg, trace=True)
    assert res["steps"] == ref["steps"] == budget
    for k in range(budget):
        r, d = O.abs_pose_error(res["trace_pose"][k], ref["trace_pose"][k])
        assert r < 0.1 and d < 1e-3, (k, r, d)
    rel = np.abs(res["trace_loss"] - ref["trace_loss"]) / ref["trace_loss"]
    assert np.max(rel) < 1e-3, rel


# ------------------------------------------------------------- optimiser
def test_pose_step_matches_oracle(G, ctx):
    R, t = O.se3_exp(np.array([0.3, -0.2, 0.5, 0.4, -0.7, 0.2]))
    p = O.pose_join(R, t)
    same, _ = G.pose_step(ctx, p, np.zeros(6), 1e-2, G.PoseAdam())
    assert same.tobytes() == p.tobytes()  # trainer.cpp:86
    g = np.array([0.3, -0.5, 0.1, 0.9, -0.2, 0.4])
    zero_lr, _ = G.pose_step(ctx, p, g, 0.0, G.PoseAdam())
    assert zero_lr.tobytes() == p.tobytes()
    st_g, st_o = G.PoseAdam(), O.PoseAdam()
    pg, po = p.copy(), p.copy()
    for k in range(20):
        gk = g * math.cos(k) + 0.1
        pg, ag = G.pose_step(ctx, pg, gk, 1e-2, st_g)
        po, ao = O.pose_step(po, gk, 1e-2, st_o)
    assert np.max(np.abs(pg - po)) < 1e-12
    assert st_g.step == st_o.step == 20


def test_estimate_pose_trajectory_matches_oracle(G, ctx):
    """pose_descent on the device vs the oracle: per-iteration poses within
    rot 0.1 deg / trans 1e-3, final errors within the same bounds."""
    rng = O.make_rng(99)
    hc = O.synth_cloud(500, 1, rng).as_float32_exact()
    poses = O.synth_poses(0, 20, rng)
    cam = O.synth_camera(64, 64, poses[0])
    target = O.render(hc, cam).image
    noisy = O.perturb_pose(poses[0], 15.0, 0.15, O.make_rng(1002))
    budget = 60
    ref = O.estimate_pose(hc, target, cam.fx, cam.fy, cam.cx, cam.cy, noisy, budget=budget)
    cloud = to_dev(G, ctx, hc)
    img = G.Image(ctx, target)
    cfg = G.PoseConfig.default(budget=budget)
    res = G.estimate_pose(ctx, cloud, img, [cam.fx, cam.fy, cam.cx, cam.cy], noisy, cfg, trace=True)
    assert res["steps"] == ref["steps"]
    for k in range(0, res["steps"], 5):
        r, d = O.abs_pose_error(res["trace_pose"][k], ref["trace_pose"][k])
        assert r < 0.1 and d < 1e-3, (k, r, d)
    assert np.max(np.abs(res["trace_loss"] - ref["trace_loss"])) < 1e-4


def test_c1_pose_descent_log_matches_oracle(G, ctx):
    """C1, the CPU-oracle parity config: 10k Gaussians SH-3,
    256x256, orbit camera 0 of seed 99, perturb 15 deg / 0.15 from Rng(1002),
    100 pose_descent iterations with the cosine schedule. The per-iteration
    pose log stays within rot 0.1 deg / trans 1e-3 of the oracle's
    (test_trainer.cpp:506-507). The loss log follows the poses (not part of
    the contract): within 5e-3 relative per iteration (measured 1.2e-3 at
    worst) and the final loss within 1e-3 relative."""
    hc, poses = synth_scene(99, 10000, 256, scale_offset=math.log(500 / 10000) / 3)
    cam = O.synth_camera(256, 256, poses[0])
    target = O.render(hc, cam).image
    noisy = O.perturb_pose(poses[0], 15.0, 0.15, O.make_rng(1002))
    budget = 100
    ref = O.estimate_pose(hc, target, cam.fx, cam.fy, cam.cx, cam.cy, noisy, budget=budget, pose_converged_eps=0.0)
    cloud = to_dev(G, ctx, hc)
    img = G.Image(ctx, target)
    cfg = G.PoseConfig.default(budget=budget, pose_converged_eps=0.0)
    res = G.estimate_pose(ctx, cloud, img, [cam.fx, cam.fy, cam.cx, cam.cy], noisy, cfg, trace=True)
    assert res["steps"] == ref["steps"] == budget
    worst = (0.0, 0.0)
    for k in range(res["steps"]):
        r, d = O.abs_pose_error(res["trace_pose"][k], ref["trace_pose"][k])
        worst = (max(worst[0], r), max(worst[1], d))
    assert worst[0] < 0.1 and worst[1] < 1e-3, worst
    rel = np.abs(res["trace_loss"] - ref["trace_loss"]) / ref["trace_loss"]
    assert np.max(rel) < 5e-3 and rel[-1] < 1e-3, (np.max(rel), rel[-1])


def test_pose_batch_bitwise_equals_sequential_sessions(G, ctx):
    """A pose batch (sessions as parallel graph branches, private forward
    states) gives bit-identical per-view trajectories to stepping each
    session alone, and each view still tracks the oracle."""
    rng = O.make_rng(99)
    hc = O.synth_cloud(2000, 3, rng).as_float32_exact()
    poses = O.synth_poses(0, 6, rng)
    cloud = to_dev(G, ctx, hc)
    noise = O.make_rng(1002)
    cams = [O.synth_camera(96, 80, poses[v]) for v in range(5)]
    targets = [O.render(hc, c).image for c in cams]
    inits = [O.perturb_pose(poses[v], 15.0, 0.15, noise) for v in range(5)]
    intr = [cams[0].fx, cams[0].fy, cams[0].cx, cams[0].cy]
    cfg = G.PoseConfig.default(budget=40, pose_converged_eps=0.0)
    imgs = [G.Image(ctx, t) for t in targets]
    seq = []
    for v in range(5):
        s = G.PoseSession(ctx, cloud, imgs[v], intr, inits[v], cfg)
        s.step(40)
        seq.append(s.read())
        del s
    sessions = [G.PoseSession(ctx, cloud, imgs[v], intr, inits[v], cfg) for v in range(5)]
    batch = G.PoseBatch(ctx, sessions)
    for _ in range(4):
        batch.step_async(10)
    batch.sync()
    for v in range(5):
        r = sessions[v].read()
        assert r["steps"] == seq[v]["steps"] == 40
        assert np.array_equal(r["pose"], seq[v]["pose"]), v
        assert np.array_equal(r["best_pose"], seq[v]["best_pose"]), v
        assert r["final_loss"] == seq[v]["final_loss"]
    batch.close()
    # the one-call form
    res = G.estimate_poses(ctx, cloud, imgs, intr, np.stack(inits), cfg)
    for v in range(5):
        assert np.array_equal(res["pose"][v], seq[v]["best_pose"]), v
        assert res["steps"][v] == 40
    # view 0 against the oracle's pose_descent
    ref = O.estimate_pose(hc, targets[0], *intr, inits[0], budget=40, pose_converged_eps=0.0)
    r, d = O.abs_pose_error(res["pose"][0], ref["pose"])
    assert r < 0.1 and d < 1e-3, (r, d)


def test_pose_batch_capacity_growth(G, ctx):
    """Sessions of a batch start with a tiny entry capacity on their private
    forward states: discarded iterations are re-run and results still equal
    the sequential ones."""
    rng = O.make_rng(7)
    hc = O.synth_cloud(4000, 1, rng).as_float32_exact()
    hc.log_scales += 0.7  # large footprints -> many tile entries
    poses = O.synth_poses(1, 3, rng)
    cloud = to_dev(G, ctx, hc)
    cams = [O.synth_camera(128, 96, poses[v]) for v in range(3)]
    imgs = [G.Image(ctx, O.render(hc, c).image) for c in cams]
    noise = O.make_rng(5)
    inits = [O.perturb_pose(poses[v], 5.0, 0.05, noise) for v in range(3)]
    intr = [cams[0].fx, cams[0].fy, cams[0].cx, cams[0].cy]
    cfg = G.PoseConfig.default(budget=12, pose_converged_eps=0.0)
    seq = [G.estimate_pose(ctx, cloud, imgs[v], intr, inits[v], cfg) for v in range(3)]
    res = G.estimate_poses(ctx, cloud, imgs, intr, np.stack(inits), cfg)
    for v in range(3):
        assert np.array_equal(res["pose"][v], seq[v]["pose"]), v


@pytest.mark.slow
def test_estimate_pose_acceptance_criterion(G, ctx):
    """tests/acceptance.cpp:74-100 on the device: >= 18/20 trials converge."""
    rng = O.make_rng(99)
    hc = O.synth_cloud(500, 1, rng).as_float32_exact()
    poses = O.synth_poses(0, 20, rng)
    cloud = to_dev(G, ctx, hc)
    noise = O.make_rng(1002)
    hits = 0
    for t in range(20):
        cam = O.synth_camera(64, 64, poses[t])
        img = G.Image(ctx, O.render(hc, cam).image)
        noisy = O.perturb_pose(poses[t], 15.0, 0.15, noise)
        res = G.estimate_pose(ctx, cloud, img, [cam.fx, cam.fy, cam.cx, cam.cy], noisy)
        r, d = O.abs_pose_error(res["pose"], poses[t])
        hits += (r < 5.0 and d < 0.05)
    assert hits >= 18


def test_cloud_adam_step_matches_oracle(G, ctx):
    hc, ocam, bg, rng = scene(64, 10, 32, conditioned=False)
    d_img = np.random.default_rng(2).uniform(-1, 1, (32, 32, 3))
    cloud = to_dev(G, ctx, hc)
    cam = dev_cam(G, ocam)
    out = G.render(ctx, cloud, cam, bg)
    grads = G.Grads(ctx, cloud)
    G.render_backward(ctx, cloud, cam, out, d_img, grads=grads)
    gd = grads.download()
    adam = G.lib()
    h = G._vp()
    G._check(adam.gsb_adam_create(ctx.h, cloud.h, G.C.byref(h)))
    lrs = np.array([1.6e-2, 1e-3, 5e-3, 5e-2, 2.5e-3, 1.25e-4])
    G._check(adam.gsb_cloud_adam_step(ctx.h, cloud.h, grads.h, h, G._p(lrs)))
    m, q, ls, op, sh = cloud.download()
    # oracle Adam on the same (FP32-rounded) gradients
    oc = hc.copy()
    og = O.Grads()
    st = (O.C.c_double * 1)
    cv = oc.c()
    n = oc.n
    gm = [np.ascontiguousarray(gd[k].reshape(-1)) for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh")]
    og.n = n
    og.sh_len = gm[4].size
    P = O.C.POINTER(O.C.c_double)
    og.d_means, og.d_rotations, og.d_log_scales, og.d_opacity_logits, og.d_sh = [a.ctypes.data_as(P) for a in gm]
    states = (O.C.c_byte * (5 * 32))()
    O.lib().orc_cloud_adam_step.argtypes = [O.C.POINTER(O.Cloud), O.C.POINTER(O.Grads), O.C.c_void_p, O.C.c_void_p]
    O.lib().orc_cloud_adam_step(cv.ref(), O.C.byref(og), states, O._p(lrs))
    want = O._from_c_cloud(cv.s)
    assert np.max(np.abs(m - want.means)) < 1e-6
    assert np.max(np.abs(q - want.rotations)) < 1e-6
    assert np.max(np.abs(ls - want.log_scales)) < 1e-6
    assert np.max(np.abs(sh - want.sh)) < 1e-6
    adam.gsb_adam_destroy(h)
    del st
