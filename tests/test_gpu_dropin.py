"""The drop-in proof: the reference's own code running on the
device through libgsb200.

* integration/_build/* — the reference library compiled from
  /root/reference/proj/src with integration/gsopt_b200.cpp (the adapter over
  the C ABI) linked INSTEAD OF src/rasterizer.cpp (integration/build.py, run
  by __graft_entry__.build() where /root/reference exists; the binaries ship
  with the snapshot). Acceptance criterion 2 (tests/acceptance.cpp:74-100:
  estimate_pose from +-15 deg / +-0.15 perturbations, >= 18/20 converge) runs
  the reference's pipelines.cpp pose_descent loop with every render /
  render_backward on the B200.
* state_fingerprint: a host-uploaded cloud's exported forward state carries
  the reference's own FNV fingerprint (rasterizer.cpp:52-73) bit for bit.
* render_expected_depth (rasterizer.cpp:283-323) against the reference build.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")


@pytest.fixture(scope="module")
def G():
    from paper_2410_08743_b200 import build, gsb
    build.build()
    return gsb


@pytest.fixture(scope="module")
def ctx(G):
    return G.Context(0)


def to_dev(G, ctx, hc):
    return G.Cloud.from_host(ctx, hc.means, hc.rotations, hc.log_scales, hc.opacity_logits, hc.sh, hc.sh_degree,
                             hc.active_sh_degree)


def dev_cam(G, ocam):
    return G.Camera.make(ocam.fx, ocam.fy, ocam.cx, ocam.cy, ocam.width, ocam.height,
                         np.array(ocam.R[:]).reshape(3, 3), np.array(ocam.t[:]))


def _run(exe, *args, timeout=450):
    path = os.path.join(BUILD, exe)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (integration/build.py needs /root/reference at build time)")
    # The reference's host code runs on its own Pool (core.cpp:39-80), whose
    # unlocked job reset can hang run() (tests/test_ref_pins.py); a hung run
    # is retried once (criterion 2 normally takes ~120 s).
    for attempt in range(2):
        try:
            r = subprocess.run([path, *map(str, args)], capture_output=True, text=True, timeout=timeout)
            break
        except subprocess.TimeoutExpired:
            if attempt == 1:
                raise
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, f"dropin_{exe}_{'_'.join(map(str, args)) or 'all'}.txt"), "w") as fh:
        fh.write(r.stdout + r.stderr)
    return r


def test_adapter_acceptance_criterion_2_pose_estimation():
    r = _run("acceptance_b200", 2)
    assert "[PASS] criterion 2" in r.stdout, r.stdout + r.stderr
    assert r.returncode == 0


def test_adapter_acceptance_criterion_8_determinism_perf():
    """tests/acceptance.cpp:451-487: bit-identical repeat renders and 100k
    Gaussians at 800x600 in under 2 s, through the adapter."""
    r = _run("acceptance_b200", 8)
    assert "[PASS] criterion 8" in r.stdout, r.stdout + r.stderr


def test_fingerprint_equals_reference(G, ctx):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = O.make_rng(31)
    hc = O.synth_cloud(700, 2, rng).as_float32_exact()
    pose = O.synth_poses(1, 1, rng)[0]
    cam = O.synth_camera(80, 64, pose)
    with O.reference_backend():
        ref = O.render(hc, cam)
    cloud = to_dev(G, ctx, hc)
    out = G.render(ctx, cloud, dev_cam(G, cam))
    assert out.frame.info().state_fingerprint == ref.fingerprint  # rasterizer.cpp:52-73 bit for bit
    assert G.state_fingerprint(cloud, dev_cam(G, cam)) == ref.fingerprint  # the same key, without rendering
    # a device-side change (here: a re-upload of different content) changes it
    hc2 = hc.copy()
    hc2.opacity_logits = hc2.opacity_logits + 0.5
    cloud.upload(hc2.means, hc2.rotations, hc2.log_scales, hc2.opacity_logits, hc2.sh, hc2.active_sh_degree)
    out2 = G.render(ctx, cloud, dev_cam(G, cam))
    with O.reference_backend():
        ref2 = O.render(hc2, cam)
    assert out2.frame.info().state_fingerprint == ref2.fingerprint != ref.fingerprint


def test_render_expected_depth_matches_reference(G, ctx):
    """Conditioned scenes (no pixel near a cutoff / termination decision):
    weights within 1e-5, depths within 1e-5 relative where the weight
    exceeds 1e-3 (the reference divides by the weight sum)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for seed in (41, 42, 43):
        rng = O.make_rng(seed)
        hc, cam, bg = O.make_conditioned_scene(rng, 12, 48)
        hc = hc.as_float32_exact()
        d_ref, w_ref = O.ref_render_expected_depth(hc, cam)
        d, w = G.render_expected_depth(ctx, to_dev(G, ctx, hc), dev_cam(G, cam))
        assert np.max(np.abs(w - w_ref)) < 1e-5
        m = w_ref > 1e-3
        assert m.any()
        assert np.max(np.abs(d[m] - d_ref[m]) / np.abs(d_ref[m])) < 1e-5
        assert np.all(d[w_ref <= 1e-8] == 0.0)


@pytest.mark.parametrize("per_index", [False, True])
def test_adam_step_bit_exact_vs_reference(G, ctx, per_index):
    """Both adam_step overloads (trainer.cpp:40-69) against the reference
    build, 5 steps: params / m / v bit for bit."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    r = np.random.default_rng(9)
    n = 1000
    p0 = r.normal(size=n)
    lrs = np.abs(r.normal(1e-2, 3e-3, n)) if per_index else None
    a = [p0.copy(), np.zeros(n), np.zeros(n)]
    b = [p0.copy(), np.zeros(n), np.zeros(n)]
    sa, sb = 0, O.C.c_int64(0)
    for _ in range(5):
        g = r.normal(size=n) * 1e-3
        sa = G.adam_step(ctx, a[0], g, a[1], a[2], sa, lrs if per_index else 5e-3)
        O.ref_lib().ref_adam_step(O._p(b[0]), O._p(g), O._p(b[1]), O._p(b[2]), O.C.byref(sb), n, 5e-3,
                                  O._p(lrs) if per_index else None)
    assert sa == sb.value == 5
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("tile", [8, 13, 32])
def test_tile_size_export_matches_reference(G, ctx, tile):
    """RasterConfig.tile_size != 16 (rasterizer.hpp:31): the device renders on
    16x16 tiles and exports the requested tile size's lists / ranges /
    contrib_count (k_export.cu). Against the reference build with the same
    tile size: tile lists and ranges bit-exact, contrib_count equal and the
    image within 1e-5 on every pixel whose decisions have a margin > 1e-4,
    the full GradientBundle unchanged vs tile 16."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    import math
    rng = O.make_rng(99)
    hc = O.synth_cloud(10000, 3, rng)
    hc.log_scales += math.log(500 / 10000) / 3
    hc = hc.as_float32_exact()
    cam = O.synth_camera(200, 152, O.synth_poses(0, 4, rng)[0])
    cfg = O.default_raster_config(tile_size=tile)
    with O.reference_backend():
        ref = O.render(hc, cam, cfg=cfg, keep_handle=True)
    cloud = to_dev(G, ctx, hc)
    gcfg = G.RasterConfig.default()
    gcfg.tile_size = tile
    out = G.render(ctx, cloud, dev_cam(G, cam), config=gcfg)
    info = out.info()
    assert (info.tiles_x, info.tiles_y) == (ref.tiles_x, ref.tiles_y)
    d = out.download()
    assert np.array_equal(d["splat_gaussian"], ref.splat_gaussian)
    assert np.array_equal(d["tile_lists"], ref.tile_lists)
    assert np.array_equal(d["tile_ranges"], ref.tile_ranges)
    margin = O.decision_margin(ref).reshape(-1)
    stable = margin > 1e-4
    assert np.mean(stable) > 0.99
    assert np.array_equal(d["contrib_count"][stable], ref.contrib_count[stable])
    err = np.max(np.abs(d["image"] - ref.image), axis=2).reshape(-1)
    assert err[stable].max() < 1e-5
    ref.free()
    # gradients do not depend on the tile size
    d_img = np.sin(np.arange(d["image"].size)).reshape(d["image"].shape) * 1e-2
    g_s, dp_s = G.render_backward(ctx, cloud, dev_cam(G, cam), out, d_img)
    out16 = G.render(ctx, cloud, dev_cam(G, cam))
    g_16, dp_16 = G.render_backward(ctx, cloud, dev_cam(G, cam), out16, d_img)
    assert np.array_equal(dp_s, dp_16)
    for k in g_16:
        assert np.array_equal(g_s[k], g_16[k]), k


def test_render_backward_device_image_equals_host(G, ctx):
    """gsb_render_backward_image: render_backward with the upstream gradient
    already on the device (a fixed d_image reused across calls, as
    tests/gradcheck.hpp:204-208 does) gives the host path's results bit for
    bit (both round the FP64 image to the same FP32 planes), and rejects a
    d_image of another size (rasterizer.cpp:341-343)."""
    import math
    rng = O.make_rng(77)
    hc = O.synth_cloud(3000, 3, rng)
    hc.log_scales += math.log(500 / 3000) / 3
    cam = O.synth_camera(96, 72, O.synth_poses(0, 3, rng)[0])
    cloud = to_dev(G, ctx, hc.as_float32_exact())
    dc = dev_cam(G, cam)
    d_img = np.random.default_rng(5).uniform(-1e-3, 1e-3, (72, 96, 3))
    dev_img = G.Image(ctx, d_img)
    for pose_only in (True, False):
        out = G.render(ctx, cloud, dc)
        g_h, dp_h = G.render_backward(ctx, cloud, dc, out, d_img, pose_only=pose_only)
        g_d, dp_d = G.render_backward(ctx, cloud, dc, out, dev_img, pose_only=pose_only)
        assert np.array_equal(dp_h, dp_d) and np.any(dp_h != 0.0)
        if not pose_only:
            for k in g_h:
                assert np.array_equal(g_h[k], g_d[k]), k
    small = G.Image(ctx, d_img[:-1])
    with pytest.raises(G.GsbError) as e:
        G.render_backward(ctx, cloud, dc, out, small, pose_only=True)
    assert e.value.code == G.ERR_DIMENSION_MISMATCH
