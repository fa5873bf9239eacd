"""The oracle pinned to the reference ITSELF (CPU, no GPU).

oracle/_ref is /root/reference/proj/src/*.cpp compiled in place against the
clean-room Eigen / doctest / libpng shim in oracle/shim (oracle/build_ref.py).
These tests
  1. run the reference's own doctest suites against that build (the shim is
     only trusted because they pass: test_lie, test_scene, test_rasterizer,
     test_losses, test_eval, test_trainer, test_io minus its PNG cases);
  2. show that the clean-room restatement (oracle/gsopt_oracle.c) equals the
     reference build bit for bit: every RenderOutput field, every
     GradientBundle group, rgb_loss and its gradient, pose_step, the scene /
     pose generators, the 100-iteration C1 pose_descent log, and
     joint_optimize (with and without densification).
The GPU parity tests compare the device path with the restatement, so these
pins carry over to the device path.
"""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import build_ref
from oracle import oracle as O

REF_DIR = os.path.join(os.path.dirname(O.__file__), "_ref")


@pytest.fixture(scope="module", autouse=True)
def _ref_build():
    build_ref.build()
    if not O.ref_available():
        pytest.skip("oracle/_ref not built and /root/reference absent")


def _both(fn):
    a = fn()
    with O.reference_backend():
        b = fn()
    return a, b


# ------------------------------------------------- the reference's own suites
PNG_CASES = "PNG round trip*,scene save/load*,load_scene error*,scenes without poses*"


@pytest.mark.parametrize("suite,args", [
    ("test_lie", []), ("test_scene", []), ("test_rasterizer", []), ("test_losses", []), ("test_eval", []),
    ("test_config", []), ("test_io", ["-tce=" + PNG_CASES]),
    pytest.param("test_trainer", ["-tce=pose_step descends a pure-translation*"], marks=pytest.mark.slow)])
def test_reference_suite_passes_under_shim(suite, args):
    """proj/tests/<suite>.cpp, unmodified, linked against the shim build.
    test_io's four PNG cases need libpng (absent; stubbed to raise
    corrupt_file), so they are excluded by name. One test_trainer case is
    excluded because the reference test itself writes out of bounds:
    test_trainer.cpp:72-77 resizes the cloud to SH degree 0 (3 coefficients)
    and then writes sh_at(0)[4] and [8] (AddressSanitizer: heap-buffer-overflow
    at test_trainer.cpp:77), which segfaults intermittently. Every other case
    of that suite is clean under ASan+UBSan with this shim."""
    exe = os.path.join(REF_DIR, suite)
    # The reference's Pool (core.cpp:39-80) lets a worker still draining one
    # job read job_n_/job_chunk_/cursor_ while run() resets them for the next
    # (outside its mutex), which can leave pending_ short and hang run(). On
    # an 8-core container it hung in about half of the unpinned test_trainer
    # runs; pinned to one core it completed 8 of 8 (same ~35 s). The suites
    # therefore run on one core of this process's affinity set, with retries.
    cpu = min(os.sched_getaffinity(0))
    for attempt in range(4):
        try:
            r = subprocess.run([exe] + args, capture_output=True, text=True, timeout=180,
                               preexec_fn=lambda: os.sched_setaffinity(0, {cpu}))
            break
        except subprocess.TimeoutExpired:
            if attempt == 3:
                raise
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "Status: SUCCESS" in r.stdout


# --------------------------------------- restatement == reference, bit for bit
RENDER_FIELDS = ["image", "final_transmittance", "accum_transmittance", "contrib_count", "overflow_mask",
                 "splat_gaussian", "splat_mu2d", "splat_depth", "splat_conic", "splat_color", "splat_opacity",
                 "splat_radius", "splat_clamped", "tile_lists", "tile_ranges"]
GRAD_FIELDS = ["d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh", "d_mu2d", "d_pose"]


def _assert_render_and_backward_equal(hc, cam, bg, d_image=None, cfg=None):
    ra, rb = _both(lambda: O.render(hc, cam, bg, cfg=cfg, keep_handle=True))
    try:
        for f in RENDER_FIELDS:
            x, y = getattr(ra, f), getattr(rb, f)
            assert x.shape == y.shape and np.array_equal(x, y), f
        assert (ra.tiles_x, ra.tiles_y) == (rb.tiles_x, rb.tiles_y)
        if d_image is None:
            d_image = np.random.default_rng(7).uniform(-1, 1, ra.image.shape)
        ga = O.render_backward(hc, cam, ra, d_image)
        gb = O.render_backward(hc, cam, rb, d_image)
        for f in GRAD_FIELDS:
            assert np.array_equal(getattr(ga, f), getattr(gb, f)), f
        return ra.image, ga
    finally:
        ra.free()
        rb.free()


@pytest.mark.parametrize("seed,n,size,conditioned", [(54, 12, 48, True), (61, 12, 48, True), (11, 10, 32, False),
                                                     (70, 200, 96, False)])
def test_gradcheck_scenes_render_and_backward_bit_exact(seed, n, size, conditioned):
    """tests/gradcheck.hpp scenes (the reference's own draw, itself bit-exact):
    splats, tile lists, ranges, contrib, every pixel and every gradient."""
    def draw():
        rng = O.make_rng(seed)
        return O.make_conditioned_scene(rng, n, size) if conditioned else O.make_gradcheck_scene(rng, n, size)
    (hc, cam, bg), (hc2, cam2, bg2) = _both(draw)
    for f in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
        assert np.array_equal(getattr(hc, f), getattr(hc2, f)), f
    assert np.array_equal(np.array(cam.R[:]), np.array(cam2.R[:])) and np.array_equal(bg, bg2)
    _assert_render_and_backward_equal(hc, cam, bg)
    _assert_render_and_backward_equal(hc.as_float32_exact(), cam, bg)


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_synth_scene_generators_bit_exact(kind):
    """synth.cpp:33-101 (cloud + trajectory, GCC argument order) and the
    rendered frames: the restated generator equals the reference's."""
    n, cams, w, h, deg, seed = 300, 5, 64, 48, 1 + kind, 40 + kind
    rc, rposes, rimgs = O.ref_synth_scene(n, cams, w, h, kind, deg, seed, with_images=True)
    rng = O.make_rng(seed)
    hc = O.synth_cloud(n, deg, rng)
    poses = O.synth_poses(kind, cams, rng)
    for f in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
        assert np.array_equal(getattr(hc, f), getattr(rc, f)), f
    assert np.array_equal(poses, rposes)
    for k in range(cams):
        img = O.render(hc, O.synth_camera(w, h, poses[k])).image
        assert np.array_equal(img, rimgs[k])


def test_synth_scene_sh_quirk_active_below_capacity():
    """Appendix A.8: active_sh_degree < sh_degree (forward indexes channel c
    at c*(d_active+1)^2, backward at c*B_capacity): restatement == reference."""
    rng = O.make_rng(5)
    hc = O.synth_cloud(150, 3, rng)
    hc.active_sh_degree = 1
    cam = O.synth_camera(64, 64, O.synth_poses(0, 1, rng)[0])
    _assert_render_and_backward_equal(hc, cam, np.array([0.1, 0.2, 0.3]))


def test_raster_config_variants_bit_exact():
    """Non-default RasterConfig fields (tile 8 / 32, cutoff, clamp,
    dilation, early termination): the reference's own behaviour."""
    rng = O.make_rng(21)
    hc = O.synth_cloud(400, 2, rng)
    hc.log_scales += math.log(500 / 400) / 3
    cam = O.synth_camera(72, 56, O.synth_poses(1, 1, rng)[0])
    for kw in (dict(tile_size=8), dict(tile_size=32), dict(cutoff_sigma=2.5, alpha_clamp=0.95),
               dict(dilation=0.0, early_termination=1e-2)):
        _assert_render_and_backward_equal(hc, cam, np.zeros(3), cfg=O.default_raster_config(**kw))


def test_perturbations_and_pose_step_bit_exact():
    rng = np.random.default_rng(3)
    for seed in range(5):
        p = O.synth_poses(2, 1, O.make_rng(seed))[0]
        (a, b) = _both(lambda: O.perturb_pose(p, 15.0, 0.15, O.make_rng(1002 + seed)))
        assert np.array_equal(a, b)
        (a, b) = _both(lambda: O.perturb_pose_tangent(p, 0.05, O.make_rng(55 + seed)))
        assert np.array_equal(a, b)
        adam_a, adam_b = O.PoseAdam(), O.PoseAdam()
        pa = pb = p
        for it in range(25):
            dp = rng.normal(size=6) * (10.0 ** rng.uniform(-6, 1))
            lr = O.schedule("cosine", 1e-2, 1e-4, it, 25)
            pa, ap_a = O.pose_step(pa, dp, lr, adam_a)
            with O.reference_backend():
                assert O.schedule("cosine", 1e-2, 1e-4, it, 25) == lr
                pb, ap_b = O.pose_step(pb, dp, lr, adam_b)
            assert np.array_equal(pa, pb) and np.array_equal(ap_a, ap_b)
        # zero gradient: the reference returns the input pose bit for bit
        with O.reference_backend():
            same, _ = O.pose_step(p, np.zeros(6), 1e-2, O.PoseAdam())
        assert np.array_equal(same, p)


def test_rgb_loss_bit_exact():
    rng = np.random.default_rng(9)
    for h, w in ((32, 32), (40, 57), (11, 11)):
        a = rng.uniform(0, 1, (h, w, 3))
        b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1)
        b[0, 0] = a[0, 0]  # an exact-zero L1 residual
        for beta in (0.0, 0.2, 1.0):
            (la, da), (lb, db) = _both(lambda: O.rgb_loss(a, b, beta))
            assert la == lb and np.array_equal(da, db)
        (la, da), (lb, db) = _both(lambda: O.rgb_loss(a, a, 0.2))
        assert la == lb == 0.0 and not da.any() and not db.any()


def _c1():
    """C1: 10k Gaussians SH-3 (density-matched log-scales),
    256x256, orbit camera 0 of seed 99, perturbed 15 deg / 0.15 from Rng(1002)."""
    rng = O.make_rng(99)
    hc = O.synth_cloud(10000, 3, rng)
    hc.log_scales += math.log(500 / 10000) / 3
    poses = O.synth_poses(0, 4, rng)
    hc = hc.as_float32_exact()
    cam = O.synth_camera(256, 256, poses[0])
    target = O.render(hc, cam).image
    noisy = O.perturb_pose(poses[0], 15.0, 0.15, O.make_rng(1002))
    return hc, cam, target, noisy


def test_c1_pose_descent_log_bit_exact():
    """The 100-iteration C1 pose_descent log: the restatement's per-iteration
    pose, loss and d_pose equal the reference's bit for bit, and the
    reference's own estimate_pose (pipelines.cpp:218-222) returns the same
    best pose and loss as the traced loop."""
    hc, cam, target, noisy = _c1()
    kw = dict(budget=100, pose_converged_eps=0.0)
    a, b = _both(lambda: O.estimate_pose(hc, target, cam.fx, cam.fy, cam.cx, cam.cy, noisy, **kw))
    assert a["steps"] == b["steps"] == 100
    for k in ("trace_pose", "trace_loss", "trace_dpose", "pose"):
        assert np.array_equal(a[k], b[k]), k
    assert a["final_loss"] == b["final_loss"]
    e = O.ref_estimate_pose(hc, target, cam.fx, cam.fy, cam.cx, cam.cy, noisy, **kw)
    assert e["steps"] == 100 and np.array_equal(e["pose"], b["pose"]) and e["final_loss"] == b["final_loss"]
    assert b["trace_loss"][-1] < b["trace_loss"][0]


@pytest.mark.parametrize("densify", [False, True])
def test_joint_optimize_bit_exact(densify):
    """pipelines.cpp:96-216 (one view per Adam step): the restatement's loss
    trace, final cloud and poses equal the reference's joint_optimize; with
    densification (trainer.cpp:134-239) every few steps when enabled."""
    rng = O.make_rng(31)
    hc = O.synth_cloud(400, 1, rng)
    views = O.synth_poses(0, 4, rng)
    imgs = [O.render(hc, O.synth_camera(48, 40, p)).image for p in views]
    init = hc.copy()
    init.log_scales += 0.2
    noisy = np.stack([O.perturb_pose_tangent(p, 0.03, O.make_rng(60 + i)) for i, p in enumerate(views)])
    kw = dict(densify_interval=3, densify_start=2, densify_stop=9, grad_threshold=1e-5, n_target=420) \
        if densify else dict(densify_interval=0)
    cfg = O.joint_config(12, sh_degree=1, sh_degree_interval=5, **kw)
    intr = (0.75 * 48, 0.75 * 48, 23.5, 19.5)
    a, b = _both(lambda: O.joint_optimize(init, imgs, intr, 48, 40, noisy, cfg, 1, O.make_rng(77)))
    assert a[0] == b[0] == 0
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
    assert np.array_equal(a[2], b[2])
    ca, cb = a[1], b[1]
    assert ca.n == cb.n
    if densify:
        assert ca.n != init.n
    for f in ("means", "rotations", "log_scales", "opacity_logits", "sh"):
        assert np.array_equal(getattr(ca, f), getattr(cb, f)), f


def test_fd_gradcheck_identical():
    """The reference's FD gate (gradcheck.hpp:201-254) run by the reference
    and by the restatement reports the same worst error and entry."""
    rng = O.make_rng(56)
    hc, cam, bg = O.make_conditioned_scene(rng, 6, 32)
    a, b = _both(lambda: O.gradcheck(hc, cam, bg, O.make_rng(3)))
    assert a == b and a[0] < 1e-5 and a[1] == 6 * (11 + 48) + 6
