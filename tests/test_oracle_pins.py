"""Pins the CPU oracle to the reference's own known-answer tests, brute-force
re-implementations, invariants and finite-difference gates.

Each test cites the reference test it restates (relative to
/root/reference/proj). These run on CPU only (no GPU, no product library).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O


def test_rng_stream_is_xorshift64star():
    # core.hpp:58-70: first outputs of seed 1 computed by hand.
    r = O.make_rng(1)
    x = 1
    outs = []
    for _ in range(4):
        x ^= x >> 12
        x ^= (x << 25) & 0xFFFFFFFFFFFFFFFF
        x ^= x >> 27
        outs.append(((x * 0x2545F4914F6CDD1D) & 0xFFFFFFFFFFFFFFFF) >> 11)
    got = [O.lib().orc_rng_uniform(O.C.byref(r)) for _ in range(4)]
    assert got == [o * 2.0 ** -53 for o in outs]


def test_project_pinhole_kat():
    # test_rasterizer.cpp:16-31
    cam = O.make_camera(1.0, 1.0, 0.0, 0.0, 8, 8)
    mu2d, depth = np.zeros(2), np.zeros(1)
    O.lib().orc_project(O._p(np.array([2.0, 4.0, 2.0])), O.C.byref(cam), O._p(mu2d), O._p(depth))
    assert mu2d.tolist() == [1.0, 2.0] and depth[0] == 2.0
    cam.cx, cam.cy = 3.5, 2.5
    O.lib().orc_project(O._p(np.array([0.0, 0.0, 5.0])), O.C.byref(cam), O._p(mu2d), O._p(depth))
    assert mu2d.tolist() == [3.5, 2.5]


def _cov2d(sigma, mu_cam, cam, dil):
    out = np.zeros(4)
    O.lib().orc_covariance2d(O._p(np.ascontiguousarray(sigma, np.float64).reshape(9)),
                             O._p(np.asarray(mu_cam, np.float64)), O.C.byref(cam), dil, O._p(out))
    return out.reshape(2, 2)


def test_covariance2d_on_axis_and_depth_scaling():
    # test_rasterizer.cpp:57-74
    cam = O.make_camera(1.0, 1.0, 0.0, 0.0, 4, 4)
    cov = _cov2d(np.eye(3), [0, 0, 1], cam, 0.3)
    assert np.linalg.norm(cov - 1.3 * np.eye(2)) < 1e-14
    cam = O.make_camera(30.0, 30.0, 0.0, 0.0, 4, 4)
    near = _cov2d(0.01 * np.eye(3), [0, 0, 1], cam, 0.0)
    far = _cov2d(0.01 * np.eye(3), [0, 0, 2], cam, 0.0)
    assert np.linalg.norm(near - 4.0 * far) < 1e-12


def test_splat_alpha_closed_forms():
    # test_rasterizer.cpp:110-125
    L = O.lib()
    P = lambda *v: O._p(np.array(v, np.float64))
    eye = P(1, 0, 0, 1)
    assert L.orc_splat_alpha(P(3, 4), eye, 0.7, P(3, 4), 0.99, 3.0) == 0.7
    assert L.orc_splat_alpha(P(3, 4), eye, 0.0, P(3.5, 4), 0.99, 3.0) == 0.0
    sig = 1.7
    ic = P(1 / sig ** 2, 0, 0, 1 / sig ** 2)
    a = L.orc_splat_alpha(P(0, 0), ic, 0.5, P(sig, 0), 0.99, 3.0)
    assert a == pytest.approx(0.5 * math.exp(-0.5), rel=1e-12)
    assert L.orc_splat_alpha(P(0, 0), ic, 0.9, P(3.0 * sig + 1e-6, 0), 0.99, 3.0) == 0.0
    assert L.orc_splat_alpha(P(0, 0), ic, 1.0, P(0, 0), 0.99, 3.0) == 0.99


def test_empty_cloud_renders_background():
    # test_rasterizer.cpp:127-142
    cloud = O.HostCloud(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3, 1)), 0, 0)
    cam = O.make_camera(20, 20, 7.5, 7.5, 16, 16)
    rr = O.render(cloud, cam, (0.3, 0.6, 0.9))
    assert np.all(rr.image == np.array([0.3, 0.6, 0.9]))
    assert np.all(rr.accum_transmittance == 0.0)


def test_single_near_opaque_gaussian():
    # test_rasterizer.cpp:144-180
    rng = O.make_rng(53)
    cloud, cam, bg = O.make_gradcheck_scene(rng, 1, 32)
    cam.R[:] = np.eye(3).reshape(9).tolist()
    cam.t[:] = [0.0, 0.0, 0.0]
    cloud.means[0] = [0, 0, 2.0]
    cloud.log_scales[0] = math.log(0.8)
    cloud.opacity_logits[0] = math.log(0.999 / 0.001)
    rr = O.render(cloud, cam, bg)
    mu2d, depth = np.zeros(2), np.zeros(1)
    O.lib().orc_project(O._p(np.ascontiguousarray(cloud.means[0])), O.C.byref(cam), O._p(mu2d), O._p(depth))
    px, py = int(round(mu2d[0])), int(round(mu2d[1]))
    dirv = cloud.means[0] / np.linalg.norm(cloud.means[0])
    rgb = np.zeros(3)
    O.lib().orc_sh_eval(O._p(np.ascontiguousarray(cloud.sh[0].reshape(-1))), O._p(dirv), 3, O._p(rgb), None)
    op = 1 / (1 + math.exp(-cloud.opacity_logits[0]))
    a = O.lib().orc_splat_alpha(O._p(mu2d), O._p(np.ascontiguousarray(rr.splat_conic[0])), op,
                                O._p(np.array([px, py], np.float64)), 0.99, 3.0)
    want = a * rgb + (1 - a) * bg
    assert np.linalg.norm(rr.image[py, px] - want) < 1e-12
    assert rr.accum_transmittance[py * 32 + px] == pytest.approx(0.99, rel=1e-9)


def _brute_force_render(cloud, cam, bg, cfg):
    """test_rasterizer.cpp:190-238: untiled per-pixel compositor over depth-sorted splats."""
    refs = []
    R, t = O.camera_pose(cam)
    cc = -R.T @ t
    for i in range(cloud.n):
        mc = R @ cloud.means[i] + t
        if not mc[2] > cfg.z_near:
            continue
        mu2d, depth = np.zeros(2), np.zeros(1)
        O.lib().orc_project(O._p(np.ascontiguousarray(cloud.means[i])), O.C.byref(cam), O._p(mu2d), O._p(depth))
        s = np.exp(cloud.log_scales[i])
        sig = np.zeros(9)
        O.lib().orc_covariance3d(O._p(np.ascontiguousarray(cloud.rotations[i])), O._p(np.ascontiguousarray(s)),
                                 O._p(sig))
        cov = _cov2d(sig, mc, cam, cfg.dilation)
        mid, diff = 0.5 * (cov[0, 0] + cov[1, 1]), 0.5 * (cov[0, 0] - cov[1, 1])
        rad = cfg.cutoff_sigma * math.sqrt(mid + math.sqrt(diff * diff + cov[0, 1] * cov[1, 0]))
        if (mu2d[0] + rad < 0 or mu2d[0] - rad > cam.width - 1 or mu2d[1] + rad < 0
                or mu2d[1] - rad > cam.height - 1):
            continue
        conic = np.linalg.inv(cov)
        d = cloud.means[i] - cc
        d = d / np.linalg.norm(d)
        rgb = np.zeros(3)
        O.lib().orc_sh_eval(O._p(np.ascontiguousarray(cloud.sh[i].reshape(-1))), O._p(d), cloud.active_sh_degree,
                            O._p(rgb), None)
        refs.append((depth[0], mu2d.copy(), conic, rgb, 1 / (1 + math.exp(-cloud.opacity_logits[i]))))
    refs.sort(key=lambda r: r[0])  # stable
    img = np.zeros((cam.height, cam.width, 3))
    for y in range(cam.height):
        for x in range(cam.width):
            col, T = np.zeros(3), 1.0
            for _, mu, conic, rgb, op in refs:
                dd = np.array([x, y]) - mu
                g = dd @ conic @ dd
                if g > cfg.cutoff_sigma ** 2:
                    continue
                a = min(cfg.alpha_clamp, op * math.exp(-0.5 * g))
                if a == 0.0:
                    continue
                col += rgb * (a * T)
                T *= 1 - a
                if T < cfg.early_termination:
                    break
            img[y, x] = np.minimum(col + bg * T, 1.0)
    return img


def test_render_matches_brute_force_compositor():
    # test_rasterizer.cpp:182-241 (4 trials, 12 Gaussians, 48x48, < 1e-12)
    rng = O.make_rng(54)
    cfg = O.default_raster_config()
    for _ in range(4):
        cloud, cam, bg = O.make_gradcheck_scene(rng, 12, 48)
        rr = O.render(cloud, cam, bg, cfg)
        ref = _brute_force_render(cloud, cam, bg, cfg)
        assert np.max(np.abs(ref - rr.image)) < 1e-12


def test_repeat_render_bit_identical_and_complement():
    # test_rasterizer.cpp:243-265
    rng = O.make_rng(55)
    cloud, cam, bg = O.make_gradcheck_scene(rng, 60, 64)
    a = O.render(cloud, cam, bg)
    b = O.render(cloud, cam, bg)
    assert a.image.tobytes() == b.image.tobytes()
    assert a.accum_transmittance.tobytes() == b.accum_transmittance.tobytes()
    rng = O.make_rng(56)
    cloud, cam, bg = O.make_gradcheck_scene(rng, 30, 32)
    o = O.render(cloud, cam, bg)
    assert np.all(o.accum_transmittance >= 0) and np.all(o.accum_transmittance <= 1)
    assert np.all(o.accum_transmittance + o.final_transmittance == 1.0)


def test_early_termination_bound():
    # test_rasterizer.cpp:267-281
    rng = O.make_rng(57)
    cloud, cam, bg = O.make_gradcheck_scene(rng, 40, 32)
    cloud.opacity_logits[:] = math.log(0.9 / 0.1)
    a = O.render(cloud, cam, bg, O.default_raster_config())
    b = O.render(cloud, cam, bg, O.default_raster_config(early_termination=0.0))
    assert np.max(np.abs(a.image - b.image)) <= 1e-4


def test_zero_upstream_and_stale_state():
    # test_rasterizer.cpp:283-306
    rng = O.make_rng(58)
    cloud, cam, bg = O.make_gradcheck_scene(rng, 8, 32)
    rr = O.render(cloud, cam, bg, keep_handle=True)
    g = O.render_backward(cloud, cam, rr, np.zeros((32, 32, 3)))
    assert np.all(g.d_means == 0) and np.all(g.d_rotations == 0) and np.all(g.d_sh == 0)
    assert np.all(g.d_pose == 0)
    rr.free()
    rng = O.make_rng(59)
    cloud, cam, bg = O.make_gradcheck_scene(rng, 8, 32)
    rr = O.render(cloud, cam, bg, keep_handle=True)
    moved = cloud.copy()
    moved.means[0] += [0.5, 0, 0]
    with pytest.raises(O.OracleError):
        O.render_backward(moved, cam, rr, np.zeros((32, 32, 3)))
    R, t = O.se3_exp(np.full(6, 0.1))
    R0, t0 = O.camera_pose(cam)
    other = O.make_camera(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, R @ R0, R @ t0 + t)
    with pytest.raises(O.OracleError):
        O.render_backward(cloud, other, rr, np.zeros((32, 32, 3)))
    rr.free()


def test_culled_gaussians_contribute_zero():
    # test_rasterizer.cpp:308-343
    rng = O.make_rng(60)
    cloud, cam, bg = O.make_gradcheck_scene(rng, 6, 32)
    base = O.render(cloud, cam, bg)
    R, t = O.camera_pose(cam)
    inv = lambda p: R.T @ (np.asarray(p) - t)
    ext = cloud.copy()
    for mean in (inv([0, 0, -2.0]), inv([50.0, 0, 2.0])):
        ext.means = np.vstack([ext.means, mean])
        ext.rotations = np.vstack([ext.rotations, [1, 0, 0, 0]])
        ext.log_scales = np.vstack([ext.log_scales, np.full(3, math.log(0.1))])
        ext.opacity_logits = np.append(ext.opacity_logits, math.log(0.9 / 0.1))
        ext.sh = np.concatenate([ext.sh, np.full((1, 3, 16), 0.3)])
    out = O.render(ext, cam, bg, keep_handle=True)
    assert np.max(np.abs(out.image - base.image)) == 0.0
    d = np.array([O.lib().orc_rng_uniform_range(O.C.byref(rng), -1, 1) for _ in range(32 * 32 * 3)]).reshape(32, 32, 3)
    g = O.render_backward(ext, cam, out, d)
    assert np.all(g.d_means[6:] == 0) and np.all(g.d_rotations[6:] == 0)
    assert np.all(g.d_log_scales[6:] == 0) and np.all(g.d_opacity_logits[6:] == 0)
    out.free()


def test_fd_gradcheck_three_conditioned_scenes():
    # test_rasterizer.cpp:345-355 (596 derivatives per scene, gate 1e-5)
    rng = O.make_rng(61)
    for _ in range(3):
        cloud, cam, bg = O.make_conditioned_scene(rng, 10, 32)
        err, checked, worst = O.gradcheck(cloud, cam, bg, rng)
        assert checked == 10 * (3 + 4 + 3 + 1 + 48) + 6
        assert err < 1e-5, worst


def test_gauge_identity():
    # test_rasterizer.cpp:377-390
    rng = O.make_rng(63)
    cloud, cam, bg = O.make_gradcheck_scene(rng, 15, 32)
    rr = O.render(cloud, cam, bg, keep_handle=True)
    d = np.array([O.lib().orc_rng_uniform_range(O.C.byref(rng), -1, 1) for _ in range(32 * 32 * 3)]).reshape(32, 32, 3)
    g = O.render_backward(cloud, cam, rr, d)
    R, _ = O.camera_pose(cam)
    expected = R @ g.d_means.sum(axis=0)
    assert np.linalg.norm(g.d_pose[:3] - expected) < 1e-10 * max(1.0, np.linalg.norm(expected))
    rr.free()


def test_sh_and_covariance_kats():
    # test_scene.cpp:19-57, 88-99
    cov = np.zeros(9)
    O.lib().orc_covariance3d(O._p(np.array([1.0, 0, 0, 0])), O._p(np.array([1.0, 2, 3])), O._p(cov))
    assert np.linalg.norm(cov.reshape(3, 3) - np.diag([1.0, 4, 9])) < 1e-14
    rgb = np.zeros(3)
    O.lib().orc_sh_eval(O._p(np.ones(3)), O._p(np.array([0.0, 0, 1])), 0, O._p(rgb), None)
    assert rgb[0] == pytest.approx(0.7820948, rel=1e-6) and rgb[1] == rgb[0]
    O.lib().orc_sh_eval(O._p(np.zeros(48)), O._p(np.array([1.0, 0, 0])), 3, O._p(rgb), None)
    assert np.all(rgb == 0.5)
    rng = O.make_rng(32)
    for _ in range(20):
        q = np.array([O.lib().orc_rng_normal(O.C.byref(rng)) for _ in range(4)])
        q /= np.linalg.norm(q)
        s = np.array([O.lib().orc_rng_uniform_range(O.C.byref(rng), 0.1, 1.0) for _ in range(3)])
        O.lib().orc_covariance3d(O._p(q), O._p(s), O._p(cov))
        ev = np.sort(np.linalg.eigvalsh(cov.reshape(3, 3)))
        assert np.linalg.norm(ev - np.sort(s ** 2)) < 1e-10


def test_quat_jacobian_fd():
    # test_scene.cpp:68-86
    rng = O.make_rng(34)
    for _ in range(10):
        q = np.array([O.lib().orc_rng_normal(O.C.byref(rng)) for _ in range(4)])
        q = q / np.linalg.norm(q) * O.lib().orc_rng_uniform_range(O.C.byref(rng), 0.8, 1.2)
        jac = np.zeros(36)
        O.lib().orc_quat_rotation_jacobian(O._p(q), O._p(jac))
        jac = jac.reshape(4, 9)
        for k in range(4):
            h = 1e-6
            qp, qm = q.copy(), q.copy()
            qp[k] += h
            qm[k] -= h
            Rp, Rm = np.zeros(9), np.zeros(9)
            O.lib().orc_quat_to_rotation(O._p(qp), O._p(Rp))
            O.lib().orc_quat_to_rotation(O._p(qm), O._p(Rm))
            fd = (Rp - Rm) / (2 * h)
            assert np.all(np.abs(jac[k] - fd) / np.maximum(np.abs(fd), 1e-3) < 1e-5)


def test_lie_kats_and_orthonormalize_drift():
    # test_lie.cpp:26-39, 231-243
    R, t = O.se3_exp(np.zeros(6))
    assert np.all(R == np.eye(3)) and np.all(t == 0)
    R, t = O.se3_exp(np.array([0, 0, 0, 0, 0, math.pi / 2]))
    assert np.linalg.norm(R @ np.array([1, 0, 0]) - np.array([0, 1, 0])) < 1e-14
    rng = O.make_rng(22)
    Rc = np.eye(3)
    for _ in range(2000):
        tau = np.array([O.lib().orc_rng_uniform_range(O.C.byref(rng), -0.05, 0.05) for _ in range(6)])
        Re, _ = O.se3_exp(tau)
        Rc = O.orthonormalize(Re @ Rc)
    assert np.linalg.norm(Rc.T @ Rc - np.eye(3)) < 1e-9
    assert abs(np.linalg.det(Rc) - 1) < 1e-9
    # polar factor of a perturbed rotation equals numpy's SVD polar factor
    A = Rc + 1e-3 * np.arange(9).reshape(3, 3) / 9
    U, _, Vt = np.linalg.svd(A)
    assert np.linalg.norm(O.orthonormalize(A) - U @ Vt) < 1e-13


def test_loss_kats():
    # test_losses.cpp:25-84
    rng = np.random.default_rng(71)
    img = rng.uniform(0, 1, (18, 24, 3))
    loss, grad = O.rgb_loss(img, img, 0.2)
    assert loss == 0.0 and np.all(grad == 0)
    a, b = np.full((16, 16, 3), 0.6), np.full((16, 16, 3), 0.5)
    assert O.rgb_loss(a, b, 0.0, want_grad=False) == pytest.approx(0.1, rel=1e-12)
    a, b = rng.uniform(0, 1, (20, 20, 3)), rng.uniform(0, 1, (20, 20, 3))
    l1 = O.rgb_loss(a, b, 0.0, False)
    ds = O.rgb_loss(a, b, 1.0, False)
    assert O.rgb_loss(a, b, 0.2, False) == pytest.approx(0.8 * l1 + 0.2 * ds, rel=1e-12)


def _brute_ssim(a, b):
    """tests/test_util.hpp:38-76."""
    w1 = np.exp(-((np.arange(11) - 5) ** 2) / (2 * 1.5 ** 2))
    w1 /= w1.sum()
    W = np.outer(w1, w1)
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    tot, cnt = 0.0, 0
    H, Wd = a.shape[:2]
    for c in range(3):
        for y in range(5, H - 5):
            for x in range(5, Wd - 5):
                pa, pb = a[y - 5:y + 6, x - 5:x + 6, c], b[y - 5:y + 6, x - 5:x + 6, c]
                ma, mb = (W * pa).sum(), (W * pb).sum()
                sa = (W * pa * pa).sum() - ma * ma
                sb = (W * pb * pb).sum() - mb * mb
                sab = (W * pa * pb).sum() - ma * mb
                tot += ((2 * ma * mb + c1) * (2 * sab + c2)) / ((ma * ma + mb * mb + c1) * (sa + sb + c2))
                cnt += 1
    return tot / cnt


def test_ssim_brute_force_and_fd():
    # test_losses.cpp:42-55, 86-107
    rng = np.random.default_rng(72)
    for _ in range(2):
        a, b = rng.uniform(0, 1, (17, 20, 3)), rng.uniform(0, 1, (17, 20, 3))
        assert abs(O.ssim(a, b) - _brute_ssim(a, b)) < 1e-6
    r = rng.uniform(0.2, 0.8, (16, 16, 3))
    tgt = np.clip(r + rng.uniform(0.02, 0.15, r.shape) * np.where(rng.uniform(size=r.shape) < 0.5, -1, 1), 0, 1)
    _, grad = O.rgb_loss(r, tgt, 0.2)
    flat = r.reshape(-1)
    for idx in rng.integers(0, flat.size, 30):
        h = 1e-6
        rp, rm = flat.copy(), flat.copy()
        rp[idx] += h
        rm[idx] -= h
        fd = (O.rgb_loss(rp.reshape(r.shape), tgt, 0.2, False) - O.rgb_loss(rm.reshape(r.shape), tgt, 0.2, False)) / (2 * h)
        assert abs(grad.reshape(-1)[idx] - fd) / max(abs(fd), 1e-4) < 1e-5


def test_schedule_and_pose_step_identities():
    # test_trainer.cpp:17-67
    assert O.schedule("cosine", 1e-2, 1e-4, 0, 100) == pytest.approx(1e-2)
    assert O.schedule("cosine", 1e-2, 1e-4, 100, 100) == pytest.approx(1e-4)
    assert O.schedule("cosine", 1e-2, 1e-4, 50, 100) == pytest.approx((1e-2 + 1e-4) / 2, rel=1e-12)
    assert O.schedule("exp", 1.6e-2, 1.6e-4, 50, 100) == pytest.approx(1.6e-3, rel=1e-12)
    R, t = O.se3_exp(np.array([0.3, -0.2, 0.5, 0.4, -0.7, 0.2]))
    p = O.pose_join(R, t)
    same, _ = O.pose_step(p, np.zeros(6), 1e-2, O.PoseAdam())
    assert same.tobytes() == p.tobytes()
    zero_lr, _ = O.pose_step(p, np.array([0.3, -0.5, 0.1, 0.9, -0.2, 0.4]), 0.0, O.PoseAdam())
    assert zero_lr.tobytes() == p.tobytes()
    g = np.array([0.3, -0.5, 0.1, 0.9, -0.2, 0.4])
    fwd, _ = O.pose_step(p, g, 1e-3, O.PoseAdam())
    back, _ = O.pose_step(fwd, -g, 1e-3, O.PoseAdam())
    assert np.linalg.norm(back - p) < 1e-6


def test_pose_descent_toy_translation():
    # test_trainer.cpp:69-107: monotone descent to < 0.005 in 40 steps
    cloud = O.HostCloud(np.array([[0, 0, 2.0]]), np.array([[1.0, 0, 0, 0]]), np.full((1, 3), math.log(0.5)),
                        np.array([math.log(0.8 / 0.2)]), np.zeros((1, 3, 1)), 0, 0)
    # The reference writes sh_at(0)[0], [4], [8] after resize(1, 0): the SH block holds 3
    # entries, so [4] and [8] land outside the vector (undefined behaviour in the reference test)
    # and only channel 0's DC coefficient is actually set. Mirror what the cloud really holds.
    cloud.sh[0, :, 0] = [(0.8 - 0.5) / 0.28209479177387814, 0.0, 0.0]
    cam = O.make_camera(24.0, 24.0, 15.5, 15.5, 32, 32)
    target = O.render(cloud, cam).image
    res = O.estimate_pose(cloud, target, 24.0, 24.0, 15.5, 15.5, O.pose_join(np.eye(3), [0.08, -0.05, 0.0]),
                          budget=40, cam_lr_start=5e-4, cam_lr_end=5e-4, beta=0.0, pose_converged_eps=0.0)
    losses = res["trace_loss"]
    assert np.all(np.diff(losses) <= 1e-12)
    assert losses[-1] < 0.005 or res["final_loss"] < 0.005


def test_estimate_pose_exact_init_converges_immediately():
    # test_trainer.cpp:327-343
    rng = O.make_rng(45)
    cloud = O.synth_cloud(30, 1, rng)
    poses = O.synth_poses(0, 2, rng)
    cam = O.synth_camera(32, 32, poses[0])
    img = O.render(cloud, cam).image
    res = O.estimate_pose(cloud, img, cam.fx, cam.fy, cam.cx, cam.cy, poses[0], budget=1000)
    assert res["converged"] and res["steps"] <= 2
    r, d = O.abs_pose_error(res["pose"], poses[0])
    assert r < 1e-6 and d < 1e-6


@pytest.mark.slow
def test_acceptance_pose_estimation_criterion():
    # tests/acceptance.cpp:74-100: >= 18/20 trials rot < 5 deg, pos < 0.05
    rng = O.make_rng(99)
    cloud = O.synth_cloud(500, 1, rng)
    poses = O.synth_poses(0, 20, rng)
    imgs = [O.render(cloud, O.synth_camera(64, 64, p)).image for p in poses]
    noise = O.make_rng(1002)
    hits = 0
    for t in range(20):
        noisy = O.perturb_pose(poses[t], 15.0, 0.15, noise)
        cam = O.synth_camera(64, 64, poses[t])
        res = O.estimate_pose(cloud, imgs[t], cam.fx, cam.fy, cam.cx, cam.cy, noisy, budget=1000)
        r, d = O.abs_pose_error(res["pose"], poses[t])
        hits += (r < 5.0 and d < 0.05)
    assert hits >= 18
