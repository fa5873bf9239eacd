"""CPU tests of the data-parallel joint loop's host logic (no GPU).

* the product's training-view schedule (gsb_joint_schedule, host code)
  equals the reference's epoch shuffles (pipelines.cpp:122-129, restated in
  the oracle), and the product's perturb_pose_tangent equals eval.cpp:148-152;
* world_size-2 gloo run of the DP step semantics the device loop implements
  (SURVEY §8e): each rank renders its slot's view, the per-Gaussian gradients
  are all-reduced (sum, then mean), regularisers are added once, Adam runs on
  every replica, and every slot's pose step is applied in slot order from
  all-gathered d_pose. Both ranks must end bit-identical, and equal to the
  oracle's single-process joint_optimize with slots=2.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def _gsb():
    from paper_2410_08743_b200 import build, gsb
    build.build()
    return gsb


@pytest.mark.parametrize("seed,n_views,count", [(11, 4, 37), (0, 20, 100), (42, 7, 70), (5, 2, 9)])
def test_joint_schedule_matches_reference_shuffle(seed, n_views, count):
    G = _gsb()
    assert np.array_equal(G.joint_schedule(seed, n_views, count), O.joint_schedule(O.make_rng(seed), n_views, count))


def test_perturb_pose_tangent_matches_reference():
    G = _gsb()
    poses = O.synth_poses(1, 5, O.make_rng(3))
    st = G.PoseRng(55)
    orng = O.make_rng(55)
    for p in poses:
        a = G.perturb_pose_tangent(p, 0.05, st)
        b = O.perturb_pose_tangent(p, 0.05, orng)
        assert np.max(np.abs(a - b)) < 1e-15


def _scene():
    rng = O.make_rng(4)
    hc = O.synth_cloud(200, 1, rng).as_float32_exact()
    poses = O.synth_poses(1, 4, rng)
    cams = [O.synth_camera(40, 32, p) for p in poses]
    imgs = [O.render(hc, c).image for c in cams]
    noise = O.make_rng(55)
    init = np.stack([O.perturb_pose_tangent(p, 0.05, noise) for p in poses])
    jit = hc.copy()
    jit.means = jit.means + 0.02 * np.sin(np.arange(jit.means.size)).reshape(jit.means.shape)
    return jit, imgs, [cams[0].fx, cams[0].fy, cams[0].cx, cams[0].cy], init


STEPS, SEED = 3, 11


def _dp_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hc, imgs, intr, init, = _scene()
        cfg = O.joint_config(STEPS, sh_degree=1, sh_degree_interval=0)
        seq = O.joint_schedule(O.make_rng(SEED), len(imgs), STEPS * world)
        adam = O.CloudAdam(hc)
        poses = init.copy()
        pads = [O.PoseAdam() for _ in imgs]
        for t in range(STEPS):
            cloud = adam.cloud()
            v = int(seq[t * world + rank])  # this rank's slot
            cam = O.make_camera(*intr, 40, 32, *O.pose_split(poses[v]))
            rr = O.render(cloud, cam, keep_handle=True)
            _, d_img = O.rgb_loss(rr.image, imgs[v], cfg.beta)
            g = O.render_backward(cloud, cam, rr, d_img)
            rr.free()
            names = ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh")
            flat = torch.from_numpy(np.concatenate([getattr(g, k).reshape(-1) for k in names]))
            dist.all_reduce(flat)  # sum over ranks
            flat = flat.numpy() * (1.0 / world)
            grads, off = {}, 0
            for k in names:
                a = getattr(g, k)
                grads[k] = flat[off:off + a.size].reshape(a.shape).copy()
                off += a.size
            _, d_an = O.anisotropy_loss(cloud.log_scales, cfg.aniso_ratio)
            grads["d_log_scales"] = grads["d_log_scales"] + d_an
            o = 1.0 / (1.0 + np.exp(-cloud.opacity_logits))
            grads["d_opacity_logits"] = grads["d_opacity_logits"] + cfg.opacity_l1_weight * (1.0 / cloud.n) * o * (1.0 - o)
            lrs = [O.schedule("exponential", cfg.pos_lr_start, cfg.pos_lr_end, t, STEPS), cfg.rot_lr, cfg.scale_lr,
                   cfg.opacity_lr, cfg.sh_dc_lr, cfg.sh_rest_lr]
            adam.step(grads, lrs)
            dp = torch.zeros(world, 6, dtype=torch.float64)
            dp[rank] = torch.from_numpy(g.d_pose)
            dist.all_reduce(dp)  # all-gather of the slots' d_pose
            lr = O.schedule("cosine", cfg.cam_lr_start, cfg.cam_lr_end, t, STEPS)
            for s in range(world):
                vs = int(seq[t * world + s])
                poses[vs], _ = O.pose_step(poses[vs], dp[s].numpy(), lr, pads[vs])
        c = adam.cloud()
        q.put((rank, np.concatenate([c.means.ravel(), c.rotations.ravel(), c.log_scales.ravel(),
                                     c.opacity_logits.ravel(), c.sh.ravel()]), poses))
    finally:
        dist.destroy_process_group()


def test_data_parallel_step_semantics_gloo_world2():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (a, P)) for r, a, P in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (a0, P0), (a1, P1) = out[0], out[1]
    assert np.array_equal(a0, a1) and np.array_equal(P0, P1)  # replicas in lock step
    hc, imgs, intr, init = _scene()
    cfg = O.joint_config(STEPS, sh_degree=1, sh_degree_interval=0)
    st, cl, P, tt, tl = O.joint_optimize(hc, imgs, intr, 40, 32, init, cfg, 2, O.make_rng(SEED))
    assert st == 0
    ref = np.concatenate([cl.means.ravel(), cl.rotations.ravel(), cl.log_scales.ravel(), cl.opacity_logits.ravel(),
                          cl.sh.ravel()])
    assert np.max(np.abs(a0 - ref)) < 1e-9
    assert np.max(np.abs(P0 - P)) < 1e-12
