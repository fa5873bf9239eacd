"""Multi-rank readiness on CPU (world_size-2 gloo).

* C3 (independent views): the bench's rank -> view partition is disjoint and
  covers C3's 64 views at 8 ranks; with 2 gloo ranks each running its own
  views' pose_descent (pipelines.cpp:58-92, the reference's loop restated in
  the oracle) and all-gathering the poses, every rank ends with exactly the
  poses a single process computes for all views — no data-path collective,
  results independent of the rank count.
* C5 (joint DP with densification): each rank renders its own training view
  and accumulates GradAccum (trainer.cpp:134-142) locally; the accumulators
  are all-reduced (sum) before densify_and_prune (trainer.cpp:144-239), which
  every replica runs with the same seeded Rng — both replicas end with the
  identical cloud, equal to the single-process reference order (view 0's
  GradAccum::add, then view 1's, then densify_and_prune).
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn(target, world, *args):
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


# ------------------------------------------------------------------ C3
def test_bench_view_partition_covers_c3():
    import bench
    for ws in (1, 2, 4, 8):
        seen = [v for r in range(ws) for v in bench.my_views(r, ws)]
        assert len(seen) == len(set(seen)) == bench.VIEWS_PER_GPU * ws  # disjoint, weak scaling
    assert sorted(v for r in range(8) for v in bench.my_views(r, 8)) == list(range(bench.TOTAL_VIEWS))


C3_VIEWS, C3_ITERS, W, H = 4, 12, 48, 40


def _c3_scene():
    rng = O.make_rng(3)
    hc = O.synth_cloud(300, 1, rng).as_float32_exact()
    gt = O.synth_poses(1, C3_VIEWS, rng)
    noise = O.make_rng(1002)
    init = np.stack([O.perturb_pose(p, 5.0, 0.05, noise) for p in gt])
    cams = [O.synth_camera(W, H, p) for p in gt]
    targets = [O.render(hc, c).image for c in cams]
    intr = (cams[0].fx, cams[0].fy, cams[0].cx, cams[0].cy)
    return hc, targets, intr, init


def _c3_views(rank, world):
    per = C3_VIEWS // world  # contiguous blocks, as bench.my_views
    return [rank * per + k for k in range(per)]


def _c3_worker(rank, world, port, q):
    import torch
    dist = _init(rank, world, port)
    try:
        hc, targets, intr, init = _c3_scene()
        mine = _c3_views(rank, world)
        local = torch.zeros(C3_VIEWS, 12, dtype=torch.float64)
        for v in mine:
            r = O.estimate_pose(hc, targets[v], *intr, init[v], budget=C3_ITERS, pose_converged_eps=0.0)
            local[v] = torch.from_numpy(r["pose"])
        gathered = [torch.zeros_like(local) for _ in range(world)]
        dist.all_gather(gathered, local)  # end of job: gather the poses (no data-path collective)
        q.put((rank, (mine, sum(gathered).numpy())))
    finally:
        dist.destroy_process_group()


def test_c3_view_sharding_gloo_world2():
    out = _spawn(_c3_worker, 2)
    (m0, p0), (m1, p1) = out[0], out[1]
    assert set(m0).isdisjoint(m1) and sorted(m0 + m1) == list(range(C3_VIEWS))
    assert np.array_equal(p0, p1)
    hc, targets, intr, init = _c3_scene()
    for v in range(C3_VIEWS):  # one process, all views: identical per-view trajectories
        r = O.estimate_pose(hc, targets[v], *intr, init[v], budget=C3_ITERS, pose_converged_eps=0.0)
        assert np.array_equal(r["pose"], p0[v]), v


# ------------------------------------------------------------------ C5
C5_W, C5_H = 64, 48


def _c5_scene():
    rng = O.make_rng(5)
    hc = O.synth_cloud(400, 1, rng).as_float32_exact()
    poses = O.synth_poses(1, 2, rng)
    cams = [O.synth_camera(C5_W, C5_H, p) for p in poses]
    targets = [O.render(hc, c).image for c in cams]
    jit = hc.copy()
    jit.means = jit.means + 0.01 * np.cos(np.arange(jit.means.size)).reshape(jit.means.shape)
    return jit, targets, cams


def _grad_accum_view(cloud, cam, target):
    """GradAccum::add (trainer.cpp:134-142) for one rendered view."""
    rr = O.render(cloud, cam, keep_handle=True)
    _, d_img = O.rgb_loss(rr.image, target, 0.2)
    g = O.render_backward(cloud, cam, rr, d_img)
    gs, ct = np.zeros(cloud.n), np.zeros(cloud.n, np.int32)
    scale = 0.5 * max(cam.width, cam.height)
    for gid in rr.splat_gaussian:
        gs[gid] += np.linalg.norm(g.d_mu2d[gid]) * scale
        ct[gid] += 1
    rr.free()
    return gs, ct


DENSIFY = dict(grad_threshold=2e-4, size_ratio=0.01, n_target=430, prune_opacity=0.005)


def _c5_worker(rank, world, port, q):
    import torch
    dist = _init(rank, world, port)
    try:
        cloud, targets, cams = _c5_scene()
        gs, ct = _grad_accum_view(cloud, cams[rank], targets[rank])  # this rank's slot
        tgs, tct = torch.from_numpy(gs), torch.from_numpy(ct)
        dist.all_reduce(tgs)  # GradAccum summed over ranks before densify_and_prune
        dist.all_reduce(tct)
        rng = O.make_rng(77)  # the run's Rng, replicated: identical split draws on every rank
        new, src, rep = O.densify_and_prune(cloud, tgs.numpy(), tct.numpy().astype(np.int32), rng=rng, **DENSIFY)
        flat = np.concatenate([new.means.ravel(), new.rotations.ravel(), new.log_scales.ravel(),
                               new.opacity_logits.ravel(), new.sh.ravel()])
        q.put((rank, (flat, src, rep)))
    finally:
        dist.destroy_process_group()


def test_c5_dp_densify_gloo_world2():
    out = _spawn(_c5_worker, 2)
    (f0, s0, r0), (f1, s1, r1) = out[0], out[1]
    assert np.array_equal(f0, f1) and np.array_equal(s0, s1) and r0 == r1  # replicas identical
    cloud, targets, cams = _c5_scene()
    gs, ct = np.zeros(cloud.n), np.zeros(cloud.n, np.int32)
    for v in range(2):  # single process, reference order
        a, b = _grad_accum_view(cloud, cams[v], targets[v])
        gs += a
        ct += b
    new, src, rep = O.densify_and_prune(cloud, gs, ct, rng=O.make_rng(77), **DENSIFY)
    ref = np.concatenate([new.means.ravel(), new.rotations.ravel(), new.log_scales.ravel(),
                          new.opacity_logits.ravel(), new.sh.ravel()])
    assert rep == r0 and sum(rep) > 0, rep  # the step densifies / prunes something
    assert np.array_equal(ref, f0) and np.array_equal(src, s0)
