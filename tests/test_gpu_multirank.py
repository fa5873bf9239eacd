"""Two-rank NCCL run of the graph-captured joint step, one
process per GPU. Skipped below 2 visible GPUs (the round's boxes have one;
the gloo world-2 tests in test_multirank_cpu.py / test_joint_cpu.py cover the
host semantics there).

Rank r renders slot r of each step; the FP32 gradient planes and the FP64
exchange slots are all-reduced by NCCL inside the step's CUDA graph. The
result must equal a single process running both slots locally (local = 2):
float addition of two addends is commutative, the exchange slots hold one
non-zero contribution each, so replicas and the local run are bitwise equal.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _scene():
    from test_gpu_joint import joint_scene
    return joint_scene(seed=4, n=400, sh=1, views=4)


def _worker(rank, world, uid, q):
    from paper_2410_08743_b200 import gsb
    from test_gpu_joint import run_device
    ctx = gsb.Context(rank)
    comm = gsb.Comm(ctx, uid, rank, world)
    hc, imgs, intr, init, _ = _scene()
    cfg = gsb.JointConfig.default(iterations=6, sh_degree=1, sh_degree_interval=0)
    res, dev = run_device(gsb, ctx, hc, imgs, intr, init, cfg, 11, 1, comm=comm)
    comm.close()
    q.put((rank, res["poses"], res["trace_total"], [np.asarray(a) for a in dev]))


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (one process per GPU)")
def test_joint_nccl_two_ranks_equals_local_two_slots():
    import torch.multiprocessing as mp
    from paper_2410_08743_b200 import build, gsb
    build.build()
    uid = gsb.Comm.unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, uid, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, rest) for r, *rest in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (P0, T0, D0), (P1, T1, D1) = out[0], out[1]
    assert np.array_equal(P0, P1) and np.array_equal(T0, T1)
    assert all(np.array_equal(a, b) for a, b in zip(D0, D1))  # replicas in lock step
    from test_gpu_joint import run_device
    hc, imgs, intr, init, _ = _scene()
    cfg = gsb.JointConfig.default(iterations=6, sh_degree=1, sh_degree_interval=0)
    res, dev = run_device(gsb, gsb.Context(0), hc, imgs, intr, init, cfg, 11, 2)
    assert np.array_equal(res["poses"], P0) and np.array_equal(res["trace_total"], T0)
    assert all(np.array_equal(np.asarray(a), b) for a, b in zip(dev, D0))
