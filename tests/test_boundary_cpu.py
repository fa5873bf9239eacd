"""CPU-side checks of the drop-in boundary (no GPU needed):
the C-ABI library loads and exports every entry point include/gsb200.h
declares, refuses to run without a device (no CPU fallback), and its host-only
helpers (synthetic input generators, schedule) equal the oracle's restatement
of the reference (synth.cpp:73-101, eval.cpp:130-146, trainer.cpp:30-38)."""
import os
import re

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def G():
    from paper_2410_08743_b200 import build, gsb
    build.build()
    return gsb


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "gsb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gsb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(G):
    import ctypes
    L = ctypes.CDLL(G.LIB_PATH)
    names = _declared_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_no_device_means_loud_failure(G):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(G.GsbError) as ei:
        G.Context(0)
    assert ei.value.code == G.ERR_NO_DEVICE


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_synth_poses_match_oracle(G, kind):
    rng = O.make_rng(7)
    O.synth_cloud(40, 1, rng)
    want = O.synth_poses(kind, 6, rng)
    got = G.synth_poses(7, 40, 1, kind, 6)
    assert np.array_equal(got, want)


def test_perturb_pose_matches_oracle(G):
    rng = O.make_rng(99)
    O.synth_cloud(20, 1, rng)
    poses = O.synth_poses(0, 4, rng)
    orng = O.make_rng(1002)
    prng = G.PoseRng(1002)
    for p in poses:
        assert np.array_equal(prng.perturb_pose(p, 15.0, 0.15), O.perturb_pose(p, 15.0, 0.15, orng))


def test_schedule_matches_reference(G):
    for step in (0, 13, 50, 99, 100, 150):
        assert G.schedule("cosine", 1e-2, 1e-4, step, 100) == O.schedule("cosine", 1e-2, 1e-4, step, 100)
        assert G.schedule("exp", 1.6e-2, 1.6e-4, step, 100) == O.schedule("exp", 1.6e-2, 1.6e-4, step, 100)
