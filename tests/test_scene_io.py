"""On-disk formats around the hot path (host C++ in
csrc/scene_io.cpp): f32map (image.cpp:105-141, tests/test_io.cpp:123-134),
pose lists (scene_io.cpp:64-79, tests/test_io.cpp:71-84) and cameras.json
(scene_io.cpp:254-279). Host-only code: runs on the CPU suite."""
import json
import os
import tempfile

import numpy as np
import pytest

from oracle import oracle as O


@pytest.fixture(scope="module")
def G():
    from paper_2410_08743_b200 import build, gsb
    build.build()
    return gsb


def test_float_map_round_trip(G):
    vals = np.array([[1.5, 2.25, 0.0], [-3.75, 100.0, 0.125]], np.float32)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "map.f32")
        G.save_float_map(vals, p)
        back = G.load_float_map(p)
        assert back.shape == (2, 3) and np.array_equal(back, vals)
        assert open(p, "rb").read().startswith(b"f32map 3 2 1\n")
        # scale applied on load, in FP32 (image.cpp:121-123)
        G.save_float_map(vals, p, scale=0.5)
        assert np.array_equal(G.load_float_map(p), (vals * 0.5).astype(np.float32))


def test_float_map_corrupt(G):
    with tempfile.TemporaryDirectory() as d:
        good = os.path.join(d, "g.f32")
        G.save_float_map(np.ones((4, 5), np.float32), good)
        blob = open(good, "rb").read()
        for name, data in {"magic": b"f64map" + blob[6:], "truncated": blob[:-3],
                           "dims": b"f32map 0 4 1\n" + blob[blob.index(b"\n") + 1:]}.items():
            p = os.path.join(d, name)
            open(p, "wb").write(data)
            with pytest.raises(G.GsbError) as e:
                G.load_float_map(p)
            assert e.value.code == G.ERR_CORRUPT_FILE, name
        with pytest.raises(G.GsbError):
            G.load_float_map(os.path.join(d, "absent.f32"))


def test_depth_map_validity(G):
    v = np.array([[1.0, 0.0, -2.0], [np.nan, np.inf, 3.5]], np.float32)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "depth.f32")
        G.save_float_map(v, p)
        dep, val = G.load_depth_map(p)
        assert np.array_equal(val, [[1, 0, 0], [0, 0, 1]])
        assert dep[0, 0] == 1.0 and dep[1, 2] == 3.5


def test_pose_json_round_trip_is_lossless(G):
    rng = O.make_rng(132)
    I = np.hstack([np.eye(3), np.zeros((3, 1))]).reshape(12)
    poses = np.stack([O.perturb_pose(I, 40.0, 1.0, rng) for _ in range(12)])
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "poses.json")
        G.save_poses_json(poses, p)
        back = G.load_poses_json(p)
        assert np.array_equal(back, poses)  # 17 digits: bit-exact
        assert np.array_equal(np.asarray(json.load(open(p))["poses"]), poses)  # plain JSON
        G.save_poses_json(np.zeros((0, 12)), p)
        assert G.load_poses_json(p).shape == (0, 12)
        for bad in ('{"poses": [[1, 2, 3]]}', '{"other": []}', '{"poses": [', '[1, 2]'):
            open(p, "w").write(bad)
            with pytest.raises(G.GsbError) as e:
                G.load_poses_json(p)
            assert e.value.code == G.ERR_CORRUPT_FILE, bad


def test_cameras_json(G):
    I = list(np.hstack([np.eye(3), np.zeros((3, 1))]).reshape(12))
    P1 = [0.0, -1.0, 0.0, 0.5, 1.0, 0.0, 0.0, -0.25, 0.0, 0.0, 1.0, 2.0]
    cam = {"fx": 756.0, "fy": 757.5, "cx": 503.5, "cy": 377.5, "width": 1008, "height": 756,
           "frames": [{"file": "a.png", "pose": I}, {"file": "bé.png", "pose": P1}]}
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "cameras.json")
        json.dump(cam, open(p, "w"), indent=2)
        c = G.load_cameras_json(p)
        assert list(c["intrinsics"]) == [756.0, 757.5, 503.5, 377.5]
        assert (c["width"], c["height"]) == (1008, 756) and c["has_poses"]
        assert c["names"] == ["a.png", "bé.png"]
        assert np.array_equal(c["poses"], np.array([I, P1]))
        cam["frames"][1].pop("pose")  # partial poses: identity, has_poses false
        json.dump(cam, open(p, "w"))
        c = G.load_cameras_json(p)
        assert not c["has_poses"] and np.array_equal(c["poses"][1], I)
        for key in ("fx", "frames", "height"):
            bad = dict(cam)
            bad.pop(key)
            json.dump(bad, open(p, "w"))
            with pytest.raises(G.GsbError) as e:
                G.load_cameras_json(p)
            assert e.value.code == G.ERR_MISSING_INTRINSICS, key
