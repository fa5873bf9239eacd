"""3DGS PLY I/O of the device cloud (gsb_cloud_{load,save}_ply) against the
reference format (src/ply.cpp:18-148, tests/test_io.cpp): an independent
numpy writer/reader of the same layout, the degree-3 zero padding on save,
the SH degree inferred from the f_rest count on load, and corrupt_file
errors."""
import os
import tempfile

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


def write_ply(path, hc, degree, extra_comment=True):
    """numpy writer of the reference layout (ply.cpp:29-60) for `degree` bands."""
    B = (degree + 1) ** 2
    names = ["x", "y", "z", "rot_0", "rot_1", "rot_2", "rot_3", "scale_0", "scale_1", "scale_2", "opacity",
             "f_dc_0", "f_dc_1", "f_dc_2"] + [f"f_rest_{k}" for k in range(3 * (B - 1))]
    sh = hc.sh[:, :, :B]
    rows = np.concatenate([hc.means, hc.rotations, hc.log_scales, hc.opacity_logits[:, None], sh[:, :, 0],
                           sh[:, :, 1:].reshape(hc.n, -1)], axis=1).astype("<f4")
    with open(path, "wb") as f:
        f.write(b"ply\nformat binary_little_endian 1.0\n")
        if extra_comment:
            f.write(b"comment written by the test\n")
        f.write(f"element vertex {hc.n}\n".encode())
        for nm in names:
            f.write(f"property float {nm}\n".encode())
        f.write(b"end_header\n")
        f.write(rows.tobytes())


def read_ply(path):
    with open(path, "rb") as f:
        data = f.read()
    head, body = data.split(b"end_header\n", 1)
    lines = head.decode().splitlines()
    n = int([ln for ln in lines if ln.startswith("element vertex")][0].split()[-1])
    cols = [ln.split()[-1] for ln in lines if ln.startswith("property")]
    return cols, np.frombuffer(body, "<f4").reshape(n, len(cols))


@pytest.mark.parametrize("degree", [0, 1, 2, 3])
def test_load_reference_layout(G, ctx, degree):
    hc = O.synth_cloud(777, 3, O.make_rng(5 + degree)).as_float32_exact()
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "c.ply")
        write_ply(p, hc, degree)
        cloud = G.Cloud.load_ply(ctx, p)
        assert cloud.n == hc.n and cloud.sh_degree == degree
        m, q, ls, op, sh = cloud.download()
        B = (degree + 1) ** 2
        assert np.array_equal(m, hc.means) and np.array_equal(q, hc.rotations)
        assert np.array_equal(ls, hc.log_scales) and np.array_equal(op, hc.opacity_logits)
        assert np.array_equal(sh, hc.sh[:, :, :B])


def test_save_pads_to_degree3_and_round_trips(G, ctx):
    hc = O.synth_cloud(1000, 1, O.make_rng(8)).as_float32_exact()
    cloud = G.Cloud.from_host(ctx, hc.means, hc.rotations, hc.log_scales, hc.opacity_logits, hc.sh, 1)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "c.ply")
        cloud.save_ply(p)
        cols, rows = read_ply(p)
        assert len(cols) == 59 and cols[14] == "f_rest_0" and cols[-1] == "f_rest_44"
        assert np.array_equal(rows[:, 0:3], hc.means.astype(np.float32))
        rest = rows[:, 14:].reshape(-1, 3, 15)
        assert np.array_equal(rest[:, :, :3], hc.sh[:, :, 1:4].astype(np.float32))
        assert np.all(rest[:, :, 3:] == 0.0)
        back = G.Cloud.load_ply(ctx, p)  # always reloads as degree 3 (tests/test_io.cpp:54)
        assert back.sh_degree == 3 and back.n == hc.n
        m, q, ls, op, sh = back.download()
        assert np.array_equal(m, hc.means) and np.array_equal(sh[:, :, :4], hc.sh)
        assert np.all(sh[:, :, 4:] == 0.0)
        # a loaded cloud renders like the uploaded one
        cam = G.Camera.from_pose12(*G.synth_intrinsics(64, 48), 64, 48, O.synth_poses(0, 1, O.make_rng(1))[0])
        a = G.render(ctx, cloud, cam).image
        b = G.render(ctx, back, cam).image
        assert np.max(np.abs(a - b)) < 1e-6


def test_corrupt_files(G, ctx):
    hc = O.synth_cloud(50, 1, O.make_rng(3)).as_float32_exact()
    with tempfile.TemporaryDirectory() as d:
        good = os.path.join(d, "g.ply")
        write_ply(good, hc, 1)
        data = open(good, "rb").read()
        cases = {
            "magic": b"plx" + data[3:],
            "ascii": data.replace(b"binary_little_endian", b"ascii", 1),
            "missing": data.replace(b"property float opacity\n", b"", 1),
            "truncated": data[:-100],
            "rest": data.replace(b"property float f_rest_8\n", b"", 1),
        }
        for name, blob in cases.items():
            p = os.path.join(d, name + ".ply")
            open(p, "wb").write(blob)
            with pytest.raises(G.GsbError) as e:
                G.Cloud.load_ply(ctx, p)
            assert e.value.code == 9, name  # ErrorCode::corrupt_file + 1
        with pytest.raises(G.GsbError) as e:
            G.Cloud.load_ply(ctx, os.path.join(d, "absent.ply"))
        assert e.value.code == 9
