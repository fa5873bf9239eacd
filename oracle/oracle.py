"""ctypes wrapper over oracle/_build/liboracle.so — TEST INFRASTRUCTURE ONLY.

The oracle is the FP64 CPU restatement of the reference hot path (see
gsopt_oracle.h). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module, and only as the
checker or the CPU baseline: nothing in paper_2410_08743_b200/ imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O3, OpenMP, no FMA contraction)."""
    src = os.path.join(HERE, "gsopt_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


class Rng(C.Structure):
    _fields_ = [("state", C.c_uint64)]


class Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("R", C.c_double * 9), ("t", C.c_double * 3)]


class RasterConfig(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("cutoff_sigma", C.c_double), ("alpha_clamp", C.c_double),
                ("dilation", C.c_double), ("early_termination", C.c_double), ("z_near", C.c_double),
                ("deterministic", C.c_int32)]


class Cloud(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_degree", C.c_int32), ("active_sh_degree", C.c_int32),
                ("means", C.POINTER(C.c_double)), ("rotations", C.POINTER(C.c_double)),
                ("log_scales", C.POINTER(C.c_double)), ("opacity_logits", C.POINTER(C.c_double)),
                ("sh", C.POINTER(C.c_double))]


class Splat(C.Structure):
    _fields_ = [("gaussian", C.c_int32), ("mu2d", C.c_double * 2), ("depth", C.c_double),
                ("conic", C.c_double * 4), ("color", C.c_double * 3), ("opacity", C.c_double),
                ("radius", C.c_double), ("color_clamped", C.c_uint8)]


class RenderOut(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("n_splats", C.c_int64), ("n_entries", C.c_int64),
                ("image", C.POINTER(C.c_double)), ("accum_transmittance", C.POINTER(C.c_double)),
                ("final_transmittance", C.POINTER(C.c_double)), ("contrib_count", C.POINTER(C.c_int32)),
                ("overflow_mask", C.POINTER(C.c_uint8)), ("splats", C.POINTER(Splat)),
                ("tile_lists", C.POINTER(C.c_int32)), ("tile_ranges", C.POINTER(C.c_int32)),
                ("camera", Camera), ("background", C.c_double * 3), ("config", RasterConfig),
                ("state_fingerprint", C.c_uint64), ("n_gaussians", C.c_int64)]


class Grads(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_len", C.c_int64), ("d_means", C.POINTER(C.c_double)),
                ("d_rotations", C.POINTER(C.c_double)), ("d_log_scales", C.POINTER(C.c_double)),
                ("d_opacity_logits", C.POINTER(C.c_double)), ("d_sh", C.POINTER(C.c_double)),
                ("d_mu2d", C.POINTER(C.c_double)), ("d_pose", C.c_double * 6)]


class PoseAdam(C.Structure):
    _fields_ = [("m", C.c_double * 6), ("v", C.c_double * 6), ("step", C.c_int64)]


class JointCfg(C.Structure):
    """orc_joint_cfg: the TrainConfig fields joint_optimize reads (trainer.hpp:21-60, losses.hpp:15-19)."""
    _fields_ = [("iterations", C.c_int32), ("cam_lr_start", C.c_double), ("cam_lr_end", C.c_double),
                ("pos_lr_start", C.c_double), ("pos_lr_end", C.c_double), ("rot_lr", C.c_double),
                ("scale_lr", C.c_double), ("opacity_lr", C.c_double), ("sh_dc_lr", C.c_double),
                ("sh_rest_lr", C.c_double), ("opacity_l1_steps", C.c_int32), ("sh_degree", C.c_int32),
                ("sh_degree_interval", C.c_int32), ("optimize_poses", C.c_int32), ("beta", C.c_double),
                ("aniso_ratio", C.c_double), ("opacity_l1_weight", C.c_double), ("background", C.c_double * 3),
                ("raster", RasterConfig), ("densify_interval", C.c_int32), ("densify_start", C.c_int32),
                ("densify_stop", C.c_int32), ("n_target", C.c_int32), ("grad_threshold", C.c_double),
                ("densify_size_ratio", C.c_double), ("prune_opacity", C.c_double)]


class FitCfg(C.Structure):
    _fields_ = [("steps", C.c_int32), ("unproject_points", C.c_int32), ("pos_lr_start", C.c_double),
                ("pos_lr_end", C.c_double), ("rot_lr", C.c_double), ("scale_lr", C.c_double),
                ("opacity_lr", C.c_double), ("sh_dc_lr", C.c_double), ("sh_rest_lr", C.c_double),
                ("beta", C.c_double), ("background", C.c_double * 3), ("raster", RasterConfig)]


class RelposeCfg(C.Structure):
    _fields_ = [("steps", C.c_int32), ("lr_start", C.c_double), ("lr_end", C.c_double), ("beta", C.c_double),
                ("mask_threshold", C.c_double), ("background", C.c_double * 3), ("raster", RasterConfig)]


class PoseCfg(C.Structure):
    _fields_ = [("cam_lr_start", C.c_double), ("cam_lr_end", C.c_double), ("beta", C.c_double),
                ("pose_converged_eps", C.c_double), ("background", C.c_double * 3), ("raster", RasterConfig)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        d, i32, i64, u64, vp = C.c_double, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
        sig = {
            "orc_rng_init": (None, [P(Rng), u64]),
            "orc_rng_uniform": (d, [P(Rng)]),
            "orc_rng_normal": (d, [P(Rng)]),
            "orc_rng_uniform_range": (d, [P(Rng), d, d]),
            "orc_default_raster_config": (None, [P(RasterConfig)]),
            "orc_quat_to_rotation": (None, [vp, vp]),
            "orc_quat_rotation_jacobian": (None, [vp, vp]),
            "orc_covariance3d": (None, [vp, vp, vp]),
            "orc_sh_basis": (None, [vp, C.c_int, vp]),
            "orc_sh_basis_gradient": (None, [vp, C.c_int, vp]),
            "orc_sh_eval": (None, [vp, vp, C.c_int, vp, vp]),
            "orc_se3_exp": (None, [vp, vp, vp]),
            "orc_so3_exp": (None, [vp, vp]),
            "orc_orthonormalize": (None, [vp]),
            "orc_rotation_angle": (d, [vp]),
            "orc_project": (None, [vp, P(Camera), vp, vp]),
            "orc_covariance2d": (None, [vp, vp, P(Camera), d, vp]),
            "orc_splat_alpha": (d, [vp, vp, d, vp, d, d]),
            "orc_fingerprint": (u64, [P(Cloud), P(Camera)]),
            "orc_render": (P(RenderOut), [P(Cloud), P(Camera), vp, P(RasterConfig)]),
            "orc_render_free": (None, [P(RenderOut)]),
            "orc_bin_records": (i64, [i64, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, i64, vp]),
            "orc_render_backward": (C.c_int, [P(Cloud), P(Camera), P(RenderOut), vp, i32, i32, P(Grads)]),
            "orc_grads_free": (None, [P(Grads)]),
            "orc_rgb_loss": (d, [vp, vp, i32, i32, d, vp]),
            "orc_ssim": (d, [vp, vp, i32, i32, vp]),
            "orc_anisotropy_loss": (d, [vp, i64, d, vp]),
            "orc_opacity_l1": (d, [vp, i64, vp]),
            "orc_schedule": (d, [C.c_int, d, d, i64, i64]),
            "orc_pose_step": (None, [vp, vp, vp, d, P(PoseAdam), vp, vp, vp]),
            "orc_estimate_pose": (i32, [P(Cloud), vp, d, d, d, d, i32, i32, vp, vp, P(PoseCfg), i32,
                                        vp, vp, vp, vp, vp, vp, vp]),
            "orc_synth_cloud": (None, [P(Cloud), i64, i32, P(Rng)]),
            "orc_look_at": (None, [vp, vp, vp, vp]),
            "orc_synth_poses": (None, [i32, i32, d, d, P(Rng), vp]),
            "orc_perturb_pose": (None, [vp, vp, d, d, P(Rng), vp, vp]),
            "orc_perturb_pose_tangent": (None, [vp, vp, d, P(Rng), vp, vp]),
            "orc_abs_pose_error": (None, [vp, vp, vp, vp, vp, vp]),
            "orc_make_gradcheck_scene": (None, [P(Rng), i32, i32, P(Cloud), P(Camera), vp]),
            "orc_scene_is_conditioned": (C.c_int, [P(Cloud), P(Camera), vp, P(RasterConfig)]),
            "orc_gradcheck": (d, [P(Cloud), P(Camera), vp, P(RasterConfig), P(Rng), d, P(i32), C.c_char_p]),
            "orc_cloud_alloc": (None, [P(Cloud), i64, i32]),
            "orc_cloud_free": (None, [P(Cloud)]),
            "orc_num_threads": (C.c_int, []),
            "orc_count_work": (None, [P(RenderOut), vp, vp]),
            "orc_decision_margin": (None, [P(RenderOut), vp]),
            "orc_joint_schedule": (None, [P(Rng), i32, i64, vp]),
            "orc_cloud_adam_step": (None, [P(Cloud), P(Grads), vp, vp]),
            "orc_densify_and_prune": (None, [P(Cloud), vp, vp, d, d, i32, d, P(Rng), P(Cloud), vp, vp]),
            "orc_free": (None, [vp]),
            "orc_transmittance_mask": (None, [vp, i64, d, vp]),
            "orc_masked_rgb_loss": (d, [vp, vp, i32, i32, vp, d, vp, P(i32)]),
            "orc_unproject": (i64, [vp, vp, i32, i32, vp, d, d, d, d, vp, vp, i32, vp, vp]),
            "orc_mean_knn_distance": (None, [vp, i64, C.c_int, vp]),
            "orc_init_from_points": (None, [vp, vp, i64, i32, P(Cloud)]),
            "orc_fit_frame_gaussians": (i32, [vp, vp, vp, i32, i32, d, d, d, d, P(FitCfg), P(Cloud)]),
            "orc_estimate_relative_pose": (i32, [P(Cloud), vp, i32, i32, d, d, d, d, P(RelposeCfg), vp, vp, P(d)]),
            "orc_bootstrap_trajectory": (i32, [vp, vp, vp, i32, i32, i32, d, d, d, d, P(FitCfg), P(RelposeCfg), vp,
                                               vp]),
            "orc_joint_optimize": (i32, [P(Cloud), vp, i32, d, d, d, d, i32, i32, vp, P(JointCfg), i32, P(Rng),
                                         vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


# ------------------------------------------------------------ backends
# "port": the clean-room restatement (liboracle.so). "reference": the
# reference's own sources compiled against oracle/shim (oracle/_ref, see
# build_ref.py); entry points with a reference counterpart route there, the
# rest (allocation helpers, work counters, generators without one) stay on
# the port. Select with `with reference_backend(): ...`.
REF_LIB_PATH = os.path.join(HERE, "_ref", "libgsopt_ref.so")
_REF_NAMES = ("render", "render_free", "render_backward", "grads_free", "rgb_loss", "schedule", "pose_step",
              "make_gradcheck_scene", "scene_is_conditioned", "gradcheck", "perturb_pose", "perturb_pose_tangent",
              "joint_optimize", "cloud_free")
_backend = ["port"]
_ref_lib = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


def ref_lib():
    """oracle/_ref/libgsopt_ref.so with argtypes (orc_* signatures, ref_* names)."""
    global _ref_lib
    if _ref_lib is None:
        L = C.CDLL(REF_LIB_PATH)
        port = lib()
        for name in _REF_NAMES:
            f, g = getattr(L, "ref_" + name), getattr(port, "orc_" + name)
            f.restype, f.argtypes = g.restype, g.argtypes
        P = C.POINTER
        d, i32, vp = C.c_double, C.c_int32, C.c_void_p
        L.ref_pose_descent_traced.restype = i32
        L.ref_pose_descent_traced.argtypes = port.orc_estimate_pose.argtypes
        L.ref_estimate_pose.restype = i32
        L.ref_estimate_pose.argtypes = port.orc_estimate_pose.argtypes[:16]
        L.ref_synth_scene.restype = None
        L.ref_synth_scene.argtypes = [i32, i32, i32, i32, i32, i32, C.c_uint64, P(Cloud), vp, vp]
        L.ref_adam_step.restype = None
        L.ref_adam_step.argtypes = [vp, vp, vp, vp, P(C.c_int64), C.c_int64, d, vp]
        L.ref_render_expected_depth.restype = None
        L.ref_render_expected_depth.argtypes = [P(Cloud), P(Camera), P(RasterConfig), vp, vp]
        L.ref_last_error.restype = C.c_char_p
        L.ref_thread_count.restype = C.c_int
        _ref_lib = L
    return _ref_lib


class _RefRouter:
    def __getattr__(self, name):
        base = name[4:] if name.startswith("orc_") else name
        if base == "estimate_pose":
            return ref_lib().ref_pose_descent_traced
        if base in _REF_NAMES:
            return getattr(ref_lib(), "ref_" + base)
        return getattr(lib(), name)


def _L():
    return _RefRouter() if _backend[0] == "reference" else lib()


class reference_backend:
    """Context manager: route the wrappers below to the reference build."""

    def __enter__(self):
        if not ref_available():
            raise FileNotFoundError(f"{REF_LIB_PATH} missing: run oracle/build_ref.py")
        self.prev = _backend[0]
        _backend[0] = "reference"
        return self

    def __exit__(self, *exc):
        _backend[0] = self.prev
        return False


def ref_estimate_pose(cloud: "HostCloud", image, fx, fy, cx, cy, init12, budget=1000, cam_lr_start=1e-2,
                      cam_lr_end=1e-4, beta=0.2, pose_converged_eps=1e-7, bg=(0, 0, 0), cfg=None):
    """The reference's own estimate_pose (pipelines.cpp:218-222 -> 58-92), no traces."""
    pc = PoseCfg()
    pc.cam_lr_start, pc.cam_lr_end, pc.beta, pc.pose_converged_eps = cam_lr_start, cam_lr_end, beta, pose_converged_eps
    for k in range(3):
        pc.background[k] = bg[k]
    pc.raster = cfg or default_raster_config()
    img = np.ascontiguousarray(image, np.float64)
    R0, t0 = pose_split(init12)
    Ro, to = np.zeros(9), np.zeros(3)
    fl, conv = C.c_double(), C.c_int32()
    steps = ref_lib().ref_estimate_pose(cloud.c().ref(), _p(img), fx, fy, cx, cy, img.shape[1], img.shape[0], _p(R0),
                                        _p(t0), C.byref(pc), budget, _p(Ro), _p(to),
                                        C.cast(C.byref(fl), C.c_void_p), C.cast(C.byref(conv), C.c_void_p))
    return dict(pose=pose_join(Ro, to), steps=steps, final_loss=fl.value, converged=bool(conv.value))


def ref_render_expected_depth(cloud: "HostCloud", cam: Camera, cfg=None):
    """The reference's own render_expected_depth (rasterizer.cpp:283-323): (depth, weight) float32 (H, W)."""
    depth = np.zeros((cam.height, cam.width), np.float32)
    weight = np.zeros((cam.height, cam.width), np.float32)
    ref_lib().ref_render_expected_depth(cloud.c().ref(), C.byref(cam), C.byref(cfg or default_raster_config()),
                                        _p(depth), _p(weight))
    return depth, weight


def ref_synth_scene(gaussians, cameras, width, height, kind, sh_degree, seed, with_images=False):
    """synth.cpp:33-135 run by the reference: (HostCloud, poses (cameras,12), images or None)."""
    cc = Cloud()
    poses = np.zeros((cameras, 12))
    imgs = np.zeros((cameras, height, width, 3)) if with_images else None
    ref_lib().ref_synth_scene(gaussians, cameras, width, height, kind, sh_degree, seed, C.byref(cc), _p(poses),
                              _p(imgs) if with_images else None)
    hc = _from_c_cloud(cc)
    lib().orc_cloud_free(C.byref(cc))
    return hc, poses, imgs


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def _arr(ptr, n, dtype=np.float64):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


# ------------------------------------------------------------------ types
def make_rng(seed: int) -> Rng:
    r = Rng()
    _L().orc_rng_init(C.byref(r), seed)
    return r


def default_raster_config(**kw) -> RasterConfig:
    c = RasterConfig()
    _L().orc_default_raster_config(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def make_camera(fx, fy, cx, cy, w, h, R=None, t=None) -> Camera:
    c = Camera()
    c.fx, c.fy, c.cx, c.cy, c.width, c.height = fx, fy, cx, cy, w, h
    R = np.eye(3) if R is None else np.asarray(R, np.float64).reshape(9)
    t = np.zeros(3) if t is None else np.asarray(t, np.float64).reshape(3)
    for k in range(9):
        c.R[k] = float(np.asarray(R).reshape(9)[k])
    for k in range(3):
        c.t[k] = float(t[k])
    return c


def camera_pose(cam: Camera):
    return np.array(cam.R[:]).reshape(3, 3), np.array(cam.t[:])


@dataclass
class HostCloud:
    """Reference-layout FP64 cloud (scene.hpp:22-46)."""
    means: np.ndarray          # (n,3)
    rotations: np.ndarray      # (n,4) wxyz
    log_scales: np.ndarray     # (n,3)
    opacity_logits: np.ndarray  # (n,)
    sh: np.ndarray             # (n,3,basis)
    sh_degree: int
    active_sh_degree: int

    @property
    def n(self):
        return self.means.shape[0]

    def copy(self):
        return HostCloud(self.means.copy(), self.rotations.copy(), self.log_scales.copy(),
                         self.opacity_logits.copy(), self.sh.copy(), self.sh_degree, self.active_sh_degree)

    def as_float32_exact(self):
        """Round every parameter to FP32 and back (what the device stores)."""
        f = lambda a: a.astype(np.float32).astype(np.float64)
        return HostCloud(f(self.means), f(self.rotations), f(self.log_scales), f(self.opacity_logits),
                         f(self.sh), self.sh_degree, self.active_sh_degree)

    def c(self) -> "CloudView":
        return CloudView(self)


class CloudView:
    """Keeps numpy buffers alive while a C Cloud struct points into them."""

    def __init__(self, hc: HostCloud):
        self.hc = hc
        self.bufs = [np.ascontiguousarray(x, np.float64) for x in
                     (hc.means, hc.rotations, hc.log_scales, hc.opacity_logits, hc.sh)]
        s = Cloud()
        s.n = hc.n
        s.sh_degree = hc.sh_degree
        s.active_sh_degree = hc.active_sh_degree
        P = C.POINTER(C.c_double)
        s.means, s.rotations, s.log_scales, s.opacity_logits, s.sh = [b.ctypes.data_as(P) for b in self.bufs]
        self.s = s

    def ref(self):
        return C.byref(self.s)


def _from_c_cloud(cc: Cloud) -> HostCloud:
    n = cc.n
    b = (cc.sh_degree + 1) ** 2
    return HostCloud(_arr(cc.means, 3 * n).reshape(n, 3), _arr(cc.rotations, 4 * n).reshape(n, 4),
                     _arr(cc.log_scales, 3 * n).reshape(n, 3), _arr(cc.opacity_logits, n),
                     _arr(cc.sh, 3 * b * n).reshape(n, 3, b), cc.sh_degree, cc.active_sh_degree)


def synth_cloud(n: int, sh_degree: int, rng: Rng) -> HostCloud:
    """synth.cpp:45-62 draws (consumes rng)."""
    cc = Cloud()
    _L().orc_synth_cloud(C.byref(cc), n, sh_degree, C.byref(rng))
    hc = _from_c_cloud(cc)
    _L().orc_cloud_free(C.byref(cc))
    return hc


def synth_poses(kind: int, cameras: int, rng: Rng, orbit_radius=2.5, orbit_arc=2 * np.pi) -> np.ndarray:
    out = np.zeros((cameras, 12))
    _L().orc_synth_poses(kind, cameras, orbit_radius, orbit_arc, C.byref(rng), _p(out))
    return out


def pose_split(p12):
    p = np.asarray(p12, np.float64).reshape(3, 4)
    return np.ascontiguousarray(p[:, :3]), np.ascontiguousarray(p[:, 3])


def pose_join(R, t):
    return np.concatenate([np.asarray(R).reshape(3, 3), np.asarray(t).reshape(3, 1)], axis=1).reshape(12)


def perturb_pose(p12, rot_deg, trans, rng: Rng):
    R, t = pose_split(p12)
    Ro, to = np.zeros(9), np.zeros(3)
    _L().orc_perturb_pose(_p(R), _p(t), rot_deg, trans, C.byref(rng), _p(Ro), _p(to))
    return pose_join(Ro, to)


def perturb_pose_tangent(p12, sigma, rng: Rng):
    R, t = pose_split(p12)
    Ro, to = np.zeros(9), np.zeros(3)
    _L().orc_perturb_pose_tangent(_p(R), _p(t), sigma, C.byref(rng), _p(Ro), _p(to))
    return pose_join(Ro, to)


def abs_pose_error(pred12, gt12):
    Rp, tp = pose_split(pred12)
    Rg, tg = pose_split(gt12)
    r, d = C.c_double(), C.c_double()
    _L().orc_abs_pose_error(_p(Rp), _p(tp), _p(Rg), _p(tg), C.cast(C.byref(r), C.c_void_p),
                             C.cast(C.byref(d), C.c_void_p))
    return r.value, d.value


def synth_camera(width, height, p12) -> Camera:
    """Intrinsics as synth.cpp:64-71: fx = fy = 0.75 W, c = (dim-1)/2."""
    R, t = pose_split(p12)
    return make_camera(0.75 * width, 0.75 * width, 0.5 * (width - 1), 0.5 * (height - 1), width, height, R, t)


# ---------------------------------------------------------------- render
@dataclass
class RenderResult:
    image: np.ndarray               # (H,W,3)
    accum_transmittance: np.ndarray  # (H*W,)
    final_transmittance: np.ndarray
    contrib_count: np.ndarray
    overflow_mask: np.ndarray
    splat_gaussian: np.ndarray      # (V,) int32, depth order
    splat_mu2d: np.ndarray          # (V,2)
    splat_depth: np.ndarray
    splat_conic: np.ndarray         # (V,4)
    splat_color: np.ndarray         # (V,3)
    splat_opacity: np.ndarray
    splat_radius: np.ndarray
    splat_clamped: np.ndarray
    tile_lists: np.ndarray          # (K,) indices into splats
    tile_ranges: np.ndarray         # (T,2)
    tiles_x: int
    tiles_y: int
    fingerprint: int
    _ptr: object = None

    _free: object = None

    def free(self):
        if self._ptr is not None:
            self._free(self._ptr)
            self._ptr = None


def render(cloud: HostCloud, cam: Camera, bg=(0.0, 0.0, 0.0), cfg: RasterConfig | None = None,
           keep_handle=False) -> RenderResult:
    cfg = cfg or default_raster_config()
    cv = cloud.c()
    bgv = np.asarray(bg, np.float64)
    ptr = _L().orc_render(cv.ref(), C.byref(cam), _p(bgv), C.byref(cfg))
    o = ptr.contents
    P = o.width * o.height
    V = o.n_splats
    K = o.n_entries
    T = o.tiles_x * o.tiles_y
    sp = np.ctypeslib.as_array(o.splats, shape=(max(V, 1),))[:V] if V else None

    def sf(name, k=None):
        if V == 0:
            return np.zeros((0,) if k is None else (0, k))
        return np.array(sp[name], copy=True)

    rr = RenderResult(
        image=_arr(o.image, 3 * P).reshape(o.height, o.width, 3),
        accum_transmittance=_arr(o.accum_transmittance, P), final_transmittance=_arr(o.final_transmittance, P),
        contrib_count=_arr(o.contrib_count, P, np.int32), overflow_mask=_arr(o.overflow_mask, P, np.uint8),
        splat_gaussian=sf("gaussian").astype(np.int32), splat_mu2d=sf("mu2d", 2), splat_depth=sf("depth"),
        splat_conic=sf("conic", 4), splat_color=sf("color", 3), splat_opacity=sf("opacity"),
        splat_radius=sf("radius"), splat_clamped=sf("color_clamped").astype(np.uint8),
        tile_lists=_arr(o.tile_lists, K, np.int32), tile_ranges=_arr(o.tile_ranges, 2 * T, np.int32).reshape(T, 2),
        tiles_x=o.tiles_x, tiles_y=o.tiles_y, fingerprint=o.state_fingerprint)
    if keep_handle:
        rr._ptr = ptr
        rr._cloud_view = cv
        rr._free = _L().orc_render_free
        rr._lib = _L()
    else:
        _L().orc_render_free(ptr)
    return rr


@dataclass
class GradResult:
    d_means: np.ndarray
    d_rotations: np.ndarray
    d_log_scales: np.ndarray
    d_opacity_logits: np.ndarray
    d_sh: np.ndarray
    d_mu2d: np.ndarray
    d_pose: np.ndarray


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def render_backward(cloud: HostCloud, cam: Camera, rr: RenderResult, d_image: np.ndarray) -> GradResult:
    assert rr._ptr is not None, "render(..., keep_handle=True) required"
    cv = cloud.c()
    d = np.ascontiguousarray(d_image, np.float64)
    h, w = (d.shape[0], d.shape[1]) if d.ndim == 3 else (cam.height, cam.width)
    g = Grads()
    L = rr._lib
    rc = L.orc_render_backward(cv.ref(), C.byref(cam), rr._ptr, _p(d), w, h, C.byref(g))
    if rc != 0:
        raise OracleError(rc, "state_mismatch" if rc == 6 else "dimension_mismatch")
    n = cloud.n
    b = (cloud.sh_degree + 1) ** 2
    out = GradResult(_arr(g.d_means, 3 * n).reshape(n, 3), _arr(g.d_rotations, 4 * n).reshape(n, 4),
                     _arr(g.d_log_scales, 3 * n).reshape(n, 3), _arr(g.d_opacity_logits, n),
                     _arr(g.d_sh, 3 * b * n).reshape(n, 3, b), _arr(g.d_mu2d, 2 * n).reshape(n, 2),
                     np.array(g.d_pose[:]))
    _L().orc_grads_free(C.byref(g))
    return out


def bin_records(keep, mu2d, radius, depth, width, height, tile_size=16):
    """rasterizer.cpp:127-168 fed externally supplied records (bit-exact check)."""
    keep = np.ascontiguousarray(keep, np.uint8)
    mu2d = np.ascontiguousarray(mu2d, np.float64).reshape(-1, 2)
    radius = np.ascontiguousarray(radius, np.float64)
    depth = np.ascontiguousarray(depth, np.float64)
    n = keep.shape[0]
    tx, ty = (width + tile_size - 1) // tile_size, (height + tile_size - 1) // tile_size
    sorted_g = np.zeros(max(n, 1), np.int32)
    nsp = C.c_int64()
    ranges = np.zeros((tx * ty, 2), np.int32)
    cap = 1 << 16
    while True:
        lists = np.zeros(cap, np.int32)
        k = _L().orc_bin_records(n, _p(keep), _p(mu2d), _p(radius), _p(depth), width, height, tile_size,
                                  _p(sorted_g), C.cast(C.byref(nsp), C.c_void_p), _p(lists), cap, _p(ranges))
        if k >= 0:
            return sorted_g[:nsp.value].copy(), lists[:k].copy(), ranges
        cap *= 4


# ------------------------------------------------------------------ losses
def rgb_loss(rendered, target, beta=0.2, want_grad=True):
    r = np.ascontiguousarray(rendered, np.float64)
    t = np.ascontiguousarray(target, np.float64)
    h, w = r.shape[0], r.shape[1]
    d = np.zeros_like(r) if want_grad else None
    loss = _L().orc_rgb_loss(_p(r), _p(t), w, h, beta, _p(d) if want_grad else None)
    return (loss, d) if want_grad else loss


def ssim(a, b, want_grad=False):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    d = np.zeros_like(a) if want_grad else None
    v = _L().orc_ssim(_p(a), _p(b), a.shape[1], a.shape[0], _p(d) if want_grad else None)
    return (v, d) if want_grad else v


def anisotropy_loss(log_scales, ratio=10.0):
    ls = np.ascontiguousarray(log_scales, np.float64)
    d = np.zeros_like(ls)
    v = _L().orc_anisotropy_loss(_p(ls), ls.shape[0], ratio, _p(d))
    return v, d


# ---------------------------------------------------------------- trainer
def schedule(kind, start, end, step, total):
    return _L().orc_schedule(0 if kind == "cosine" else 1, start, end, step, total)


def pose_step(p12, d_pose, lr, adam: PoseAdam):
    R, t = pose_split(p12)
    dp = np.ascontiguousarray(d_pose, np.float64)
    Ro, to, ap = np.zeros(9), np.zeros(3), np.zeros(6)
    _L().orc_pose_step(_p(R), _p(t), _p(dp), lr, C.byref(adam), _p(Ro), _p(to), _p(ap))
    return pose_join(Ro, to), ap


def se3_exp(tau):
    tau = np.ascontiguousarray(tau, np.float64)
    R, t = np.zeros(9), np.zeros(3)
    _L().orc_se3_exp(_p(tau), _p(R), _p(t))
    return R.reshape(3, 3), t


def orthonormalize(R):
    R = np.ascontiguousarray(np.asarray(R, np.float64).reshape(9)).copy()
    _L().orc_orthonormalize(_p(R))
    return R.reshape(3, 3)


def estimate_pose(cloud: HostCloud, image, fx, fy, cx, cy, init12, budget=1000, cam_lr_start=1e-2,
                  cam_lr_end=1e-4, beta=0.2, pose_converged_eps=1e-7, bg=(0, 0, 0), cfg=None):
    """pipelines.cpp:58-92 with per-iteration traces."""
    pc = PoseCfg()
    pc.cam_lr_start, pc.cam_lr_end, pc.beta, pc.pose_converged_eps = cam_lr_start, cam_lr_end, beta, pose_converged_eps
    for k in range(3):
        pc.background[k] = bg[k]
    pc.raster = cfg or default_raster_config()
    img = np.ascontiguousarray(image, np.float64)
    h, w = img.shape[0], img.shape[1]
    R0, t0 = pose_split(init12)
    Ro, to = np.zeros(9), np.zeros(3)
    fl = C.c_double()
    conv = C.c_int32()
    tp, tl, td = np.zeros((budget, 12)), np.zeros(budget), np.zeros((budget, 6))
    cv = cloud.c()
    steps = _L().orc_estimate_pose(cv.ref(), _p(img), fx, fy, cx, cy, w, h, _p(R0), _p(t0), C.byref(pc), budget,
                                    _p(Ro), _p(to), C.cast(C.byref(fl), C.c_void_p),
                                    C.cast(C.byref(conv), C.c_void_p), _p(tp), _p(tl), _p(td))
    return dict(pose=pose_join(Ro, to), steps=steps, final_loss=fl.value, converged=bool(conv.value),
                trace_pose=tp[:steps], trace_loss=tl[:steps], trace_dpose=td[:steps])


class CloudAdam:
    """cloud_adam_step (pipelines.cpp:18-41) over a persistent FP64 cloud and
    its five AdamStates (trainer.hpp:69-78): step(grads, lrs) updates in place."""

    def __init__(self, cloud: HostCloud):
        self.view = cloud.copy().c()
        self.states = (C.c_byte * (5 * 32))()  # 5 x {double* m, *v; int64 n, step}

    def step(self, g: dict, lrs):
        n = self.view.s.n
        bufs = [np.ascontiguousarray(g[k], np.float64).reshape(-1)
                for k in ("d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh")]
        og = Grads()
        og.n, og.sh_len = n, bufs[4].size
        P = C.POINTER(C.c_double)
        og.d_means, og.d_rotations, og.d_log_scales, og.d_opacity_logits, og.d_sh = [b.ctypes.data_as(P) for b in bufs]
        lrs = np.ascontiguousarray(lrs, np.float64)
        _L().orc_cloud_adam_step(self.view.ref(), C.byref(og), C.cast(self.states, C.c_void_p), _p(lrs))

    def cloud(self) -> HostCloud:
        hc = self.view.hc
        return HostCloud(*[b.reshape(a.shape).copy() for b, a in zip(self.view.bufs, (
            hc.means, hc.rotations, hc.log_scales, hc.opacity_logits, hc.sh))], hc.sh_degree, hc.active_sh_degree)


def densify_and_prune(cloud: HostCloud, grad_sum, count, grad_threshold=2e-4, size_ratio=0.01, n_target=256000,
                      prune_opacity=0.005, rng: Rng | None = None):
    """trainer.cpp:144-239. Returns (new HostCloud, final_source int32[n'], (cloned, split, pruned))."""
    cv = cloud.c()
    gs = np.ascontiguousarray(grad_sum, np.float64)
    ct = np.ascontiguousarray(count, np.int32)
    out = Cloud()
    fs = C.POINTER(C.c_int32)()
    rep = np.zeros(3, np.int32)
    _L().orc_densify_and_prune(cv.ref(), _p(gs), _p(ct), grad_threshold, size_ratio, n_target, prune_opacity,
                                C.byref(rng), C.byref(out), C.cast(C.byref(fs), C.c_void_p), _p(rep))
    res = _from_c_cloud(out)
    src = np.ctypeslib.as_array(fs, shape=(max(out.n, 1),))[:out.n].copy() if out.n else np.zeros(0, np.int32)
    _L().orc_free(C.cast(fs, C.c_void_p))
    _L().orc_cloud_free(C.byref(out))
    return res, src, tuple(int(x) for x in rep)


def joint_config(iterations, **kw) -> JointCfg:
    """TrainConfig defaults (trainer.hpp:21-60, losses.hpp:15-19) with overrides."""
    c = JointCfg()
    c.iterations = iterations
    c.cam_lr_start, c.cam_lr_end, c.pos_lr_start, c.pos_lr_end = 1e-2, 1e-4, 1.6e-2, 1.6e-4
    c.rot_lr, c.scale_lr, c.opacity_lr, c.sh_dc_lr, c.sh_rest_lr = 1e-3, 5e-3, 5e-2, 2.5e-3, 2.5e-3 / 20.0
    c.opacity_l1_steps, c.sh_degree, c.sh_degree_interval, c.optimize_poses = 10000, 3, 1000, 1
    c.beta, c.aniso_ratio, c.opacity_l1_weight = 0.2, 10.0, 0.01
    c.raster = default_raster_config()
    c.densify_interval, c.densify_start, c.densify_stop, c.n_target = 100, 500, 15000, 256000
    c.grad_threshold, c.densify_size_ratio, c.prune_opacity = 2e-4, 0.01, 0.005
    for k, v in kw.items():
        if k == "background":
            for i in range(3):
                c.background[i] = v[i]
        else:
            setattr(c, k, v)
    return c


def joint_schedule(rng: Rng, n_views: int, count: int) -> np.ndarray:
    """pipelines.cpp:122-129 view sequence (epoch shuffles in place)."""
    out = np.zeros(count, np.int32)
    _L().orc_joint_schedule(C.byref(rng), n_views, count, _p(out))
    return out


def _alloc_c_cloud(hc: HostCloud) -> Cloud:
    """A malloc-backed copy (orc_cloud_alloc) the oracle may reallocate."""
    cc = Cloud()
    _L().orc_cloud_alloc(C.byref(cc), hc.n, hc.sh_degree)
    cc.active_sh_degree = hc.active_sh_degree
    for name, arr in (("means", hc.means), ("rotations", hc.rotations), ("log_scales", hc.log_scales),
                      ("opacity_logits", hc.opacity_logits), ("sh", hc.sh)):
        a = np.ascontiguousarray(arr, np.float64).reshape(-1)
        if a.size:
            C.memmove(getattr(cc, name), a.ctypes.data, a.nbytes)
    return cc


def joint_optimize(cloud: HostCloud, images, intr, width, height, poses, cfg: JointCfg, slots: int, rng: Rng):
    """pipelines.cpp:96-216 (+ densify_and_prune), `slots` views per step. Returns
    (status, cloud, poses, trace_total, trace_l1); cloud/poses are new arrays."""
    cc = _alloc_c_cloud(cloud)
    imgs = [np.ascontiguousarray(im, np.float64) for im in images]
    ptrs = (C.c_void_p * len(imgs))(*[im.ctypes.data for im in imgs])
    P = np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, 12)).copy()
    tt, tl = np.zeros(cfg.iterations), np.zeros(cfg.iterations)
    st = _L().orc_joint_optimize(C.byref(cc), C.cast(ptrs, C.c_void_p), len(imgs), intr[0], intr[1], intr[2],
                                  intr[3], width, height, _p(P), C.byref(cfg), slots, C.byref(rng), _p(tt), _p(tl))
    out = _from_c_cloud(cc)
    _L().orc_cloud_free(C.byref(cc))
    return st, out, P, tt, tl


# ---------------------------------------------------------- bootstrap
def fit_config(steps=100, unproject_points=50000, **kw) -> FitCfg:
    """TrainConfig defaults of fit_frame_gaussians (trainer.hpp:21-60)."""
    c = FitCfg()
    c.steps, c.unproject_points = steps, unproject_points
    c.pos_lr_start, c.pos_lr_end, c.rot_lr, c.scale_lr = 1.6e-2, 1.6e-4, 1e-3, 5e-3
    c.opacity_lr, c.sh_dc_lr, c.sh_rest_lr, c.beta = 5e-2, 2.5e-3, 2.5e-3 / 20.0, 0.2
    c.raster = default_raster_config()
    for k, v in kw.items():
        if k == "background":
            for i in range(3):
                c.background[i] = v[i]
        else:
            setattr(c, k, v)
    return c


def relpose_config(steps=200, **kw) -> RelposeCfg:
    """TrainConfig / LossConfig defaults of estimate_relative_pose (trainer.hpp:43-45, losses.hpp:19)."""
    c = RelposeCfg()
    c.steps, c.lr_start, c.lr_end, c.beta, c.mask_threshold = steps, 1e-3, 1e-4, 0.2, 0.99
    c.raster = default_raster_config()
    for k, v in kw.items():
        if k == "background":
            for i in range(3):
                c.background[i] = v[i]
        else:
            setattr(c, k, v)
    return c


def masked_rgb_loss(rendered, target, mask, beta=0.2, want_grad=True):
    """losses.cpp:273-289; raises OracleError(5) on an empty mask."""
    r = np.ascontiguousarray(rendered, np.float64)
    t = np.ascontiguousarray(target, np.float64)
    m = np.ascontiguousarray(mask, np.uint8).reshape(-1)
    d = np.zeros_like(r) if want_grad else None
    st = C.c_int32()
    loss = _L().orc_masked_rgb_loss(_p(r), _p(t), r.shape[1], r.shape[0], _p(m), beta,
                                     _p(d) if d is not None else None, C.byref(st))
    if st.value:
        raise OracleError(st.value, "masked_l1: no pixel passes the mask")
    return (loss, d) if want_grad else loss


def unproject(depth, valid, frame, intr, R, t, max_points):
    dep = np.ascontiguousarray(depth, np.float64)
    val = np.ascontiguousarray(valid, np.uint8)
    img = np.ascontiguousarray(frame, np.float64)
    H, W = dep.shape
    pts, cols = np.zeros((max_points, 3)), np.zeros((max_points, 3))
    Rm = np.ascontiguousarray(R, np.float64).reshape(9)
    tv = np.ascontiguousarray(t, np.float64).reshape(3)
    n = _L().orc_unproject(_p(dep), _p(val), W, H, _p(img), intr[0], intr[1], intr[2], intr[3], _p(Rm), _p(tv),
                            max_points, _p(pts), _p(cols))
    if n < 0:
        raise OracleError(3, "unproject: empty validity mask")
    return pts[:n].copy(), cols[:n].copy()


def mean_knn_distance(points, k=3):
    p = np.ascontiguousarray(points, np.float64)
    out = np.zeros(p.shape[0])
    _L().orc_mean_knn_distance(_p(p), p.shape[0], k, _p(out))
    return out


def init_from_points(points, colors, sh_degree=0) -> HostCloud:
    p = np.ascontiguousarray(points, np.float64)
    c = np.ascontiguousarray(colors, np.float64)
    out = Cloud()
    _L().orc_init_from_points(_p(p), _p(c), p.shape[0], sh_degree, C.byref(out))
    res = _from_c_cloud(out)
    _L().orc_cloud_free(C.byref(out))
    return res


def fit_frame_gaussians(frame, depth, valid, intr, cfg: FitCfg) -> HostCloud:
    img = np.ascontiguousarray(frame, np.float64)
    dep = np.ascontiguousarray(depth, np.float64)
    val = np.ascontiguousarray(valid, np.uint8)
    out = Cloud()
    st = _L().orc_fit_frame_gaussians(_p(img), _p(dep), _p(val), img.shape[1], img.shape[0], intr[0], intr[1],
                                       intr[2], intr[3], C.byref(cfg), C.byref(out))
    if st:
        raise OracleError(3, "unproject: empty validity mask")
    res = _from_c_cloud(out)
    _L().orc_cloud_free(C.byref(out))
    return res


def estimate_relative_pose(cloud: HostCloud, frame_next, intr, cfg: RelposeCfg):
    """-> (pose12, ok, final_loss)."""
    cv = cloud.c()
    img = np.ascontiguousarray(frame_next, np.float64)
    R, t, fl = np.zeros(9), np.zeros(3), C.c_double()
    ok = _L().orc_estimate_relative_pose(cv.ref(), _p(img), img.shape[1], img.shape[0], intr[0], intr[1], intr[2],
                                          intr[3], C.byref(cfg), _p(R), _p(t), C.byref(fl))
    return pose_join(R.reshape(3, 3), t), bool(ok), fl.value


def bootstrap_trajectory(frames, depths, valids, intr, fit: FitCfg, rel: RelposeCfg):
    n = len(frames)
    fr = [np.ascontiguousarray(f, np.float64) for f in frames]
    de = [np.ascontiguousarray(d, np.float64) for d in depths]
    va = [np.ascontiguousarray(v, np.uint8) for v in valids]
    arr = lambda xs: C.cast((C.c_void_p * n)(*[x.ctypes.data for x in xs]), C.c_void_p)  # noqa: E731
    poses, ok = np.zeros((n, 12)), np.zeros(max(n - 1, 1), np.int32)
    st = _L().orc_bootstrap_trajectory(arr(fr), arr(de), arr(va), n, fr[0].shape[1], fr[0].shape[0], intr[0],
                                        intr[1], intr[2], intr[3], C.byref(fit), C.byref(rel), _p(poses), _p(ok))
    if st:
        raise OracleError(3, "unproject: empty validity mask")
    return poses, ok[:n - 1].astype(bool)


# --------------------------------------------------------------- gradcheck
def make_gradcheck_scene(rng: Rng, n, image_size):
    cc = Cloud()
    cam = Camera()
    bg = np.zeros(3)
    _L().orc_make_gradcheck_scene(C.byref(rng), n, image_size, C.byref(cc), C.byref(cam), _p(bg))
    hc = _from_c_cloud(cc)
    _L().orc_cloud_free(C.byref(cc))
    return hc, cam, bg


def scene_is_conditioned(cloud: HostCloud, cam: Camera, bg, cfg=None) -> bool:
    cfg = cfg or default_raster_config()
    bgv = np.ascontiguousarray(bg, np.float64)
    return bool(_L().orc_scene_is_conditioned(cloud.c().ref(), C.byref(cam), _p(bgv), C.byref(cfg)))


def make_conditioned_scene(rng: Rng, n, image_size, cfg=None, max_attempts=64):
    for _ in range(max_attempts):
        sc = make_gradcheck_scene(rng, n, image_size)
        if scene_is_conditioned(*sc, cfg=cfg):
            return sc
    raise RuntimeError("make_conditioned_scene: rejection sampling failed")


def gradcheck(cloud: HostCloud, cam: Camera, bg, rng: Rng, cfg=None, step=1e-5):
    cfg = cfg or default_raster_config()
    bgv = np.ascontiguousarray(bg, np.float64)
    checked = C.c_int32()
    label = C.create_string_buffer(32)
    err = _L().orc_gradcheck(cloud.c().ref(), C.byref(cam), _p(bgv), C.byref(cfg), C.byref(rng), step,
                              C.byref(checked), label)
    return err, checked.value, label.value.decode()


def count_work(rr: RenderResult, d_image=None):
    """(H_f, C_f, H_b, C_b) for the roofline's algorithmic FLOPs."""
    assert rr._ptr is not None, "render(..., keep_handle=True) required"
    out = np.zeros(4, np.int64)
    d = None if d_image is None else np.ascontiguousarray(d_image, np.float64)
    _L().orc_count_work(rr._ptr, _p(d) if d is not None else None, _p(out))
    return tuple(int(v) for v in out)


def decision_margin(rr: RenderResult) -> np.ndarray:
    """Per-pixel relative margin (H, W) of the FP64 forward's discrete decisions
    (cutoff test, early termination): pixels above a threshold cannot flip in FP32."""
    m = np.zeros(rr.image.shape[0] * rr.image.shape[1])
    lib().orc_decision_margin(rr._ptr, _p(m))
    return m.reshape(rr.image.shape[:2])


def num_threads() -> int:
    return _L().orc_num_threads()
