"""Host-side Python mirror of the reference's hot-path API over libgsb200.so.

The functions mirror gsopt's C++ interface for the pose-gradient path
(/root/reference/proj/include/gsopt/rasterizer.hpp:98-113, losses.hpp:37,
trainer.hpp:85-100, trainer.hpp:170-171): same names, same argument meaning,
same error behaviour (``GsbError`` carries the reference ``ErrorCode`` + 1).
Every call goes through the C ABI declared in include/gsb200.h; there is no
CPU implementation behind any of them — without the built library or without
a B200 the calls raise instead of falling back.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libgsb200.so")

# include/gsb200.h status codes
OK = 0
ERR_DEGENERATE_CLOUD = 2
ERR_NO_VALID_DEPTH = 3
ERR_EMPTY_MASK = 5
ERR_STATE_MISMATCH = 6
ERR_MISSING_INTRINSICS = 7
ERR_CORRUPT_FILE = 9
ERR_DIMENSION_MISMATCH = 4
ERR_DIVERGED = 10
ERR_INVALID_CONFIG = 11
ERR_CUDA = 100
ERR_INVALID_ARGUMENT = 101
ERR_NO_DEVICE = 103
BWD_POSE_ONLY = 1
BWD_FAST_ATOMIC = 2

_ERR_NAMES = {1: "angle_near_pi", 2: "degenerate_cloud", 3: "no_valid_depth", 4: "dimension_mismatch",
              5: "empty_mask", 6: "state_mismatch", 7: "missing_intrinsics", 8: "image_size_mismatch",
              9: "corrupt_file", 10: "diverged", 11: "invalid_config", 100: "cuda", 101: "invalid_argument",
              102: "out_of_memory", 103: "no_device"}


class GsbError(RuntimeError):
    """gsopt::Error equivalent (core.hpp:49-52): ``code`` is the C ABI status."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{_ERR_NAMES.get(code, code)}] {msg}")
        self.code = code


class Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("R", C.c_double * 9), ("t", C.c_double * 3)]

    @staticmethod
    def make(fx, fy, cx, cy, width, height, R=None, t=None) -> "Camera":
        c = Camera()
        c.fx, c.fy, c.cx, c.cy, c.width, c.height = fx, fy, cx, cy, width, height
        R = np.eye(3) if R is None else np.asarray(R, np.float64)
        t = np.zeros(3) if t is None else np.asarray(t, np.float64)
        c.R[:] = [float(v) for v in R.reshape(9)]
        c.t[:] = [float(v) for v in t.reshape(3)]
        return c

    @staticmethod
    def from_pose12(fx, fy, cx, cy, width, height, pose12) -> "Camera":
        p = np.asarray(pose12, np.float64).reshape(3, 4)
        return Camera.make(fx, fy, cx, cy, width, height, p[:, :3], p[:, 3])

    def pose12(self) -> np.ndarray:
        return np.concatenate([np.array(self.R[:]).reshape(3, 3), np.array(self.t[:]).reshape(3, 1)], 1).reshape(12)


class RasterConfig(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("cutoff_sigma", C.c_double), ("alpha_clamp", C.c_double),
                ("dilation", C.c_double), ("early_termination", C.c_double), ("z_near", C.c_double),
                ("deterministic", C.c_int32)]

    @staticmethod
    def default(**kw) -> "RasterConfig":
        c = RasterConfig()
        lib().gsb_default_raster_config(C.byref(c))
        for k, v in kw.items():
            setattr(c, k, v)
        return c


class PoseAdam(C.Structure):
    _fields_ = [("m", C.c_double * 6), ("v", C.c_double * 6), ("step", C.c_int64)]


class FrameInfo(C.Structure):
    _fields_ = [("n_gaussians", C.c_int64), ("n_splats", C.c_int64), ("n_entries", C.c_int64),
                ("width", C.c_int32), ("height", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("state_fingerprint", C.c_uint64), ("binning", C.c_int32), ("reserved", C.c_int32)]


class PoseConfig(C.Structure):
    _fields_ = [("cam_lr_start", C.c_double), ("cam_lr_end", C.c_double), ("beta", C.c_double),
                ("pose_converged_eps", C.c_double), ("background", C.c_double * 3), ("raster", RasterConfig),
                ("budget", C.c_int32)]

    @staticmethod
    def default(**kw) -> "PoseConfig":
        c = PoseConfig()
        lib().gsb_default_pose_config(C.byref(c))
        for k, v in kw.items():
            if k == "background":
                c.background[:] = list(v)
            else:
                setattr(c, k, v)
        return c


_lib = None
_vp = C.c_void_p


class JointConfig(C.Structure):
    """gsb_joint_config: the TrainConfig fields joint_optimize reads (trainer.hpp:21-60)."""
    _fields_ = [("iterations", C.c_int32), ("cam_lr_start", C.c_double), ("cam_lr_end", C.c_double),
                ("pos_lr_start", C.c_double), ("pos_lr_end", C.c_double), ("rot_lr", C.c_double),
                ("scale_lr", C.c_double), ("opacity_lr", C.c_double), ("sh_dc_lr", C.c_double),
                ("sh_rest_lr", C.c_double), ("opacity_l1_steps", C.c_int32), ("sh_degree", C.c_int32),
                ("sh_degree_interval", C.c_int32), ("optimize_poses", C.c_int32), ("beta", C.c_double),
                ("aniso_ratio", C.c_double), ("opacity_l1_weight", C.c_double), ("background", C.c_double * 3),
                ("raster", RasterConfig), ("densify_interval", C.c_int32), ("densify_start", C.c_int32),
                ("densify_stop", C.c_int32), ("n_target", C.c_int32), ("grad_threshold", C.c_double),
                ("densify_size_ratio", C.c_double), ("prune_opacity", C.c_double)]

    @staticmethod
    def default(**kw) -> "JointConfig":
        c = JointConfig()
        lib().gsb_default_joint_config(C.byref(c))
        for k, v in kw.items():
            if k == "background":
                for i in range(3):
                    c.background[i] = v[i]
            else:
                setattr(c, k, v)
        return c


class BootstrapConfig(C.Structure):
    """gsb_bootstrap_config: the TrainConfig / LossConfig knobs of the bootstrap path
    (trainer.hpp:21-60, losses.hpp:19)."""
    _fields_ = [("per_frame_fit_steps", C.c_int32), ("relpose_steps", C.c_int32), ("unproject_points", C.c_int32),
                ("pos_lr_start", C.c_double), ("pos_lr_end", C.c_double), ("rot_lr", C.c_double),
                ("scale_lr", C.c_double), ("opacity_lr", C.c_double), ("sh_dc_lr", C.c_double),
                ("sh_rest_lr", C.c_double), ("relpose_lr_start", C.c_double), ("relpose_lr_end", C.c_double),
                ("beta", C.c_double), ("mask_threshold", C.c_double), ("background", C.c_double * 3),
                ("raster", RasterConfig)]

    @staticmethod
    def default(**kw) -> "BootstrapConfig":
        c = BootstrapConfig()
        lib().gsb_default_bootstrap_config(C.byref(c))
        for k, v in kw.items():
            if k == "background":
                for i in range(3):
                    c.background[i] = v[i]
            else:
                setattr(c, k, v)
        return c


def _sigs():
    P = C.POINTER
    d, i32, i64, u32, u64 = C.c_double, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
    return {
        "gsb_last_error": (C.c_char_p, []),
        "gsb_version": (C.c_char_p, []),
        "gsb_default_raster_config": (None, [P(RasterConfig)]),
        "gsb_default_pose_config": (None, [P(PoseConfig)]),
        "gsb_ctx_create": (C.c_int, [i32, P(_vp)]),
        "gsb_ctx_destroy": (C.c_int, [_vp]),
        "gsb_ctx_synchronize": (C.c_int, [_vp]),
        "gsb_ctx_set_profiling": (C.c_int, [_vp, i32]),
        "gsb_ctx_set_binning": (C.c_int, [_vp, i32]),
        "gsb_ctx_stage_times": (C.c_int, [_vp, _vp, _vp, i32]),
        "gsb_ctx_launch_count": (i64, [_vp]),
        "gsb_measure_fp32_peaks": (C.c_int, [i32, P(d), P(d)]),
        "gsb_build_id": (C.c_char_p, []),
        "gsb_cloud_create": (C.c_int, [_vp, i64, i32, P(_vp)]),
        "gsb_cloud_destroy": (C.c_int, [_vp]),
        "gsb_cloud_upload": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, i32]),
        "gsb_cloud_download": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
        "gsb_cloud_info": (C.c_int, [_vp, _vp, _vp, _vp]),
        "gsb_cloud_set_active_sh_degree": (C.c_int, [_vp, i32]),
        "gsb_cloud_synth": (C.c_int, [_vp, u64, d]),
        "gsb_synth_poses": (C.c_int, [u64, i64, i32, i32, i32, d, d, _vp]),
        "gsb_perturb_pose": (C.c_int, [_vp, d, d, P(u64), _vp]),
        "gsb_frame_create": (C.c_int, [_vp, P(_vp)]),
        "gsb_frame_destroy": (C.c_int, [_vp]),
        "gsb_render": (C.c_int, [_vp, _vp, P(Camera), _vp, P(RasterConfig), _vp, _vp]),
        "gsb_frame_get_info": (C.c_int, [_vp, P(FrameInfo)]),
        "gsb_state_fingerprint": (C.c_int, [_vp, P(Camera), P(C.c_uint64)]),
        "gsb_frame_download": (C.c_int, [_vp] + [_vp] * 15),
        "gsb_rgb_loss": (C.c_int, [_vp, _vp, _vp, i32, i32, d, P(d), _vp]),
        "gsb_image_create": (C.c_int, [_vp, _vp, i32, i32, P(_vp)]),
        "gsb_image_destroy": (C.c_int, [_vp]),
        "gsb_frame_rgb_loss": (C.c_int, [_vp, _vp, _vp, d, P(d)]),
        "gsb_grads_create": (C.c_int, [_vp, _vp, P(_vp)]),
        "gsb_grads_destroy": (C.c_int, [_vp]),
        "gsb_grads_download": (C.c_int, [_vp] + [_vp] * 7),
        "gsb_render_backward": (C.c_int, [_vp, _vp, P(Camera), _vp, _vp, i32, i32, u32, _vp, _vp]),
        "gsb_render_backward_device": (C.c_int, [_vp, _vp, P(Camera), _vp, u32, _vp, _vp]),
        "gsb_render_backward_image": (C.c_int, [_vp, _vp, P(Camera), _vp, _vp, u32, _vp, _vp]),
        "gsb_schedule": (d, [i32, d, d, i64, i64]),
        "gsb_pose_step": (C.c_int, [_vp, _vp, _vp, d, P(PoseAdam), _vp, _vp]),
        "gsb_adam_step": (C.c_int, [_vp, _vp, _vp, _vp, _vp, P(i64), i64, d]),
        "gsb_adam_step_lrs": (C.c_int, [_vp, _vp, _vp, _vp, _vp, P(i64), i64, _vp]),
        "gsb_adam_create": (C.c_int, [_vp, _vp, P(_vp)]),
        "gsb_adam_destroy": (C.c_int, [_vp]),
        "gsb_cloud_adam_step": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
        "gsb_estimate_pose": (C.c_int, [_vp, _vp, _vp, _vp, _vp, P(PoseConfig), _vp, P(d), P(i32), P(i32), _vp, _vp]),
        "gsb_ctx_timer_start": (C.c_int, [_vp]),
        "gsb_ctx_timer_stop": (C.c_int, [_vp, P(d)]),
        "gsb_session_create": (C.c_int, [_vp, _vp, _vp, _vp, _vp, P(PoseConfig), P(_vp)]),
        "gsb_session_destroy": (C.c_int, [_vp]),
        "gsb_session_step": (C.c_int, [_vp, _vp, i32]),
        "gsb_session_read": (C.c_int, [_vp, _vp, _vp, P(d), P(i32), P(i32), P(i32)]),
        "gsb_session_frame_info": (C.c_int, [_vp, P(FrameInfo)]),
        "gsb_session_step_async": (C.c_int, [_vp, _vp, i32]),
        "gsb_session_stage_times": (C.c_int, [_vp, _vp]),
        "gsb_pose_batch_create": (C.c_int, [_vp, _vp, i32, P(_vp)]),
        "gsb_pose_batch_destroy": (C.c_int, [_vp]),
        "gsb_pose_batch_step": (C.c_int, [_vp, _vp, i32]),
        "gsb_pose_batch_step_async": (C.c_int, [_vp, _vp, i32]),
        "gsb_pose_batch_sync": (C.c_int, [_vp, _vp]),
        "gsb_pose_batch_discarded": (C.c_int, [_vp, P(i64)]),
        "gsb_estimate_poses": (C.c_int, [_vp, _vp, _vp, _vp, _vp, i32, P(PoseConfig), _vp, _vp, _vp]),
        "gsb_comm_unique_id": (C.c_int, [_vp]),
        "gsb_comm_create": (C.c_int, [_vp, _vp, i32, i32, P(_vp)]),
        "gsb_comm_destroy": (C.c_int, [_vp]),
        "gsb_comm_allreduce_f32": (C.c_int, [_vp, _vp, i64]),
        "gsb_default_joint_config": (None, [P(JointConfig)]),
        "gsb_joint_schedule": (C.c_int, [u64, i32, i64, _vp]),
        "gsb_joint_rng_state": (C.c_int, [_vp, P(u64)]),
        "gsb_render_expected_depth": (C.c_int, [_vp, _vp, P(Camera), _vp, _vp, _vp]),
        "gsb_joint_create": (C.c_int, [_vp, _vp, _vp, i32, _vp, _vp, P(JointConfig), u64, i32, _vp, P(_vp)]),
        "gsb_joint_destroy": (C.c_int, [_vp]),
        "gsb_joint_step": (C.c_int, [_vp, _vp, i32]),
        "gsb_joint_read": (C.c_int, [_vp, _vp, P(i64), _vp, _vp]),
        "gsb_joint_info": (C.c_int, [_vp, P(i64), P(i32), _vp]),
        "gsb_perturb_pose_tangent": (C.c_int, [_vp, d, P(u64), _vp]),
        "gsb_cloud_jitter": (C.c_int, [_vp, u64, d, d]),
        "gsb_densify_and_prune": (C.c_int, [_vp, _vp, _vp, _vp, d, d, i32, d, P(u64), _vp, _vp]),
        "gsb_rng_child_normals": (C.c_int, [P(u64), i64, _vp]),
        "gsb_rng_shuffle": (C.c_int, [P(u64), i32, _vp]),
        "gsb_cloud_load_ply": (C.c_int, [_vp, C.c_char_p, P(_vp)]),
        "gsb_cloud_save_ply": (C.c_int, [_vp, C.c_char_p]),
        "gsb_load_float_map": (C.c_int, [C.c_char_p, _vp, i64, P(i32), P(i32)]),
        "gsb_save_float_map": (C.c_int, [_vp, i32, i32, C.c_char_p, d]),
        "gsb_load_depth_map": (C.c_int, [C.c_char_p, _vp, _vp, i64, P(i32), P(i32)]),
        "gsb_save_poses_json": (C.c_int, [_vp, i32, C.c_char_p]),
        "gsb_load_poses_json": (C.c_int, [C.c_char_p, _vp, i32, P(i32)]),
        "gsb_load_cameras_json": (C.c_int, [C.c_char_p, _vp, _vp, _vp, i32, P(i32), P(i32), C.c_char_p, i64]),
        "gsb_masked_rgb_loss": (C.c_int, [_vp, _vp, _vp, i32, i32, _vp, d, P(d), _vp]),
        "gsb_frame_masked_rgb_loss": (C.c_int, [_vp, _vp, _vp, d, d, P(d), P(i64)]),
        "gsb_default_bootstrap_config": (None, [P(BootstrapConfig)]),
        "gsb_unproject": (C.c_int, [_vp, _vp, i32, i32, _vp, _vp, _vp, i32, _vp, _vp, P(i64)]),
        "gsb_init_from_points": (C.c_int, [_vp, _vp, _vp, i64, i32, P(_vp)]),
        "gsb_fit_frame_gaussians": (C.c_int, [_vp, _vp, _vp, _vp, i32, i32, _vp, P(BootstrapConfig), P(_vp)]),
        "gsb_estimate_relative_pose": (C.c_int, [_vp, _vp, _vp, i32, i32, _vp, P(BootstrapConfig), _vp, P(i32),
                                                 P(d)]),
        "gsb_bootstrap_trajectory": (C.c_int, [_vp, _vp, _vp, _vp, i32, i32, i32, _vp, P(BootstrapConfig), _vp,
                                               _vp]),
    }


def lib():
    """Loads libgsb200.so (built in-tree by __graft_entry__.build()). Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GsbError(ERR_NO_DEVICE, f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _sigs().items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        raise GsbError(rc, lib().gsb_last_error().decode())


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays must be C contiguous"
    return a.ctypes.data_as(_vp)


# ----------------------------------------------------------------- objects
class Context:
    """One device + one CUDA stream (gsb_ctx)."""

    def __init__(self, device: int = 0):
        h = _vp()
        _check(lib().gsb_ctx_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().gsb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(lib().gsb_ctx_synchronize(self.h))

    BINNING_TILE_LOCAL = 0
    BINNING_GLOBAL = 1

    def set_binning(self, mode: int):
        """K2 strategy: BINNING_TILE_LOCAL (default) or BINNING_GLOBAL."""
        _check(lib().gsb_ctx_set_binning(self.h, int(mode)))

    def set_profiling(self, on: bool):
        _check(lib().gsb_ctx_set_profiling(self.h, 1 if on else 0))

    STAGES = ("preprocess", "sort", "composite", "loss", "bwd_raster", "bwd_geom", "optim", "other")

    def stage_times(self, reset=True):
        ms = np.zeros(8)
        cnt = np.zeros(8, np.int64)
        _check(lib().gsb_ctx_stage_times(self.h, _p(ms), _p(cnt), 1 if reset else 0))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(self.STAGES)}

    def launch_count(self) -> int:
        return int(lib().gsb_ctx_launch_count(self.h))

    def timer_start(self):
        _check(lib().gsb_ctx_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_double()
        _check(lib().gsb_ctx_timer_stop(self.h, C.byref(ms)))
        return ms.value


class Cloud:
    """GaussianCloud (scene.hpp:22-46), FP32 planes on the device."""

    def __init__(self, ctx: Context, n: int, sh_degree: int):
        h = _vp()
        _check(lib().gsb_cloud_create(ctx.h, n, sh_degree, C.byref(h)))
        self.h, self.ctx, self.n, self.sh_degree = h, ctx, n, sh_degree

    def __del__(self):
        try:
            if self.h:
                lib().gsb_cloud_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @staticmethod
    def from_host(ctx: Context, means, rotations, log_scales, opacity_logits, sh, sh_degree, active_sh_degree=None):
        n = int(np.asarray(means).shape[0])
        c = Cloud(ctx, n, sh_degree)
        c.upload(means, rotations, log_scales, opacity_logits, sh,
                 sh_degree if active_sh_degree is None else active_sh_degree)
        return c

    def upload(self, means, rotations, log_scales, opacity_logits, sh, active_sh_degree):
        arrs = [np.ascontiguousarray(a, np.float64) for a in (means, rotations, log_scales, opacity_logits, sh)]
        _check(lib().gsb_cloud_upload(self.h, *[_p(a) for a in arrs], int(active_sh_degree)))

    def download(self):
        n, b = self.n, (self.sh_degree + 1) ** 2
        out = [np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3, b))]
        _check(lib().gsb_cloud_download(self.h, *[_p(a) for a in out]))
        return out

    @staticmethod
    def load_ply(ctx: Context, path: str) -> "Cloud":
        """load_cloud_ply (src/ply.cpp:62-148) straight into the device layout."""
        h = _vp()
        _check(lib().gsb_cloud_load_ply(ctx.h, os.fsencode(path), C.byref(h)))
        return Cloud._wrap(ctx, h)

    @staticmethod
    def _wrap(ctx: Context, h) -> "Cloud":
        c = Cloud.__new__(Cloud)
        c.h, c.ctx = h, ctx
        n, dd, ad = C.c_int64(), C.c_int32(), C.c_int32()
        _check(lib().gsb_cloud_info(h, C.byref(n), C.byref(dd), C.byref(ad)))
        c.n, c.sh_degree = n.value, dd.value
        return c

    def save_ply(self, path: str):
        """save_cloud_ply (src/ply.cpp:29-60)."""
        _check(lib().gsb_cloud_save_ply(self.h, os.fsencode(path)))

    def refresh(self):
        """Re-reads the size (changed by densify_and_prune on the device)."""
        n, dd, ad = C.c_int64(), C.c_int32(), C.c_int32()
        _check(lib().gsb_cloud_info(self.h, C.byref(n), C.byref(dd), C.byref(ad)))
        self.n = n.value

    def jitter(self, seed: int, mean_sigma: float, log_scale_range: float = 0.0):
        """tests/test_trainer.cpp:598-601 initial-cloud jitter (gsb_cloud_jitter)."""
        _check(lib().gsb_cloud_jitter(self.h, seed, mean_sigma, log_scale_range))

    def synth(self, seed: int, log_scale_offset: float = 0.0):
        _check(lib().gsb_cloud_synth(self.h, seed, log_scale_offset))

    def set_active_sh_degree(self, d: int):
        _check(lib().gsb_cloud_set_active_sh_degree(self.h, d))


@dataclass
class RenderOutput:
    """RenderOutput (rasterizer.hpp:66-82) with its device-resident forward state."""
    frame: "Frame"
    image: np.ndarray | None

    def info(self) -> FrameInfo:
        return self.frame.info()

    def download(self):
        return self.frame.download()


class Frame:
    def __init__(self, ctx: Context):
        h = _vp()
        _check(lib().gsb_frame_create(ctx.h, C.byref(h)))
        self.h, self.ctx = h, ctx

    def __del__(self):
        try:
            if self.h:
                lib().gsb_frame_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def info(self) -> FrameInfo:
        fi = FrameInfo()
        _check(lib().gsb_frame_get_info(self.h, C.byref(fi)))
        return fi

    def download(self) -> dict:
        fi = self.info()
        P, V, K, T = fi.width * fi.height, fi.n_splats, fi.n_entries, fi.tiles_x * fi.tiles_y
        o = dict(image=np.zeros((fi.height, fi.width, 3)), accum_transmittance=np.zeros(P),
                 final_transmittance=np.zeros(P), contrib_count=np.zeros(P, np.int32),
                 overflow_mask=np.zeros(P, np.uint8), splat_gaussian=np.zeros(V, np.int32),
                 splat_mu2d=np.zeros((V, 2)), splat_depth=np.zeros(V), splat_conic=np.zeros((V, 4)),
                 splat_color=np.zeros((V, 3)), splat_opacity=np.zeros(V), splat_radius=np.zeros(V),
                 splat_clamped=np.zeros(V, np.uint8), tile_lists=np.zeros(K, np.int32),
                 tile_ranges=np.zeros((T, 2), np.int32))
        keys = ["image", "accum_transmittance", "final_transmittance", "contrib_count", "overflow_mask",
                "splat_gaussian", "splat_mu2d", "splat_depth", "splat_conic", "splat_color", "splat_opacity",
                "splat_radius", "splat_clamped", "tile_lists", "tile_ranges"]
        _check(lib().gsb_frame_download(self.h, *[_p(o[k]) for k in keys]))
        o.update(tiles_x=fi.tiles_x, tiles_y=fi.tiles_y, fingerprint=fi.state_fingerprint)
        return o


class Grads:
    """GradientBundle (rasterizer.hpp:84-94), device resident."""

    def __init__(self, ctx: Context, cloud: Cloud):
        h = _vp()
        _check(lib().gsb_grads_create(ctx.h, cloud.h, C.byref(h)))
        self.h, self.ctx, self.n, self.sh_degree = h, ctx, cloud.n, cloud.sh_degree

    def __del__(self):
        try:
            if self.h:
                lib().gsb_grads_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def download(self) -> dict:
        n, b = self.n, (self.sh_degree + 1) ** 2
        o = dict(d_means=np.zeros((n, 3)), d_rotations=np.zeros((n, 4)), d_log_scales=np.zeros((n, 3)),
                 d_opacity_logits=np.zeros(n), d_sh=np.zeros((n, 3, b)), d_mu2d=np.zeros((n, 2)), d_pose=np.zeros(6))
        keys = ["d_means", "d_rotations", "d_log_scales", "d_opacity_logits", "d_sh", "d_mu2d", "d_pose"]
        _check(lib().gsb_grads_download(self.h, *[_p(o[k]) for k in keys]))
        return o


class Image:
    """Device-resident target frame (H, W, 3)."""

    def __init__(self, ctx: Context, img: np.ndarray):
        img = np.ascontiguousarray(img, np.float64)
        h = _vp()
        _check(lib().gsb_image_create(ctx.h, _p(img), img.shape[1], img.shape[0], C.byref(h)))
        self.h, self.ctx, self.width, self.height = h, ctx, img.shape[1], img.shape[0]

    def __del__(self):
        try:
            if self.h:
                lib().gsb_image_destroy(self.h)
                self.h = None
        except Exception:
            pass


# -------------------------------------------------------- reference API
def render(ctx: Context, cloud: Cloud, cam: Camera, background=(0.0, 0.0, 0.0), config: RasterConfig | None = None,
           frame: Frame | None = None, want_image=True) -> RenderOutput:
    """gsopt::render (rasterizer.hpp:98-99)."""
    frame = frame or Frame(ctx)
    bg = np.ascontiguousarray(background, np.float64)
    img = np.zeros((cam.height, cam.width, 3)) if want_image else None
    cfg = config or RasterConfig.default()
    _check(lib().gsb_render(ctx.h, cloud.h, C.byref(cam), _p(bg), C.byref(cfg), frame.h, _p(img)))
    return RenderOutput(frame, img)


def state_fingerprint(cloud: Cloud, cam: Camera) -> int:
    """The RenderOutput::state_fingerprint render(cloud, cam) stamps
    (rasterizer.cpp:52-73), without rendering."""
    fp = C.c_uint64()
    _check(lib().gsb_state_fingerprint(cloud.h, C.byref(cam), C.byref(fp)))
    return int(fp.value)


def adam_step(ctx: Context, params, grads, m, v, step: int, lr) -> int:
    """gsopt::adam_step (trainer.hpp:85-87): params / m / v (FP64 arrays) updated in
    place; lr a scalar or a per-index array (the lr_of overload). Returns the new step."""
    st = C.c_int64(step)
    g = np.ascontiguousarray(grads, np.float64)
    for a in (params, m, v):
        assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    if np.ndim(lr) == 0:
        _check(lib().gsb_adam_step(ctx.h, _p(params), _p(g), _p(m), _p(v), C.byref(st), params.size, float(lr)))
    else:
        lrs = np.ascontiguousarray(lr, np.float64)
        _check(lib().gsb_adam_step_lrs(ctx.h, _p(params), _p(g), _p(m), _p(v), C.byref(st), params.size, _p(lrs)))
    return int(st.value)


def render_expected_depth(ctx: Context, cloud: Cloud, cam: Camera, config: RasterConfig | None = None):
    """gsopt::render_expected_depth (rasterizer.cpp:283-323): (depth, weight), each (H, W) float32."""
    cfg = config or RasterConfig.default()
    depth = np.zeros((cam.height, cam.width), np.float32)
    weight = np.zeros((cam.height, cam.width), np.float32)
    _check(lib().gsb_render_expected_depth(ctx.h, cloud.h, C.byref(cam), C.byref(cfg), _p(depth), _p(weight)))
    return depth, weight


def render_backward(ctx: Context, cloud: Cloud, cam: Camera, out: RenderOutput, d_image,
                    pose_only=False, grads: Grads | None = None):
    """gsopt::render_backward (rasterizer.hpp:112-113). d_image: host (H, W, 3)
    FP64 array, or an `Image` already on the device. Returns (grads dict | None, d_pose)."""
    flags = BWD_POSE_ONLY if pose_only else 0
    if not pose_only and grads is None:
        grads = Grads(ctx, cloud)
    dp = np.zeros(6)
    gh = grads.h if grads is not None else None
    if isinstance(d_image, Image):
        _check(lib().gsb_render_backward_image(ctx.h, cloud.h, C.byref(cam), out.frame.h, d_image.h, flags, gh,
                                               _p(dp)))
        return (grads.download() if (grads is not None and not pose_only) else None), dp
    d = np.ascontiguousarray(d_image, np.float64)
    h, w = (d.shape[0], d.shape[1]) if d.ndim == 3 else (0, 0)
    _check(lib().gsb_render_backward(ctx.h, cloud.h, C.byref(cam), out.frame.h, _p(d), w, h, flags, gh, _p(dp)))
    return (grads.download() if (grads is not None and not pose_only) else None), dp


def rgb_loss(ctx: Context, rendered: np.ndarray, target: np.ndarray, beta: float = 0.2, want_grad=True):
    """gsopt::rgb_loss (losses.hpp:37)."""
    r = np.ascontiguousarray(rendered, np.float64)
    t = np.ascontiguousarray(target, np.float64)
    if r.shape != t.shape:
        raise GsbError(ERR_DIMENSION_MISMATCH, "rgb_loss: image shapes differ")
    loss = C.c_double()
    d = np.zeros_like(r) if want_grad else None
    _check(lib().gsb_rgb_loss(ctx.h, _p(r), _p(t), r.shape[1], r.shape[0], beta, C.byref(loss), _p(d)))
    return (loss.value, d) if want_grad else loss.value


def schedule(kind: str, start: float, end: float, step: int, total: int) -> float:
    """gsopt::schedule (trainer.hpp:62-63)."""
    return lib().gsb_schedule(0 if kind == "cosine" else 1, start, end, step, total)


def pose_step(ctx: Context, pose12, d_pose, lr: float, state: PoseAdam):
    """gsopt::pose_step (trainer.hpp:99-100). Returns (pose12, applied_update)."""
    p = np.ascontiguousarray(pose12, np.float64).reshape(12)
    g = np.ascontiguousarray(d_pose, np.float64).reshape(6)
    out, ap = np.zeros(12), np.zeros(6)
    _check(lib().gsb_pose_step(ctx.h, _p(p), _p(g), lr, C.byref(state), _p(out), _p(ap)))
    return out, ap


def estimate_pose(ctx: Context, cloud: Cloud, target: Image, intr, init_pose12, config: PoseConfig | None = None,
                  trace=False):
    """gsopt::estimate_pose (trainer.hpp:170-171) = pose_descent (pipelines.cpp:58-92) on the device."""
    cfg = config or PoseConfig.default()
    intr = np.ascontiguousarray(intr, np.float64)
    init = np.ascontiguousarray(init_pose12, np.float64).reshape(12)
    out = np.zeros(12)
    fl, su, cv = C.c_double(), C.c_int32(), C.c_int32()
    tp = np.zeros((cfg.budget, 12)) if trace else None
    tl = np.zeros(cfg.budget) if trace else None
    _check(lib().gsb_estimate_pose(ctx.h, cloud.h, target.h, _p(intr), _p(init), C.byref(cfg), _p(out),
                                   C.byref(fl), C.byref(su), C.byref(cv), _p(tp), _p(tl)))
    res = dict(pose=out, final_loss=fl.value, steps=su.value, converged=bool(cv.value))
    if trace:
        res.update(trace_pose=tp[:su.value], trace_loss=tl[:su.value])
    return res


class PoseSession:
    """One view's device-resident pose_descent state (gsb_session)."""

    def __init__(self, ctx: Context, cloud: Cloud, target: Image, intr, init_pose12, config: PoseConfig | None = None):
        self.cfg = config or PoseConfig.default()
        intr = np.ascontiguousarray(intr, np.float64)
        init = np.ascontiguousarray(init_pose12, np.float64).reshape(12)
        h = _vp()
        _check(lib().gsb_session_create(ctx.h, cloud.h, target.h, _p(intr), _p(init), C.byref(self.cfg), C.byref(h)))
        self.h, self.ctx, self._keep = h, ctx, (cloud, target)

    def __del__(self):
        try:
            if self.h:
                lib().gsb_session_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def step(self, iterations: int = 1):
        _check(lib().gsb_session_step(self.ctx.h, self.h, iterations))

    def step_async(self, iterations: int = 1):
        _check(lib().gsb_session_step_async(self.ctx.h, self.h, iterations))

    def stage_times(self) -> dict:
        ms = np.zeros(8)
        _check(lib().gsb_session_stage_times(self.h, _p(ms)))
        return {k: float(ms[i]) for i, k in enumerate(Context.STAGES)}

    def read(self) -> dict:
        pose, best = np.zeros(12), np.zeros(12)
        fl, su, cv, st = C.c_double(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().gsb_session_read(self.h, _p(pose), _p(best), C.byref(fl), C.byref(su), C.byref(cv), C.byref(st)))
        return dict(pose=pose, best_pose=best, final_loss=fl.value, steps=su.value, converged=bool(cv.value),
                    stopped=bool(st.value))

    def frame_info(self) -> FrameInfo:
        fi = FrameInfo()
        _check(lib().gsb_session_frame_info(self.h, C.byref(fi)))
        return fi


def measure_fp32_peaks(device: int = 0) -> dict:
    """FFMA TFLOP/s and MUFU ex2 Tops/s of the device by microbenchmark (gsb_measure_fp32_peaks)."""
    f, m = C.c_double(), C.c_double()
    _check(lib().gsb_measure_fp32_peaks(device, C.byref(f), C.byref(m)))
    return {"ffma_tflops": f.value, "mufu_tops": m.value}


def build_id() -> str:
    return lib().gsb_build_id().decode()


class PoseBatch:
    """Several sessions advanced by one CUDA-graph replay per iteration (gsb_pose_batch)."""

    def __init__(self, ctx: Context, sessions):
        self.sessions = list(sessions)
        arr = (_vp * len(self.sessions))(*[s.h for s in self.sessions])
        h = _vp()
        _check(lib().gsb_pose_batch_create(ctx.h, arr, len(self.sessions), C.byref(h)))
        self.h, self.ctx = h, ctx

    def close(self):
        if self.h:
            lib().gsb_pose_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, iterations: int = 1):
        _check(lib().gsb_pose_batch_step(self.ctx.h, self.h, iterations))

    def step_async(self, iterations: int = 1):
        _check(lib().gsb_pose_batch_step_async(self.ctx.h, self.h, iterations))

    def sync(self):
        _check(lib().gsb_pose_batch_sync(self.ctx.h, self.h))

    def discarded(self) -> int:
        """Iterations discarded for entry-capacity growth (and re-run by sync) so far."""
        v = C.c_int64()
        _check(lib().gsb_pose_batch_discarded(self.h, C.byref(v)))
        return int(v.value)


def estimate_poses(ctx: Context, cloud: Cloud, targets, intr, init_poses, config: PoseConfig | None = None):
    """estimate_pose for several views of one cloud at once (gsb_estimate_poses)."""
    cfg = config or PoseConfig.default()
    intr = np.ascontiguousarray(intr, np.float64)
    init = np.ascontiguousarray(init_poses, np.float64).reshape(-1, 12)
    n = init.shape[0]
    assert len(targets) == n
    arr = (_vp * n)(*[t.h for t in targets])
    out, fl, su = np.zeros((n, 12)), np.zeros(n), np.zeros(n, np.int32)
    _check(lib().gsb_estimate_poses(ctx.h, cloud.h, arr, _p(intr), _p(init), n, C.byref(cfg), _p(out), _p(fl),
                                    _p(su)))
    return dict(pose=out, final_loss=fl, steps=su)


class Comm:
    """NCCL communicator for data-parallel joint training (gsb_comm). Rank 0
    creates the unique id; the caller distributes it (e.g. torch.distributed)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().gsb_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, uid: bytes, rank: int, world: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = _vp()
        _check(lib().gsb_comm_create(ctx.h, buf, rank, world, C.byref(h)))
        self.h, self.ctx, self.rank, self.world = h, ctx, rank, world

    def close(self):
        if self.h:
            lib().gsb_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def joint_schedule(seed: int, n_views: int, count: int) -> np.ndarray:
    """joint_optimize's training-view sequence (pipelines.cpp:122-129)."""
    out = np.zeros(count, np.int32)
    _check(lib().gsb_joint_schedule(seed, n_views, count, _p(out)))
    return out


class JointOptimizer:
    """joint_optimize (pipelines.cpp:96-216, densification off) on the device,
    `local_views` views per rank per step, data parallel over `comm`."""

    def __init__(self, ctx: Context, cloud: Cloud, targets, intr, init_poses, config: JointConfig, seed: int,
                 local_views: int = 1, comm: Comm | None = None):
        self.cfg = config
        intr = np.ascontiguousarray(intr, np.float64)
        init = np.ascontiguousarray(init_poses, np.float64).reshape(-1, 12)
        self.n_views = init.shape[0]
        arr = (_vp * self.n_views)(*[t.h for t in targets])
        h = _vp()
        _check(lib().gsb_joint_create(ctx.h, cloud.h, arr, self.n_views, _p(intr), _p(init), C.byref(config), seed,
                                      local_views, comm.h if comm else None, C.byref(h)))
        self.h, self.ctx, self._keep = h, ctx, (cloud, list(targets), comm)

    def close(self):
        if self.h:
            lib().gsb_joint_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rng_state(self) -> int:
        """The run's Rng state (gsb_joint_rng_state): continue the caller's Rng from it."""
        v = C.c_uint64()
        _check(lib().gsb_joint_rng_state(self.h, C.byref(v)))
        return int(v.value)

    def step(self, steps: int = 1):
        _check(lib().gsb_joint_step(self.ctx.h, self.h, steps))

    def read(self) -> dict:
        poses = np.zeros((self.n_views, 12))
        done = C.c_int64()
        tt, tl = np.zeros(max(self.cfg.iterations, 1)), np.zeros(max(self.cfg.iterations, 1))
        _check(lib().gsb_joint_read(self.h, _p(poses), C.byref(done), _p(tt), _p(tl)))
        n, ev, rep = C.c_int64(), C.c_int32(), np.zeros(3, np.int32)
        _check(lib().gsb_joint_info(self.h, C.byref(n), C.byref(ev), _p(rep)))
        self._keep[0].refresh()
        return dict(poses=poses, steps=done.value, trace_total=tt[:done.value], trace_l1=tl[:done.value],
                    n_gaussians=n.value, densify_events=ev.value, densify_report=tuple(int(x) for x in rep))


def densify_and_prune(ctx: Context, cloud: Cloud, grad_sum, count, grad_threshold=2e-4, densify_size_ratio=0.01,
                      n_target=256000, prune_opacity=0.005, rng: "PoseRng" = None, adam_handle=None):
    """gsopt::densify_and_prune (trainer.hpp:130-133) on the device; returns
    (cloned, split, pruned). The cloud's size changes in place."""
    gs = np.ascontiguousarray(grad_sum, np.float64)
    ct = np.ascontiguousarray(count, np.int32)
    rep = np.zeros(3, np.int32)
    _check(lib().gsb_densify_and_prune(ctx.h, cloud.h, _p(gs), _p(ct), grad_threshold, densify_size_ratio, n_target,
                                       prune_opacity, C.byref(rng.state), adam_handle, _p(rep)))
    cloud.refresh()
    return tuple(int(x) for x in rep)


def perturb_pose_tangent(pose12, sigma, state: "PoseRng"):
    p = np.ascontiguousarray(pose12, np.float64).reshape(12)
    out = np.zeros(12)
    _check(lib().gsb_perturb_pose_tangent(_p(p), sigma, C.byref(state.state), _p(out)))
    return out


def synth_poses(seed: int, n: int, sh_degree: int, kind: int, cameras: int, orbit_radius=2.5,
                orbit_arc=2 * np.pi) -> np.ndarray:
    out = np.zeros((cameras, 12))
    _check(lib().gsb_synth_poses(seed, n, sh_degree, kind, cameras, orbit_radius, orbit_arc, _p(out)))
    return out


class PoseRng:
    """Holds the xorshift64* state perturb_pose draws from (core.hpp:58-70)."""

    def __init__(self, seed: int):
        self.state = C.c_uint64(seed if seed else 0x9E3779B97F4A7C15)

    def perturb_pose(self, pose12, rot_deg, trans):
        p = np.ascontiguousarray(pose12, np.float64).reshape(12)
        out = np.zeros(12)
        _check(lib().gsb_perturb_pose(_p(p), rot_deg, trans, C.byref(self.state), _p(out)))
        return out


def synth_intrinsics(width: int, height: int):
    """synth.cpp:64-71: fx = fy = 0.75 W, c = (dim - 1) / 2."""
    return np.array([0.75 * width, 0.75 * width, 0.5 * (width - 1), 0.5 * (height - 1)])


# ------------------------------------------------------- bootstrap path
def masked_rgb_loss(ctx: Context, rendered: np.ndarray, target: np.ndarray, mask: np.ndarray, beta: float = 0.2,
                    want_grad=True):
    """gsopt::masked_rgb_loss (losses.cpp:273-289); mask: (H, W) or (H*W,) of 0/1."""
    r = np.ascontiguousarray(rendered, np.float64)
    t = np.ascontiguousarray(target, np.float64)
    if r.shape != t.shape:
        raise GsbError(ERR_DIMENSION_MISMATCH, "masked_rgb_loss: image shapes differ")
    m = np.ascontiguousarray(mask, np.uint8).reshape(-1)
    if m.size != r.shape[0] * r.shape[1]:
        raise GsbError(ERR_DIMENSION_MISMATCH, "masked_l1: mask size mismatch")
    loss = C.c_double()
    d = np.zeros_like(r) if want_grad else None
    _check(lib().gsb_masked_rgb_loss(ctx.h, _p(r), _p(t), r.shape[1], r.shape[0], _p(m), beta, C.byref(loss),
                                     _p(d)))
    return (loss.value, d) if want_grad else loss.value


def frame_masked_rgb_loss(ctx: Context, frame: Frame, target: Image, beta: float, threshold: float):
    """masked_rgb_loss(out.image, target, transmittance_mask(out.accum_transmittance, threshold))
    on the device; returns (loss, masked pixel count)."""
    loss, cnt = C.c_double(), C.c_int64()
    _check(lib().gsb_frame_masked_rgb_loss(ctx.h, frame.h, target.h, beta, threshold, C.byref(loss),
                                           C.byref(cnt)))
    return loss.value, cnt.value


def unproject(depth: np.ndarray, valid: np.ndarray, frame: np.ndarray, intr, world_to_cam12, max_points: int):
    """gsopt::unproject (scene.cpp:209-243) -> (points (n,3), colors (n,3))."""
    dep = np.ascontiguousarray(depth, np.float64)
    val = np.ascontiguousarray(valid, np.uint8)
    img = np.ascontiguousarray(frame, np.float64)
    H, W = dep.shape
    i4 = np.ascontiguousarray(intr, np.float64)
    pose = np.ascontiguousarray(world_to_cam12, np.float64).reshape(12)
    pts, cols, n = np.zeros((max(max_points, 1), 3)), np.zeros((max(max_points, 1), 3)), C.c_int64()
    _check(lib().gsb_unproject(_p(dep), _p(val), W, H, _p(img), _p(i4), _p(pose), max_points, _p(pts), _p(cols),
                               C.byref(n)))
    return pts[:n.value].copy(), cols[:n.value].copy()


def init_from_points(ctx: Context, points, colors, sh_degree: int = 0) -> Cloud:
    """gsopt::init_from_points (scene.cpp:182-207), kNN scales computed on the device."""
    p = np.ascontiguousarray(points, np.float64)
    c = np.ascontiguousarray(colors, np.float64)
    if p.shape != c.shape:
        raise GsbError(ERR_DIMENSION_MISMATCH, "init_from_points: points/colors size mismatch")
    h = _vp()
    _check(lib().gsb_init_from_points(ctx.h, _p(p), _p(c), p.shape[0], sh_degree, C.byref(h)))
    return Cloud._wrap(ctx, h)


def fit_frame_gaussians(ctx: Context, frame, depth, valid, intr, config: BootstrapConfig | None = None) -> Cloud:
    """gsopt::fit_frame_gaussians (pipelines.cpp:224-250)."""
    cfg = config or BootstrapConfig.default()
    img = np.ascontiguousarray(frame, np.float64)
    dep = np.ascontiguousarray(depth, np.float64)
    val = np.ascontiguousarray(valid, np.uint8)
    i4 = np.ascontiguousarray(intr, np.float64)
    h = _vp()
    _check(lib().gsb_fit_frame_gaussians(ctx.h, _p(img), _p(dep), _p(val), img.shape[1], img.shape[0], _p(i4),
                                         C.byref(cfg), C.byref(h)))
    return Cloud._wrap(ctx, h)


def estimate_relative_pose(ctx: Context, cloud: Cloud, frame_next, intr, config: BootstrapConfig | None = None):
    """gsopt::estimate_relative_pose (pipelines.cpp:252-290) -> (pose12, ok, final_loss)."""
    cfg = config or BootstrapConfig.default()
    img = np.ascontiguousarray(frame_next, np.float64)
    i4 = np.ascontiguousarray(intr, np.float64)
    pose, ok, fl = np.zeros(12), C.c_int32(), C.c_double()
    _check(lib().gsb_estimate_relative_pose(ctx.h, cloud.h, _p(img), img.shape[1], img.shape[0], _p(i4),
                                            C.byref(cfg), _p(pose), C.byref(ok), C.byref(fl)))
    return pose, bool(ok.value), fl.value


def bootstrap_trajectory(ctx: Context, frames, depths, valids, intr, config: BootstrapConfig | None = None):
    """gsopt::bootstrap_trajectory (pipelines.cpp:292-312) -> (world_to_cam (n,12), pair_ok (n-1,))."""
    cfg = config or BootstrapConfig.default()
    n = len(frames)
    if n < 2 or len(depths) != n or len(valids) != n:
        raise GsbError(ERR_INVALID_CONFIG, "bootstrap_trajectory: need >= 2 frames with depths")
    fr = [np.ascontiguousarray(f, np.float64) for f in frames]
    de = [np.ascontiguousarray(d, np.float64) for d in depths]
    va = [np.ascontiguousarray(v, np.uint8) for v in valids]
    arr = lambda xs: (C.c_void_p * n)(*[x.ctypes.data for x in xs])  # noqa: E731
    i4 = np.ascontiguousarray(intr, np.float64)
    poses, ok = np.zeros((n, 12)), np.zeros(n - 1, np.int32)
    _check(lib().gsb_bootstrap_trajectory(ctx.h, arr(fr), arr(de), arr(va), n, fr[0].shape[1], fr[0].shape[0],
                                          _p(i4), C.byref(cfg), _p(poses), _p(ok)))
    return poses, ok.astype(bool)


# ------------------------------------------------------- on-disk formats
def load_float_map(path: str) -> np.ndarray:
    """load_float_map (image.cpp:105-126) -> float32 (H, W)."""
    w, h = C.c_int32(), C.c_int32()
    _check(lib().gsb_load_float_map(os.fsencode(path), None, 0, C.byref(w), C.byref(h)))
    out = np.zeros((h.value, w.value), np.float32)
    _check(lib().gsb_load_float_map(os.fsencode(path), _p(out), out.size, C.byref(w), C.byref(h)))
    return out


def save_float_map(values, path: str, scale: float = 1.0):
    """save_float_map (image.cpp:128-141); values (H, W)."""
    v = np.ascontiguousarray(values, np.float32)
    _check(lib().gsb_save_float_map(_p(v), v.shape[1], v.shape[0], os.fsencode(path), scale))


def load_depth_map(path: str):
    """depth/<stem>.f32 as load_scene reads it -> (depth FP64 (H, W), valid uint8 (H, W))."""
    w, h = C.c_int32(), C.c_int32()
    _check(lib().gsb_load_depth_map(os.fsencode(path), None, None, 0, C.byref(w), C.byref(h)))
    dep, val = np.zeros((h.value, w.value)), np.zeros((h.value, w.value), np.uint8)
    _check(lib().gsb_load_depth_map(os.fsencode(path), _p(dep), _p(val), dep.size, C.byref(w), C.byref(h)))
    return dep, val


def save_poses_json(poses, path: str):
    """save_poses_json (scene_io.cpp:64-68); poses (n, 12) row-major [R|t]."""
    P_ = np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, 12))
    _check(lib().gsb_save_poses_json(_p(P_), P_.shape[0], os.fsencode(path)))


def load_poses_json(path: str) -> np.ndarray:
    """load_poses_json (scene_io.cpp:70-79) -> (n, 12)."""
    n = C.c_int32()
    _check(lib().gsb_load_poses_json(os.fsencode(path), None, 0, C.byref(n)))
    out = np.zeros((n.value, 12))
    _check(lib().gsb_load_poses_json(os.fsencode(path), _p(out), n.value, C.byref(n)))
    return out


def load_cameras_json(path: str) -> dict:
    """load_cameras_json (scene_io.cpp:254-279) -> dict(intrinsics, width, height, poses, names, has_poses)."""
    intr, size, n, hp = np.zeros(4), np.zeros(2, np.int32), C.c_int32(), C.c_int32()
    _check(lib().gsb_load_cameras_json(os.fsencode(path), _p(intr), _p(size), None, 0, C.byref(n), C.byref(hp),
                                       None, 0))
    poses = np.zeros((n.value, 12))
    cap = max(os.path.getsize(path) + 1, 1)
    names = C.create_string_buffer(cap)
    _check(lib().gsb_load_cameras_json(os.fsencode(path), _p(intr), _p(size), _p(poses), n.value, C.byref(n),
                                       C.byref(hp), names, cap))
    nm = names.value.decode()
    return dict(intrinsics=intr, width=int(size[0]), height=int(size[1]), poses=poses,
                names=nm.split("\n") if n.value else [], has_poses=bool(hp.value))
