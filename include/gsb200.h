/*
 * gsb200.h — C ABI of the B200-native pose-gradient Gaussian-splatting hot
 * path (libgsb200.so). Plain pointers and sizes only; no C++ or torch types.
 *
 * Drop-in boundary. Each entry point replaces one reference
 * interface (paths relative to /root/reference/proj):
 *
 *   gsb_render            <- gsopt::render            include/gsopt/rasterizer.hpp:98-99
 *   gsb_frame_download    <- RenderOutput fields       include/gsopt/rasterizer.hpp:66-82
 *   gsb_render_backward   <- gsopt::render_backward   include/gsopt/rasterizer.hpp:112-113
 *   gsb_render_expected_depth <- gsopt::render_expected_depth rasterizer.hpp:101-107
 *                            (src/rasterizer.cpp:283-323; dataset generation, synth.cpp:117-127)
 *   gsb_rgb_loss          <- gsopt::rgb_loss          include/gsopt/losses.hpp:37
 *   gsb_pose_step         <- gsopt::pose_step         include/gsopt/trainer.hpp:99-100
 *   gsb_adam_step         <- gsopt::adam_step (both)  include/gsopt/trainer.hpp:85-87
 *   gsb_cloud_adam_step   <- cloud_adam_step          src/pipelines.cpp:18-41
 *   gsb_schedule          <- gsopt::schedule          include/gsopt/trainer.hpp:62-63
 *   gsb_estimate_pose     <- gsopt::estimate_pose     include/gsopt/trainer.hpp:170-171
 *                            (pose_descent, src/pipelines.cpp:58-92, device resident)
 *   gsb_cloud_*           <- GaussianCloud            include/gsopt/scene.hpp:22-46
 *   gsb_cloud_{load,save}_ply <- load/save_cloud_ply  include/gsopt/scene_io.hpp (src/ply.cpp:29-148)
 *   gsb_densify_and_prune <- gsopt::densify_and_prune include/gsopt/trainer.hpp:130-133
 *   gsb_joint_*           <- gsopt::joint_optimize    include/gsopt/trainer.hpp:155-163
 *                            (src/pipelines.cpp:96-216, densification off), data parallel
 *                            over training views with an NCCL all-reduce (gsb_comm_*)
 *
 * Status codes: 0 = OK; reference ErrorCode value + 1 (core.hpp:35-47) for
 * the reference's own failure modes; >= 100 for CUDA / argument / memory
 * failures. gsb_last_error() returns a thread-local message for the last
 * non-zero status. No call ever falls back to a CPU path: without a usable
 * sm_100 device every call that needs one returns GSB_ERR_NO_DEVICE.
 *
 * Threading: one context = one device + one CUDA stream; calls on a context
 * are stream ordered and blocking for host outputs. A context must not be
 * used from two threads at once without external locking (the reference's
 * pool is not re-entrant either, core.cpp:39-58).
 */
#ifndef GSB200_H
#define GSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSB_OK 0
#define GSB_ERR_ANGLE_NEAR_PI 1
#define GSB_ERR_DEGENERATE_CLOUD 2
#define GSB_ERR_NO_VALID_DEPTH 3
#define GSB_ERR_DIMENSION_MISMATCH 4
#define GSB_ERR_EMPTY_MASK 5
#define GSB_ERR_STATE_MISMATCH 6
#define GSB_ERR_MISSING_INTRINSICS 7
#define GSB_ERR_IMAGE_SIZE_MISMATCH 8
#define GSB_ERR_CORRUPT_FILE 9
#define GSB_ERR_DIVERGED 10
#define GSB_ERR_INVALID_CONFIG 11
#define GSB_ERR_CUDA 100
#define GSB_ERR_INVALID_ARGUMENT 101
#define GSB_ERR_OUT_OF_MEMORY 102
#define GSB_ERR_NO_DEVICE 103

/* render_backward flags */
#define GSB_BWD_POSE_ONLY 1u   /* estimate_pose only consumes d_pose (pipelines.cpp:84) */
/* RasterConfig::deterministic == false selects the reference's atomic
 * phase-2 reduction (rasterizer.cpp:419-431). Accepted and has no effect:
 * libgsb200's reduction is always the fixed-order one (no floating-point
 * atomics anywhere), which the reference's own test requires to agree with
 * the atomic mode within 1e-10 (test_rasterizer.cpp:357-375). */
#define GSB_BWD_FAST_ATOMIC 2u

typedef struct gsb_ctx gsb_ctx;
typedef struct gsb_cloud gsb_cloud;
typedef struct gsb_frame gsb_frame;   /* RenderOutput's cached forward state, device resident */
typedef struct gsb_grads gsb_grads;   /* GradientBundle, device resident */
typedef struct gsb_image gsb_image;   /* a device-resident H x W x 3 target frame */
typedef struct gsb_adam gsb_adam;     /* CloudAdam, device resident */

/* Camera (rasterizer.hpp:19-28): pinhole intrinsics + world_to_cam [R|t], R row-major. */
typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
  double R[9];
  double t[3];
} gsb_camera;

/* RasterConfig (rasterizer.hpp:30-38). */
typedef struct {
  int32_t tile_size; /* must be 16 */
  double cutoff_sigma, alpha_clamp, dilation, early_termination, z_near;
  int32_t deterministic;
} gsb_raster_config;

/* PoseAdam (trainer.hpp:90-94). */
typedef struct {
  double m[6], v[6];
  int64_t step;
} gsb_pose_adam;

/* Forward-state sizes (RenderOutput bookkeeping). */
typedef struct {
  int64_t n_gaussians, n_splats, n_entries;
  int32_t width, height, tiles_x, tiles_y;
  uint64_t state_fingerprint;
  int32_t binning; /* GSB_BINNING_* used for this state */
  int32_t reserved;
} gsb_frame_info;

/* The pose_descent knobs of TrainConfig (trainer.hpp:21-60) that estimate_pose reads. */
typedef struct {
  double cam_lr_start, cam_lr_end; /* cosine schedule (pipelines.cpp:82) */
  double beta;                     /* LossConfig::beta */
  double pose_converged_eps;       /* 0 disables the early exit */
  double background[3];
  gsb_raster_config raster;
  int32_t budget;                  /* estimate_pose_steps */
} gsb_pose_config;

const char* gsb_last_error(void);
const char* gsb_version(void);
void gsb_default_raster_config(gsb_raster_config* cfg);
void gsb_default_pose_config(gsb_pose_config* cfg);

/* ---- context ---- */
int gsb_ctx_create(int32_t device, gsb_ctx** out);
int gsb_ctx_destroy(gsb_ctx* ctx);
int gsb_ctx_synchronize(gsb_ctx* ctx);
/* K2 binning strategy (both give the reference's tile lists bit for bit,
 * rasterizer.cpp:127-168). TILE_LOCAL (default): per-tile (depth, gid) sort
 * in shared memory, falling back to GLOBAL for a frame once any tile holds
 * more than 8192 entries. GLOBAL: global stable depth sort + rank-major
 * duplication + stable tile sort. */
#define GSB_BINNING_TILE_LOCAL 0
#define GSB_BINNING_GLOBAL 1
int gsb_ctx_set_binning(gsb_ctx* ctx, int32_t mode);
/* Device time of the kernels launched on the context stream since the last
 * reset, split by stage (ms): preprocess, sort/bin, composite, loss,
 * backward raster, backward geometry, optimizer. Enabled by
 * gsb_ctx_set_profiling(ctx, 1); used by bench.py for the roofline line. */
int gsb_ctx_set_profiling(gsb_ctx* ctx, int32_t enable);
int gsb_ctx_stage_times(gsb_ctx* ctx, double* ms_out /* 8 */, int64_t* launches_out /* 8 */, int32_t reset);
/* Number of kernel launches issued by this context so far. */
int64_t gsb_ctx_launch_count(gsb_ctx* ctx);
/* CUDA-event interval on the context stream (device time, ms). */
int gsb_ctx_timer_start(gsb_ctx* ctx);
int gsb_ctx_timer_stop(gsb_ctx* ctx, double* ms_out);

/* ---- measurement aids (no reference counterpart) ----
 * FP32 FFMA throughput (TFLOP/s, FMA = 2 FLOP) and MUFU ex2 throughput
 * (T ops/s) of `device`, measured by microbenchmark kernels at the clock the
 * device runs at now: the denominators of the FP32-bound kernels' roofline. */
int gsb_measure_fp32_peaks(int32_t device, double* ffma_tflops, double* mufu_tops);
/* SHA-256 (hex) of the sources + flags this libgsb200.so was compiled from. */
const char* gsb_build_id(void);

/* ---- cloud (GaussianCloud, scene.hpp:22-46), stored as FP32 planes on device ---- */
int gsb_cloud_create(gsb_ctx* ctx, int64_t n, int32_t sh_degree, gsb_cloud** out);
int gsb_cloud_destroy(gsb_cloud* cloud);
/* Reference FP64 layout: means n*3, rotations n*4 (w,x,y,z), log_scales n*3,
 * opacity_logits n, sh n*3*(sh_degree+1)^2 channel-major per Gaussian. */
int gsb_cloud_upload(gsb_cloud* cloud, const double* means, const double* rotations,
                     const double* log_scales, const double* opacity_logits, const double* sh,
                     int32_t active_sh_degree);
int gsb_cloud_download(gsb_cloud* cloud, double* means, double* rotations, double* log_scales,
                       double* opacity_logits, double* sh);
int gsb_cloud_info(gsb_cloud* cloud, int64_t* n, int32_t* sh_degree, int32_t* active_sh_degree);
int gsb_cloud_set_active_sh_degree(gsb_cloud* cloud, int32_t active_sh_degree);
/* 3DGS PLY I/O straight to / from the device layout: load_cloud_ply
 * (src/ply.cpp:62-148; the SH degree follows the f_rest count, active = it)
 * and save_cloud_ply (29-60; higher bands zero-padded to degree 3). Bad files
 * return GSB_ERR_CORRUPT_FILE. */
int gsb_cloud_load_ply(gsb_ctx* ctx, const char* path, gsb_cloud** out);
int gsb_cloud_save_ply(gsb_cloud* cloud, const char* path);
/* Fills the cloud with the synth.cpp:45-62 draw sequence (GCC argument order)
 * from seed, plus log_scale_offset added to every log-scale (SURVEY §8d
 * density matching). Host generator, then one upload. */
int gsb_cloud_synth(gsb_cloud* cloud, uint64_t seed, double log_scale_offset);
/* Generates `cameras` poses exactly as synth_scene (synth.cpp:73-101) would
 * after drawing an n-Gaussian cloud of degree sh_degree from seed.
 * kind: 0 orbit, 1 forward-facing, 2 random-walk. poses: cameras*12 row-major [R|t]. */
int gsb_synth_poses(uint64_t seed, int64_t n, int32_t sh_degree, int32_t kind, int32_t cameras,
                    double orbit_radius, double orbit_arc, double* poses);
/* Rng helpers on a caller-held xorshift64* state (core.hpp:58-102): the split
 * children's normal3 draws of densify_and_prune (children x 3, GCC draw
 * order) and one epoch shuffle of pipelines.cpp:123-129. Host only. */
int gsb_rng_child_normals(uint64_t* rng_state, int64_t children, double* out);
int gsb_rng_shuffle(uint64_t* rng_state, int32_t n, int32_t* order);
/* perturb_pose_tangent (eval.cpp:148-152), same rng convention as gsb_perturb_pose. */
int gsb_perturb_pose_tangent(const double pose[12], double sigma, uint64_t* rng_state, double out[12]);
/* Joint-test initial cloud (tests/test_trainer.cpp:598-601): means += mean_sigma
 * * normal3, then log-scales += log_scale_range * uniform(-1, 1) per Gaussian. */
int gsb_cloud_jitter(gsb_cloud* cloud, uint64_t seed, double mean_sigma, double log_scale_range);
/* perturb_pose (eval.cpp:130-146) with a caller-held rng state (init with seed). */
int gsb_perturb_pose(const double pose[12], double rot_deg, double trans, uint64_t* rng_state,
                     double out[12]);

/* ---- forward (render, rasterizer.cpp:209-281) ---- */
int gsb_frame_create(gsb_ctx* ctx, gsb_frame** out);
int gsb_frame_destroy(gsb_frame* frame);
/* image_out: optional host H*W*3 interleaved FP64 (Image layout, image.hpp:15-37). */
int gsb_render(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, const double background[3],
               const gsb_raster_config* cfg, gsb_frame* frame, double* image_out);
int gsb_frame_get_info(gsb_frame* frame, gsb_frame_info* info);
/* The state_fingerprint gsb_render(cloud, cam, ...) stamps on its forward
 * state (rasterizer.cpp:52-73), without rendering: lets a caller that keys
 * forward states by fingerprint re-render into the state it already holds. */
int gsb_state_fingerprint(gsb_cloud* cloud, const gsb_camera* cam, uint64_t* out);
/* render_expected_depth (rasterizer.cpp:283-323): per-pixel alpha-weighted
 * mean view-space depth (0 where the weight sum is <= 1e-8) and the weight
 * sum, host H*W FP32 each. Same cutoff / alpha decisions as gsb_render. */
int gsb_render_expected_depth(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam,
                              const gsb_raster_config* cfg, float* depth_out, float* weight_out);
/* Copies every RenderOutput field to host (any pointer may be NULL). Per-splat
 * arrays are in depth order (n_splats), tile_lists holds indices into them
 * (n_entries), tile_ranges is tiles*2 (begin,end). conic is 2x2 row-major. */
int gsb_frame_download(gsb_frame* frame, double* image, double* accum_transmittance,
                       double* final_transmittance, int32_t* contrib_count, uint8_t* overflow_mask,
                       int32_t* splat_gaussian, double* splat_mu2d, double* splat_depth,
                       double* splat_conic, double* splat_color, double* splat_opacity,
                       double* splat_radius, uint8_t* splat_clamped, int32_t* tile_lists,
                       int32_t* tile_ranges);

/* ---- loss (rgb_loss, losses.cpp:201-215) ---- */
/* Host FP64 HWC images; d_rendered optional. */
int gsb_rgb_loss(gsb_ctx* ctx, const double* rendered, const double* target, int32_t width,
                 int32_t height, double beta, double* loss_out, double* d_rendered);
int gsb_image_create(gsb_ctx* ctx, const double* image_hwc, int32_t width, int32_t height,
                     gsb_image** out);
int gsb_image_destroy(gsb_image* image);
/* Loss of the frame's rendered image against a device target; the gradient
 * stays on device inside the frame (consumed by gsb_render_backward_device). */
int gsb_frame_rgb_loss(gsb_ctx* ctx, gsb_frame* frame, gsb_image* target, double beta,
                       double* loss_out);

/* masked_rgb_loss (losses.cpp:273-289): mask = host uint8 H*W; GSB_ERR_EMPTY_MASK
 * when no pixel is set (masked_l1's empty_mask). d_rendered optional. */
int gsb_masked_rgb_loss(gsb_ctx* ctx, const double* rendered, const double* target, int32_t width,
                        int32_t height, const uint8_t* mask, double beta, double* loss_out,
                        double* d_rendered);
/* Same on the frame's image with its own transmittance_mask(accum, threshold)
 * (losses.cpp:259-263, accum = 1 - final transmittance); the gradient stays in
 * the frame. masked_out: pixels that passed (0 -> GSB_ERR_EMPTY_MASK). */
int gsb_frame_masked_rgb_loss(gsb_ctx* ctx, gsb_frame* frame, gsb_image* target, double beta,
                              double threshold, double* loss_out, int64_t* masked_out);

/* ---- backward (render_backward, rasterizer.cpp:336-540) ---- */
int gsb_grads_create(gsb_ctx* ctx, gsb_cloud* cloud, gsb_grads** out);
int gsb_grads_destroy(gsb_grads* grads);
int gsb_grads_download(gsb_grads* grads, double* d_means, double* d_rotations,
                       double* d_log_scales, double* d_opacity_logits, double* d_sh,
                       double* d_mu2d, double d_pose[6]);
/* d_image: host H*W*3 FP64. grads may be NULL with GSB_BWD_POSE_ONLY. */
int gsb_render_backward(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, gsb_frame* frame,
                        const double* d_image, int32_t width, int32_t height, uint32_t flags,
                        gsb_grads* grads, double d_pose_out[6]);
/* Same, upstream gradient = the one left in the frame by gsb_frame_rgb_loss. */
int gsb_render_backward_device(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam,
                               gsb_frame* frame, uint32_t flags, gsb_grads* grads,
                               double d_pose_out[6]);

/* Same, upstream gradient = a device-resident Image (gsb_image_create, e.g. a
 * fixed d_image reused across calls as tests/gradcheck.hpp:204-208 does):
 * render_backward(cloud, camera, fwd, d_image) with d_image already on the
 * device; GSB_ERR_DIMENSION_MISMATCH when its size differs from the camera's
 * (rasterizer.cpp:341-343). */
int gsb_render_backward_image(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, gsb_frame* frame,
                              const gsb_image* d_image, uint32_t flags, gsb_grads* grads, double d_pose_out[6]);

/* ---- optimiser (trainer.cpp:30-90, pipelines.cpp:18-41) ---- */
double gsb_schedule(int32_t kind /* 0 cosine, 1 exponential */, double start, double end,
                    int64_t step, int64_t total);
/* Runs on the device (FP64), like the batched step inside gsb_estimate_pose. */
int gsb_pose_step(gsb_ctx* ctx, const double pose[12], const double d_pose[6], double lr,
                  gsb_pose_adam* state, double pose_out[12], double applied_update[6]);
/* adam_step (trainer.hpp:85 / trainer.cpp:40-53): AdamState = (m, v, step),
 * the caller's n-element arrays (zero-initialised before the first step, as
 * AdamState::resize); updated in place, bit for bit the reference's FP64. */
int gsb_adam_step(gsb_ctx* ctx, double* params, const double* grads, double* m, double* v,
                  int64_t* step, int64_t n, double lr);
/* The per-index overload adam_step(..., lr_of) (trainer.hpp:86-87 /
 * trainer.cpp:55-69): lr_of[i] is the learning rate of element i. */
int gsb_adam_step_lrs(gsb_ctx* ctx, double* params, const double* grads, double* m, double* v,
                      int64_t* step, int64_t n, const double* lr_of);
int gsb_adam_create(gsb_ctx* ctx, gsb_cloud* cloud, gsb_adam** out);
int gsb_adam_destroy(gsb_adam* adam);
/* lrs = {pos, rot, scale, opacity, sh_dc, sh_rest} (pipelines.cpp:14-16). */
int gsb_cloud_adam_step(gsb_ctx* ctx, gsb_cloud* cloud, gsb_grads* grads, gsb_adam* adam,
                        const double lrs[6]);

/* ---- pose estimation (pose_descent, pipelines.cpp:58-92), device resident ---- */
/* intr = {fx, fy, cx, cy}; trace_* optional (budget entries): pose before each
 * step (12), loss (1). Returns best pose (pipelines.cpp:71-75). */
int gsb_estimate_pose(gsb_ctx* ctx, gsb_cloud* cloud, gsb_image* target, const double intr[4],
                      const double init_pose[12], const gsb_pose_config* cfg, double pose_out[12],
                      double* final_loss, int32_t* steps_used, int32_t* converged,
                      double* trace_pose, double* trace_loss);

/* ---- pose session: one view's pose_descent state kept on the device ----
 * A session holds the view's target, pose, PoseAdam and best-loss pose; each
 * gsb_session_step runs `iterations` pose_descent iterations (render ->
 * rgb_loss -> render_backward(pose only) -> pose_step) without copying any
 * image to the host. Sessions of one context share its scratch forward state.
 * gsb_estimate_pose == create + step(budget) + read + destroy. */
typedef struct gsb_session gsb_session;
int gsb_session_create(gsb_ctx* ctx, gsb_cloud* cloud, gsb_image* target, const double intr[4],
                       const double init_pose[12], const gsb_pose_config* cfg, gsb_session** out);
int gsb_session_destroy(gsb_session* s);
int gsb_session_step(gsb_ctx* ctx, gsb_session* s, int32_t iterations);
/* Enqueue iterations without waiting (the next gsb_session_step / _read
 * synchronises; early exits are then honoured on the device). */
int gsb_session_step_async(gsb_ctx* ctx, gsb_session* s, int32_t iterations);
/* Per-stage device time (ms, 8 stages as gsb_ctx_stage_times) of the session's
 * last iteration, recorded by events inside its CUDA graph while profiling. */
int gsb_session_stage_times(gsb_session* s, double* ms_out);
/* current pose, best pose, best loss, steps used, converged, stopped (any may be NULL) */
int gsb_session_read(gsb_session* s, double pose[12], double best_pose[12], double* final_loss,
                     int32_t* steps_used, int32_t* converged, int32_t* stopped);
/* Forward-state sizes of the session's last iteration (V, K) for work accounting. */
int gsb_session_frame_info(gsb_session* s, gsb_frame_info* info);

/* ---- pose batch: several sessions advanced by one graph replay ----
 * Config C3 (independent views of one cloud). Each session gets a private
 * forward state for the batch's lifetime; one replay runs one pose_descent
 * iteration of every session, the sessions' launch sequences being parallel
 * branches of one CUDA graph. Per-session results are identical to stepping
 * the sessions one by one. No reference counterpart: the reference runs
 * estimate_pose once per view (pipelines.cpp:218-222). */
typedef struct gsb_pose_batch gsb_pose_batch;
int gsb_pose_batch_create(gsb_ctx* ctx, gsb_session* const* sessions, int32_t count, gsb_pose_batch** out);
int gsb_pose_batch_destroy(gsb_pose_batch* b);
int gsb_pose_batch_step(gsb_ctx* ctx, gsb_pose_batch* b, int32_t iterations);
int gsb_pose_batch_step_async(gsb_ctx* ctx, gsb_pose_batch* b, int32_t iterations);
/* waits for the batch; re-runs any iteration a session discarded (capacity growth) */
int gsb_pose_batch_sync(gsb_ctx* ctx, gsb_pose_batch* b);
/* Iterations the device discarded for entry-capacity growth (and the host
 * re-ran in gsb_pose_batch_sync) since the batch's sessions were created.
 * Measurement aid: a timed region must see 0. */
int gsb_pose_batch_discarded(const gsb_pose_batch* b, int64_t* out);
/* estimate_pose for `count` views of one cloud as one pose batch: init_poses /
 * poses_out are count x 12 (best pose per view); final_losses, steps_used optional. */
int gsb_estimate_poses(gsb_ctx* ctx, gsb_cloud* cloud, gsb_image* const* targets, const double intr[4],
                       const double* init_poses, int32_t count, const gsb_pose_config* cfg, double* poses_out,
                       double* final_losses, int32_t* steps_used);

/* ---- densify_and_prune (trainer.hpp:130-133, trainer.cpp:144-239) ----
 * grad_sum / count: the GradAccum arrays (host, cloud n entries). The cloud is
 * rebuilt on the device (its size changes); adam (optional) is remapped like
 * CloudAdam::remap. rng_state: the run's Rng (split children draw normal3).
 * report = {cloned, split, pruned}. */
int gsb_densify_and_prune(gsb_ctx* ctx, gsb_cloud* cloud, const double* grad_sum, const int32_t* count,
                          double grad_threshold, double densify_size_ratio, int32_t n_target, double prune_opacity,
                          uint64_t* rng_state, gsb_adam* adam, int32_t report[3]);

/* ---- communicator: NCCL over NVLink for data-parallel training ----
 * libnccl.so.2 is loaded at run time (dlopen); without it gsb_comm_* return
 * GSB_ERR_NO_DEVICE. One rank per GPU. The 128-byte unique id is created on
 * rank 0 and distributed by the caller (e.g. torch.distributed broadcast). */
typedef struct gsb_comm gsb_comm;
int gsb_comm_unique_id(uint8_t id_out[128]);
int gsb_comm_create(gsb_ctx* ctx, const uint8_t id[128], int32_t rank, int32_t world, gsb_comm** out);
int gsb_comm_destroy(gsb_comm* c);
/* in-place sum over ranks of n device floats (stream ordered on ctx) */
int gsb_comm_allreduce_f32(gsb_comm* c, float* dev_buf, int64_t n);

/* ---- joint reconstruction + pose refinement (joint_optimize) ----
 * The TrainConfig fields joint_optimize reads (trainer.hpp:21-60,
 * losses.hpp:15-19); densification is not part of this loop. */
typedef struct {
  int32_t iterations;
  double cam_lr_start, cam_lr_end, pos_lr_start, pos_lr_end;
  double rot_lr, scale_lr, opacity_lr, sh_dc_lr, sh_rest_lr;
  int32_t opacity_l1_steps, sh_degree, sh_degree_interval, optimize_poses;
  double beta, aniso_ratio, opacity_l1_weight;
  double background[3];
  gsb_raster_config raster;
  /* densification (trainer.hpp:35-42): after step t when densify_start <= t <=
   * densify_stop, t > 0 and (t - densify_start) % densify_interval == 0;
   * densify_interval <= 0 disables it */
  int32_t densify_interval, densify_start, densify_stop, n_target;
  double grad_threshold, densify_size_ratio, prune_opacity;
} gsb_joint_config;
void gsb_default_joint_config(gsb_joint_config* c);
/* The training-view sequence of joint_optimize (pipelines.cpp:122-129: epoch
 * permutations shuffled in place from Rng(seed)); step t of a data-parallel
 * run with S slots per step uses seq[t*S .. t*S+S-1], rank r the slots
 * r*local .. r*local+local-1. Host only. */
int gsb_joint_schedule(uint64_t seed, int32_t n_views, int64_t count, int32_t* seq_out);
/* One step = `local` views rendered on this rank (local * world slots in
 * all); the Adam gradient is the slots' mean plus the regularisers, then each
 * slot's pose step in slot order. local = world = 1 is joint_optimize's loop.
 * The cloud is optimised in place; targets stay owned by the caller.
 * comm may be NULL (single rank). */
typedef struct gsb_joint gsb_joint;
/* rng_state: the caller's Rng (core.hpp:58-102, xorshift64*) state — the
 * reference's joint_optimize(..., Rng& rng, ...) draws its epoch shuffles and
 * densify normals from it (pipelines.cpp:123-129, trainer.cpp:186-205); 0
 * means Rng(0)'s state as in the Rng constructor. The run advances its own
 * copy; gsb_joint_rng_state returns it so the caller's Rng can continue. */
int gsb_joint_create(gsb_ctx* ctx, gsb_cloud* cloud, gsb_image* const* targets, int32_t n_views,
                     const double intr[4], const double* init_poses, const gsb_joint_config* cfg,
                     uint64_t rng_state, int32_t local_views, gsb_comm* comm, gsb_joint** out);
/* The joint run's Rng state after the steps run so far (write it back into the
 * caller's Rng). */
int gsb_joint_rng_state(const gsb_joint* j, uint64_t* rng_state);
int gsb_joint_destroy(gsb_joint* j);
/* runs `steps` steps (blocking); GSB_ERR_DIVERGED at a non-finite total loss */
int gsb_joint_step(gsb_ctx* ctx, gsb_joint* j, int32_t steps);
/* poses_out n_views x 12 (optional), steps done, per-step total / L1 traces
 * (iterations entries each, optional) */
int gsb_joint_read(gsb_joint* j, double* poses_out, int64_t* steps_done, double* trace_total, double* trace_l1);
/* current cloud size, densify_and_prune events so far, last event's {cloned, split, pruned} */
int gsb_joint_info(gsb_joint* j, int64_t* n_gaussians, int32_t* densify_events, int32_t last_report[3]);

/* ---- small on-disk formats (host only; scene_io.cpp, image.cpp:105-141) ----
 * f32map: "f32map W H scale\n" + W*H little-endian floats (values * scale on
 * load). Pass values/depth = NULL to query the size first. */
int gsb_load_float_map(const char* path, float* values, int64_t capacity, int32_t* width,
                       int32_t* height);
int gsb_save_float_map(const float* values, int32_t width, int32_t height, const char* path,
                       double scale);
/* f32map as load_scene's depth (scene_io.cpp:203-215): valid = finite && > 0. */
int gsb_load_depth_map(const char* path, double* depth, uint8_t* valid, int64_t capacity,
                       int32_t* width, int32_t* height);
/* {"poses": [[12 numbers: row-major R|t world_to_cam], ...]} (scene_io.cpp:64-79),
 * 17 significant digits (lossless). poses = NULL queries n. */
int gsb_save_poses_json(const double* poses, int32_t n, const char* path);
int gsb_load_poses_json(const char* path, double* poses, int32_t capacity, int32_t* n);
/* cameras.json (load_cameras_json, scene_io.cpp:254-279): GSB_ERR_MISSING_INTRINSICS
 * if fx/fy/cx/cy/width/height/frames is absent. poses / names optional. */
int gsb_load_cameras_json(const char* path, double intr[4], int32_t size[2], double* poses,
                          int32_t capacity, int32_t* n_frames, int32_t* has_poses, char* names,
                          int64_t names_capacity);

/* ---- bootstrap path (pipelines.cpp:224-312, scene.cpp:115-243) ----
 * RGB-D frames -> per-frame clouds -> relative poses -> an initial trajectory.
 * The TrainConfig knobs these read (trainer.hpp:21-60, losses.hpp:19). */
typedef struct {
  int32_t per_frame_fit_steps, relpose_steps, unproject_points;
  double pos_lr_start, pos_lr_end, rot_lr, scale_lr, opacity_lr, sh_dc_lr, sh_rest_lr;
  double relpose_lr_start, relpose_lr_end;
  double beta, mask_threshold;
  double background[3];
  gsb_raster_config raster;
} gsb_bootstrap_config;
void gsb_default_bootstrap_config(gsb_bootstrap_config* cfg);
/* unproject (scene.cpp:209-243): every ceil(valid / max_points)-th valid pixel
 * (valid != 0, finite, > 0; row-major) lifted to world by world_to_cam^-1.
 * points_out / colors_out: max_points * 3. GSB_ERR_NO_VALID_DEPTH if none. */
int gsb_unproject(const double* depth, const uint8_t* valid, int32_t width, int32_t height,
                  const double* frame_hwc, const double intr[4], const double world_to_cam[12],
                  int32_t max_points, double* points_out, double* colors_out, int64_t* n_out);
/* init_from_points (scene.cpp:182-207): log-scale = log(max(mean 3-NN distance,
 * 1e-7)) (kNN on the device), identity rotation, opacity logit(0.1), SH DC
 * from colour, active degree 0. GSB_ERR_DEGENERATE_CLOUD below 4 points. */
int gsb_init_from_points(gsb_ctx* ctx, const double* points, const double* colors, int64_t n,
                         int32_t sh_degree, gsb_cloud** out);
/* fit_frame_gaussians (pipelines.cpp:224-250): SH-0 cloud from the frame at the
 * identity pose, per_frame_fit_steps of render -> rgb_loss -> backward -> Adam. */
int gsb_fit_frame_gaussians(gsb_ctx* ctx, const double* frame_hwc, const double* depth,
                            const uint8_t* valid, int32_t width, int32_t height, const double intr[4],
                            const gsb_bootstrap_config* cfg, gsb_cloud** out);
/* estimate_relative_pose (pipelines.cpp:252-290): masked pose-only descent from
 * the identity; best-loss pose, ok = 0 (identity) once the mask empties. */
int gsb_estimate_relative_pose(gsb_ctx* ctx, gsb_cloud* cloud, const double* frame_next_hwc,
                               int32_t width, int32_t height, const double intr[4],
                               const gsb_bootstrap_config* cfg, double pose_out[12], int32_t* ok,
                               double* final_loss);
/* bootstrap_trajectory (pipelines.cpp:292-312): poses_out n_frames x 12
 * world_to_cam (frame 0 = identity), pair_ok n_frames - 1 (optional). */
int gsb_bootstrap_trajectory(gsb_ctx* ctx, const double* const* frames, const double* const* depths,
                             const uint8_t* const* valids, int32_t n_frames, int32_t width,
                             int32_t height, const double intr[4], const gsb_bootstrap_config* cfg,
                             double* poses_out, int32_t* pair_ok);

#ifdef __cplusplus
}
#endif
#endif
