/*
 * gsopt_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A clean-room, double-precision CPU restatement of the reference (gsopt,
 * arxiv/paper_2410_08743, /root/reference/proj) hot path: render (cull /
 * project / sort / bin / composite), rgb_loss (L1 + SSIM fwd/bwd),
 * render_backward (3-phase backward + SE(3) pose gradient), pose_step, Adam,
 * and the pose_descent loop, plus the deterministic synthetic-scene
 * generator the benchmark inputs follow.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the CPU baseline. The product (paper_2410_08743_b200/) never links it.
 *
 * Every function cites the reference file:line it restates. Arithmetic
 * order follows the reference expressions left to right with no FMA
 * contraction (-ffp-contract=off). Argument evaluation order of the
 * reference's Vec3(rng..., rng..., rng...) constructors follows GCC/x86-64
 * (right to left), i.e. the order a g++ build of the reference draws in.
 */
#ifndef GSOPT_ORACLE_H
#define GSOPT_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* core.hpp:58-102 */
typedef struct { uint64_t state; } orc_rng;
void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_uniform_range(orc_rng* r, double lo, double hi);
int64_t orc_rng_uniform_int(orc_rng* r, int64_t lo, int64_t hi);
double orc_rng_normal(orc_rng* r);

/* rasterizer.hpp:19-38; scene.hpp:22-46 (flattened) */
typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
  double R[9]; /* world_to_cam rotation, row-major */
  double t[3]; /* world_to_cam translation */
} orc_camera;

typedef struct {
  int32_t tile_size;
  double cutoff_sigma, alpha_clamp, dilation, early_termination, z_near;
  int32_t deterministic;
} orc_raster_config;

typedef struct {
  int64_t n;
  int32_t sh_degree;        /* capacity */
  int32_t active_sh_degree;
  double* means;            /* n*3 */
  double* rotations;        /* n*4 (w,x,y,z) */
  double* log_scales;       /* n*3 */
  double* opacity_logits;   /* n   */
  double* sh;               /* n*3*basis, channel-major per Gaussian */
} orc_cloud;

/* rasterizer.hpp:55-64 */
typedef struct {
  int32_t gaussian;
  double mu2d[2];
  double depth;
  double conic[4]; /* row-major 2x2 */
  double color[3];
  double opacity;
  double radius;
  uint8_t color_clamped;
} orc_splat;

/* rasterizer.hpp:66-82 */
typedef struct {
  int32_t width, height, tiles_x, tiles_y;
  int64_t n_splats, n_entries;
  double* image;                /* H*W*3 interleaved */
  double* accum_transmittance;  /* H*W */
  double* final_transmittance;  /* H*W */
  int32_t* contrib_count;       /* H*W */
  uint8_t* overflow_mask;       /* H*W */
  orc_splat* splats;            /* n_splats, depth sorted */
  int32_t* tile_lists;          /* n_entries, indices into splats */
  int32_t* tile_ranges;         /* tiles*2 (begin, end) */
  orc_camera camera;
  double background[3];
  orc_raster_config config;
  uint64_t state_fingerprint;
  int64_t n_gaussians;
} orc_render_out;

/* rasterizer.hpp:84-94 */
typedef struct {
  int64_t n, sh_len;
  double* d_means, *d_rotations, *d_log_scales, *d_opacity_logits, *d_sh, *d_mu2d;
  double d_pose[6];
} orc_grads;

void orc_default_raster_config(orc_raster_config* c);

/* scene/sh/lie primitives */
void orc_quat_to_rotation(const double q[4], double R[9]);
void orc_quat_rotation_jacobian(const double q[4], double out[36]);
void orc_covariance3d(const double q[4], const double s[3], double out[9]);
void orc_sh_basis(const double dir[3], int degree, double* out);
void orc_sh_basis_gradient(const double dir[3], int degree, double* out /* 16*3 */);
void orc_sh_eval(const double* coeffs, const double dir[3], int degree, double rgb[3], uint8_t* mask);
void orc_se3_exp(const double tau[6], double R[9], double t[3]);
void orc_so3_exp(const double w[3], double R[9]);
void orc_orthonormalize(double R[9]);
double orc_rotation_angle(const double R[9]);
void orc_project(const double mu[3], const orc_camera* cam, double mu2d[2], double* depth);
void orc_covariance2d(const double sigma[9], const double mu_cam[3], const orc_camera* cam,
                      double dilation, double out[4]);
double orc_splat_alpha(const double mu2d[2], const double conic[4], double opacity,
                       const double pixel[2], double alpha_clamp, double cutoff_sigma);

/* rasterizer.cpp:41-73 */
uint64_t orc_fingerprint(const orc_cloud* cloud, const orc_camera* cam);

/* rasterizer.cpp:209-281 */
orc_render_out* orc_render(const orc_cloud* cloud, const orc_camera* cam, const double bg[3],
                           const orc_raster_config* cfg);
void orc_render_free(orc_render_out* out);

/* rasterizer.cpp:83-170 binning half only, fed externally supplied per-splat
 * (keep, mu2d, radius, depth) records — the FP-agnostic bit-exactness check
 * for the device sort/bin. Writes n_entries; tile_lists (indices into the
 * depth-sorted kept list), tile_ranges and the sorted Gaussian ids. Returns
 * the number of entries, or -1 if cap is too small. */
int64_t orc_bin_records(int64_t n, const uint8_t* keep, const double* mu2d, const double* radius,
                        const double* depth, int32_t width, int32_t height, int32_t tile_size,
                        int32_t* sorted_gaussian, int64_t* n_splats, int32_t* tile_lists,
                        int64_t cap, int32_t* tile_ranges);

/* rasterizer.cpp:336-540; returns 0 ok, 6 = state_mismatch, 4 = dimension_mismatch
 * (ErrorCode + 1) */
int orc_render_backward(const orc_cloud* cloud, const orc_camera* cam, const orc_render_out* out,
                        const double* d_image, int32_t d_w, int32_t d_h, orc_grads* grads);
void orc_grads_alloc(orc_grads* g, const orc_cloud* cloud);
void orc_grads_free(orc_grads* g);

/* losses.cpp:201-215, 74-155, 158-192 */
double orc_rgb_loss(const double* rendered, const double* target, int32_t w, int32_t h,
                    double beta, double* d_rendered /* nullable */);
double orc_ssim(const double* a, const double* b, int32_t w, int32_t h, double* d_a);
/* losses.cpp:217-257 */
double orc_anisotropy_loss(const double* log_scales, int64_t n, double ratio, double* d_log_scales);
double orc_opacity_l1(const double* opacities, int64_t n, double* d_opacities);

/* trainer.cpp:30-90 */
double orc_schedule(int kind /*0 cosine,1 exp*/, double start, double end, int64_t step, int64_t total);
typedef struct { double m[6], v[6]; int64_t step; } orc_pose_adam;
void orc_pose_step(const double R[9], const double t[3], const double d_pose[6], double lr,
                   orc_pose_adam* state, double R_out[9], double t_out[3], double applied[6]);
typedef struct { double* m; double* v; int64_t n; int64_t step; } orc_adam_state;
void orc_adam_step(orc_adam_state* s, double* params, const double* grads, int64_t n, double lr);
/* pipelines.cpp:18-41; lrs = {pos, rot, scale, opacity, sh_dc, sh_rest} */
void orc_cloud_adam_step(orc_cloud* cloud, const orc_grads* g, orc_adam_state st[5], const double lrs[6]);

/* pipelines.cpp:58-92. trace_* (nullable, length budget) receive the pose
 * (12 doubles, row-major [R|t]) and loss BEFORE each iteration's step.
 * Returns steps_used; best pose in R_out/t_out. */
typedef struct { double cam_lr_start, cam_lr_end, beta, pose_converged_eps; double background[3]; orc_raster_config raster; } orc_pose_cfg;
int32_t orc_estimate_pose(const orc_cloud* cloud, const double* image, double fx, double fy,
                          double cx, double cy, int32_t w, int32_t h, const double R0[9],
                          const double t0[3], const orc_pose_cfg* cfg, int32_t budget,
                          double R_out[9], double t_out[3], double* final_loss, int32_t* converged,
                          double* trace_pose, double* trace_loss, double* trace_dpose);

/* trainer.cpp:134-142 GradAccum::add for one rendered view */
void orc_grad_accum_add(const orc_render_out* out, const orc_grads* g, int32_t image_max_dim, double* grad_sum,
                        int32_t* count);
/* trainer.cpp:144-239; `out` allocated inside (orc_cloud_free), *final_source
 * (out->n, -1 = fresh) freed with orc_free; report = {cloned, split, pruned} */
void orc_densify_and_prune(const orc_cloud* cloud, const double* grad_sum, const int32_t* count,
                           double grad_threshold, double size_ratio, int32_t n_target, double prune_opacity,
                           orc_rng* rng, orc_cloud* out, int32_t** final_source, int32_t report[3]);
void orc_free(void* p);
/* pipelines.cpp:122-129 epoch shuffles -> view sequence (count entries) */
void orc_joint_schedule(orc_rng* rng, int32_t n_views, int64_t count, int32_t* seq);
/* TrainConfig fields joint_optimize reads (trainer.hpp:21-60, losses.hpp:15-19) */
typedef struct {
  int32_t iterations;
  double cam_lr_start, cam_lr_end, pos_lr_start, pos_lr_end, rot_lr, scale_lr, opacity_lr, sh_dc_lr, sh_rest_lr;
  int32_t opacity_l1_steps, sh_degree, sh_degree_interval, optimize_poses;
  double beta, aniso_ratio, opacity_l1_weight;
  double background[3];
  orc_raster_config raster;
  /* densification (trainer.hpp:35-42); densify_interval <= 0 disables */
  int32_t densify_interval, densify_start, densify_stop, n_target;
  double grad_threshold, densify_size_ratio, prune_opacity;
} orc_joint_cfg;
/* pipelines.cpp:96-216 without gt stats; `slots` views per step (1 = the
 * reference loop). The cloud may change size (densify_and_prune): it is
 * reallocated in place (orc_cloud_alloc'ed memory). Returns 0 or 10 (diverged). */
int32_t orc_joint_optimize(orc_cloud* cloud, const double* const* images, int32_t n_views, double fx, double fy,
                           double cx, double cy, int32_t w, int32_t h, double* poses, const orc_joint_cfg* cfg,
                           int32_t slots, orc_rng* rng, double* trace_total, double* trace_l1);

/* ---- bootstrap path (pipelines.cpp:224-312, losses.cpp:259-289, scene.cpp:115-243) ---- */
void orc_transmittance_mask(const double* accum, int64_t n, double threshold, uint8_t* mask);
double orc_masked_rgb_loss(const double* rendered, const double* target, int32_t w, int32_t h, const uint8_t* mask,
                           double beta, double* d_rendered, int32_t* status);
int64_t orc_unproject(const double* depth, const uint8_t* valid, int32_t w, int32_t h, const double* frame,
                      double fx, double fy, double cx, double cy, const double R[9], const double t[3],
                      int32_t max_points, double* points, double* colors);
void orc_mean_knn_distance(const double* pts, int64_t n, int k, double* out);
void orc_init_from_points(const double* pts, const double* cols, int64_t n, int32_t sh_degree, orc_cloud* out);
typedef struct {
  int32_t steps, unproject_points;
  double pos_lr_start, pos_lr_end, rot_lr, scale_lr, opacity_lr, sh_dc_lr, sh_rest_lr, beta;
  double background[3];
  orc_raster_config raster;
} orc_fit_cfg;
typedef struct {
  int32_t steps;
  double lr_start, lr_end, beta, mask_threshold;
  double background[3];
  orc_raster_config raster;
} orc_relpose_cfg;
int32_t orc_fit_frame_gaussians(const double* frame, const double* depth, const uint8_t* valid, int32_t w, int32_t h,
                                double fx, double fy, double cx, double cy, const orc_fit_cfg* cfg, orc_cloud* out);
int32_t orc_estimate_relative_pose(const orc_cloud* cloud, const double* frame, int32_t w, int32_t h, double fx,
                                   double fy, double cx, double cy, const orc_relpose_cfg* cfg, double R_out[9],
                                   double t_out[3], double* final_loss);
int32_t orc_bootstrap_trajectory(const double* const* frames, const double* const* depths,
                                 const uint8_t* const* valids, int32_t n, int32_t w, int32_t h, double fx, double fy,
                                 double cx, double cy, const orc_fit_cfg* fit, const orc_relpose_cfg* rel,
                                 double* poses, int32_t* pair_ok);

/* synth.cpp:33-101 + eval.cpp:122-152 */
void orc_synth_cloud(orc_cloud* cloud, int64_t n, int32_t sh_degree, orc_rng* rng);
void orc_look_at(const double eye[3], const double target[3], double R[9], double t[3]);
/* kind: 0 orbit, 1 forward-facing, 2 random-walk. Draws cameras after the
 * cloud from the same rng, exactly like synth_scene. poses: cameras*12 */
void orc_synth_poses(int32_t kind, int32_t cameras, double orbit_radius, double orbit_arc,
                     orc_rng* rng, double* poses);
void orc_perturb_pose(const double R[9], const double t[3], double rot_deg, double trans,
                      orc_rng* rng, double R_out[9], double t_out[3]);
void orc_perturb_pose_tangent(const double R[9], const double t[3], double sigma, orc_rng* rng,
                              double R_out[9], double t_out[3]);
void orc_abs_pose_error(const double R_pred_w2c[9], const double t_pred_w2c[3],
                        const double R_gt_w2c[9], const double t_gt_w2c[3], double* rot_deg,
                        double* trans);

/* tests/gradcheck.hpp:67-170 (scene draw + conditioning) and 201-254 (FD) */
void orc_make_gradcheck_scene(orc_rng* rng, int32_t n, int32_t image_size, orc_cloud* cloud,
                              orc_camera* cam, double bg[3]);
int orc_scene_is_conditioned(const orc_cloud* cloud, const orc_camera* cam, const double bg[3],
                             const orc_raster_config* cfg);
/* max_err over all params (reference gate), n checked */
double orc_gradcheck(const orc_cloud* cloud, const orc_camera* cam, const double bg[3],
                     const orc_raster_config* cfg, orc_rng* rng, double step, int32_t* checked,
                     char* worst_label /* >= 32 bytes */);

/* Work counts for the roofline: forward (pixel, entry) pairs with
 * e < contrib_count that pass (H_f) / fail (C_f) the g <= cutoff^2 test, and
 * the same over pixels with a non-zero (unclamped) upstream gradient (H_b,
 * C_b). d_image may be NULL (then H_b = C_b = 0). */
void orc_count_work(const orc_render_out* out, const double* d_image, int64_t counts[4]);
void orc_decision_margin(const orc_render_out* out, double* margin);

/* helpers for ctypes users */
void orc_cloud_alloc(orc_cloud* c, int64_t n, int32_t sh_degree);
void orc_cloud_free(orc_cloud* c);
int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
