// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C ABI over the reference's OWN functions (/root/reference/proj/src/*.cpp,
// compiled in place against oracle/shim by oracle/build_ref.py into
// oracle/_ref/libgsopt_ref.so). Entry points mirror the orc_* signatures of
// oracle/gsopt_oracle.h so the tests can run the clean-room restatement and
// the reference itself on the same inputs and compare field by field.
//
// Nothing here re-implements reference arithmetic: every number comes from a
// reference call (render, render_backward, rgb_loss, pose_step, schedule,
// estimate_pose, joint_optimize, densify_and_prune, synth_scene,
// perturb_pose, make_gradcheck_scene, gradcheck_scene). ref_pose_descent_traced
// repeats the 20-line loop body of pose_descent (pipelines.cpp:58-92, which is
// in an anonymous namespace) with the public calls so per-iteration traces can
// be recorded, and ref_estimate_pose runs the reference's own estimate_pose so
// the traced loop is itself checked against it.
#include "gsopt_oracle.h"

#include "gsopt/eval.hpp"
#include "gsopt/losses.hpp"
#include "gsopt/rasterizer.hpp"
#include "gsopt/synth.hpp"
#include "gsopt/trainer.hpp"

#include "gradcheck.hpp"

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace gsopt;

namespace {

GaussianCloud to_cloud(const orc_cloud* c) {
  GaussianCloud g;
  g.resize(static_cast<int>(c->n), c->sh_degree);
  g.active_sh_degree = c->active_sh_degree;
  for (int64_t i = 0; i < c->n; ++i) {
    for (int k = 0; k < 3; ++k) g.means[i](k) = c->means[3 * i + k];
    for (int k = 0; k < 4; ++k) g.rotations[i](k) = c->rotations[4 * i + k];
    for (int k = 0; k < 3; ++k) g.log_scales[i](k) = c->log_scales[3 * i + k];
    g.opacity_logits[i] = c->opacity_logits[i];
  }
  if (!g.sh.empty()) std::memcpy(g.sh.data(), c->sh, g.sh.size() * sizeof(double));
  return g;
}

extern "C" void ref_cloud_alloc(orc_cloud* c, int64_t n, int32_t sh_degree);

void from_cloud(const GaussianCloud& g, orc_cloud* c) {
  ref_cloud_alloc(c, g.size(), g.sh_degree);
  c->active_sh_degree = g.active_sh_degree;
  for (int i = 0; i < g.size(); ++i) {
    for (int k = 0; k < 3; ++k) c->means[3 * i + k] = g.means[i](k);
    for (int k = 0; k < 4; ++k) c->rotations[4 * i + k] = g.rotations[i](k);
    for (int k = 0; k < 3; ++k) c->log_scales[3 * i + k] = g.log_scales[i](k);
    c->opacity_logits[i] = g.opacity_logits[i];
  }
  if (!g.sh.empty()) std::memcpy(c->sh, g.sh.data(), g.sh.size() * sizeof(double));
}

Se3Pose to_pose(const double R[9], const double t[3]) {
  Se3Pose p;
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) p.rotation(r, k) = R[3 * r + k];
    p.translation(r) = t[r];
  }
  return p;
}

void from_pose(const Se3Pose& p, double R[9], double t[3]) {
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) R[3 * r + k] = p.rotation(r, k);
    t[r] = p.translation(r);
  }
}

void to_pose12(const Se3Pose& p, double* out12) {
  std::array<Scalar, 12> f = p.flatten();
  for (int k = 0; k < 12; ++k) out12[k] = f[k];
}

Camera to_camera(const orc_camera* c) {
  Camera cam;
  cam.fx = c->fx;
  cam.fy = c->fy;
  cam.cx = c->cx;
  cam.cy = c->cy;
  cam.width = c->width;
  cam.height = c->height;
  cam.world_to_cam = to_pose(c->R, c->t);
  return cam;
}

void from_camera(const Camera& cam, orc_camera* c) {
  c->fx = cam.fx;
  c->fy = cam.fy;
  c->cx = cam.cx;
  c->cy = cam.cy;
  c->width = cam.width;
  c->height = cam.height;
  from_pose(cam.world_to_cam, c->R, c->t);
}

RasterConfig to_config(const orc_raster_config* c) {
  RasterConfig r;
  if (c == nullptr) return r;
  r.tile_size = c->tile_size;
  r.cutoff_sigma = c->cutoff_sigma;
  r.alpha_clamp = c->alpha_clamp;
  r.dilation = c->dilation;
  r.early_termination = c->early_termination;
  r.z_near = c->z_near;
  r.deterministic = c->deterministic != 0;
  return r;
}

Image to_image(const double* data, int w, int h) {
  Image img(w, h);
  std::memcpy(img.data.data(), data, img.data.size() * sizeof(double));
  return img;
}

// orc_render_out first, so the pointer handed out is an orc_render_out*.
struct RefRender {
  orc_render_out out;
  RenderOutput ro;
};

template <typename T>
T* dup(const T* src, std::size_t n) {
  T* p = static_cast<T*>(std::malloc(std::max<std::size_t>(n, 1) * sizeof(T)));
  if (n) std::memcpy(p, src, n * sizeof(T));
  return p;
}

void fill_grads(const GradientBundle& g, orc_grads* o) {
  const std::size_t n = g.d_means.size();
  o->n = static_cast<int64_t>(n);
  o->sh_len = static_cast<int64_t>(g.d_sh.size());
  o->d_means = dup(g.d_means.data()->data(), 3 * n);
  o->d_rotations = dup(g.d_rotations.data()->data(), 4 * n);
  o->d_log_scales = dup(g.d_log_scales.data()->data(), 3 * n);
  o->d_opacity_logits = dup(g.d_opacity_logits.data(), n);
  o->d_sh = dup(g.d_sh.data(), g.d_sh.size());
  o->d_mu2d = dup(g.d_mu2d.data()->data(), 2 * n);
  for (int k = 0; k < 6; ++k) o->d_pose[k] = g.d_pose(k);
}

thread_local std::string g_last_error;

}  // namespace

extern "C" {
// calloc-backed arrays, freed with free() (interchangeable with
// orc_cloud_alloc / orc_cloud_free).
void ref_cloud_alloc(orc_cloud* c, int64_t n, int32_t sh_degree) {
  const int64_t basis = static_cast<int64_t>(sh_degree + 1) * (sh_degree + 1);
  c->n = n;
  c->sh_degree = sh_degree;
  c->active_sh_degree = sh_degree;
  c->means = static_cast<double*>(std::calloc(3 * n + 1, sizeof(double)));
  c->rotations = static_cast<double*>(std::calloc(4 * n + 1, sizeof(double)));
  c->log_scales = static_cast<double*>(std::calloc(3 * n + 1, sizeof(double)));
  c->opacity_logits = static_cast<double*>(std::calloc(n + 1, sizeof(double)));
  c->sh = static_cast<double*>(std::calloc(3 * basis * n + 1, sizeof(double)));
}
void ref_cloud_free(orc_cloud* c) {
  std::free(c->means);
  std::free(c->rotations);
  std::free(c->log_scales);
  std::free(c->opacity_logits);
  std::free(c->sh);
  c->means = c->rotations = c->log_scales = c->opacity_logits = c->sh = nullptr;
  c->n = 0;
}
}

extern "C" {

const char* ref_last_error(void) { return g_last_error.c_str(); }
int ref_thread_count(void) { return thread_count(); }

// rasterizer.cpp:209-281 (render) — every RenderOutput field copied out.
orc_render_out* ref_render(const orc_cloud* cloud, const orc_camera* cam, const double bg[3],
                           const orc_raster_config* cfg) {
  auto* h = new RefRender();
  h->ro = render(to_cloud(cloud), to_camera(cam), Vec3(bg[0], bg[1], bg[2]), to_config(cfg));
  const RenderOutput& r = h->ro;
  orc_render_out& o = h->out;
  o.width = r.image.width;
  o.height = r.image.height;
  o.tiles_x = r.tiles_x;
  o.tiles_y = r.tiles_y;
  o.n_splats = static_cast<int64_t>(r.splats.size());
  o.n_entries = static_cast<int64_t>(r.tile_lists.size());
  o.image = const_cast<double*>(r.image.data.data());
  o.accum_transmittance = const_cast<double*>(r.accum_transmittance.data());
  o.final_transmittance = const_cast<double*>(r.final_transmittance.data());
  o.contrib_count = const_cast<int32_t*>(r.contrib_count.data());
  o.overflow_mask = const_cast<uint8_t*>(r.overflow_mask.data());
  o.splats = static_cast<orc_splat*>(std::calloc(std::max<std::size_t>(r.splats.size(), 1), sizeof(orc_splat)));
  for (std::size_t s = 0; s < r.splats.size(); ++s) {
    const SplatRecord& a = r.splats[s];
    orc_splat& b = o.splats[s];
    b.gaussian = a.gaussian;
    b.mu2d[0] = a.mu2d(0);
    b.mu2d[1] = a.mu2d(1);
    b.depth = a.depth;
    b.conic[0] = a.conic(0, 0);
    b.conic[1] = a.conic(0, 1);
    b.conic[2] = a.conic(1, 0);
    b.conic[3] = a.conic(1, 1);
    for (int c = 0; c < 3; ++c) b.color[c] = a.color(c);
    b.opacity = a.opacity;
    b.radius = a.radius;
    b.color_clamped = a.color_clamped;
  }
  o.tile_lists = const_cast<int32_t*>(r.tile_lists.data());
  static_assert(sizeof(std::pair<int32_t, int32_t>) == 8, "tile range layout");
  o.tile_ranges = reinterpret_cast<int32_t*>(const_cast<std::pair<int32_t, int32_t>*>(r.tile_ranges.data()));
  from_camera(r.camera, &o.camera);
  for (int c = 0; c < 3; ++c) o.background[c] = r.background(c);
  if (cfg != nullptr) {
    o.config = *cfg;
  } else {
    RasterConfig d;
    o.config = {d.tile_size, d.cutoff_sigma, d.alpha_clamp, d.dilation, d.early_termination, d.z_near,
                d.deterministic ? 1 : 0};
  }
  o.state_fingerprint = r.state_fingerprint;
  o.n_gaussians = r.n_gaussians;
  return &h->out;
}

// rasterizer.cpp:283-323 (render_expected_depth): depth / weight, H*W floats each.
void ref_render_expected_depth(const orc_cloud* cloud, const orc_camera* cam, const orc_raster_config* cfg,
                               float* depth_out, float* weight_out) {
  std::vector<float> d, w;
  render_expected_depth(to_cloud(cloud), to_camera(cam), to_config(cfg), &d, &w);
  std::memcpy(depth_out, d.data(), d.size() * sizeof(float));
  std::memcpy(weight_out, w.data(), w.size() * sizeof(float));
}

void ref_render_free(orc_render_out* out) {
  if (out == nullptr) return;
  auto* h = reinterpret_cast<RefRender*>(out);
  std::free(h->out.splats);
  delete h;
}

// rasterizer.cpp:336-540. Returns 0, or ErrorCode + 1 on a reference throw.
int ref_render_backward(const orc_cloud* cloud, const orc_camera* cam, const orc_render_out* out,
                        const double* d_image, int32_t d_w, int32_t d_h, orc_grads* grads) {
  const auto* h = reinterpret_cast<const RefRender*>(out);
  try {
    GradientBundle g = render_backward(to_cloud(cloud), to_camera(cam), h->ro, to_image(d_image, d_w, d_h));
    fill_grads(g, grads);
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return static_cast<int>(e.code) + 1;
  }
}

void ref_grads_free(orc_grads* g) {
  std::free(g->d_means);
  std::free(g->d_rotations);
  std::free(g->d_log_scales);
  std::free(g->d_opacity_logits);
  std::free(g->d_sh);
  std::free(g->d_mu2d);
  std::memset(g, 0, sizeof *g);
}

// losses.cpp:201-215
double ref_rgb_loss(const double* rendered, const double* target, int32_t w, int32_t h, double beta,
                    double* d_rendered) {
  Image d;
  Scalar loss = rgb_loss(to_image(rendered, w, h), to_image(target, w, h), beta, d_rendered ? &d : nullptr);
  if (d_rendered) std::memcpy(d_rendered, d.data.data(), d.data.size() * sizeof(double));
  return loss;
}

// trainer.cpp:30-38
double ref_schedule(int kind, double start, double end, int64_t step, int64_t total) {
  return schedule(kind == 0 ? ScheduleKind::cosine : ScheduleKind::exponential, start, end, step, total);
}

// trainer.cpp:71-90
void ref_pose_step(const double R[9], const double t[3], const double d_pose[6], double lr, orc_pose_adam* state,
                   double R_out[9], double t_out[3], double applied[6]) {
  PoseAdam adam;
  for (int k = 0; k < 6; ++k) {
    adam.m(k) = state->m[k];
    adam.v(k) = state->v[k];
  }
  adam.step = state->step;
  Tangent6 dp;
  for (int k = 0; k < 6; ++k) dp(k) = d_pose[k];
  Tangent6 ap;
  Se3Pose next = pose_step(to_pose(R, t), dp, lr, &adam, &ap);
  from_pose(next, R_out, t_out);
  for (int k = 0; k < 6; ++k) {
    state->m[k] = adam.m(k);
    state->v[k] = adam.v(k);
    if (applied) applied[k] = ap(k);
  }
  state->step = adam.step;
}

// trainer.cpp:40-69: both adam_step overloads; lrs == nullptr -> scalar lr.
void ref_adam_step(double* params, const double* grads, double* m, double* v, int64_t* step, int64_t n, double lr,
                   const double* lrs) {
  AdamState st;
  st.m.assign(m, m + n);
  st.v.assign(v, v + n);
  st.step = *step;
  if (lrs)
    adam_step(&st, params, grads, static_cast<std::size_t>(n), [lrs](std::size_t i) { return lrs[i]; });
  else
    adam_step(&st, params, grads, static_cast<std::size_t>(n), lr);
  std::memcpy(m, st.m.data(), sizeof(double) * n);
  std::memcpy(v, st.v.data(), sizeof(double) * n);
  *step = st.step;
}

// pipelines.cpp:218-222 -> 58-92: the reference's own estimate_pose. Returns
// steps_used; best pose out.
int32_t ref_estimate_pose(const orc_cloud* cloud, const double* image, double fx, double fy, double cx, double cy,
                          int32_t w, int32_t h, const double R0[9], const double t0[3], const orc_pose_cfg* pc,
                          int32_t budget, double R_out[9], double t_out[3], double* final_loss,
                          int32_t* converged) {
  TrainConfig cfg;
  cfg.estimate_pose_steps = budget;
  cfg.cam_lr_start = pc->cam_lr_start;
  cfg.cam_lr_end = pc->cam_lr_end;
  cfg.loss.beta = pc->beta;
  cfg.pose_converged_eps = pc->pose_converged_eps;
  cfg.background = Vec3(pc->background[0], pc->background[1], pc->background[2]);
  cfg.raster = to_config(&pc->raster);
  Intrinsics intr{fx, fy, cx, cy, w, h};
  PoseEstimate est = estimate_pose(to_cloud(cloud), to_image(image, w, h), intr, to_pose(R0, t0), cfg);
  from_pose(est.pose, R_out, t_out);
  if (final_loss) *final_loss = est.final_loss;
  if (converged) *converged = est.converged ? 1 : 0;
  return est.steps_used;
}

// The body of pose_descent (pipelines.cpp:66-90) over the public calls, with
// traces of the pose / loss / d_pose BEFORE each step (the orc_estimate_pose
// trace convention). Returns steps_used; best pose out.
int32_t ref_pose_descent_traced(const orc_cloud* cloud, const double* image, double fx, double fy, double cx,
                                double cy, int32_t w, int32_t h, const double R0[9], const double t0[3],
                                const orc_pose_cfg* pc, int32_t budget, double R_out[9], double t_out[3],
                                double* final_loss, int32_t* converged, double* trace_pose, double* trace_loss,
                                double* trace_dpose) {
  const GaussianCloud g = to_cloud(cloud);
  const Image target = to_image(image, w, h);
  const RasterConfig rc = to_config(&pc->raster);
  const Vec3 bg(pc->background[0], pc->background[1], pc->background[2]);
  Se3Pose pose = to_pose(R0, t0), best = pose;
  PoseAdam adam;
  Scalar best_loss = std::numeric_limits<Scalar>::infinity(), best_value = 0.0;
  bool conv = false;
  int used = 0;
  for (int t = 0; t < budget; ++t) {
    Camera cam;
    cam.fx = fx;
    cam.fy = fy;
    cam.cx = cx;
    cam.cy = cy;
    cam.width = w;
    cam.height = h;
    cam.world_to_cam = pose;
    RenderOutput out = render(g, cam, bg, rc);
    Image d_image;
    Scalar loss = rgb_loss(out.image, target, pc->beta, &d_image);
    if (trace_pose) to_pose12(pose, trace_pose + 12 * t);
    if (trace_loss) trace_loss[t] = loss;
    if (loss < best_loss) {
      best_loss = loss;
      best = pose;
      best_value = loss;
    }
    if (loss < 1e-14) {
      conv = true;
      used = t + 1;
      if (trace_dpose) std::memset(trace_dpose + 6 * t, 0, 6 * sizeof(double));
      break;
    }
    GradientBundle grads = render_backward(g, cam, out, d_image);
    if (trace_dpose)
      for (int k = 0; k < 6; ++k) trace_dpose[6 * t + k] = grads.d_pose(k);
    Scalar lr = schedule(ScheduleKind::cosine, pc->cam_lr_start, pc->cam_lr_end, t, budget);
    Tangent6 applied;
    pose = pose_step(pose, grads.d_pose, lr, &adam, &applied);
    used = t + 1;
    if (applied.norm() < pc->pose_converged_eps) {
      conv = true;
      break;
    }
  }
  from_pose(best, R_out, t_out);
  if (final_loss) *final_loss = best_value;
  if (converged) *converged = conv ? 1 : 0;
  return used;
}

// tests/gradcheck.hpp:28-67 — the reference's own scene draw.
void ref_make_gradcheck_scene(orc_rng* rng, int32_t n, int32_t image_size, orc_cloud* cloud, orc_camera* cam,
                              double bg[3]) {
  Rng r(1);
  std::memcpy(static_cast<void*>(&r), &rng->state, sizeof(uint64_t));
  testing::GradCheckScene s = testing::make_gradcheck_scene(r, n, image_size);
  std::memcpy(&rng->state, static_cast<void*>(&r), sizeof(uint64_t));
  from_cloud(s.cloud, cloud);
  from_camera(s.camera, cam);
  for (int c = 0; c < 3; ++c) bg[c] = s.background(c);
}

// tests/gradcheck.hpp:69-161
int ref_scene_is_conditioned(const orc_cloud* cloud, const orc_camera* cam, const double bg[3],
                             const orc_raster_config* cfg) {
  testing::GradCheckScene s{to_cloud(cloud), to_camera(cam), Vec3(bg[0], bg[1], bg[2])};
  return testing::gradcheck_scene_is_conditioned(s, to_config(cfg)) ? 1 : 0;
}

// tests/gradcheck.hpp:201-254 — the reference's FD gate.
double ref_gradcheck(const orc_cloud* cloud, const orc_camera* cam, const double bg[3], const orc_raster_config* cfg,
                     orc_rng* rng, double step, int32_t* checked, char* worst_label) {
  testing::GradCheckScene s{to_cloud(cloud), to_camera(cam), Vec3(bg[0], bg[1], bg[2])};
  Rng r(1);
  std::memcpy(static_cast<void*>(&r), &rng->state, sizeof(uint64_t));
  testing::GradCheckResult res = testing::gradcheck_scene(s, to_config(cfg), r, step);
  std::memcpy(&rng->state, static_cast<void*>(&r), sizeof(uint64_t));
  if (checked) *checked = res.checked;
  if (worst_label) {
    std::strncpy(worst_label, res.worst.c_str(), 31);
    worst_label[31] = 0;
  }
  return res.max_err;
}

// synth.cpp:33-135: cloud + poses (+ images when `images` is non-null,
// cameras*H*W*3). kind: 0 orbit, 1 forward-facing, 2 random-walk.
void ref_synth_scene(int32_t gaussians, int32_t cameras, int32_t width, int32_t height, int32_t kind,
                     int32_t sh_degree, uint64_t seed, orc_cloud* cloud, double* poses, double* images) {
  SynthSpec spec;
  spec.gaussians = gaussians;
  spec.cameras = cameras;
  spec.width = width;
  spec.height = height;
  spec.trajectory = kind == 0 ? TrajectoryKind::orbit
                              : (kind == 1 ? TrajectoryKind::forward_facing : TrajectoryKind::random_walk);
  spec.sh_degree = sh_degree;
  SynthScene s = synth_scene(spec, seed);
  from_cloud(s.gt_cloud, cloud);
  for (int k = 0; k < cameras; ++k) {
    to_pose12(s.bundle.poses[k], poses + 12 * k);
    if (images)
      std::memcpy(images + static_cast<std::size_t>(k) * width * height * 3, s.bundle.images[k].data.data(),
                  s.bundle.images[k].data.size() * sizeof(double));
  }
}

// eval.cpp:130-152
void ref_perturb_pose(const double R[9], const double t[3], double rot_deg, double trans, orc_rng* rng,
                      double R_out[9], double t_out[3]) {
  Rng r(1);
  std::memcpy(static_cast<void*>(&r), &rng->state, sizeof(uint64_t));
  Se3Pose p = perturb_pose(to_pose(R, t), rot_deg, trans, r);
  std::memcpy(&rng->state, static_cast<void*>(&r), sizeof(uint64_t));
  from_pose(p, R_out, t_out);
}

void ref_perturb_pose_tangent(const double R[9], const double t[3], double sigma, orc_rng* rng, double R_out[9],
                              double t_out[3]) {
  Rng r(1);
  std::memcpy(static_cast<void*>(&r), &rng->state, sizeof(uint64_t));
  Se3Pose p = perturb_pose_tangent(to_pose(R, t), sigma, r);
  std::memcpy(&rng->state, static_cast<void*>(&r), sizeof(uint64_t));
  from_pose(p, R_out, t_out);
}

// pipelines.cpp:96-216: the reference's joint_optimize (optimize_poses as
// configured, no gt stats, no checkpoints). The cloud is replaced in place
// (the input's arrays are freed with free(): pass calloc/orc_cloud_alloc
// memory). trace_total / trace_l1 (iterations) from the StepStats history.
int32_t ref_joint_optimize(orc_cloud* cloud, const double* const* images, int32_t n_views, double fx, double fy,
                           double cx, double cy, int32_t w, int32_t h, double* poses, const orc_joint_cfg* jc,
                           int32_t slots, orc_rng* rng, double* trace_total, double* trace_l1) {
  if (slots != 1) {  // the reference loop trains one view per step (pipelines.cpp:120-180)
    g_last_error = "ref_joint_optimize: the reference loop has exactly one slot per step";
    return static_cast<int>(ErrorCode::invalid_config) + 1;
  }
  TrainConfig cfg;
  cfg.iterations = jc->iterations;
  cfg.cam_lr_start = jc->cam_lr_start;
  cfg.cam_lr_end = jc->cam_lr_end;
  cfg.pos_lr_start = jc->pos_lr_start;
  cfg.pos_lr_end = jc->pos_lr_end;
  cfg.rot_lr = jc->rot_lr;
  cfg.scale_lr = jc->scale_lr;
  cfg.opacity_lr = jc->opacity_lr;
  cfg.sh_dc_lr = jc->sh_dc_lr;
  cfg.sh_rest_lr = jc->sh_rest_lr;
  cfg.opacity_l1_steps = jc->opacity_l1_steps;
  cfg.sh_degree = jc->sh_degree;
  cfg.sh_degree_interval = jc->sh_degree_interval;
  cfg.loss.beta = jc->beta;
  cfg.loss.aniso_ratio = jc->aniso_ratio;
  cfg.loss.opacity_l1_weight = jc->opacity_l1_weight;
  cfg.background = Vec3(jc->background[0], jc->background[1], jc->background[2]);
  cfg.raster = to_config(&jc->raster);
  // densify_interval <= 0 means "off" in orc_joint_cfg; the reference has no
  // off switch (pipelines.cpp:182-183 takes t % interval), so start past the end.
  cfg.densify_interval = jc->densify_interval > 0 ? jc->densify_interval : 100;
  cfg.densify_start = jc->densify_interval > 0 ? jc->densify_start : jc->iterations + 1;
  cfg.densify_stop = jc->densify_interval > 0 ? jc->densify_stop : jc->iterations + 1;
  cfg.n_target = jc->n_target;
  cfg.grad_threshold = jc->grad_threshold;
  cfg.densify_size_ratio = jc->densify_size_ratio;
  cfg.prune_opacity = jc->prune_opacity;
  std::vector<Image> imgs;
  for (int v = 0; v < n_views; ++v) imgs.push_back(to_image(images[v], w, h));
  std::vector<Se3Pose> init;
  for (int v = 0; v < n_views; ++v) init.push_back(Se3Pose::from_flat(poses + 12 * v));
  Intrinsics intr{fx, fy, cx, cy, w, h};
  Rng r(1);
  std::memcpy(static_cast<void*>(&r), &rng->state, sizeof(uint64_t));
  try {
    JointResult res = joint_optimize(imgs, intr, init, to_cloud(cloud), cfg, r, nullptr, nullptr,
                                     jc->optimize_poses != 0);
    std::memcpy(&rng->state, static_cast<void*>(&r), sizeof(uint64_t));
    ref_cloud_free(cloud);
    from_cloud(res.cloud, cloud);
    for (int v = 0; v < n_views; ++v) to_pose12(res.poses[v], poses + 12 * v);
    for (std::size_t s = 0; s < res.history.size() && s < static_cast<std::size_t>(cfg.iterations); ++s) {
      if (trace_total) trace_total[s] = res.history[s].total;
      if (trace_l1) trace_l1[s] = res.history[s].l1;
    }
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return static_cast<int>(e.code) + 1;
  }
}

}  // extern "C"
