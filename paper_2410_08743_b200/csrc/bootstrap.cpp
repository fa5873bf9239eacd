// bootstrap.cpp — the bootstrap path: the callers on
// either side of pose_descent that turn RGB-D frames into an initial
// trajectory. Host orchestration over the public C-ABI only; every render,
// loss, backward and optimiser step runs in the device kernels of the hot path.
//
//   gsb_unproject              scene.cpp:209-243 (host: an O(pixels) gather)
//   gsb_init_from_points       scene.cpp:182-207, kNN on the device
//   gsb_fit_frame_gaussians    pipelines.cpp:224-250
//   gsb_estimate_relative_pose pipelines.cpp:252-290
//   gsb_bootstrap_trajectory   pipelines.cpp:292-312
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "gsb_internal.cuh"

namespace gsb {
int launch_knn3_mean(cudaStream_t st, const double* pts, int64_t n, double* out);
}

namespace {

struct ErrGuard {  // destroys what a bootstrap step created on every exit
  gsb_frame* frame = nullptr;
  gsb_grads* grads = nullptr;
  gsb_adam* adam = nullptr;
  gsb_image* image = nullptr;
  ~ErrGuard() {
    gsb_grads_destroy(grads);
    gsb_adam_destroy(adam);
    gsb_image_destroy(image);
    gsb_frame_destroy(frame);
  }
};

gsb_camera make_camera(const double intr[4], int32_t W, int32_t H, const double R[9], const double t[3]) {
  gsb_camera c;
  c.fx = intr[0];
  c.fy = intr[1];
  c.cx = intr[2];
  c.cy = intr[3];
  c.width = W;
  c.height = H;
  std::memcpy(c.R, R, sizeof c.R);
  std::memcpy(c.t, t, sizeof c.t);
  return c;
}

void to_pose12(const double R[9], const double t[3], double* p) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) p[r * 4 + c] = R[r * 3 + c];
    p[r * 4 + 3] = t[r];
  }
}

void from_pose12(const double* p, double R[9], double t[3]) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) R[r * 3 + c] = p[r * 4 + c];
    t[r] = p[r * 4 + 3];
  }
}

const double kI[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
const double kZ[3] = {0, 0, 0};

}  // namespace

extern "C" {

void gsb_default_bootstrap_config(gsb_bootstrap_config* c) {  // trainer.hpp:21-60, losses.hpp:15-19
  c->per_frame_fit_steps = 100;
  c->relpose_steps = 200;
  c->unproject_points = 50000;
  c->pos_lr_start = 1.6e-2;
  c->pos_lr_end = 1.6e-4;
  c->rot_lr = 1e-3;
  c->scale_lr = 5e-3;
  c->opacity_lr = 5e-2;
  c->sh_dc_lr = 2.5e-3;
  c->sh_rest_lr = 2.5e-3 / 20.0;
  c->relpose_lr_start = 1e-3;
  c->relpose_lr_end = 1e-4;
  c->beta = 0.2;
  c->mask_threshold = 0.99;
  c->background[0] = c->background[1] = c->background[2] = 0.0;
  gsb_default_raster_config(&c->raster);
}

int gsb_unproject(const double* depth, const uint8_t* valid, int32_t W, int32_t H, const double* frame,
                  const double intr[4], const double world_to_cam[12], int32_t max_points, double* points_out,
                  double* colors_out, int64_t* n_out) {
  if (!depth || !valid || !frame || !intr || !world_to_cam || !points_out || !colors_out || !n_out || W <= 0 ||
      H <= 0)
    return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "unproject: null argument");
  if (max_points < 1) return gsb::fail(GSB_ERR_INVALID_CONFIG, "unproject: max_points must be >= 1");
  const int64_t P = (int64_t)W * H;
  std::vector<int64_t> pix;
  pix.reserve((size_t)P);
  for (int64_t p = 0; p < P; ++p)
    if (valid[p] && std::isfinite(depth[p]) && depth[p] > 0.0) pix.push_back(p);
  if (pix.empty()) return gsb::fail(GSB_ERR_NO_VALID_DEPTH, "unproject: empty validity mask");
  const int64_t count = (int64_t)pix.size();
  const int64_t stride = (count + max_points - 1) / max_points;
  double R[9], t[3], Ri[9], ti[3];
  from_pose12(world_to_cam, R, t);
  for (int i = 0; i < 3; ++i)  // cam_to_world = (R^T, -R^T t) (lie.hpp inverse)
    for (int j = 0; j < 3; ++j) Ri[i * 3 + j] = R[j * 3 + i];
  for (int i = 0; i < 3; ++i) ti[i] = -(Ri[i * 3] * t[0] + Ri[i * 3 + 1] * t[1] + Ri[i * 3 + 2] * t[2]);
  int64_t out = 0;
  for (int64_t idx = 0; idx < count; idx += stride) {
    const int64_t p = pix[idx];
    const int x = (int)(p % W), y = (int)(p / W);
    const double d = depth[p];
    const double ray[3] = {(x - intr[2]) / intr[0], (y - intr[3]) / intr[1], 1.0};
    const double q[3] = {d * ray[0], d * ray[1], d * ray[2]};
    for (int k = 0; k < 3; ++k) {
      points_out[3 * out + k] = (Ri[k * 3] * q[0] + Ri[k * 3 + 1] * q[1] + Ri[k * 3 + 2] * q[2]) + ti[k];
      colors_out[3 * out + k] = frame[p * 3 + k];
    }
    ++out;
  }
  *n_out = out;
  return GSB_OK;
}

int gsb_init_from_points(gsb_ctx* ctx, const double* points, const double* colors, int64_t n, int32_t sh_degree,
                         gsb_cloud** out) {
  if (!ctx || !points || !colors || !out) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (n < 4) return gsb::fail(GSB_ERR_DEGENERATE_CLOUD, "init_from_points: need at least 4 points");
  if (sh_degree < 0 || sh_degree > 3) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "sh_degree");
  cudaSetDevice(ctx->device);
  // mean_knn_distance(points, 3) on the device: exact k nearest distances,
  // FP64 with the reference's rounding
  gsb::DevBuf d_pts, d_nn;
  GSB_CUDA(d_pts.reserve(sizeof(double) * 3 * n));
  GSB_CUDA(d_nn.reserve(sizeof(double) * n));
  GSB_CUDA(cudaMemcpyAsync(d_pts.p, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->stream));
  if (int r = gsb::launch_knn3_mean(ctx->stream, d_pts.as<double>(), n, d_nn.as<double>())) return r;
  ctx->launches += 1;
  std::vector<double> nn(n);
  GSB_CUDA(cudaMemcpyAsync(nn.data(), d_nn.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  d_pts.release();
  d_nn.release();
  const int B = (sh_degree + 1) * (sh_degree + 1);
  std::vector<double> rot(4 * n, 0.0), ls(3 * n), op(n, std::log(0.1 / (1.0 - 0.1))), sh(3 * B * n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    rot[4 * i] = 1.0;
    const double s = std::log(std::fmax(nn[i], 1e-7));
    ls[3 * i] = ls[3 * i + 1] = ls[3 * i + 2] = s;
    for (int c = 0; c < 3; ++c) sh[(size_t)i * 3 * B + c * B] = (colors[3 * i + c] - 0.5) / 0.28209479177387814;
  }
  gsb_cloud* cloud = nullptr;
  if (int r = gsb_cloud_create(ctx, n, sh_degree, &cloud)) return r;
  if (int r = gsb_cloud_upload(cloud, points, rot.data(), ls.data(), op.data(), sh.data(), 0)) {
    gsb_cloud_destroy(cloud);
    return r;
  }
  *out = cloud;
  return GSB_OK;
}

int gsb_fit_frame_gaussians(gsb_ctx* ctx, const double* frame, const double* depth, const uint8_t* valid, int32_t W,
                            int32_t H, const double intr[4], const gsb_bootstrap_config* cfg, gsb_cloud** out) {
  if (!ctx || !frame || !depth || !valid || !intr || !cfg || !out)
    return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  const int32_t maxp = cfg->unproject_points;
  if (maxp < 1) return gsb::fail(GSB_ERR_INVALID_CONFIG, "unproject: max_points must be >= 1");
  std::vector<double> pts(3 * (size_t)maxp), cols(3 * (size_t)maxp);
  int64_t np = 0;
  double I12[12];
  to_pose12(kI, kZ, I12);
  if (int r = gsb_unproject(depth, valid, W, H, frame, intr, I12, maxp, pts.data(), cols.data(), &np)) return r;
  gsb_cloud* cloud = nullptr;
  if (int r = gsb_init_from_points(ctx, pts.data(), cols.data(), np, 0, &cloud)) return r;
  ErrGuard g;
  int r = gsb_frame_create(ctx, &g.frame);
  if (!r) r = gsb_grads_create(ctx, cloud, &g.grads);
  if (!r) r = gsb_adam_create(ctx, cloud, &g.adam);
  if (!r) r = gsb_image_create(ctx, frame, W, H, &g.image);
  const gsb_camera cam = make_camera(intr, W, H, kI, kZ);
  for (int32_t t = 0; !r && t < cfg->per_frame_fit_steps; ++t) {
    r = gsb_render(ctx, cloud, &cam, cfg->background, &cfg->raster, g.frame, nullptr);
    if (!r) r = gsb_frame_rgb_loss(ctx, g.frame, g.image, cfg->beta, nullptr);
    if (!r) r = gsb_render_backward_device(ctx, cloud, &cam, g.frame, 0u, g.grads, nullptr);
    if (r) break;
    const double lrs[6] = {gsb_schedule(1, cfg->pos_lr_start, cfg->pos_lr_end, t, cfg->per_frame_fit_steps),
                           cfg->rot_lr, cfg->scale_lr, cfg->opacity_lr, cfg->sh_dc_lr, cfg->sh_rest_lr};
    r = gsb_cloud_adam_step(ctx, cloud, g.grads, g.adam, lrs);
  }
  if (r) {
    gsb_cloud_destroy(cloud);
    return r;
  }
  *out = cloud;
  return GSB_OK;
}

int gsb_estimate_relative_pose(gsb_ctx* ctx, gsb_cloud* cloud, const double* frame_next, int32_t W, int32_t H,
                               const double intr[4], const gsb_bootstrap_config* cfg, double pose_out[12],
                               int32_t* ok_out, double* final_loss) {
  if (!ctx || !cloud || !frame_next || !intr || !cfg || !pose_out)
    return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  to_pose12(kI, kZ, pose_out);
  if (ok_out) *ok_out = 0;
  if (final_loss) *final_loss = 0.0;
  ErrGuard g;
  if (int r = gsb_frame_create(ctx, &g.frame)) return r;
  if (int r = gsb_image_create(ctx, frame_next, W, H, &g.image)) return r;
  gsb_pose_adam adam;
  std::memset(&adam, 0, sizeof adam);
  double pose[12];
  to_pose12(kI, kZ, pose);
  double best = INFINITY, lr_scale = 1.0;
  const double n_pix = (double)W * (double)H;
  for (int32_t t = 0; t < cfg->relpose_steps; ++t) {
    double R[9], tr[3];
    from_pose12(pose, R, tr);
    const gsb_camera cam = make_camera(intr, W, H, R, tr);
    if (int r = gsb_render(ctx, cloud, &cam, cfg->background, &cfg->raster, g.frame, nullptr)) return r;
    double loss = 0.0;
    int64_t masked = 0;
    int r = gsb_frame_masked_rgb_loss(ctx, g.frame, g.image, cfg->beta, cfg->mask_threshold, &loss, &masked);
    if (r == GSB_ERR_EMPTY_MASK) {  // diverged out of the rendered geometry: failure, identity
      to_pose12(kI, kZ, pose_out);
      if (ok_out) *ok_out = 0;
      return GSB_OK;
    }
    if (r) return r;
    if ((double)masked < 0.05 * n_pix) lr_scale *= 0.5;  // divergence guard
    if (loss < best) {
      best = loss;
      std::memcpy(pose_out, pose, sizeof pose);
      if (final_loss) *final_loss = loss;
    }
    double d_pose[6];
    if (int r2 = gsb_render_backward_device(ctx, cloud, &cam, g.frame, GSB_BWD_POSE_ONLY, nullptr, d_pose)) return r2;
    const double lr = lr_scale * gsb_schedule(0, cfg->relpose_lr_start, cfg->relpose_lr_end, t, cfg->relpose_steps);
    double next[12], applied[6];
    if (int r2 = gsb_pose_step(ctx, pose, d_pose, lr, &adam, next, applied)) return r2;
    std::memcpy(pose, next, sizeof pose);
  }
  if (ok_out) *ok_out = 1;
  return GSB_OK;
}

int gsb_bootstrap_trajectory(gsb_ctx* ctx, const double* const* frames, const double* const* depths,
                             const uint8_t* const* valids, int32_t n_frames, int32_t W, int32_t H,
                             const double intr[4], const gsb_bootstrap_config* cfg, double* poses_out,
                             int32_t* pair_ok) {
  if (!ctx || !frames || !depths || !valids || !intr || !cfg || !poses_out)
    return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (n_frames < 2) return gsb::fail(GSB_ERR_INVALID_CONFIG, "bootstrap_trajectory: need >= 2 frames with depths");
  double R[9], t[3];
  std::memcpy(R, kI, sizeof R);
  std::memcpy(t, kZ, sizeof t);
  to_pose12(R, t, poses_out);
  for (int32_t f = 0; f + 1 < n_frames; ++f) {
    gsb_cloud* cloud = nullptr;
    if (int r = gsb_fit_frame_gaussians(ctx, frames[f], depths[f], valids[f], W, H, intr, cfg, &cloud)) return r;
    double rel[12];
    int32_t ok = 0;
    double fl = 0.0;
    const int r = gsb_estimate_relative_pose(ctx, cloud, frames[f + 1], W, H, intr, cfg, rel, &ok, &fl);
    gsb_cloud_destroy(cloud);
    if (r) return r;
    if (pair_ok) pair_ok[f] = ok;
    double Rr[9], trr[3], Rn[9], tn[3];  // world_to_cam[f+1] = rel * world_to_cam[f] (lie.hpp:48-53)
    from_pose12(rel, Rr, trr);
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) Rn[i * 3 + j] = Rr[i * 3] * R[j] + Rr[i * 3 + 1] * R[3 + j] + Rr[i * 3 + 2] * R[6 + j];
      tn[i] = (Rr[i * 3] * t[0] + Rr[i * 3 + 1] * t[1] + Rr[i * 3 + 2] * t[2]) + trr[i];
    }
    std::memcpy(R, Rn, sizeof R);
    std::memcpy(t, tn, sizeof t);
    to_pose12(R, t, poses_out + 12 * (f + 1));
  }
  return GSB_OK;
}

}  // extern "C"
