// synth.cpp — deterministic synthetic inputs for benchmarks and tests:
// the reference's cloud / camera draw sequence (synth.cpp:33-101), its Rng
// (core.hpp:58-102) and perturb_pose (eval.cpp:130-146). Input generation
// only; nothing here is on the hot path. Vec3(rng(), rng(), rng())
// constructor arguments are drawn right to left, matching a GCC x86-64
// build of the reference.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "gsb_internal.cuh"

namespace {

struct Rng {  // core.hpp:58-102
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed ? seed : 0x9e3779b97f4a7c15ull) {}
  uint64_t next() {
    uint64_t x = s;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    s = x;
    return x * 0x2545f4914f6cdd1dull;
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    double u1 = uniform();
    double u2 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
  void unit_quaternion(double q[4]) {
    for (;;) {
      q[3] = normal();
      q[2] = normal();
      q[1] = normal();
      q[0] = normal();
      if (!(std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) < 1e-12)) break;
    }
    const double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int k = 0; k < 4; ++k) q[k] = q[k] / n;
  }
};

constexpr double kSh0 = 0.28209479177387814;

// synth.cpp:45-62 for one Gaussian.
void draw_gaussian(Rng& rng, int basis, double* mean, double* q, double* ls, double* op, double* sh) {
  mean[2] = rng.uniform(-0.8, 0.8);
  mean[1] = rng.uniform(-0.8, 0.8);
  mean[0] = rng.uniform(-0.8, 0.8);
  rng.unit_quaternion(q);
  const double base = std::exp(rng.uniform(std::log(0.03), std::log(0.10)));
  for (int k = 0; k < 3; ++k) ls[k] = std::log(base) + rng.uniform(-0.35, 0.35);
  const double o = rng.uniform(0.55, 0.9);
  *op = std::log(o / (1.0 - o));
  for (int c = 0; c < 3; ++c) {
    sh[c * basis] = (rng.uniform(0.15, 0.85) - 0.5) / kSh0;
    for (int b = 1; b < basis; ++b) {
      const double scale = b < 4 ? 0.08 : 0.03;
      sh[c * basis + b] = rng.uniform(-scale, scale);
    }
  }
}

void mat3_vec(const double* a, const double* v, double* out) {
  double r[3];
  for (int i = 0; i < 3; ++i) r[i] = a[i * 3] * v[0] + a[i * 3 + 1] * v[1] + a[i * 3 + 2] * v[2];
  for (int i = 0; i < 3; ++i) out[i] = r[i];
}
void mat3_mul(const double* a, const double* b, double* out) {
  double r[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i * 3 + j] = a[i * 3] * b[j] + a[i * 3 + 1] * b[3 + j] + a[i * 3 + 2] * b[6 + j];
  for (int k = 0; k < 9; ++k) out[k] = r[k];
}

// synth.cpp:19-31
void look_at(const double eye[3], const double target[3], double R[9], double t[3]) {
  double f[3] = {target[0] - eye[0], target[1] - eye[1], target[2] - eye[2]};
  const double fn = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
  for (double& v : f) v /= fn;
  double up[3] = {0, 1, 0};
  if (std::fabs(f[0] * up[0] + f[1] * up[1] + f[2] * up[2]) > 0.999) {
    up[0] = 1;
    up[1] = 0;
  }
  double right[3] = {up[1] * f[2] - up[2] * f[1], up[2] * f[0] - up[0] * f[2], up[0] * f[1] - up[1] * f[0]};
  const double rn = std::sqrt(right[0] * right[0] + right[1] * right[1] + right[2] * right[2]);
  for (double& v : right) v /= rn;
  const double down[3] = {f[1] * right[2] - f[2] * right[1], f[2] * right[0] - f[0] * right[2],
                          f[0] * right[1] - f[1] * right[0]};
  for (int k = 0; k < 3; ++k) {
    R[k] = right[k];
    R[3 + k] = down[k];
    R[6 + k] = f[k];
  }
  double re[3];
  mat3_vec(R, eye, re);
  for (int k = 0; k < 3; ++k) t[k] = -re[k];
}

// so3_exp (lie.cpp:55-60) with series_coeffs (26-43)
void so3_exp(const double w[3], double R[9]) {
  const double th = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  const double t2 = th * th;
  double a, b;
  if (th < 1e-8) {
    a = 1.0 - t2 / 6.0;
    b = 0.5 - t2 / 24.0;
  } else {
    const double hs = std::sin(0.5 * th);
    a = std::sin(th) / th;
    b = 2.0 * hs * hs / t2;
  }
  const double W[9] = {0.0, -w[2], w[1], w[2], 0.0, -w[0], -w[1], w[0], 0.0};
  double W2[9];
  mat3_mul(W, W, W2);
  for (int k = 0; k < 9; ++k) R[k] = ((k % 4 == 0) ? 1.0 : 0.0) + a * W[k] + b * W2[k];
}

// se3_exp (lie.cpp:117-129): rotation as so3_exp, translation V(omega) v
void se3_exp(const double tau[6], double R[9], double t[3]) {
  const double* w = tau + 3;
  so3_exp(w, R);
  const double th = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  const double t2 = th * th;
  double b, d;
  if (th < 1e-8) {
    b = 0.5 - t2 / 24.0;
  } else {
    const double hs = std::sin(0.5 * th);
    b = 2.0 * hs * hs / t2;
  }
  d = th < 1e-2 ? 1.0 / 6.0 - t2 / 120.0 + t2 * t2 / 5040.0 : (th - std::sin(th)) / (t2 * th);
  const double W[9] = {0.0, -w[2], w[1], w[2], 0.0, -w[0], -w[1], w[0], 0.0};
  double W2[9], V[9];
  mat3_mul(W, W, W2);
  for (int k = 0; k < 9; ++k) V[k] = ((k % 4 == 0) ? 1.0 : 0.0) + b * W[k] + d * W2[k];
  mat3_vec(V, tau, t);
}

}  // namespace

extern "C" {

// pipelines.cpp:122-129: `order` starts as iota and is shuffled in place at
// every epoch start (j = rng.uniform_int(0, i) for i = n-1 .. 1).
int gsb_joint_schedule(uint64_t seed, int32_t n_views, int64_t count, int32_t* seq_out) {
  if (n_views <= 0 || count < 0 || (count > 0 && !seq_out))
    return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "bad joint schedule arguments");
  Rng rng(seed);
  std::vector<int32_t> order(n_views);
  for (int32_t i = 0; i < n_views; ++i) order[i] = i;
  for (int64_t k = 0; k < count; ++k) {
    if (k % n_views == 0)
      for (int32_t i = n_views - 1; i > 0; --i) {
        const int32_t j = (int32_t)(rng.next() % (uint64_t)(i + 1));  // core.hpp:78-80
        std::swap(order[i], order[j]);
      }
    seq_out[k] = order[k % n_views];
  }
  return GSB_OK;
}

// The split children's normals of densify_and_prune (trainer.cpp:215-219):
// per child one rng->normal3(), whose Vec3(normal(), normal(), normal())
// arguments a GCC build draws right to left. out: children x 3 (x, y, z).
int gsb_rng_child_normals(uint64_t* rng_state, int64_t children, double* out) {
  if (!rng_state || children < 0 || (children > 0 && !out)) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  Rng rng(1);
  rng.s = *rng_state ? *rng_state : 0x9e3779b97f4a7c15ull;
  for (int64_t c = 0; c < children; ++c) {
    out[3 * c + 2] = rng.normal();
    out[3 * c + 1] = rng.normal();
    out[3 * c + 0] = rng.normal();
  }
  *rng_state = rng.s;
  return GSB_OK;
}

// Epoch shuffle of pipelines.cpp:123-129 on a caller-held order and rng state.
int gsb_rng_shuffle(uint64_t* rng_state, int32_t n, int32_t* order) {
  if (!rng_state || n < 0 || (n > 0 && !order)) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  Rng rng(1);
  rng.s = *rng_state ? *rng_state : 0x9e3779b97f4a7c15ull;
  for (int32_t i = n - 1; i > 0; --i) {
    const int32_t j = (int32_t)(rng.next() % (uint64_t)(i + 1));
    std::swap(order[i], order[j]);
  }
  *rng_state = rng.s;
  return GSB_OK;
}

// perturb_pose_tangent (eval.cpp:148-152): Exp(sigma * N(0, I_6)) * pose
int gsb_perturb_pose_tangent(const double pose[12], double sigma, uint64_t* rng_state, double out[12]) {
  if (!pose || !rng_state || !out) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  Rng rng(1);
  rng.s = *rng_state ? *rng_state : 0x9e3779b97f4a7c15ull;
  double tau[6];
  for (int k = 0; k < 6; ++k) tau[k] = sigma * rng.normal();
  *rng_state = rng.s;
  double Re[9], te[3], R[9], t[3], Rn[9], tn[3];
  se3_exp(tau, Re, te);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) R[r * 3 + c] = pose[r * 4 + c];
    t[r] = pose[r * 4 + 3];
  }
  mat3_mul(Re, R, Rn);
  mat3_vec(Re, t, tn);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) out[r * 4 + c] = Rn[r * 3 + c];
    out[r * 4 + 3] = tn[r] + te[r];
  }
  return GSB_OK;
}

// Initial cloud of the joint tests (tests/test_trainer.cpp:598-601): means +=
// mean_sigma * normal3 (GCC draws z, y, x), then per Gaussian log-scales +=
// log_scale_range * uniform(-1, 1) (one draw for all three axes).
int gsb_cloud_jitter(gsb_cloud* cloud, uint64_t seed, double mean_sigma, double log_scale_range) {
  if (!cloud) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null cloud");
  const int64_t n = cloud->n;
  const int basis = (cloud->sh_degree + 1) * (cloud->sh_degree + 1);
  std::vector<double> means(3 * n), rot(4 * n), ls(3 * n), op(n), sh((size_t)3 * basis * n);
  if (int r = gsb_cloud_download(cloud, means.data(), rot.data(), ls.data(), op.data(), sh.data())) return r;
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) {
    const double z = rng.normal(), y = rng.normal(), x = rng.normal();
    means[3 * i] += mean_sigma * x;
    means[3 * i + 1] += mean_sigma * y;
    means[3 * i + 2] += mean_sigma * z;
  }
  if (log_scale_range != 0.0)
    for (int64_t i = 0; i < n; ++i) {
      const double u = log_scale_range * rng.uniform(-1.0, 1.0);
      for (int k = 0; k < 3; ++k) ls[3 * i + k] += u;
    }
  return gsb_cloud_upload(cloud, means.data(), rot.data(), ls.data(), op.data(), sh.data(), cloud->active_sh_degree);
}


int gsb_cloud_synth(gsb_cloud* cloud, uint64_t seed, double log_scale_offset) {
  if (!cloud) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null cloud");
  const int64_t n = cloud->n;
  const int basis = (cloud->sh_degree + 1) * (cloud->sh_degree + 1);
  std::vector<double> means(3 * n), rot(4 * n), ls(3 * n), op(n), sh((size_t)3 * basis * n);
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) {
    draw_gaussian(rng, basis, &means[3 * i], &rot[4 * i], &ls[3 * i], &op[i], &sh[(size_t)3 * basis * i]);
    for (int k = 0; k < 3; ++k) ls[3 * i + k] += log_scale_offset;
  }
  return gsb_cloud_upload(cloud, means.data(), rot.data(), ls.data(), op.data(), sh.data(), cloud->sh_degree);
}

int gsb_synth_poses(uint64_t seed, int64_t n, int32_t sh_degree, int32_t kind, int32_t cameras, double orbit_radius,
                    double orbit_arc, double* poses) {
  if (!poses || cameras < 0 || n < 0 || sh_degree < 0 || sh_degree > 3)
    return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "bad synth_poses arguments");
  const int basis = (sh_degree + 1) * (sh_degree + 1);
  Rng rng(seed);
  std::vector<double> scratch(3 * basis);
  double mean[3], q[4], ls[3], op;
  for (int64_t i = 0; i < n; ++i) draw_gaussian(rng, basis, mean, q, ls, &op, scratch.data());
  double walker[3] = {0, 0, -orbit_radius};
  for (int k = 0; k < cameras; ++k) {  // synth.cpp:73-101
    double eye[3];
    if (kind == 0) {
      const double theta = orbit_arc * (double)k / (double)(cameras > 1 ? cameras : 1);
      const double phi = 0.25 * std::sin(3.0 * theta);
      eye[0] = orbit_radius * (std::sin(theta) * std::cos(phi));
      eye[1] = orbit_radius * std::sin(phi);
      eye[2] = orbit_radius * (-std::cos(theta) * std::cos(phi));
    } else if (kind == 1) {
      eye[2] = -orbit_radius + rng.uniform(-0.15, 0.15);
      eye[1] = rng.uniform(-0.4, 0.4);
      eye[0] = rng.uniform(-0.4, 0.4);
    } else {
      if (k > 0) {
        const double n2 = rng.normal(), n1 = rng.normal(), n0 = rng.normal();
        walker[0] += 0.08 * n0;
        walker[1] += 0.08 * n1;
        walker[2] += 0.08 * n2;
      }
      for (int j = 0; j < 3; ++j) eye[j] = walker[j];
    }
    double target[3] = {0, 0, 0};
    if (kind == 2) {
      const double jy = 0.05 * rng.normal();
      const double jx = 0.05 * rng.normal();
      target[0] = jx;
      target[1] = jy;
    }
    double R[9], t[3];
    look_at(eye, target, R, t);
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) poses[12 * k + r * 4 + c] = R[r * 3 + c];
      poses[12 * k + r * 4 + 3] = t[r];
    }
  }
  return GSB_OK;
}

int gsb_perturb_pose(const double pose[12], double rot_deg, double trans, uint64_t* rng_state, double out[12]) {
  if (!pose || !rng_state || !out) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  Rng rng(1);
  rng.s = *rng_state ? *rng_state : 0x9e3779b97f4a7c15ull;
  const double to_rad = M_PI / 180.0;
  const double ax = rng.uniform(-rot_deg, rot_deg) * to_rad;
  const double ay = rng.uniform(-rot_deg, rot_deg) * to_rad;
  const double az = rng.uniform(-rot_deg, rot_deg) * to_rad;
  double off[3];
  off[2] = rng.uniform(-trans, trans);
  off[1] = rng.uniform(-trans, trans);
  off[0] = rng.uniform(-trans, trans);
  *rng_state = rng.s;
  const double wz[3] = {0, 0, az}, wy[3] = {0, ay, 0}, wx[3] = {ax, 0, 0};
  double Rz[9], Ry[9], Rx[9], tmp[9], rot[9];
  so3_exp(wz, Rz);
  so3_exp(wy, Ry);
  so3_exp(wx, Rx);
  mat3_mul(Rz, Ry, tmp);
  mat3_mul(tmp, Rx, rot);
  double R[9], t[3], Rcw[9], tcw[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) R[r * 3 + c] = pose[r * 4 + c];
    t[r] = pose[r * 4 + 3];
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rcw[i * 3 + j] = R[j * 3 + i];
  for (int i = 0; i < 3; ++i) tcw[i] = -(R[0 * 3 + i] * t[0] + R[1 * 3 + i] * t[1] + R[2 * 3 + i] * t[2]);
  double Rn[9];
  mat3_mul(Rcw, rot, Rn);
  for (int k = 0; k < 3; ++k) tcw[k] += off[k];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) out[i * 4 + j] = Rn[j * 3 + i];
    out[i * 4 + 3] = -(Rn[0 * 3 + i] * tcw[0] + Rn[1 * 3 + i] * tcw[1] + Rn[2 * 3 + i] * tcw[2]);
  }
  return GSB_OK;
}

}  // extern "C"
