/*
 * gsopt_oracle.c — TEST INFRASTRUCTURE ONLY (see gsopt_oracle.h).
 *
 * Clean-room FP64 CPU restatement of the reference hot path. Citations are
 * relative to /root/reference/proj. Parallel loops mirror the reference's
 * parallel_for fan-out (core.cpp:101-117) with OpenMP over disjoint outputs,
 * so results are schedule independent exactly as in the reference.
 *
 * Third-party arithmetic: the reference uses Eigen3 (>= 3.3, unpinned, not
 * vendored). Its small fixed-size products are restated as left-to-right
 * sums; JacobiSVD (used by Se3Pose::orthonormalize, lie.cpp:87-97) is
 * restated from Eigen's published two-sided Jacobi algorithm below.
 */
#include "gsopt_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------ core */
/* core.hpp:58-102 */
void orc_rng_init(orc_rng* r, uint64_t seed) { r->state = seed ? seed : 0x9e3779b97f4a7c15ull; }
uint64_t orc_rng_next(orc_rng* r) {
  uint64_t x = r->state;
  x ^= x >> 12;
  x ^= x << 25;
  x ^= x >> 27;
  r->state = x;
  return x * 0x2545f4914f6cdd1dull;
}
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }
double orc_rng_uniform_range(orc_rng* r, double lo, double hi) { return lo + (hi - lo) * orc_rng_uniform(r); }
int64_t orc_rng_uniform_int(orc_rng* r, int64_t lo, int64_t hi) {
  return lo + (int64_t)(orc_rng_next(r) % (uint64_t)(hi - lo + 1));
}
double orc_rng_normal(orc_rng* r) {
  double u1 = orc_rng_uniform(r);
  double u2 = orc_rng_uniform(r);
  while (u1 <= 0.0) u1 = orc_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * ORC_PI * u2);
}
/* Vec3(normal(), normal(), normal()) under GCC's right-to-left argument
 * evaluation (core.hpp:91). */
static void rng_normal3(orc_rng* r, double out[3]) {
  out[2] = orc_rng_normal(r);
  out[1] = orc_rng_normal(r);
  out[0] = orc_rng_normal(r);
}
static double norm4(const double q[4]) { return sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]); }
/* core.hpp:94-98 */
static void rng_unit_quaternion(orc_rng* r, double q[4]) {
  for (;;) {
    q[3] = orc_rng_normal(r);
    q[2] = orc_rng_normal(r);
    q[1] = orc_rng_normal(r);
    q[0] = orc_rng_normal(r);
    if (!(norm4(q) < 1e-12)) break;
  }
  double n = norm4(q);
  for (int k = 0; k < 4; ++k) q[k] = q[k] / n;
}
static inline double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); } /* core.hpp:112 */
static inline double logit(double p) { return log(p / (1.0 - p)); }    /* core.hpp:113 */

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------ small linalg */
static void mat3_mul(const double a[9], const double b[9], double out[9]) {
  double r[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i * 3 + j] = a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j] + a[i * 3 + 2] * b[2 * 3 + j];
  memcpy(out, r, sizeof r);
}
static void mat3_T(const double a[9], double out[9]) {
  double r[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i * 3 + j] = a[j * 3 + i];
  memcpy(out, r, sizeof r);
}
static void mat3_vec(const double a[9], const double v[3], double out[3]) {
  double r[3];
  for (int i = 0; i < 3; ++i) r[i] = a[i * 3 + 0] * v[0] + a[i * 3 + 1] * v[1] + a[i * 3 + 2] * v[2];
  memcpy(out, r, sizeof r);
}
static void mat3T_vec(const double a[9], const double v[3], double out[3]) {
  double r[3];
  for (int i = 0; i < 3; ++i) r[i] = a[0 * 3 + i] * v[0] + a[1 * 3 + i] * v[1] + a[2 * 3 + i] * v[2];
  memcpy(out, r, sizeof r);
}
static double det3(const double a[9]) {
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) + a[2] * (a[3] * a[7] - a[4] * a[6]);
}
static void skew3(const double v[3], double s[9]) { /* lie.cpp:47-53 */
  s[0] = 0.0; s[1] = -v[2]; s[2] = v[1];
  s[3] = v[2]; s[4] = 0.0; s[5] = -v[0];
  s[6] = -v[1]; s[7] = v[0]; s[8] = 0.0;
}
static double norm3(const double v[3]) { return sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }
/* Se3Pose::act (lie.hpp:38) */
static void pose_act(const double R[9], const double t[3], const double p[3], double out[3]) {
  double r[3];
  mat3_vec(R, p, r);
  out[0] = r[0] + t[0];
  out[1] = r[1] + t[1];
  out[2] = r[2] + t[2];
}
/* Camera::center (rasterizer.hpp:24) */
static void cam_center(const orc_camera* cam, double c[3]) {
  double r[3];
  mat3T_vec(cam->R, cam->t, r);
  c[0] = -r[0];
  c[1] = -r[1];
  c[2] = -r[2];
}

/* ------------------------------------------------------------------ lie */
/* lie.cpp:26-43 */
typedef struct { double a, b, d; } series_t;
static series_t series_coeffs(double theta) {
  series_t o;
  double t2 = theta * theta;
  if (theta < 1e-8) {
    o.a = 1.0 - t2 / 6.0;
    o.b = 0.5 - t2 / 24.0;
  } else {
    double half_sin = sin(0.5 * theta);
    o.a = sin(theta) / theta;
    o.b = 2.0 * half_sin * half_sin / t2;
  }
  if (theta < 1e-2) o.d = 1.0 / 6.0 - t2 / 120.0 + t2 * t2 / 5040.0;
  else o.d = (theta - sin(theta)) / (t2 * theta);
  return o;
}
/* lie.cpp:55-60 */
void orc_so3_exp(const double w[3], double R[9]) {
  double theta = norm3(w);
  series_t c = series_coeffs(theta);
  double W[9], W2[9];
  skew3(w, W);
  mat3_mul(W, W, W2);
  for (int k = 0; k < 9; ++k) R[k] = ((k % 4 == 0) ? 1.0 : 0.0) + c.a * W[k] + c.b * W2[k];
}
/* lie.cpp:117-129 */
void orc_se3_exp(const double tau[6], double R[9], double t[3]) {
  const double* v = tau;
  const double* w = tau + 3;
  double theta = norm3(w);
  series_t c = series_coeffs(theta);
  double W[9], W2[9], V[9];
  skew3(w, W);
  mat3_mul(W, W, W2);
  for (int k = 0; k < 9; ++k) {
    double I = (k % 4 == 0) ? 1.0 : 0.0;
    R[k] = I + c.a * W[k] + c.b * W2[k];
    V[k] = I + c.b * W[k] + c.d * W2[k];
  }
  mat3_vec(V, v, t);
}
/* lie.cpp:79-85 */
double orc_rotation_angle(const double R[9]) {
  double sa[3] = {R[7] - R[5], R[2] - R[6], R[3] - R[1]};
  double s = 0.5 * norm3(sa);
  double c = ((R[0] + R[4] + R[8]) - 1.0) * 0.5;
  if (c < -1.0) c = -1.0;
  if (c > 1.0) c = 1.0;
  return atan2(s, c);
}

/* Eigen JacobiSVD (two-sided Jacobi, real 3x3) restated: real_2x2_jacobi_svd,
 * JacobiRotation::makeJacobi, applyOnTheLeft/Right, sign fix and descending
 * sort. Used by orthonormalize (lie.cpp:87-97). */
typedef struct { double c, s; } jrot;
static void rot_rows(double M[9], int p, int q, jrot j) { /* applyOnTheLeft(p,q,j) */
  for (int i = 0; i < 3; ++i) {
    double x = M[p * 3 + i], y = M[q * 3 + i];
    M[p * 3 + i] = j.c * x + j.s * y;
    M[q * 3 + i] = -j.s * x + j.c * y;
  }
}
static void rot_cols(double M[9], int p, int q, jrot j) { /* applyOnTheRight(p,q,j) */
  jrot t = {j.c, -j.s};
  for (int i = 0; i < 3; ++i) {
    double x = M[i * 3 + p], y = M[i * 3 + q];
    M[i * 3 + p] = t.c * x + t.s * y;
    M[i * 3 + q] = -t.s * x + t.c * y;
  }
}
static void jacobi_svd3(const double A[9], double U[9], double S[3], double V[9]) {
  const double eps = 2.220446049250313e-16, min_pos = 2.2250738585072014e-308;
  double M[9];
  double scale = 0.0;
  for (int k = 0; k < 9; ++k) scale = fmax(scale, fabs(A[k]));
  if (scale == 0.0) scale = 1.0;
  for (int k = 0; k < 9; ++k) M[k] = A[k] / scale;
  for (int k = 0; k < 9; ++k) U[k] = V[k] = (k % 4 == 0) ? 1.0 : 0.0;
  double precision = 2.0 * eps;
  double max_diag = fmax(fabs(M[0]), fmax(fabs(M[4]), fabs(M[8])));
  int finished = 0, sweeps = 0;
  while (!finished && sweeps < 100) {
    finished = 1;
    ++sweeps;
    for (int p = 1; p < 3; ++p) {
      for (int q = 0; q < p; ++q) {
        double threshold = fmax(min_pos, precision * max_diag);
        if (fabs(M[p * 3 + q]) > threshold || fabs(M[q * 3 + p]) > threshold) {
          finished = 0;
          /* real_2x2_jacobi_svd(M, p, q) */
          double m00 = M[p * 3 + p], m01 = M[p * 3 + q], m10 = M[q * 3 + p], m11 = M[q * 3 + q];
          jrot rot1;
          double tt = m00 + m11, d = m10 - m01;
          if (fabs(d) < min_pos) {
            rot1.s = 0.0;
            rot1.c = 1.0;
          } else {
            double u = tt / d;
            double tmp = sqrt(1.0 + u * u);
            rot1.s = 1.0 / tmp;
            rot1.c = u / tmp;
          }
          /* m.applyOnTheLeft(0,1,rot1) */
          double n00 = rot1.c * m00 + rot1.s * m10, n01 = rot1.c * m01 + rot1.s * m11;
          double n11 = -rot1.s * m01 + rot1.c * m11;
          /* j_right.makeJacobi(m,0,1) on (x=n00, y=n01, z=n11) */
          jrot jr;
          double deno = 2.0 * fabs(n01);
          if (deno < min_pos) {
            jr.c = 1.0;
            jr.s = 0.0;
          } else {
            double tau = (n00 - n11) / deno;
            double w = sqrt(tau * tau + 1.0);
            double t = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
            double sign_t = t > 0.0 ? 1.0 : -1.0;
            double n = 1.0 / sqrt(t * t + 1.0);
            jr.s = -sign_t * (n01 / fabs(n01)) * fabs(t) * n;
            jr.c = n;
          }
          /* j_left = rot1 * j_right.transpose() */
          jrot jrt = {jr.c, -jr.s};
          jrot jl = {rot1.c * jrt.c - rot1.s * jrt.s, rot1.c * jrt.s + rot1.s * jrt.c};
          rot_rows(M, p, q, jl);
          jrot jlt = {jl.c, -jl.s};
          rot_cols(U, p, q, jlt);
          rot_cols(M, p, q, jr);
          rot_cols(V, p, q, jr);
          max_diag = fmax(max_diag, fmax(fabs(M[p * 3 + p]), fabs(M[q * 3 + q])));
        }
      }
    }
  }
  for (int i = 0; i < 3; ++i) {
    double a = M[i * 3 + i];
    S[i] = fabs(a);
    if (a < 0.0)
      for (int r = 0; r < 3; ++r) U[r * 3 + i] = -U[r * 3 + i];
  }
  for (int i = 0; i < 3; ++i) S[i] *= scale;
  /* sort descending (selection, swapping columns of U and V) */
  for (int i = 0; i < 3; ++i) {
    int best = i;
    for (int k = i + 1; k < 3; ++k)
      if (S[k] > S[best]) best = k;
    if (best != i) {
      double ts = S[i]; S[i] = S[best]; S[best] = ts;
      for (int r = 0; r < 3; ++r) {
        double tu = U[r * 3 + i]; U[r * 3 + i] = U[r * 3 + best]; U[r * 3 + best] = tu;
        double tv = V[r * 3 + i]; V[r * 3 + i] = V[r * 3 + best]; V[r * 3 + best] = tv;
      }
    }
  }
}
/* lie.cpp:87-97 */
void orc_orthonormalize(double R[9]) {
  double U[9], S[3], V[9], Vt[9], r[9];
  jacobi_svd3(R, U, S, V);
  mat3_T(V, Vt);
  mat3_mul(U, Vt, r);
  if (det3(r) < 0.0) {
    for (int k = 0; k < 3; ++k) U[k * 3 + 2] *= -1.0;
    mat3_mul(U, Vt, r);
  }
  memcpy(R, r, sizeof r);
}

/* ---------------------------------------------------------------- scene */
/* scene.cpp:46-54 */
void orc_quat_to_rotation(const double qr[4], double R[9]) {
  double n = norm4(qr);
  double w = qr[0] / n, x = qr[1] / n, y = qr[2] / n, z = qr[3] / n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}
/* scene.cpp:56-88; out = 4 matrices of 9 */
void orc_quat_rotation_jacobian(const double qr[4], double out[36]) {
  double norm = norm4(qr);
  double q[4] = {qr[0] / norm, qr[1] / norm, qr[2] / norm, qr[3] / norm};
  double w = q[0], x = q[1], y = q[2], z = q[3];
  double unit[4][9] = {
      {0, -z, y, z, 0, -x, -y, x, 0},
      {0, y, z, y, -2 * x, -w, z, w, -2 * x},
      {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
      {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
  for (int m = 0; m < 4; ++m)
    for (int k = 0; k < 9; ++k) unit[m][k] *= 2.0;
  for (int k = 0; k < 4; ++k) {
    double acc[9] = {0};
    for (int j = 0; j < 4; ++j) {
      double dj = ((j == k) ? 1.0 : 0.0) - q[j] * q[k];
      double f = dj / norm;
      for (int e = 0; e < 9; ++e) acc[e] += unit[j][e] * f;
    }
    memcpy(out + 9 * k, acc, sizeof acc);
  }
}
/* scene.cpp:90-94 */
void orc_covariance3d(const double q[4], const double s[3], double out[9]) {
  double r[9], m[9];
  orc_quat_to_rotation(q, r);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i * 3 + j] = r[i * 3 + j] * s[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) out[i * 3 + j] = m[i * 3 + 0] * m[j * 3 + 0] + m[i * 3 + 1] * m[j * 3 + 1] + m[i * 3 + 2] * m[j * 3 + 2];
}

/* ------------------------------------------------------------------- sh */
/* sh.cpp:9-14 */
static const double kC1 = 0.4886025119029199;
static const double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                              -1.0925484305920792, 0.5462742152960396};
static const double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                              0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                              -0.5900435899266435};
static const double kSh0 = 0.28209479177387814; /* sh.hpp:13 */
static inline int sh_count(int d) { return (d + 1) * (d + 1); }

/* sh.cpp:18-40 */
void orc_sh_basis(const double dir[3], int degree, double* out) {
  const double x = dir[0], y = dir[1], z = dir[2];
  out[0] = kSh0;
  if (degree < 1) return;
  out[1] = -kC1 * y;
  out[2] = kC1 * z;
  out[3] = -kC1 * x;
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  out[4] = kC2[0] * x * y;
  out[5] = kC2[1] * y * z;
  out[6] = kC2[2] * (2.0 * zz - xx - yy);
  out[7] = kC2[3] * x * z;
  out[8] = kC2[4] * (xx - yy);
  if (degree < 3) return;
  out[9] = kC3[0] * y * (3.0 * xx - yy);
  out[10] = kC3[1] * x * y * z;
  out[11] = kC3[2] * y * (4.0 * zz - xx - yy);
  out[12] = kC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  out[13] = kC3[4] * x * (4.0 * zz - xx - yy);
  out[14] = kC3[5] * z * (xx - yy);
  out[15] = kC3[6] * x * (xx - 3.0 * yy);
}
/* sh.cpp:42-64; out[b*3 + k] */
void orc_sh_basis_gradient(const double dir[3], int degree, double* g) {
  const double x = dir[0], y = dir[1], z = dir[2];
#define SETG(b, a0, a1, a2, s) do { g[(b)*3+0] = (s) * (a0); g[(b)*3+1] = (s) * (a1); g[(b)*3+2] = (s) * (a2); } while (0)
  g[0] = g[1] = g[2] = 0.0;
  if (degree < 1) return;
  g[3] = 0.0; g[4] = -kC1; g[5] = 0.0;
  g[6] = 0.0; g[7] = 0.0; g[8] = kC1;
  g[9] = -kC1; g[10] = 0.0; g[11] = 0.0;
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  SETG(4, y, x, 0.0, kC2[0]);
  SETG(5, 0.0, z, y, kC2[1]);
  SETG(6, -2.0 * x, -2.0 * y, 4.0 * z, kC2[2]);
  SETG(7, z, 0.0, x, kC2[3]);
  SETG(8, 2.0 * x, -2.0 * y, 0.0, kC2[4]);
  if (degree < 3) return;
  SETG(9, 6.0 * x * y, 3.0 * xx - 3.0 * yy, 0.0, kC3[0]);
  SETG(10, y * z, x * z, x * y, kC3[1]);
  SETG(11, -2.0 * x * y, 4.0 * zz - xx - 3.0 * yy, 8.0 * y * z, kC3[2]);
  SETG(12, -6.0 * x * z, -6.0 * y * z, 6.0 * zz - 3.0 * xx - 3.0 * yy, kC3[3]);
  SETG(13, 4.0 * zz - 3.0 * xx - yy, -2.0 * x * y, 8.0 * x * z, kC3[4]);
  SETG(14, 2.0 * x * z, -2.0 * y * z, xx - yy, kC3[5]);
  SETG(15, 3.0 * xx - 3.0 * yy, -6.0 * x * y, 0.0, kC3[6]);
#undef SETG
}
/* sh.cpp:66-84 (channel stride = (degree+1)^2 — the reference's forward quirk) */
void orc_sh_eval(const double* coeffs, const double dir[3], int degree, double rgb[3], uint8_t* mask) {
  double basis[16];
  const int n = sh_count(degree);
  orc_sh_basis(dir, degree, basis);
  uint8_t m = 0;
  for (int c = 0; c < 3; ++c) {
    double v = 0.5;
    const double* ch = coeffs + c * n;
    for (int b = 0; b < n; ++b) v += ch[b] * basis[b];
    if (v < 0.0) {
      m |= (uint8_t)(1u << c);
      v = 0.0;
    }
    rgb[c] = v;
  }
  if (mask) *mask = m;
}

/* ----------------------------------------------------------- rasterizer */
void orc_default_raster_config(orc_raster_config* c) { /* rasterizer.hpp:30-38 */
  c->tile_size = 16;
  c->cutoff_sigma = 3.0;
  c->alpha_clamp = 0.99;
  c->dilation = 0.3;
  c->early_termination = 1e-4;
  c->z_near = 0.01;
  c->deterministic = 1;
}
/* rasterizer.cpp:31-39 */
static void projection_jacobian(const double mu_cam[3], const orc_camera* cam, double J[6]) {
  const double x = mu_cam[0], y = mu_cam[1], z = mu_cam[2];
  const double iz = 1.0 / z;
  const double iz2 = iz * iz;
  J[0] = cam->fx * iz; J[1] = 0.0; J[2] = -cam->fx * x * iz2;
  J[3] = 0.0; J[4] = cam->fy * iz; J[5] = -cam->fy * y * iz2;
}
/* rasterizer.cpp:185-190 */
void orc_project(const double mu[3], const orc_camera* cam, double mu2d[2], double* depth) {
  double mc[3];
  pose_act(cam->R, cam->t, mu, mc);
  *depth = mc[2];
  mu2d[0] = cam->fx * mc[0] / mc[2] + cam->cx;
  mu2d[1] = cam->fy * mc[1] / mc[2] + cam->cy;
}
/* rasterizer.cpp:192-199: m = J R, cov = (m Sigma) m^T + dilation I */
void orc_covariance2d(const double sigma[9], const double mu_cam[3], const orc_camera* cam,
                      double dilation, double out[4]) {
  double J[6], m[6], ms[6];
  projection_jacobian(mu_cam, cam, J);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j) m[i * 3 + j] = J[i * 3 + 0] * cam->R[0 * 3 + j] + J[i * 3 + 1] * cam->R[1 * 3 + j] + J[i * 3 + 2] * cam->R[2 * 3 + j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j) ms[i * 3 + j] = m[i * 3 + 0] * sigma[0 * 3 + j] + m[i * 3 + 1] * sigma[1 * 3 + j] + m[i * 3 + 2] * sigma[2 * 3 + j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) out[i * 2 + j] = ms[i * 3 + 0] * m[j * 3 + 0] + ms[i * 3 + 1] * m[j * 3 + 1] + ms[i * 3 + 2] * m[j * 3 + 2];
  out[0] += dilation;
  out[3] += dilation;
}
/* rasterizer.cpp:201-207 */
double orc_splat_alpha(const double mu2d[2], const double conic[4], double opacity,
                       const double pixel[2], double alpha_clamp, double cutoff_sigma) {
  double d0 = pixel[0] - mu2d[0], d1 = pixel[1] - mu2d[1];
  double c0 = conic[0] * d0 + conic[1] * d1, c1 = conic[2] * d0 + conic[3] * d1;
  double g = d0 * c0 + d1 * c1;
  if (g > cutoff_sigma * cutoff_sigma) return 0.0;
  double a = opacity * exp(-0.5 * g);
  return a < alpha_clamp ? a : alpha_clamp;
}

/* rasterizer.cpp:41-48 */
static uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
/* rasterizer.cpp:52-73. Eigen Mat3 is column-major: rotation.data() hashes
 * the column-major sequence. */
uint64_t orc_fingerprint(const orc_cloud* cloud, const orc_camera* cam) {
  uint64_t h = 0xcbf29ce484222325ull;
  int64_t n = cloud->n;
  h = fnv1a(h, &n, sizeof n);
  h = fnv1a(h, &cloud->sh_degree, sizeof(int32_t));
  h = fnv1a(h, &cloud->active_sh_degree, sizeof(int32_t));
  double f4[4] = {cam->fx, cam->fy, cam->cx, cam->cy};
  h = fnv1a(h, f4, sizeof f4);
  int32_t wh[2] = {cam->width, cam->height};
  h = fnv1a(h, wh, sizeof wh);
  double colmajor[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) colmajor[j * 3 + i] = cam->R[i * 3 + j];
  h = fnv1a(h, colmajor, sizeof colmajor);
  h = fnv1a(h, cam->t, sizeof(double) * 3);
  if (n > 0) {
    const int basis = sh_count(cloud->sh_degree);
    int64_t stride = n / 64 > 1 ? n / 64 : 1;
    for (int64_t i = 0; i < n; i += stride) {
      h = fnv1a(h, cloud->means + 3 * i, sizeof(double) * 3);
      h = fnv1a(h, cloud->rotations + 4 * i, sizeof(double) * 4);
      h = fnv1a(h, cloud->log_scales + 3 * i, sizeof(double) * 3);
      h = fnv1a(h, cloud->opacity_logits + i, sizeof(double));
      h = fnv1a(h, cloud->sh + (size_t)i * 3 * basis, sizeof(double) * 3 * basis);
    }
  }
  return h;
}

/* stable sort of splats by depth (rasterizer.cpp:131-132): merge sort */
static void merge_sort_splats(orc_splat* a, orc_splat* tmp, int64_t n) {
  if (n < 2) return;
  int64_t h = n / 2;
  merge_sort_splats(a, tmp, h);
  merge_sort_splats(a + h, tmp, n - h);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) {
    if (a[j].depth < a[i].depth) tmp[k++] = a[j++];
    else tmp[k++] = a[i++];
  }
  while (i < h) tmp[k++] = a[i++];
  while (j < n) tmp[k++] = a[j++];
  memcpy(a, tmp, sizeof(orc_splat) * n);
}

static inline int clampi_d(double v, int n_tiles) { /* rasterizer.cpp:140-143 */
  double hi = n_tiles - 1.0;
  double c = v < 0.0 ? 0.0 : (v > hi ? hi : v);
  return (int)c;
}
static void tile_span(double mux, double muy, double r, int tile, int tx_n, int ty_n, int* tx0, int* tx1,
                      int* ty0, int* ty1) {
  double t = (double)tile;
  *tx0 = clampi_d(floor((mux - r) / t), tx_n);
  *tx1 = clampi_d(floor((mux + r) / t), tx_n);
  *ty0 = clampi_d(floor((muy - r) / t), ty_n);
  *ty1 = clampi_d(floor((muy + r) / t), ty_n);
}

/* rasterizer.cpp:134-168 — count / prefix / fill over depth-sorted records */
static int32_t* bin_splats(const double* mux, const double* muy, const double* rad, int64_t n_splats, int tile,
                           int tiles_x, int tiles_y, int32_t* ranges, int64_t* total_out) {
  const int n_tiles = tiles_x * tiles_y;
  int32_t* counts = (int32_t*)calloc(n_tiles > 0 ? n_tiles : 1, sizeof(int32_t));
  for (int64_t s = 0; s < n_splats; ++s) {
    int tx0, tx1, ty0, ty1;
    tile_span(mux[s], muy[s], rad[s], tile, tiles_x, tiles_y, &tx0, &tx1, &ty0, &ty1);
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) ++counts[ty * tiles_x + tx];
  }
  int64_t total = 0;
  for (int t = 0; t < n_tiles; ++t) {
    ranges[2 * t] = (int32_t)total;
    total += counts[t];
    ranges[2 * t + 1] = (int32_t)total;
  }
  int32_t* lists = (int32_t*)malloc(sizeof(int32_t) * (total > 0 ? total : 1));
  for (int t = 0; t < n_tiles; ++t) counts[t] = ranges[2 * t];
  for (int64_t s = 0; s < n_splats; ++s) {
    int tx0, tx1, ty0, ty1;
    tile_span(mux[s], muy[s], rad[s], tile, tiles_x, tiles_y, &tx0, &tx1, &ty0, &ty1);
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) lists[counts[ty * tiles_x + tx]++] = (int32_t)s;
  }
  free(counts);
  *total_out = total;
  return lists;
}

/* rasterizer.cpp:83-170 */
static void prepare(const orc_cloud* cloud, const orc_camera* cam, const orc_raster_config* cfg,
                    orc_render_out* out) {
  const int64_t n = cloud->n;
  double cc[3];
  cam_center(cam, cc);
  const int degree = cloud->active_sh_degree < cloud->sh_degree ? cloud->active_sh_degree : cloud->sh_degree;
  const int basis_cap = sh_count(cloud->sh_degree);
  out->tiles_x = (cam->width + cfg->tile_size - 1) / cfg->tile_size;
  out->tiles_y = (cam->height + cfg->tile_size - 1) / cfg->tile_size;

  orc_splat* cand = (orc_splat*)malloc(sizeof(orc_splat) * (n > 0 ? n : 1));
  uint8_t* keep = (uint8_t*)calloc(n > 0 ? n : 1, 1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* mean = cloud->means + 3 * i;
    double mu_cam[3];
    pose_act(cam->R, cam->t, mean, mu_cam);
    if (!(mu_cam[2] > cfg->z_near)) continue;
    double mu2d[2], depth;
    orc_project(mean, cam, mu2d, &depth);
    if (!isfinite(mu2d[0]) || !isfinite(mu2d[1])) continue;
    double s[3] = {exp(cloud->log_scales[3 * i]), exp(cloud->log_scales[3 * i + 1]), exp(cloud->log_scales[3 * i + 2])};
    double sigma[9], cov[4];
    orc_covariance3d(cloud->rotations + 4 * i, s, sigma);
    orc_covariance2d(sigma, mu_cam, cam, cfg->dilation, cov);
    /* max_eigenvalue_2x2 (rasterizer.cpp:24-28) */
    double mid = 0.5 * (cov[0] + cov[3]);
    double diff = 0.5 * (cov[0] - cov[3]);
    double lmax = mid + sqrt(diff * diff + cov[1] * cov[2]);
    double radius = cfg->cutoff_sigma * sqrt(lmax);
    if (!(radius > 0.0) || !isfinite(radius)) continue;
    if (mu2d[0] + radius < 0.0 || mu2d[0] - radius > cam->width - 1 || mu2d[1] + radius < 0.0 ||
        mu2d[1] - radius > cam->height - 1)
      continue;
    orc_splat rec;
    memset(&rec, 0, sizeof rec);
    rec.gaussian = (int32_t)i;
    rec.mu2d[0] = mu2d[0];
    rec.mu2d[1] = mu2d[1];
    rec.depth = depth;
    /* invert_spd2 (rasterizer.cpp:17-22) */
    double det = cov[0] * cov[3] - cov[1] * cov[2];
    rec.conic[0] = cov[3] / det;
    rec.conic[1] = -cov[1] / det;
    rec.conic[2] = -cov[2] / det;
    rec.conic[3] = cov[0] / det;
    double dir[3] = {mean[0] - cc[0], mean[1] - cc[1], mean[2] - cc[2]};
    double dn = norm3(dir);
    dir[0] /= dn; dir[1] /= dn; dir[2] /= dn;
    orc_sh_eval(cloud->sh + (size_t)i * 3 * basis_cap, dir, degree, rec.color, &rec.color_clamped);
    rec.opacity = sigmoid(cloud->opacity_logits[i]);
    rec.radius = radius;
    cand[i] = rec;
    keep[i] = 1;
  }
  int64_t v = 0;
  for (int64_t i = 0; i < n; ++i) if (keep[i]) cand[v++] = cand[i];
  orc_splat* tmp = (orc_splat*)malloc(sizeof(orc_splat) * (v > 0 ? v : 1));
  merge_sort_splats(cand, tmp, v);
  free(tmp);
  free(keep);
  out->splats = cand;
  out->n_splats = v;

  double* mux = (double*)malloc(sizeof(double) * (v > 0 ? v : 1));
  double* muy = (double*)malloc(sizeof(double) * (v > 0 ? v : 1));
  double* rad = (double*)malloc(sizeof(double) * (v > 0 ? v : 1));
  for (int64_t s2 = 0; s2 < v; ++s2) {
    mux[s2] = cand[s2].mu2d[0];
    muy[s2] = cand[s2].mu2d[1];
    rad[s2] = cand[s2].radius;
  }
  const int n_tiles = out->tiles_x * out->tiles_y;
  out->tile_ranges = (int32_t*)malloc(sizeof(int32_t) * 2 * (n_tiles > 0 ? n_tiles : 1));
  out->tile_lists = bin_splats(mux, muy, rad, v, cfg->tile_size, out->tiles_x, out->tiles_y, out->tile_ranges,
                               &out->n_entries);
  free(mux);
  free(muy);
  free(rad);
}

int64_t orc_bin_records(int64_t n, const uint8_t* keep, const double* mu2d, const double* radius,
                        const double* depth, int32_t width, int32_t height, int32_t tile_size,
                        int32_t* sorted_gaussian, int64_t* n_splats, int32_t* tile_lists, int64_t cap,
                        int32_t* tile_ranges) {
  orc_splat* cand = (orc_splat*)malloc(sizeof(orc_splat) * (n > 0 ? n : 1));
  int64_t v = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!keep[i]) continue;
    memset(&cand[v], 0, sizeof(orc_splat));
    cand[v].gaussian = (int32_t)i;
    cand[v].mu2d[0] = mu2d[2 * i];
    cand[v].mu2d[1] = mu2d[2 * i + 1];
    cand[v].radius = radius[i];
    cand[v].depth = depth[i];
    ++v;
  }
  orc_splat* tmp = (orc_splat*)malloc(sizeof(orc_splat) * (v > 0 ? v : 1));
  merge_sort_splats(cand, tmp, v);
  free(tmp);
  double* mux = (double*)malloc(sizeof(double) * (v > 0 ? v : 1));
  double* muy = (double*)malloc(sizeof(double) * (v > 0 ? v : 1));
  double* rad = (double*)malloc(sizeof(double) * (v > 0 ? v : 1));
  for (int64_t s = 0; s < v; ++s) {
    mux[s] = cand[s].mu2d[0];
    muy[s] = cand[s].mu2d[1];
    rad[s] = cand[s].radius;
    sorted_gaussian[s] = cand[s].gaussian;
  }
  int tx = (width + tile_size - 1) / tile_size, ty = (height + tile_size - 1) / tile_size;
  int64_t total = 0;
  int32_t* lists = bin_splats(mux, muy, rad, v, tile_size, tx, ty, tile_ranges, &total);
  *n_splats = v;
  if (total <= cap) memcpy(tile_lists, lists, sizeof(int32_t) * total);
  free(lists);
  free(mux);
  free(muy);
  free(rad);
  free(cand);
  return total <= cap ? total : -1;
}

/* rasterizer.cpp:209-281 */
orc_render_out* orc_render(const orc_cloud* cloud, const orc_camera* cam, const double bg[3],
                           const orc_raster_config* cfg) {
  orc_render_out* out = (orc_render_out*)calloc(1, sizeof(orc_render_out));
  out->camera = *cam;
  memcpy(out->background, bg, sizeof(double) * 3);
  out->config = *cfg;
  out->n_gaussians = cloud->n;
  out->state_fingerprint = orc_fingerprint(cloud, cam);
  out->width = cam->width;
  out->height = cam->height;
  prepare(cloud, cam, cfg, out);

  const size_t n_pix = (size_t)cam->width * cam->height;
  out->image = (double*)calloc(n_pix * 3 + 1, sizeof(double));
  out->accum_transmittance = (double*)calloc(n_pix + 1, sizeof(double));
  out->final_transmittance = (double*)malloc(sizeof(double) * (n_pix + 1));
  out->contrib_count = (int32_t*)calloc(n_pix + 1, sizeof(int32_t));
  out->overflow_mask = (uint8_t*)calloc(n_pix + 1, 1);
  for (size_t p = 0; p < n_pix; ++p) out->final_transmittance[p] = 1.0;

  const double cutoff2 = cfg->cutoff_sigma * cfg->cutoff_sigma;
  const int n_tiles = out->tiles_x * out->tiles_y;
#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < n_tiles; ++t) {
    const int tx = t % out->tiles_x, ty = t / out->tiles_x;
    const int x0 = tx * cfg->tile_size, y0 = ty * cfg->tile_size;
    const int x1 = x0 + cfg->tile_size < cam->width ? x0 + cfg->tile_size : cam->width;
    const int y1 = y0 + cfg->tile_size < cam->height ? y0 + cfg->tile_size : cam->height;
    const int32_t lb = out->tile_ranges[2 * t], le = out->tile_ranges[2 * t + 1];
    for (int y = y0; y < y1; ++y) {
      for (int x = x0; x < x1; ++x) {
        const double px = (double)x, py = (double)y;
        double T = 1.0, col[3] = {0, 0, 0};
        int32_t processed = 0;
        for (int32_t e = lb; e < le; ++e) {
          const orc_splat* rec = &out->splats[out->tile_lists[e]];
          processed = e - lb + 1;
          double d0 = px - rec->mu2d[0], d1 = py - rec->mu2d[1];
          double c0 = rec->conic[0] * d0 + rec->conic[1] * d1, c1 = rec->conic[2] * d0 + rec->conic[3] * d1;
          double g = d0 * c0 + d1 * c1;
          if (g > cutoff2) continue;
          double a = rec->opacity * exp(-0.5 * g);
          double alpha = cfg->alpha_clamp < a ? cfg->alpha_clamp : a;
          double w = alpha * T;
          col[0] += rec->color[0] * w;
          col[1] += rec->color[1] * w;
          col[2] += rec->color[2] * w;
          T *= (1.0 - alpha);
          if (T < cfg->early_termination) break;
        }
        col[0] += bg[0] * T;
        col[1] += bg[1] * T;
        col[2] += bg[2] * T;
        const size_t pix = (size_t)y * cam->width + x;
        uint8_t of = 0;
        for (int c = 0; c < 3; ++c)
          if (col[c] > 1.0) {
            col[c] = 1.0;
            of |= (uint8_t)(1u << c);
          }
        out->image[pix * 3 + 0] = col[0];
        out->image[pix * 3 + 1] = col[1];
        out->image[pix * 3 + 2] = col[2];
        out->final_transmittance[pix] = T;
        out->accum_transmittance[pix] = 1.0 - T;
        out->contrib_count[pix] = processed;
        out->overflow_mask[pix] = of;
      }
    }
  }
  return out;
}

void orc_render_free(orc_render_out* out) {
  if (!out) return;
  free(out->image);
  free(out->accum_transmittance);
  free(out->final_transmittance);
  free(out->contrib_count);
  free(out->overflow_mask);
  free(out->splats);
  free(out->tile_lists);
  free(out->tile_ranges);
  free(out);
}

void orc_grads_alloc(orc_grads* g, const orc_cloud* cloud) { /* rasterizer.cpp:174-183 */
  const int64_t n = cloud->n;
  g->n = n;
  g->sh_len = n * 3 * sh_count(cloud->sh_degree);
  g->d_means = (double*)calloc(n * 3 + 1, sizeof(double));
  g->d_rotations = (double*)calloc(n * 4 + 1, sizeof(double));
  g->d_log_scales = (double*)calloc(n * 3 + 1, sizeof(double));
  g->d_opacity_logits = (double*)calloc(n + 1, sizeof(double));
  g->d_sh = (double*)calloc(g->sh_len + 1, sizeof(double));
  g->d_mu2d = (double*)calloc(n * 2 + 1, sizeof(double));
  memset(g->d_pose, 0, sizeof g->d_pose);
}
void orc_grads_free(orc_grads* g) {
  free(g->d_means); free(g->d_rotations); free(g->d_log_scales);
  free(g->d_opacity_logits); free(g->d_sh); free(g->d_mu2d);
  memset(g, 0, sizeof *g);
}

typedef struct { double d_mu2d[2], d_conic[4], d_color[3], d_opacity; } partial_t; /* rasterizer.cpp:327-332 */

/* rasterizer.cpp:336-540 */
int orc_render_backward(const orc_cloud* cloud, const orc_camera* cam, const orc_render_out* out,
                        const double* d_image, int32_t d_w, int32_t d_h, orc_grads* grads) {
  if (out->state_fingerprint != orc_fingerprint(cloud, cam) || out->n_gaussians != cloud->n) return 6;
  if (d_w != cam->width || d_h != cam->height) return 4;
  orc_grads_alloc(grads, cloud);
  const orc_raster_config* cfg = &out->config;
  const double cutoff2 = cfg->cutoff_sigma * cfg->cutoff_sigma;
  const int n_tiles = out->tiles_x * out->tiles_y;
  const int64_t n_entries = out->n_entries, n_splats = out->n_splats;

  /* Phase 1 (rasterizer.cpp:354-405) */
  partial_t* partials = (partial_t*)calloc(n_entries + 1, sizeof(partial_t));
#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < n_tiles; ++t) {
    const int tx = t % out->tiles_x, ty = t / out->tiles_x;
    const int x1 = (tx + 1) * cfg->tile_size < cam->width ? (tx + 1) * cfg->tile_size : cam->width;
    const int y1 = (ty + 1) * cfg->tile_size < cam->height ? (ty + 1) * cfg->tile_size : cam->height;
    const int32_t lb = out->tile_ranges[2 * t];
    for (int y = ty * cfg->tile_size; y < y1; ++y) {
      for (int x = tx * cfg->tile_size; x < x1; ++x) {
        const size_t pix = (size_t)y * cam->width + x;
        double dp[3] = {d_image[pix * 3], d_image[pix * 3 + 1], d_image[pix * 3 + 2]};
        const uint8_t of = out->overflow_mask[pix];
        for (int c = 0; c < 3; ++c)
          if (of & (1u << c)) dp[c] = 0.0;
        if (dp[0] == 0.0 && dp[1] == 0.0 && dp[2] == 0.0) continue;
        const double px = (double)x, py = (double)y;
        double t_run = out->final_transmittance[pix];
        double behind[3] = {out->background[0] * t_run, out->background[1] * t_run, out->background[2] * t_run};
        for (int32_t j = out->contrib_count[pix] - 1; j >= 0; --j) {
          const int32_t entry = lb + j;
          const orc_splat* rec = &out->splats[out->tile_lists[entry]];
          double d0 = px - rec->mu2d[0], d1 = py - rec->mu2d[1];
          double c0 = rec->conic[0] * d0 + rec->conic[1] * d1, c1 = rec->conic[2] * d0 + rec->conic[3] * d1;
          double g = d0 * c0 + d1 * c1;
          if (g > cutoff2) continue;
          double alpha_raw = rec->opacity * exp(-0.5 * g);
          double alpha = cfg->alpha_clamp < alpha_raw ? cfg->alpha_clamp : alpha_raw;
          double t_before = t_run / (1.0 - alpha);
          double weight = alpha * t_before;
          partial_t* p = &partials[entry];
          p->d_color[0] += weight * dp[0];
          p->d_color[1] += weight * dp[1];
          p->d_color[2] += weight * dp[2];
          double om = 1.0 - alpha;
          double d_alpha = dp[0] * (rec->color[0] * t_before - behind[0] / om) +
                           dp[1] * (rec->color[1] * t_before - behind[1] / om) +
                           dp[2] * (rec->color[2] * t_before - behind[2] / om);
          if (alpha_raw < cfg->alpha_clamp) {
            double expg = exp(-0.5 * g);
            p->d_opacity += d_alpha * expg;
            double d_g = d_alpha * (-0.5 * alpha_raw);
            double k = -2.0 * d_g;
            p->d_mu2d[0] += k * c0;
            p->d_mu2d[1] += k * c1;
            p->d_conic[0] += d_g * (d0 * d0);
            p->d_conic[1] += d_g * (d0 * d1);
            p->d_conic[2] += d_g * (d1 * d0);
            p->d_conic[3] += d_g * (d1 * d1);
          }
          t_run = t_before;
          behind[0] += rec->color[0] * weight;
          behind[1] += rec->color[1] * weight;
          behind[2] += rec->color[2] * weight;
        }
      }
    }
  }

  /* Phase 2 (rasterizer.cpp:407-418; deterministic order; the fast atomic
   * mode differs only in summation order) */
  partial_t* sums = (partial_t*)calloc(n_splats + 1, sizeof(partial_t));
  for (int64_t e = 0; e < n_entries; ++e) {
    const partial_t* p = &partials[e];
    partial_t* s = &sums[out->tile_lists[e]];
    s->d_mu2d[0] += p->d_mu2d[0]; s->d_mu2d[1] += p->d_mu2d[1];
    for (int k = 0; k < 4; ++k) s->d_conic[k] += p->d_conic[k];
    for (int k = 0; k < 3; ++k) s->d_color[k] += p->d_color[k];
    s->d_opacity += p->d_opacity;
  }
  free(partials);

  /* Phase 3 (rasterizer.cpp:433-535) */
  const double* Rc = cam->R;
  double cc[3];
  cam_center(cam, cc);
  const int degree = cloud->active_sh_degree < cloud->sh_degree ? cloud->active_sh_degree : cloud->sh_degree;
  const int basis_n = sh_count(degree);
  const int basis_cap = sh_count(cloud->sh_degree);
  double rot_blocks[3][9]; /* lie.cpp:173-181 */
  for (int k = 0; k < 3; ++k) {
    double e[3] = {0, 0, 0}, S[9];
    e[k] = 1.0;
    skew3(e, S);
    mat3_mul(S, Rc, rot_blocks[k]);
  }
  double* pose_contrib = (double*)calloc(6 * (n_splats + 1), sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < n_splats; ++s) {
    const orc_splat* rec = &out->splats[s];
    const partial_t* acc = &sums[s];
    const int64_t i = rec->gaussian;
    const double* mean = cloud->means + 3 * i;
    double mu_cam[3];
    pose_act(Rc, cam->t, mean, mu_cam);
    const double z = mu_cam[2];
    double J[6], m[6];
    projection_jacobian(mu_cam, cam, J);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) m[a * 3 + b] = J[a * 3 + 0] * Rc[0 * 3 + b] + J[a * 3 + 1] * Rc[1 * 3 + b] + J[a * 3 + 2] * Rc[2 * 3 + b];
    const double sc[3] = {exp(cloud->log_scales[3 * i]), exp(cloud->log_scales[3 * i + 1]), exp(cloud->log_scales[3 * i + 2])};
    double Rg[9], RS[9], sigma[9];
    orc_quat_to_rotation(cloud->rotations + 4 * i, Rg);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) RS[a * 3 + b] = Rg[a * 3 + b] * sc[b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) sigma[a * 3 + b] = RS[a * 3 + 0] * RS[b * 3 + 0] + RS[a * 3 + 1] * RS[b * 3 + 1] + RS[a * 3 + 2] * RS[b * 3 + 2];
    /* d_cov2d = -(conic * d_conic * conic) */
    const double* C = rec->conic;
    const double* D = acc->d_conic;
    double CD[4], dcov[4];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) CD[a * 2 + b] = C[a * 2 + 0] * D[0 * 2 + b] + C[a * 2 + 1] * D[1 * 2 + b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) dcov[a * 2 + b] = -(CD[a * 2 + 0] * C[0 * 2 + b] + CD[a * 2 + 1] * C[1 * 2 + b]);
    /* d_m = ((2 d_cov2d) m) sigma */
    double dc2[4] = {2.0 * dcov[0], 2.0 * dcov[1], 2.0 * dcov[2], 2.0 * dcov[3]};
    double t23[6], d_m[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) t23[a * 3 + b] = dc2[a * 2 + 0] * m[0 * 3 + b] + dc2[a * 2 + 1] * m[1 * 3 + b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) d_m[a * 3 + b] = t23[a * 3 + 0] * sigma[0 * 3 + b] + t23[a * 3 + 1] * sigma[1 * 3 + b] + t23[a * 3 + 2] * sigma[2 * 3 + b];
    /* d_sigma3d = (m^T d_cov2d) m */
    double t32[6], dS[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 2; ++b) t32[a * 2 + b] = m[0 * 3 + a] * dcov[0 * 2 + b] + m[1 * 3 + a] * dcov[1 * 2 + b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) dS[a * 3 + b] = t32[a * 2 + 0] * m[0 * 3 + b] + t32[a * 2 + 1] * m[1 * 3 + b];
    /* d_jac = d_m R^T ; d_rot_c = J^T d_m */
    double d_jac[6], d_rot_c[9];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) d_jac[a * 3 + b] = d_m[a * 3 + 0] * Rc[b * 3 + 0] + d_m[a * 3 + 1] * Rc[b * 3 + 1] + d_m[a * 3 + 2] * Rc[b * 3 + 2];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) d_rot_c[a * 3 + b] = J[0 * 3 + a] * d_m[0 * 3 + b] + J[1 * 3 + a] * d_m[1 * 3 + b];
    const double iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
    const double fx = cam->fx, fy = cam->fy;
    double dmc[3];
    dmc[0] = d_jac[2] * (-fx * iz2);
    dmc[1] = d_jac[5] * (-fy * iz2);
    dmc[2] = d_jac[0] * (-fx * iz2) + d_jac[4] * (-fy * iz2) + d_jac[2] * (2.0 * fx * mu_cam[0] * iz3) +
             d_jac[5] * (2.0 * fy * mu_cam[1] * iz3);
    dmc[0] += acc->d_mu2d[0] * fx * iz;
    dmc[1] += acc->d_mu2d[1] * fy * iz;
    dmc[2] += -acc->d_mu2d[0] * fx * mu_cam[0] * iz2 - acc->d_mu2d[1] * fy * mu_cam[1] * iz2;
    /* d_rot_g = ((2 dS) Rg) diag(s^2); rt_ds_r = (Rg^T dS) Rg */
    double dS2[9], t33[9], d_rot_g[9], RgT[9], rtds[9], rtdsr[9];
    for (int k = 0; k < 9; ++k) dS2[k] = 2.0 * dS[k];
    mat3_mul(dS2, Rg, t33);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) d_rot_g[a * 3 + b] = t33[a * 3 + b] * (sc[b] * sc[b]);
    mat3_T(Rg, RgT);
    mat3_mul(RgT, dS, rtds);
    mat3_mul(rtds, Rg, rtdsr);
    double d_log_scale[3];
    for (int k = 0; k < 3; ++k) {
      double d_s = 2.0 * sc[k] * rtdsr[k * 3 + k];
      d_log_scale[k] = d_s * sc[k];
    }
    double qj[36], d_quat[4];
    orc_quat_rotation_jacobian(cloud->rotations + 4 * i, qj);
    for (int k = 0; k < 4; ++k) {
      double acc9 = 0.0;
      for (int b = 0; b < 3; ++b) /* column-major traversal as Eigen's redux */
        for (int a = 0; a < 3; ++a) acc9 += d_rot_g[a * 3 + b] * qj[9 * k + a * 3 + b];
      d_quat[k] = acc9;
    }
    /* SH colour chain */
    double tg[3] = {mean[0] - cc[0], mean[1] - cc[1], mean[2] - cc[2]};
    const double dist = norm3(tg);
    const double dir[3] = {tg[0] / dist, tg[1] / dist, tg[2] / dist};
    double basis[16], bgrad[48];
    orc_sh_basis(dir, degree, basis);
    orc_sh_basis_gradient(dir, degree, bgrad);
    double* d_sh = grads->d_sh + (size_t)i * 3 * basis_cap;
    const double* coeffs = cloud->sh + (size_t)i * 3 * basis_cap;
    double d_dir[3] = {0, 0, 0};
    for (int c = 0; c < 3; ++c) {
      if (rec->color_clamped & (1u << c)) continue;
      const double* coeff = coeffs + c * basis_cap;
      for (int b = 0; b < basis_n; ++b) {
        d_sh[c * basis_cap + b] += acc->d_color[c] * basis[b];
        double f = acc->d_color[c] * coeff[b];
        d_dir[0] += f * bgrad[b * 3 + 0];
        d_dir[1] += f * bgrad[b * 3 + 1];
        d_dir[2] += f * bgrad[b * 3 + 2];
      }
    }
    /* (I - dir dir^T) d_dir / dist */
    double P[9], dtg[3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) P[a * 3 + b] = ((a == b) ? 1.0 : 0.0) - dir[a] * dir[b];
    mat3_vec(P, d_dir, dtg);
    dtg[0] /= dist; dtg[1] /= dist; dtg[2] /= dist;
    double rt_dmc[3];
    mat3T_vec(Rc, dmc, rt_dmc);
    for (int k = 0; k < 3; ++k) grads->d_means[3 * i + k] += rt_dmc[k] + dtg[k];
    grads->d_mu2d[2 * i] += acc->d_mu2d[0];
    grads->d_mu2d[2 * i + 1] += acc->d_mu2d[1];
    for (int k = 0; k < 3; ++k) grads->d_log_scales[3 * i + k] += d_log_scale[k];
    for (int k = 0; k < 4; ++k) grads->d_rotations[4 * i + k] += d_quat[k];
    const double o = rec->opacity;
    grads->d_opacity_logits[i] += acc->d_opacity * o * (1.0 - o);
    /* pose (rasterizer.cpp:523-533) */
    double r_dtg[3];
    mat3_vec(Rc, dtg, r_dtg);
    double* pc = pose_contrib + 6 * s;
    pc[0] = dmc[0] + r_dtg[0];
    pc[1] = dmc[1] + r_dtg[1];
    pc[2] = dmc[2] + r_dtg[2];
    pc[3] = mu_cam[1] * dmc[2] - mu_cam[2] * dmc[1];
    pc[4] = mu_cam[2] * dmc[0] - mu_cam[0] * dmc[2];
    pc[5] = mu_cam[0] * dmc[1] - mu_cam[1] * dmc[0];
    for (int k = 0; k < 3; ++k) {
      double a9 = 0.0;
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) a9 += d_rot_c[a * 3 + b] * rot_blocks[k][a * 3 + b];
      pc[3 + k] += a9;
    }
  }
  /* rasterizer.cpp:537-538 */
  for (int64_t s = 0; s < n_splats; ++s)
    for (int k = 0; k < 6; ++k) grads->d_pose[k] += pose_contrib[6 * s + k];
  free(pose_contrib);
  free(sums);
  return 0;
}

void orc_count_work(const orc_render_out* out, const double* d_image, int64_t counts[4]) {
  const double cutoff2 = out->config.cutoff_sigma * out->config.cutoff_sigma;
  const int tile = out->config.tile_size;
  int64_t hf = 0, cf = 0, hb = 0, cb = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : hf, cf, hb, cb)
  for (int y = 0; y < out->height; ++y) {
    for (int x = 0; x < out->width; ++x) {
      const size_t pix = (size_t)y * out->width + x;
      const int t = (y / tile) * out->tiles_x + x / tile;
      const int32_t lb = out->tile_ranges[2 * t];
      int bwd = 0;
      if (d_image) {
        const uint8_t of = out->overflow_mask[pix];
        for (int c = 0; c < 3; ++c)
          if (!(of & (1u << c)) && d_image[pix * 3 + c] != 0.0) bwd = 1;
      }
      for (int32_t j = 0; j < out->contrib_count[pix]; ++j) {
        const orc_splat* rec = &out->splats[out->tile_lists[lb + j]];
        double d0 = x - rec->mu2d[0], d1 = y - rec->mu2d[1];
        double c0 = rec->conic[0] * d0 + rec->conic[1] * d1, c1 = rec->conic[2] * d0 + rec->conic[3] * d1;
        const int hit = !(d0 * c0 + d1 * c1 > cutoff2);
        hf += hit;
        cf += !hit;
        if (bwd) {
          hb += hit;
          cb += !hit;
        }
      }
    }
  }
  counts[0] = hf;
  counts[1] = cf;
  counts[2] = hb;
  counts[3] = cb;
}

/* Test aid (no reference counterpart): per-pixel relative distance of the
 * FP64 forward pass from its discrete decisions — min over the examined
 * entries (j < contrib) of |g - cutoff^2| / cutoff^2 (rasterizer.cpp:254) and,
 * over the hits, of |T - early_termination| / early_termination after the
 * update (258). An FP32 evaluation can only take a different decision where
 * this margin is below its rounding error; parity tests hold pixels with a
 * margin above a stated threshold to the image tolerance and report the rest. */
void orc_decision_margin(const orc_render_out* out, double* margin) {
  const double cutoff2 = out->config.cutoff_sigma * out->config.cutoff_sigma;
  const double et = out->config.early_termination, clampa = out->config.alpha_clamp;
  const int tile = out->config.tile_size;
#pragma omp parallel for schedule(dynamic, 4)
  for (int y = 0; y < out->height; ++y) {
    for (int x = 0; x < out->width; ++x) {
      const size_t pix = (size_t)y * out->width + x;
      const int t = (y / tile) * out->tiles_x + x / tile;
      const int32_t lb = out->tile_ranges[2 * t];
      double m = INFINITY, T = 1.0;
      for (int32_t j = 0; j < out->contrib_count[pix]; ++j) {
        const orc_splat* rec = &out->splats[out->tile_lists[lb + j]];
        const double d0 = x - rec->mu2d[0], d1 = y - rec->mu2d[1];
        const double c0 = rec->conic[0] * d0 + rec->conic[1] * d1, c1 = rec->conic[2] * d0 + rec->conic[3] * d1;
        const double g = d0 * c0 + d1 * c1;
        const double mg = fabs(g - cutoff2) / cutoff2;
        if (mg < m) m = mg;
        if (g > cutoff2) continue;
        double a = rec->opacity * exp(-0.5 * g);
        if (a > clampa) a = clampa;
        T *= 1.0 - a;
        const double mt = fabs(T - et) / et;
        if (mt < m) m = mt;
      }
      margin[pix] = m;
    }
  }
}

/* ---------------------------------------------------------------- losses */
#define KWIN 11
#define KHALF 5
static void gaussian_window(double w[KWIN]) { /* losses.cpp:19-32 */
  double sum = 0.0;
  for (int i = 0; i < KWIN; ++i) {
    double d = i - KHALF;
    w[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
    sum += w[i];
  }
  for (int i = 0; i < KWIN; ++i) w[i] /= sum;
}
/* losses.cpp:37-63 */
static void conv_window(const double* src, int width, int height, double* dst, double* tmp) {
  double w[KWIN];
  gaussian_window(w);
  for (int y = 0; y < height; ++y) {
    const double* row = src + (size_t)y * width;
    double* trow = tmp + (size_t)y * width;
    for (int x = 0; x < width; ++x) {
      double acc = 0.0;
      int k0 = KHALF - x > 0 ? KHALF - x : 0;
      int k1 = width - x + KHALF < KWIN ? width - x + KHALF : KWIN;
      for (int k = k0; k < k1; ++k) acc += w[k] * row[x + k - KHALF];
      trow[x] = acc;
    }
  }
  for (int y = 0; y < height; ++y) {
    double* drow = dst + (size_t)y * width;
    int k0 = KHALF - y > 0 ? KHALF - y : 0;
    int k1 = height - y + KHALF < KWIN ? height - y + KHALF : KWIN;
    for (int x = 0; x < width; ++x) {
      double acc = 0.0;
      for (int k = k0; k < k1; ++k) acc += w[k] * tmp[(size_t)(y + k - KHALF) * width + x];
      drow[x] = acc;
    }
  }
}
/* losses.cpp:74-155 (mask == nullptr path) */
/* losses.cpp:74-155 (ssim_core): mask (nullable) selects the valid-window
 * pixels that enter the mean */
static double ssim_core_m(const double* a, const double* b, int32_t width, int32_t height, const uint8_t* mask,
                          double* d_a) {
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  const int x0 = KHALF, x1 = width - KHALF, y0 = KHALF, y1 = height - KHALF;
  const size_t P = (size_t)width * height;
  if (d_a) memset(d_a, 0, sizeof(double) * P * 3);
  int64_t count = 0;
  if (x1 > x0 && y1 > y0)
    for (int y = y0; y < y1; ++y)
      for (int x = x0; x < x1; ++x) count += (!mask || mask[(size_t)y * width + x]) ? 1 : 0;
  if (count == 0) return 1.0;
  const double scale = 1.0 / (3.0 * (double)count);
  double total = 0.0;
  double* buf = (double*)malloc(sizeof(double) * P * 17);
  double *pa = buf, *pb = buf + P, *paa = buf + 2 * P, *pbb = buf + 3 * P, *pab = buf + 4 * P;
  double *mu_a = buf + 5 * P, *mu_b = buf + 6 * P, *e_aa = buf + 7 * P, *e_bb = buf + 8 * P, *e_ab = buf + 9 * P;
  double *g_mu = buf + 10 * P, *g_eaa = buf + 11 * P, *g_eab = buf + 12 * P, *tmp = buf + 13 * P;
  double *c_mu = buf + 14 * P, *c_eaa = buf + 15 * P, *c_eab = buf + 16 * P;
  for (int c = 0; c < 3; ++c) {
    for (size_t p = 0; p < P; ++p) {
      pa[p] = a[p * 3 + c];
      pb[p] = b[p * 3 + c];
      paa[p] = pa[p] * pa[p];
      pbb[p] = pb[p] * pb[p];
      pab[p] = pa[p] * pb[p];
    }
    conv_window(pa, width, height, mu_a, tmp);
    conv_window(pb, width, height, mu_b, tmp);
    conv_window(paa, width, height, e_aa, tmp);
    conv_window(pbb, width, height, e_bb, tmp);
    conv_window(pab, width, height, e_ab, tmp);
    if (d_a) {
      memset(g_mu, 0, sizeof(double) * P);
      memset(g_eaa, 0, sizeof(double) * P);
      memset(g_eab, 0, sizeof(double) * P);
    }
    for (int y = y0; y < y1; ++y) {
      for (int x = x0; x < x1; ++x) {
        const size_t p = (size_t)y * width + x;
        if (mask && !mask[p]) continue;
        const double ma = mu_a[p], mb = mu_b[p];
        const double va = e_aa[p] - ma * ma;
        const double vb = e_bb[p] - mb * mb;
        const double vab = e_ab[p] - ma * mb;
        const double a1 = 2.0 * ma * mb + C1;
        const double a2 = 2.0 * vab + C2;
        const double b1 = ma * ma + mb * mb + C1;
        const double b2 = va + vb + C2;
        const double s = (a1 * a2) / (b1 * b2);
        total += s;
        if (!d_a) continue;
        g_mu[p] = scale * (2.0 * mb * (a2 - a1) + 2.0 * ma * s * (b1 - b2)) / (b1 * b2);
        const double q = a1 / (b1 * b2);
        g_eaa[p] = -(scale * q) * (a2 / b2);
        g_eab[p] = 2.0 * (scale * q);
      }
    }
    if (d_a) {
      conv_window(g_mu, width, height, c_mu, tmp);
      conv_window(g_eaa, width, height, c_eaa, tmp);
      conv_window(g_eab, width, height, c_eab, tmp);
      for (size_t p = 0; p < P; ++p) d_a[p * 3 + c] = c_mu[p] + 2.0 * pa[p] * c_eaa[p] + pb[p] * c_eab[p];
    }
  }
  free(buf);
  return total * scale;
}
double orc_ssim(const double* a, const double* b, int32_t width, int32_t height, double* d_a) {
  return ssim_core_m(a, b, width, height, NULL, d_a);
}
/* losses.cpp:158-192 with a mask: masked pixels only, norm over their count */
static double l1_core_m(const double* r, const double* t, int32_t w, int32_t h, const uint8_t* mask, double* d,
                        int64_t* count_out) {
  const int64_t P = (int64_t)w * h;
  int64_t count = 0;
  for (int64_t p = 0; p < P; ++p) count += mask[p] != 0;
  *count_out = count;
  if (d) memset(d, 0, sizeof(double) * P * 3);
  if (count == 0) return 0.0;
  const double norm = 1.0 / (3.0 * (double)count);
  double total = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    if (!mask[p]) continue;
    for (int c = 0; c < 3; ++c) {
      double diff = r[p * 3 + c] - t[p * 3 + c];
      total += fabs(diff);
      if (d && diff != 0.0) d[p * 3 + c] = diff > 0.0 ? norm : -norm;
    }
  }
  return total * norm;
}
/* losses.cpp:259-263 */
void orc_transmittance_mask(const double* accum, int64_t n, double threshold, uint8_t* mask) {
  for (int64_t i = 0; i < n; ++i) mask[i] = accum[i] > threshold ? 1 : 0;
}
/* losses.cpp:273-289; returns the loss, *status = 5 (empty_mask + 1) when no pixel passes */
double orc_masked_rgb_loss(const double* rendered, const double* target, int32_t w, int32_t h, const uint8_t* mask,
                           double beta, double* d_rendered, int32_t* status) {
  const size_t n = (size_t)w * h * 3;
  double* d_l1 = d_rendered ? (double*)malloc(sizeof(double) * n) : NULL;
  double* d_ss = d_rendered ? (double*)malloc(sizeof(double) * n) : NULL;
  int64_t cnt = 0;
  double l1 = l1_core_m(rendered, target, w, h, mask, d_l1, &cnt);
  *status = cnt == 0 ? 5 : 0;
  double s = cnt ? ssim_core_m(rendered, target, w, h, mask, d_ss) : 1.0;
  double loss = (1.0 - beta) * l1 + beta * (1.0 - s);
  if (d_rendered)
    for (size_t i = 0; i < n; ++i) d_rendered[i] = cnt ? (1.0 - beta) * d_l1[i] - beta * d_ss[i] : 0.0;
  free(d_l1);
  free(d_ss);
  return loss;
}
/* losses.cpp:158-192 */
static double l1_core(const double* r, const double* t, int32_t w, int32_t h, double* d) {
  const int64_t count = (int64_t)w * h;
  if (d) memset(d, 0, sizeof(double) * count * 3);
  const double norm = 1.0 / (3.0 * (double)count);
  double total = 0.0;
  for (int64_t p = 0; p < count; ++p)
    for (int c = 0; c < 3; ++c) {
      double diff = r[p * 3 + c] - t[p * 3 + c];
      total += fabs(diff);
      if (d && diff != 0.0) d[p * 3 + c] = diff > 0.0 ? norm : -norm;
    }
  return total * norm;
}
/* losses.cpp:201-215 */
double orc_rgb_loss(const double* rendered, const double* target, int32_t w, int32_t h, double beta,
                    double* d_rendered) {
  const size_t n = (size_t)w * h * 3;
  double* d_l1 = d_rendered ? (double*)malloc(sizeof(double) * n) : NULL;
  double* d_ss = d_rendered ? (double*)malloc(sizeof(double) * n) : NULL;
  double l1 = l1_core(rendered, target, w, h, d_l1);
  double s = orc_ssim(rendered, target, w, h, d_ss);
  double loss = (1.0 - beta) * l1 + beta * (1.0 - s);
  if (d_rendered)
    for (size_t i = 0; i < n; ++i) d_rendered[i] = (1.0 - beta) * d_l1[i] - beta * d_ss[i];
  free(d_l1);
  free(d_ss);
  return loss;
}
/* losses.cpp:217-244 */
double orc_anisotropy_loss(const double* ls, int64_t n, double ratio, double* d) {
  if (d) memset(d, 0, sizeof(double) * 3 * n);
  if (n == 0) return 0.0;
  double total = 0.0;
  const double inv_n = 1.0 / (double)n;
  for (int64_t i = 0; i < n; ++i) {
    double s[3] = {exp(ls[3 * i]), exp(ls[3 * i + 1]), exp(ls[3 * i + 2])};
    int amax = 0, amin = 0;
    for (int k = 1; k < 3; ++k) {
      if (s[k] > s[amax]) amax = k;
      if (s[k] < s[amin]) amin = k;
    }
    double r = s[amax] / s[amin];
    if (r > ratio) {
      total += (r - ratio) * inv_n;
      if (d) {
        double d_max = inv_n / s[amin];
        double d_min = -inv_n * s[amax] / (s[amin] * s[amin]);
        d[3 * i + amax] += d_max * s[amax];
        d[3 * i + amin] += d_min * s[amin];
      }
    }
  }
  return total;
}
/* losses.cpp:246-257 */
double orc_opacity_l1(const double* op, int64_t n, double* d) {
  if (d) memset(d, 0, sizeof(double) * n);
  if (n == 0) return 0.0;
  const double inv_n = 1.0 / (double)n;
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    total += op[i] * inv_n;
    if (d) d[i] = inv_n;
  }
  return total;
}

/* --------------------------------------------------------------- trainer */
static const double kB1 = 0.9, kB2 = 0.999, kEps = 1e-15; /* trainer.hpp:80-82 */
/* trainer.cpp:30-38 */
double orc_schedule(int kind, double start, double end, int64_t step, int64_t total) {
  if (total <= 0) return end;
  double s = (double)step / (double)total;
  if (s < 0.0) s = 0.0;
  if (s > 1.0) s = 1.0;
  if (kind == 0) return end + (start - end) * 0.5 * (1.0 + cos(ORC_PI * s));
  return start * pow(end / start, s);
}
/* trainer.cpp:71-90 */
void orc_pose_step(const double R[9], const double t[3], const double d_pose[6], double lr,
                   orc_pose_adam* st, double R_out[9], double t_out[3], double applied[6]) {
  ++st->step;
  const double bc1 = 1.0 - pow(kB1, (double)st->step);
  const double bc2 = 1.0 - pow(kB2, (double)st->step);
  double delta[6];
  for (int k = 0; k < 6; ++k) {
    double g = d_pose[k];
    st->m[k] = kB1 * st->m[k] + (1.0 - kB1) * g;
    st->v[k] = kB2 * st->v[k] + (1.0 - kB2) * g * g;
    double m_hat = st->m[k] / bc1;
    double v_hat = st->v[k] / bc2;
    delta[k] = -lr * m_hat / (sqrt(v_hat) + kEps);
  }
  if (applied) memcpy(applied, delta, sizeof delta);
  int zero = 1;
  for (int k = 0; k < 6; ++k) if (delta[k] != 0.0) zero = 0;
  if (zero) {
    memcpy(R_out, R, sizeof(double) * 9);
    memcpy(t_out, t, sizeof(double) * 3);
    return;
  }
  double Re[9], te[3], Rn[9], tn[3];
  orc_se3_exp(delta, Re, te);
  mat3_mul(Re, R, Rn); /* Se3Pose::operator* (lie.hpp:48-53) */
  mat3_vec(Re, t, tn);
  tn[0] += te[0]; tn[1] += te[1]; tn[2] += te[2];
  orc_orthonormalize(Rn);
  memcpy(R_out, Rn, sizeof Rn);
  memcpy(t_out, tn, sizeof tn);
}
/* trainer.cpp:40-53 */
void orc_adam_step(orc_adam_state* s, double* params, const double* grads, int64_t n, double lr) {
  if (s->n != n) {
    free(s->m); free(s->v);
    s->m = (double*)calloc(n + 1, sizeof(double));
    s->v = (double*)calloc(n + 1, sizeof(double));
    s->n = n;
    s->step = 0;
  }
  ++s->step;
  const double bc1 = 1.0 - pow(kB1, (double)s->step);
  const double bc2 = 1.0 - pow(kB2, (double)s->step);
  for (int64_t i = 0; i < n; ++i) {
    double g = grads[i];
    s->m[i] = kB1 * s->m[i] + (1.0 - kB1) * g;
    s->v[i] = kB2 * s->v[i] + (1.0 - kB2) * g * g;
    double m_hat = s->m[i] / bc1, v_hat = s->v[i] / bc2;
    params[i] -= lr * m_hat / (sqrt(v_hat) + kEps);
  }
}
/* pipelines.cpp:18-41 with adam_step's lr_of overload (trainer.cpp:55-69) */
void orc_cloud_adam_step(orc_cloud* cloud, const orc_grads* g, orc_adam_state st[5], const double lrs[6]) {
  const int64_t n = cloud->n;
  if (n == 0) return;
  orc_adam_step(&st[0], cloud->means, g->d_means, n * 3, lrs[0]);
  double* before = (double*)malloc(sizeof(double) * 4 * n);
  memcpy(before, cloud->rotations, sizeof(double) * 4 * n);
  orc_adam_step(&st[1], cloud->rotations, g->d_rotations, n * 4, lrs[1]);
  orc_adam_step(&st[2], cloud->log_scales, g->d_log_scales, n * 3, lrs[2]);
  orc_adam_step(&st[3], cloud->opacity_logits, g->d_opacity_logits, n, lrs[3]);
  const int basis = sh_count(cloud->sh_degree);
  const int64_t L = n * 3 * basis;
  orc_adam_state* s = &st[4];
  if (s->n != L) {
    free(s->m); free(s->v);
    s->m = (double*)calloc(L + 1, sizeof(double));
    s->v = (double*)calloc(L + 1, sizeof(double));
    s->n = L;
    s->step = 0;
  }
  ++s->step;
  const double bc1 = 1.0 - pow(kB1, (double)s->step), bc2 = 1.0 - pow(kB2, (double)s->step);
  for (int64_t k = 0; k < L; ++k) {
    double gk = g->d_sh[k];
    s->m[k] = kB1 * s->m[k] + (1.0 - kB1) * gk;
    s->v[k] = kB2 * s->v[k] + (1.0 - kB2) * gk * gk;
    double m_hat = s->m[k] / bc1, v_hat = s->v[k] / bc2;
    double lr = (k % basis == 0) ? lrs[4] : lrs[5];
    cloud->sh[k] -= lr * m_hat / (sqrt(v_hat) + kEps);
  }
  for (int64_t i = 0; i < n; ++i) {
    double* q = cloud->rotations + 4 * i;
    if (q[0] != before[4 * i] || q[1] != before[4 * i + 1] || q[2] != before[4 * i + 2] || q[3] != before[4 * i + 3]) {
      double nn = norm4(q);
      for (int k = 0; k < 4; ++k) q[k] /= nn;
    }
  }
  free(before);
}

/* pipelines.cpp:58-92 */
int32_t orc_estimate_pose(const orc_cloud* cloud, const double* image, double fx, double fy, double cx,
                          double cy, int32_t w, int32_t h, const double R0[9], const double t0[3],
                          const orc_pose_cfg* cfg, int32_t budget, double R_out[9], double t_out[3],
                          double* final_loss, int32_t* converged, double* trace_pose, double* trace_loss,
                          double* trace_dpose) {
  orc_pose_adam adam;
  memset(&adam, 0, sizeof adam);
  double R[9], t[3];
  memcpy(R, R0, sizeof R);
  memcpy(t, t0, sizeof t);
  memcpy(R_out, R0, sizeof R);
  memcpy(t_out, t0, sizeof t);
  *final_loss = 0.0;
  *converged = 0;
  double best = INFINITY;
  int32_t steps_used = 0;
  double* d_image = (double*)malloc(sizeof(double) * (size_t)w * h * 3);
  for (int32_t it = 0; it < budget; ++it) {
    orc_camera cam;
    cam.fx = fx; cam.fy = fy; cam.cx = cx; cam.cy = cy; cam.width = w; cam.height = h;
    memcpy(cam.R, R, sizeof R);
    memcpy(cam.t, t, sizeof t);
    orc_render_out* out = orc_render(cloud, &cam, cfg->background, &cfg->raster);
    double loss = orc_rgb_loss(out->image, image, w, h, cfg->beta, d_image);
    if (trace_pose) {
      for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) trace_pose[12 * it + r * 4 + c] = R[r * 3 + c];
        trace_pose[12 * it + r * 4 + 3] = t[r];
      }
    }
    if (trace_loss) trace_loss[it] = loss;
    if (loss < best) {
      best = loss;
      memcpy(R_out, R, sizeof R);
      memcpy(t_out, t, sizeof t);
      *final_loss = loss;
    }
    if (loss < 1e-14) {
      *converged = 1;
      steps_used = it + 1;
      orc_render_free(out);
      break;
    }
    orc_grads g;
    orc_render_backward(cloud, &cam, out, d_image, w, h, &g);
    if (trace_dpose) memcpy(trace_dpose + 6 * it, g.d_pose, sizeof(double) * 6);
    double lr = orc_schedule(0, cfg->cam_lr_start, cfg->cam_lr_end, it, budget);
    double applied[6], Rn[9], tn[3];
    orc_pose_step(R, t, g.d_pose, lr, &adam, Rn, tn, applied);
    memcpy(R, Rn, sizeof R);
    memcpy(t, tn, sizeof t);
    orc_grads_free(&g);
    orc_render_free(out);
    steps_used = it + 1;
    double an = sqrt(applied[0] * applied[0] + applied[1] * applied[1] + applied[2] * applied[2] +
                     applied[3] * applied[3] + applied[4] * applied[4] + applied[5] * applied[5]);
    if (an < cfg->pose_converged_eps) {
      *converged = 1;
      break;
    }
  }
  free(d_image);
  return steps_used;
}

/* trainer.cpp:134-142 (GradAccum::add) for one view: visible splats only. */
void orc_grad_accum_add(const orc_render_out* out, const orc_grads* g, int32_t image_max_dim, double* grad_sum,
                        int32_t* count) {
  const double norm_scale = 0.5 * (double)image_max_dim;
  for (int64_t s = 0; s < out->n_splats; ++s) {
    const int32_t i = out->splats[s].gaussian;
    const double x = g->d_mu2d[2 * i], y = g->d_mu2d[2 * i + 1];
    grad_sum[i] += sqrt(x * x + y * y) * norm_scale;
    count[i] += 1;
  }
}

static int cmp_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x > y ? -1 : (x < y ? 1 : 0);
}

/* trainer.cpp:144-239 (densify_and_prune): clone small / split large
 * Gaussians whose mean normalised screen gradient reaches grad_threshold
 * (kept originals first, then clones and split children in index order,
 * children drawn rot * (scale .* normal3) with log-scale - ln 1.6), then prune
 * to opacity > max(prune_opacity, (n_target+1)-th largest opacity). `out` is
 * allocated here (free with orc_cloud_free); *final_source (out->n entries,
 * -1 = fresh) with orc_free. report = {cloned, split, pruned}. */
void orc_densify_and_prune(const orc_cloud* cloud, const double* grad_sum, const int32_t* count,
                           double grad_threshold, double size_ratio, int32_t n_target, double prune_opacity,
                           orc_rng* rng, orc_cloud* out, int32_t** final_source, int32_t report[3]) {
  const int64_t n = cloud->n;
  const int basis = sh_count(cloud->sh_degree);
  const int64_t shs = 3 * basis;
  report[0] = report[1] = report[2] = 0;
  double lo[3] = {cloud->means[0], cloud->means[1], cloud->means[2]}, hi[3] = {lo[0], lo[1], lo[2]};
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], cloud->means[3 * i + k]);
      hi[k] = fmax(hi[k], cloud->means[3 * i + k]);
    }
  const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  const double extent = sqrt(dx * dx + dy * dy + dz * dz);
  const double size_threshold = size_ratio * fmax(extent, 1e-6);
  uint8_t* action = (uint8_t*)calloc((size_t)n + 1, 1); /* 0 keep, 1 clone, 2 split */
  int64_t extra = 0, kept = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (count[i] > 0) {
      const double avg = grad_sum[i] / (double)count[i];
      if (!(avg < grad_threshold)) {
        double mx = exp(cloud->log_scales[3 * i]);
        mx = fmax(mx, exp(cloud->log_scales[3 * i + 1]));
        mx = fmax(mx, exp(cloud->log_scales[3 * i + 2]));
        action[i] = mx <= size_threshold ? 1 : 2;
      }
    }
    kept += action[i] != 2;
    extra += action[i] == 1 ? 1 : (action[i] == 2 ? 2 : 0);
  }
  const int64_t total = kept + extra;
  orc_cloud nx;
  orc_cloud_alloc(&nx, total, cloud->sh_degree);
  nx.active_sh_degree = cloud->active_sh_degree;
  int32_t* src = (int32_t*)malloc(sizeof(int32_t) * (size_t)(total + 1));
  int64_t j = 0;
  #define ORC_APPEND(I, FRESH)                                                              \
    do {                                                                                    \
      memcpy(nx.rotations + 4 * j, cloud->rotations + 4 * (I), 4 * sizeof(double));         \
      nx.opacity_logits[j] = cloud->opacity_logits[I];                                      \
      memcpy(nx.sh + shs * j, cloud->sh + shs * (I), (size_t)shs * sizeof(double));         \
      src[j] = (FRESH) ? -1 : (int32_t)(I);                                                 \
    } while (0)
  for (int64_t i = 0; i < n; ++i) {
    if (action[i] == 2) continue;
    memcpy(nx.means + 3 * j, cloud->means + 3 * i, 3 * sizeof(double));
    memcpy(nx.log_scales + 3 * j, cloud->log_scales + 3 * i, 3 * sizeof(double));
    ORC_APPEND(i, 0);
    ++j;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (action[i] == 1) {
      memcpy(nx.means + 3 * j, cloud->means + 3 * i, 3 * sizeof(double));
      memcpy(nx.log_scales + 3 * j, cloud->log_scales + 3 * i, 3 * sizeof(double));
      ORC_APPEND(i, 1);
      ++j;
      ++report[0];
    } else if (action[i] == 2) {
      double R[9];
      orc_quat_to_rotation(cloud->rotations + 4 * i, R);
      const double sc[3] = {exp(cloud->log_scales[3 * i]), exp(cloud->log_scales[3 * i + 1]),
                            exp(cloud->log_scales[3 * i + 2])};
      for (int c = 0; c < 2; ++c) {
        double nrm[3];
        nrm[2] = orc_rng_normal(rng); /* Vec3(normal(), normal(), normal()): GCC draws right to left */
        nrm[1] = orc_rng_normal(rng);
        nrm[0] = orc_rng_normal(rng);
        const double v[3] = {sc[0] * nrm[0], sc[1] * nrm[1], sc[2] * nrm[2]};
        double smp[3];
        mat3_vec(R, v, smp);
        for (int k = 0; k < 3; ++k) {
          nx.means[3 * j + k] = cloud->means[3 * i + k] + smp[k];
          nx.log_scales[3 * j + k] = cloud->log_scales[3 * i + k] - log(1.6);
        }
        ORC_APPEND(i, 1);
        ++j;
      }
      ++report[1];
    }
  }
  #undef ORC_APPEND
  double* op = (double*)malloc(sizeof(double) * (size_t)(total + 1));
  for (int64_t i = 0; i < total; ++i) op[i] = sigmoid(nx.opacity_logits[i]);
  double threshold = prune_opacity;
  if (total > n_target) {
    double* sorted = (double*)malloc(sizeof(double) * (size_t)total);
    memcpy(sorted, op, sizeof(double) * (size_t)total);
    qsort(sorted, (size_t)total, sizeof(double), cmp_desc);
    threshold = fmax(threshold, sorted[n_target]); /* (n_target+1)-th largest */
    free(sorted);
  }
  int64_t m = 0;
  for (int64_t i = 0; i < total; ++i) m += op[i] > threshold;
  orc_cloud_alloc(out, m, cloud->sh_degree);
  out->active_sh_degree = cloud->active_sh_degree;
  int32_t* fs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
  int64_t q = 0;
  for (int64_t i = 0; i < total; ++i) {
    if (!(op[i] > threshold)) {
      ++report[2];
      continue;
    }
    memcpy(out->means + 3 * q, nx.means + 3 * i, 3 * sizeof(double));
    memcpy(out->rotations + 4 * q, nx.rotations + 4 * i, 4 * sizeof(double));
    memcpy(out->log_scales + 3 * q, nx.log_scales + 3 * i, 3 * sizeof(double));
    out->opacity_logits[q] = nx.opacity_logits[i];
    memcpy(out->sh + shs * q, nx.sh + shs * i, (size_t)shs * sizeof(double));
    fs[q] = src[i];
    ++q;
  }
  *final_source = fs;
  free(op);
  free(src);
  free(action);
  orc_cloud_free(&nx);
}

void orc_free(void* p) { free(p); }

/* pipelines.cpp:122-129: the training-view sequence. `order` starts as iota
 * and is re-shuffled IN PLACE (Fisher-Yates from the back with
 * rng.uniform_int(0, i)) at the start of every epoch; the sequence is the
 * concatenation of the epoch orders. seq receives `count` view indices. */
void orc_joint_schedule(orc_rng* rng, int32_t n_views, int64_t count, int32_t* seq) {
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_views > 0 ? n_views : 1));
  for (int32_t i = 0; i < n_views; ++i) order[i] = i;
  for (int64_t k = 0; k < count; ++k) {
    if (k % n_views == 0) {
      for (int32_t i = n_views - 1; i > 0; --i) {
        const int32_t j = (int32_t)orc_rng_uniform_int(rng, 0, i);
        const int32_t tmp = order[i];
        order[i] = order[j];
        order[j] = tmp;
      }
    }
    seq[k] = order[k % n_views];
  }
  free(order);
}

/* Epoch-shuffle state of pipelines.cpp:122-129, consumed lazily so that its
 * draws interleave with densify_and_prune's exactly as in the reference. */
typedef struct {
  int32_t n, *order;
  int64_t next; /* next slot index to produce */
} orc_sched;

static int32_t sched_slot(orc_sched* sc, orc_rng* rng) {
  const int64_t k = sc->next++;
  if (k % sc->n == 0)
    for (int32_t i = sc->n - 1; i > 0; --i) {
      const int32_t j = (int32_t)orc_rng_uniform_int(rng, 0, i);
      const int32_t tmp = sc->order[i];
      sc->order[i] = sc->order[j];
      sc->order[j] = tmp;
    }
  return sc->order[k % sc->n];
}

/* CloudAdam::remap (trainer.cpp:101-132) for one flat AdamState of `width`
 * entries per Gaussian. */
static void adam_remap(orc_adam_state* s, const int32_t* src, int64_t n_new, int64_t width) {
  if (!s->m) return;
  double* m = (double*)calloc((size_t)(n_new * width + 1), sizeof(double));
  double* v = (double*)calloc((size_t)(n_new * width + 1), sizeof(double));
  for (int64_t j = 0; j < n_new; ++j) {
    if (src[j] < 0) continue;
    memcpy(m + j * width, s->m + (int64_t)src[j] * width, sizeof(double) * (size_t)width);
    memcpy(v + j * width, s->v + (int64_t)src[j] * width, sizeof(double) * (size_t)width);
  }
  free(s->m);
  free(s->v);
  s->m = m;
  s->v = v;
  s->n = n_new * width;
}

/* pipelines.cpp:96-216 (joint_optimize) without the ground-truth pose
 * statistics, generalised to `slots` training views per step (the
 * data-parallel semantics of the B200 build): step t renders the
 * next `slots` views of the epoch-shuffle sequence, the Adam gradient is the
 * MEAN of the slots' render gradients plus the regularisers (anisotropy
 * 217-244, opacity L1 246-257, both added once, on the pre-step parameters),
 * GradAccum adds every slot's view (trainer.cpp:134-142), the slots' pose
 * steps are applied in slot order with each view's own PoseAdam, and
 * densify_and_prune runs after step t when t is a densification step
 * (182-186). slots == 1 is the reference loop exactly. Returns 0, or 10
 * (ErrorCode::diverged + 1) at a non-finite total loss (160-162).
 * trace_total / trace_l1 (iterations, nullable) receive the step's mean total
 * loss and mean L1. poses: n_views x 12, updated in place. */
int32_t orc_joint_optimize(orc_cloud* cloud, const double* const* images, int32_t n_views, double fx, double fy,
                           double cx, double cy, int32_t w, int32_t h, double* poses, const orc_joint_cfg* cfg,
                           int32_t slots, orc_rng* rng, double* trace_total, double* trace_l1) {
  const int32_t iters = cfg->iterations;
  orc_sched sc;
  sc.n = n_views;
  sc.next = 0;
  sc.order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_views);
  for (int32_t i = 0; i < n_views; ++i) sc.order[i] = i;
  int32_t* vs = (int32_t*)malloc(sizeof(int32_t) * (size_t)slots);
  orc_adam_state st[5];
  memset(st, 0, sizeof st);
  orc_pose_adam* pad = (orc_pose_adam*)calloc((size_t)n_views, sizeof(orc_pose_adam));
  double* d_image = (double*)malloc(sizeof(double) * (size_t)w * h * 3);
  double* dpose = (double*)malloc(sizeof(double) * 6 * (size_t)slots);
  double* acc_sum = (double*)calloc((size_t)cloud->n + 1, sizeof(double));
  int32_t* acc_cnt = (int32_t*)calloc((size_t)cloud->n + 1, sizeof(int32_t));
  int32_t status = 0;
  for (int32_t t = 0; t < iters && status == 0; ++t) {
    const int64_t n = cloud->n;
    const int basis = sh_count(cloud->sh_degree);
    for (int32_t s = 0; s < slots; ++s) vs[s] = sched_slot(&sc, rng);
    if (cfg->sh_degree_interval > 0 && t > 0 && t % cfg->sh_degree_interval == 0) {
      const int32_t a = cloud->active_sh_degree + 1;
      cloud->active_sh_degree = a < cfg->sh_degree ? a : cfg->sh_degree;
    }
    orc_grads acc;
    orc_grads_alloc(&acc, cloud);
    double rgb_sum = 0.0, l1_sum = 0.0;
    for (int32_t s = 0; s < slots; ++s) {
      const int32_t v = vs[s];
      orc_camera cam;
      cam.fx = fx; cam.fy = fy; cam.cx = cx; cam.cy = cy; cam.width = w; cam.height = h;
      for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) cam.R[r * 3 + c] = poses[12 * v + r * 4 + c];
        cam.t[r] = poses[12 * v + r * 4 + 3];
      }
      orc_render_out* out = orc_render(cloud, &cam, cfg->background, &cfg->raster);
      l1_sum += orc_rgb_loss(out->image, images[v], w, h, 0.0, NULL);
      rgb_sum += orc_rgb_loss(out->image, images[v], w, h, cfg->beta, d_image);
      orc_grads g;
      orc_render_backward(cloud, &cam, out, d_image, w, h, &g);
      const double inv = 1.0 / (double)slots;
      for (int64_t k = 0; k < 3 * n; ++k) acc.d_means[k] += g.d_means[k] * inv;
      for (int64_t k = 0; k < 4 * n; ++k) acc.d_rotations[k] += g.d_rotations[k] * inv;
      for (int64_t k = 0; k < 3 * n; ++k) acc.d_log_scales[k] += g.d_log_scales[k] * inv;
      for (int64_t k = 0; k < n; ++k) acc.d_opacity_logits[k] += g.d_opacity_logits[k] * inv;
      for (int64_t k = 0; k < 3 * basis * n; ++k) acc.d_sh[k] += g.d_sh[k] * inv;
      memcpy(dpose + 6 * s, g.d_pose, sizeof(double) * 6);
      orc_grad_accum_add(out, &g, w > h ? w : h, acc_sum, acc_cnt);
      orc_grads_free(&g);
      orc_render_free(out);
    }
    /* regularisers on the pre-step parameters (pipelines.cpp:144-157) */
    double* d_aniso = (double*)malloc(sizeof(double) * (3 * n + 1));
    const double aniso = orc_anisotropy_loss(cloud->log_scales, n, cfg->aniso_ratio, d_aniso);
    for (int64_t k = 0; k < 3 * n; ++k) acc.d_log_scales[k] += d_aniso[k];
    free(d_aniso);
    double op_l1 = 0.0;
    if (t < cfg->opacity_l1_steps && cfg->opacity_l1_weight > 0.0) {
      double* ops = (double*)malloc(sizeof(double) * (n + 1));
      double* d_ops = (double*)malloc(sizeof(double) * (n + 1));
      for (int64_t i = 0; i < n; ++i) ops[i] = sigmoid(cloud->opacity_logits[i]);
      op_l1 = orc_opacity_l1(ops, n, d_ops);
      for (int64_t i = 0; i < n; ++i)
        acc.d_opacity_logits[i] += cfg->opacity_l1_weight * d_ops[i] * ops[i] * (1.0 - ops[i]);
      free(ops);
      free(d_ops);
    }
    const double total = rgb_sum / slots + aniso + cfg->opacity_l1_weight * op_l1;
    if (trace_total) trace_total[t] = total;
    if (trace_l1) trace_l1[t] = l1_sum / slots;
    if (!isfinite(total)) {
      status = 10;
      orc_grads_free(&acc);
      break;
    }
    double lrs[6];
    lrs[0] = orc_schedule(1, cfg->pos_lr_start, cfg->pos_lr_end, t, iters);
    lrs[1] = cfg->rot_lr;
    lrs[2] = cfg->scale_lr;
    lrs[3] = cfg->opacity_lr;
    lrs[4] = cfg->sh_dc_lr;
    lrs[5] = cfg->sh_rest_lr;
    orc_cloud_adam_step(cloud, &acc, st, lrs);
    orc_grads_free(&acc);
    if (cfg->optimize_poses) {
      const double cam_lr = orc_schedule(0, cfg->cam_lr_start, cfg->cam_lr_end, t, iters);
      for (int32_t s = 0; s < slots; ++s) {
        const int32_t v = vs[s];
        double R[9], tt[3], Rn[9], tn[3], applied[6];
        for (int r = 0; r < 3; ++r) {
          for (int c = 0; c < 3; ++c) R[r * 3 + c] = poses[12 * v + r * 4 + c];
          tt[r] = poses[12 * v + r * 4 + 3];
        }
        orc_pose_step(R, tt, dpose + 6 * s, cam_lr, &pad[v], Rn, tn, applied);
        for (int r = 0; r < 3; ++r) {
          for (int c = 0; c < 3; ++c) poses[12 * v + r * 4 + c] = Rn[r * 3 + c];
          poses[12 * v + r * 4 + 3] = tn[r];
        }
      }
    }
    if (cfg->densify_interval > 0 && t >= cfg->densify_start && t <= cfg->densify_stop && t > 0 &&
        (t - cfg->densify_start) % cfg->densify_interval == 0) {
      orc_cloud out;
      int32_t* src = NULL;
      int32_t rep[3];
      orc_densify_and_prune(cloud, acc_sum, acc_cnt, cfg->grad_threshold, cfg->densify_size_ratio, cfg->n_target,
                            cfg->prune_opacity, rng, &out, &src, rep);
      const int64_t nn = out.n, bw = 3 * (int64_t)sh_count(cloud->sh_degree);
      adam_remap(&st[0], src, nn, 3);
      adam_remap(&st[1], src, nn, 4);
      adam_remap(&st[2], src, nn, 3);
      adam_remap(&st[3], src, nn, 1);
      adam_remap(&st[4], src, nn, bw);
      free(src);
      orc_cloud_free(cloud);
      *cloud = out;
      free(acc_sum);
      free(acc_cnt);
      acc_sum = (double*)calloc((size_t)nn + 1, sizeof(double));
      acc_cnt = (int32_t*)calloc((size_t)nn + 1, sizeof(int32_t));
    }
  }
  for (int k = 0; k < 5; ++k) {
    free(st[k].m);
    free(st[k].v);
  }
  free(pad);
  free(d_image);
  free(dpose);
  free(vs);
  free(sc.order);
  free(acc_sum);
  free(acc_cnt);
  return status;
}

/* ------------------------------------------------------------ bootstrap */
/* scene.cpp:209-243: valid pixels (valid != 0, finite, d > 0) in row-major
 * order, every ceil(count / max_points)-th one lifted to cam_to_world (d * ray).
 * points / colors: caller buffers of max_points * 3. Returns the number of
 * points, -1 for no valid depth (ErrorCode::no_valid_depth). */
int64_t orc_unproject(const double* depth, const uint8_t* valid, int32_t w, int32_t h, const double* frame,
                      double fx, double fy, double cx, double cy, const double R[9], const double t[3],
                      int32_t max_points, double* points, double* colors) {
  int64_t count = 0;
  for (int64_t p = 0; p < (int64_t)w * h; ++p)
    if (valid[p] && isfinite(depth[p]) && depth[p] > 0.0) ++count;
  if (count == 0) return -1;
  const int64_t stride = (count + max_points - 1) / max_points;
  /* cam_to_world = (R^T, -R^T t) */
  double Rt[9], ti[3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rt[i * 3 + j] = R[j * 3 + i];
  mat3_vec(Rt, t, ti);
  for (int k = 0; k < 3; ++k) ti[k] = -ti[k];
  int64_t idx = 0, out = 0;
  for (int64_t p = 0; p < (int64_t)w * h; ++p) {
    if (!(valid[p] && isfinite(depth[p]) && depth[p] > 0.0)) continue;
    if (idx % stride == 0) {
      const int x = (int)(p % w), y = (int)(p / w);
      const double d = depth[p];
      const double ray[3] = {(x - cx) / fx, (y - cy) / fy, 1.0};
      const double q[3] = {d * ray[0], d * ray[1], d * ray[2]};
      double wpt[3];
      mat3_vec(Rt, q, wpt);
      for (int k = 0; k < 3; ++k) {
        points[3 * out + k] = wpt[k] + ti[k];
        colors[3 * out + k] = frame[p * 3 + k];
      }
      ++out;
    }
    ++idx;
  }
  return out;
}

/* scene.cpp:115-180: mean distance to the k nearest other points (exact;
 * restated as brute force, which selects the same k distances). */
void orc_mean_knn_distance(const double* pts, int64_t n, int k, double* out) {
  double best[8];
  for (int64_t i = 0; i < n; ++i) {
    for (int b = 0; b < k; ++b) best[b] = INFINITY;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const double dx = pts[3 * j] - pts[3 * i], dy = pts[3 * j + 1] - pts[3 * i + 1],
                   dz = pts[3 * j + 2] - pts[3 * i + 2];
      const double d = sqrt(dx * dx + dy * dy + dz * dz);
      if (d < best[k - 1]) {
        best[k - 1] = d;
        for (int b = k - 1; b > 0 && best[b] < best[b - 1]; --b) {
          const double tmp = best[b];
          best[b] = best[b - 1];
          best[b - 1] = tmp;
        }
      }
    }
    double sum = 0.0;
    for (int b = 0; b < k; ++b) sum += best[b];
    out[i] = sum / k;
  }
}

/* scene.cpp:182-207 */
void orc_init_from_points(const double* pts, const double* cols, int64_t n, int32_t sh_degree, orc_cloud* out) {
  double* nn = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  orc_mean_knn_distance(pts, n, 3, nn);
  orc_cloud_alloc(out, n, sh_degree);
  out->active_sh_degree = 0;
  const int basis = sh_count(sh_degree);
  const double op = log(0.1 / (1.0 - 0.1)); /* logit(0.1), core.hpp:113 */
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) out->means[3 * i + k] = pts[3 * i + k];
    out->rotations[4 * i] = 1.0;
    out->rotations[4 * i + 1] = out->rotations[4 * i + 2] = out->rotations[4 * i + 3] = 0.0;
    const double sc = log(fmax(nn[i], 1e-7));
    for (int k = 0; k < 3; ++k) out->log_scales[3 * i + k] = sc;
    out->opacity_logits[i] = op;
    for (int c = 0; c < 3; ++c) out->sh[(size_t)i * 3 * basis + c * basis] = (cols[3 * i + c] - 0.5) / 0.28209479177387814;
  }
  free(nn);
}

/* pipelines.cpp:224-250: unproject at the identity pose, SH-0 cloud, steps of
 * render -> rgb_loss -> render_backward -> cloud_adam_step (position lr
 * exponential over the fit). Returns 0, or -1 (no valid depth). */
int32_t orc_fit_frame_gaussians(const double* frame, const double* depth, const uint8_t* valid, int32_t w, int32_t h,
                                double fx, double fy, double cx, double cy, const orc_fit_cfg* cfg, orc_cloud* out) {
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, z[3] = {0, 0, 0};
  double* pts = (double*)malloc(sizeof(double) * 3 * (size_t)cfg->unproject_points);
  double* cols = (double*)malloc(sizeof(double) * 3 * (size_t)cfg->unproject_points);
  const int64_t np = orc_unproject(depth, valid, w, h, frame, fx, fy, cx, cy, I, z, cfg->unproject_points, pts, cols);
  if (np < 0) {
    free(pts);
    free(cols);
    return -1;
  }
  orc_init_from_points(pts, cols, np, 0, out);
  free(pts);
  free(cols);
  orc_adam_state st[5];
  memset(st, 0, sizeof st);
  orc_camera cam;
  cam.fx = fx; cam.fy = fy; cam.cx = cx; cam.cy = cy; cam.width = w; cam.height = h;
  memcpy(cam.R, I, sizeof I);
  memcpy(cam.t, z, sizeof z);
  double* d_image = (double*)malloc(sizeof(double) * (size_t)w * h * 3);
  for (int32_t t = 0; t < cfg->steps; ++t) {
    orc_render_out* ro = orc_render(out, &cam, cfg->background, &cfg->raster);
    orc_rgb_loss(ro->image, frame, w, h, cfg->beta, d_image);
    orc_grads g;
    orc_render_backward(out, &cam, ro, d_image, w, h, &g);
    const double lrs[6] = {orc_schedule(1, cfg->pos_lr_start, cfg->pos_lr_end, t, cfg->steps), cfg->rot_lr,
                           cfg->scale_lr, cfg->opacity_lr, cfg->sh_dc_lr, cfg->sh_rest_lr};
    orc_cloud_adam_step(out, &g, st, lrs);
    orc_grads_free(&g);
    orc_render_free(ro);
  }
  for (int k = 0; k < 5; ++k) {
    free(st[k].m);
    free(st[k].v);
  }
  free(d_image);
  return 0;
}

/* pipelines.cpp:252-290: transmittance-masked pose-only descent from the
 * identity; failure (ok = 0, identity) once the mask empties; lr halves
 * whenever fewer than 5% of the pixels pass. Returns ok. */
int32_t orc_estimate_relative_pose(const orc_cloud* cloud, const double* frame, int32_t w, int32_t h, double fx,
                                   double fy, double cx, double cy, const orc_relpose_cfg* cfg, double R_out[9],
                                   double t_out[3], double* final_loss) {
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double R[9], t[3] = {0, 0, 0};
  memcpy(R, I, sizeof R);
  memcpy(R_out, I, sizeof R);
  memset(t_out, 0, sizeof(double) * 3);
  *final_loss = 0.0;
  orc_pose_adam adam;
  memset(&adam, 0, sizeof adam);
  double best = INFINITY, lr_scale = 1.0;
  const size_t P = (size_t)w * h;
  uint8_t* mask = (uint8_t*)malloc(P);
  double* d_image = (double*)malloc(sizeof(double) * P * 3);
  int32_t ok = 1;
  for (int32_t it = 0; it < cfg->steps; ++it) {
    orc_camera cam;
    cam.fx = fx; cam.fy = fy; cam.cx = cx; cam.cy = cy; cam.width = w; cam.height = h;
    memcpy(cam.R, R, sizeof R);
    memcpy(cam.t, t, sizeof t);
    orc_render_out* ro = orc_render(cloud, &cam, cfg->background, &cfg->raster);
    orc_transmittance_mask(ro->accum_transmittance, (int64_t)P, cfg->mask_threshold, mask);
    size_t masked = 0;
    for (size_t p = 0; p < P; ++p) masked += mask[p];
    if (masked == 0) {
      memcpy(R_out, I, sizeof R);
      memset(t_out, 0, sizeof(double) * 3);
      ok = 0;
      orc_render_free(ro);
      break;
    }
    if ((double)masked < 0.05 * (double)P) lr_scale *= 0.5;
    int32_t st = 0;
    const double loss = orc_masked_rgb_loss(ro->image, frame, w, h, mask, cfg->beta, d_image, &st);
    if (loss < best) {
      best = loss;
      memcpy(R_out, R, sizeof R);
      memcpy(t_out, t, sizeof t);
      *final_loss = loss;
    }
    orc_grads g;
    orc_render_backward(cloud, &cam, ro, d_image, w, h, &g);
    const double lr = lr_scale * orc_schedule(0, cfg->lr_start, cfg->lr_end, it, cfg->steps);
    double Rn[9], tn[3], applied[6];
    orc_pose_step(R, t, g.d_pose, lr, &adam, Rn, tn, applied);
    memcpy(R, Rn, sizeof R);
    memcpy(t, tn, sizeof t);
    orc_grads_free(&g);
    orc_render_free(ro);
  }
  free(mask);
  free(d_image);
  return ok;
}

/* pipelines.cpp:292-312: per consecutive pair, fit frame t, estimate the
 * relative pose into frame t+1, compose (lie.hpp:48-53). poses: n x 12. */
int32_t orc_bootstrap_trajectory(const double* const* frames, const double* const* depths,
                                 const uint8_t* const* valids, int32_t n, int32_t w, int32_t h, double fx, double fy,
                                 double cx, double cy, const orc_fit_cfg* fit, const orc_relpose_cfg* rel,
                                 double* poses, int32_t* pair_ok) {
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, t[3] = {0, 0, 0};
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) poses[r * 4 + c] = R[r * 3 + c];
    poses[r * 4 + 3] = t[r];
  }
  for (int32_t f = 0; f + 1 < n; ++f) {
    orc_cloud cl;
    if (orc_fit_frame_gaussians(frames[f], depths[f], valids[f], w, h, fx, fy, cx, cy, fit, &cl) != 0) return -1;
    double Rr[9], tr[3], fl;
    pair_ok[f] = orc_estimate_relative_pose(&cl, frames[f + 1], w, h, fx, fy, cx, cy, rel, Rr, tr, &fl);
    orc_cloud_free(&cl);
    double Rn[9], tn[3];
    mat3_mul(Rr, R, Rn);
    mat3_vec(Rr, t, tn);
    for (int k = 0; k < 3; ++k) tn[k] += tr[k];
    memcpy(R, Rn, sizeof R);
    memcpy(t, tn, sizeof t);
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) poses[12 * (f + 1) + r * 4 + c] = R[r * 3 + c];
      poses[12 * (f + 1) + r * 4 + 3] = t[r];
    }
  }
  return 0;
}

/* ----------------------------------------------------------------- synth */
void orc_cloud_alloc(orc_cloud* c, int64_t n, int32_t sh_degree) { /* scene.cpp:14-24 */
  const int basis = sh_count(sh_degree);
  c->n = n;
  c->sh_degree = sh_degree;
  c->active_sh_degree = sh_degree;
  c->means = (double*)calloc(3 * n + 1, sizeof(double));
  c->rotations = (double*)calloc(4 * n + 1, sizeof(double));
  for (int64_t i = 0; i < n; ++i) c->rotations[4 * i] = 1.0;
  c->log_scales = (double*)calloc(3 * n + 1, sizeof(double));
  c->opacity_logits = (double*)calloc(n + 1, sizeof(double));
  c->sh = (double*)calloc((size_t)n * 3 * basis + 1, sizeof(double));
}
void orc_cloud_free(orc_cloud* c) {
  free(c->means); free(c->rotations); free(c->log_scales); free(c->opacity_logits); free(c->sh);
  memset(c, 0, sizeof *c);
}
/* synth.cpp:45-62 (cloud draws), active degree = capacity (synth.cpp:42) */
void orc_synth_cloud(orc_cloud* cloud, int64_t n, int32_t sh_degree, orc_rng* rng) {
  orc_cloud_alloc(cloud, n, sh_degree);
  const int basis = sh_count(sh_degree);
  for (int64_t i = 0; i < n; ++i) {
    double* m = cloud->means + 3 * i;
    m[2] = orc_rng_uniform_range(rng, -0.8, 0.8); /* right-to-left Vec3 args */
    m[1] = orc_rng_uniform_range(rng, -0.8, 0.8);
    m[0] = orc_rng_uniform_range(rng, -0.8, 0.8);
    rng_unit_quaternion(rng, cloud->rotations + 4 * i);
    double base = exp(orc_rng_uniform_range(rng, log(0.03), log(0.10)));
    for (int k = 0; k < 3; ++k) cloud->log_scales[3 * i + k] = log(base) + orc_rng_uniform_range(rng, -0.35, 0.35);
    cloud->opacity_logits[i] = logit(orc_rng_uniform_range(rng, 0.55, 0.9));
    double* sh = cloud->sh + (size_t)i * 3 * basis;
    for (int c = 0; c < 3; ++c) {
      sh[c * basis] = (orc_rng_uniform_range(rng, 0.15, 0.85) - 0.5) / kSh0;
      for (int b = 1; b < basis; ++b) {
        double scale = b < 4 ? 0.08 : 0.03;
        sh[c * basis + b] = orc_rng_uniform_range(rng, -scale, scale);
      }
    }
  }
}
/* synth.cpp:19-31 */
void orc_look_at(const double eye[3], const double target[3], double R[9], double t[3]) {
  double f[3] = {target[0] - eye[0], target[1] - eye[1], target[2] - eye[2]};
  double fn = norm3(f);
  f[0] /= fn; f[1] /= fn; f[2] /= fn;
  double up[3] = {0, 1, 0};
  if (fabs(f[0] * up[0] + f[1] * up[1] + f[2] * up[2]) > 0.999) { up[0] = 1; up[1] = 0; up[2] = 0; }
  double right[3] = {up[1] * f[2] - up[2] * f[1], up[2] * f[0] - up[0] * f[2], up[0] * f[1] - up[1] * f[0]};
  double rn = norm3(right);
  right[0] /= rn; right[1] /= rn; right[2] /= rn;
  double down[3] = {f[1] * right[2] - f[2] * right[1], f[2] * right[0] - f[0] * right[2], f[0] * right[1] - f[1] * right[0]};
  for (int k = 0; k < 3; ++k) { R[k] = right[k]; R[3 + k] = down[k]; R[6 + k] = f[k]; }
  double re[3];
  mat3_vec(R, eye, re);
  t[0] = -re[0]; t[1] = -re[1]; t[2] = -re[2];
}
/* synth.cpp:73-101 */
void orc_synth_poses(int32_t kind, int32_t cameras, double orbit_radius, double orbit_arc, orc_rng* rng,
                     double* poses) {
  double walker[3] = {0, 0, -orbit_radius};
  for (int k = 0; k < cameras; ++k) {
    double eye[3];
    if (kind == 0) {
      double theta = orbit_arc * (double)k / (double)(cameras > 1 ? cameras : 1);
      double phi = 0.25 * sin(3.0 * theta);
      eye[0] = orbit_radius * (sin(theta) * cos(phi));
      eye[1] = orbit_radius * sin(phi);
      eye[2] = orbit_radius * (-cos(theta) * cos(phi));
    } else if (kind == 1) {
      eye[2] = -orbit_radius + orc_rng_uniform_range(rng, -0.15, 0.15);
      eye[1] = orc_rng_uniform_range(rng, -0.4, 0.4);
      eye[0] = orc_rng_uniform_range(rng, -0.4, 0.4);
    } else {
      if (k > 0) {
        double nrm[3];
        rng_normal3(rng, nrm);
        for (int j = 0; j < 3; ++j) walker[j] += 0.08 * nrm[j];
      }
      memcpy(eye, walker, sizeof eye);
    }
    double target[3] = {0, 0, 0};
    if (kind == 2) {
      double jy = 0.05 * orc_rng_normal(rng);
      double jx = 0.05 * orc_rng_normal(rng);
      target[0] = jx;
      target[1] = jy;
    }
    double R[9], t[3];
    orc_look_at(eye, target, R, t);
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) poses[12 * k + r * 4 + c] = R[r * 3 + c];
      poses[12 * k + r * 4 + 3] = t[r];
    }
  }
}
/* eval.cpp:130-146 */
void orc_perturb_pose(const double R[9], const double t[3], double rot_deg, double trans, orc_rng* rng,
                      double R_out[9], double t_out[3]) {
  const double to_rad = ORC_PI / 180.0;
  double ax = orc_rng_uniform_range(rng, -rot_deg, rot_deg) * to_rad;
  double ay = orc_rng_uniform_range(rng, -rot_deg, rot_deg) * to_rad;
  double az = orc_rng_uniform_range(rng, -rot_deg, rot_deg) * to_rad;
  double off[3];
  off[2] = orc_rng_uniform_range(rng, -trans, trans);
  off[1] = orc_rng_uniform_range(rng, -trans, trans);
  off[0] = orc_rng_uniform_range(rng, -trans, trans);
  double wz[3] = {0, 0, az}, wy[3] = {0, ay, 0}, wx[3] = {ax, 0, 0};
  double Rz[9], Ry[9], Rx[9], tmp[9], rot[9];
  orc_so3_exp(wz, Rz);
  orc_so3_exp(wy, Ry);
  orc_so3_exp(wx, Rx);
  mat3_mul(Rz, Ry, tmp);
  mat3_mul(tmp, Rx, rot);
  /* cam_to_world = inverse */
  double Rcw[9], tcw[3];
  mat3_T(R, Rcw);
  mat3T_vec(R, t, tcw);
  tcw[0] = -tcw[0]; tcw[1] = -tcw[1]; tcw[2] = -tcw[2];
  double Rn[9];
  mat3_mul(Rcw, rot, Rn);
  tcw[0] += off[0]; tcw[1] += off[1]; tcw[2] += off[2];
  /* back to world_to_cam */
  mat3_T(Rn, R_out);
  double tt[3];
  mat3T_vec(Rn, tcw, tt);
  t_out[0] = -tt[0]; t_out[1] = -tt[1]; t_out[2] = -tt[2];
}
/* eval.cpp:148-152 */
void orc_perturb_pose_tangent(const double R[9], const double t[3], double sigma, orc_rng* rng, double R_out[9],
                              double t_out[3]) {
  double noise[6], Re[9], te[3];
  for (int k = 0; k < 6; ++k) noise[k] = sigma * orc_rng_normal(rng);
  orc_se3_exp(noise, Re, te);
  double Rn[9], tn[3];
  mat3_mul(Re, R, Rn);
  mat3_vec(Re, t, tn);
  tn[0] += te[0]; tn[1] += te[1]; tn[2] += te[2];
  memcpy(R_out, Rn, sizeof Rn);
  memcpy(t_out, tn, sizeof tn);
}
/* eval.cpp:122-128 on cam_to_world poses (callers pass inverse()) */
void orc_abs_pose_error(const double Rp[9], const double tp[3], const double Rg[9], const double tg[3],
                        double* rot_deg, double* trans) {
  /* pred_c2w.R * gt_c2w.R^T = Rp^T Rg */
  double RpT[9], rel[9];
  mat3_T(Rp, RpT);
  mat3_mul(RpT, Rg, rel);
  *rot_deg = orc_rotation_angle(rel) * 180.0 / ORC_PI;
  double cp[3], cg[3];
  mat3T_vec(Rp, tp, cp);
  mat3T_vec(Rg, tg, cg);
  double d[3] = {-cp[0] + cg[0], -cp[1] + cg[1], -cp[2] + cg[2]};
  *trans = norm3(d);
}

/* --------------------------------------------------- gradcheck (tests/) */
/* tests/gradcheck.hpp:26-61 */
void orc_make_gradcheck_scene(orc_rng* rng, int32_t n, int32_t image_size, orc_cloud* cloud, orc_camera* cam,
                              double bg[3]) {
  cam->width = cam->height = image_size;
  cam->fx = cam->fy = 0.75 * image_size;
  cam->cx = cam->cy = 0.5 * (image_size - 1);
  double tau[6];
  for (int k = 0; k < 3; ++k) tau[k] = orc_rng_uniform_range(rng, -0.2, 0.2);
  for (int k = 3; k < 6; ++k) tau[k] = orc_rng_uniform_range(rng, -0.3, 0.3);
  orc_se3_exp(tau, cam->R, cam->t);
  bg[0] = 0.2; bg[1] = 0.25; bg[2] = 0.3;
  orc_cloud_alloc(cloud, n, 3);
  cloud->active_sh_degree = 3;
  double Rcw[9], tcw[3];
  mat3_T(cam->R, Rcw);
  mat3T_vec(cam->R, cam->t, tcw);
  tcw[0] = -tcw[0]; tcw[1] = -tcw[1]; tcw[2] = -tcw[2];
  const int basis = 16;
  for (int i = 0; i < n; ++i) {
    double z = orc_rng_uniform_range(rng, 1.5, 3.0);
    double px = orc_rng_uniform_range(rng, 0.2, 0.8) * (image_size - 1);
    double py = orc_rng_uniform_range(rng, 0.2, 0.8) * (image_size - 1);
    double mc[3] = {(px - cam->cx) * z / cam->fx, (py - cam->cy) * z / cam->fy, z};
    pose_act(Rcw, tcw, mc, cloud->means + 3 * i);
    rng_unit_quaternion(rng, cloud->rotations + 4 * i);
    double base = orc_rng_uniform_range(rng, 0.12, 0.3);
    for (int k = 0; k < 3; ++k) cloud->log_scales[3 * i + k] = log(base) + orc_rng_uniform_range(rng, -0.35, 0.35);
    cloud->opacity_logits[i] = logit(orc_rng_uniform_range(rng, 0.25, 0.75));
    double* sh = cloud->sh + (size_t)i * 3 * basis;
    for (int c = 0; c < 3; ++c) {
      sh[c * basis] = (orc_rng_uniform_range(rng, 0.3, 0.7) - 0.5) / kSh0;
      for (int b = 1; b < basis; ++b) sh[c * basis + b] = orc_rng_uniform_range(rng, -0.03, 0.03);
    }
  }
}

typedef struct { double mu2d[2], conic[4], color[3], opacity, depth, radius; } flat_t;
static int cmp_flat(const void* a, const void* b) {
  double da = ((const flat_t*)a)->depth, db = ((const flat_t*)b)->depth;
  return (da > db) - (da < db);
}
/* tests/gradcheck.hpp:67-161 */
int orc_scene_is_conditioned(const orc_cloud* cloud, const orc_camera* cam, const double bg[3],
                             const orc_raster_config* cfg) {
  const double cutoff2 = cfg->cutoff_sigma * cfg->cutoff_sigma;
  const double margin_g = 1e-3, margin_alpha = 1e-3, margin_term = 1e-6, margin_edge_px = 1e-2, margin_color = 1e-3;
  double cc[3];
  cam_center(cam, cc);
  flat_t* flats = (flat_t*)malloc(sizeof(flat_t) * (cloud->n + 1));
  int64_t nf = 0;
  int ok = 1;
  const int basis = sh_count(cloud->sh_degree);
  for (int64_t i = 0; i < cloud->n && ok; ++i) {
    double mc[3];
    pose_act(cam->R, cam->t, cloud->means + 3 * i, mc);
    if (!(mc[2] > cfg->z_near + 1e-3)) { ok = 0; break; }
    flat_t f;
    orc_project(cloud->means + 3 * i, cam, f.mu2d, &f.depth);
    double s[3] = {exp(cloud->log_scales[3 * i]), exp(cloud->log_scales[3 * i + 1]), exp(cloud->log_scales[3 * i + 2])};
    double sigma[9], cov[4];
    orc_covariance3d(cloud->rotations + 4 * i, s, sigma);
    orc_covariance2d(sigma, mc, cam, cfg->dilation, cov);
    double mid = 0.5 * (cov[0] + cov[3]), diff = 0.5 * (cov[0] - cov[3]);
    double lmax = mid + sqrt(diff * diff + cov[1] * cov[2]);
    f.radius = cfg->cutoff_sigma * sqrt(lmax);
    double det = cov[0] * cov[3] - cov[1] * cov[2];
    f.conic[0] = cov[3] / det; f.conic[1] = -cov[1] / det; f.conic[2] = -cov[2] / det; f.conic[3] = cov[0] / det;
    double dir[3] = {cloud->means[3 * i] - cc[0], cloud->means[3 * i + 1] - cc[1], cloud->means[3 * i + 2] - cc[2]};
    double dn = norm3(dir);
    dir[0] /= dn; dir[1] /= dn; dir[2] /= dn;
    uint8_t cm;
    orc_sh_eval(cloud->sh + (size_t)i * 3 * basis, dir, cloud->active_sh_degree, f.color, &cm);
    double bv[16];
    orc_sh_basis(dir, cloud->active_sh_degree, bv);
    for (int c = 0; c < 3 && ok; ++c) {
      double v = 0.5;
      for (int b = 0; b < basis; ++b) v += cloud->sh[(size_t)i * 3 * basis + c * basis + b] * bv[b];
      if (fabs(v) < margin_color) ok = 0;
    }
    f.opacity = sigmoid(cloud->opacity_logits[i]);
    double ex[2] = {f.mu2d[0] - f.radius, f.mu2d[0] + f.radius};
    double ey[2] = {f.mu2d[1] - f.radius, f.mu2d[1] + f.radius};
    for (int k = 0; k < 2 && ok; ++k) {
      double nearest = round(ex[k] / cfg->tile_size) * cfg->tile_size;
      if (fabs(ex[k] - nearest) < margin_edge_px) ok = 0;
      if (fabs(ex[k] - (cam->width - 1)) < margin_edge_px || fabs(ex[k]) < margin_edge_px) ok = 0;
    }
    for (int k = 0; k < 2 && ok; ++k) {
      double nearest = round(ey[k] / cfg->tile_size) * cfg->tile_size;
      if (fabs(ey[k] - nearest) < margin_edge_px) ok = 0;
      if (fabs(ey[k] - (cam->height - 1)) < margin_edge_px || fabs(ey[k]) < margin_edge_px) ok = 0;
    }
    flats[nf++] = f;
  }
  if (ok) {
    /* stable sort by depth: insertion sort (n is tiny) */
    for (int64_t a = 1; a < nf; ++a) {
      flat_t key = flats[a];
      int64_t b = a - 1;
      while (b >= 0 && flats[b].depth > key.depth) { flats[b + 1] = flats[b]; --b; }
      flats[b + 1] = key;
    }
    (void)cmp_flat;
    for (int y = 0; y < cam->height && ok; ++y) {
      for (int x = 0; x < cam->width && ok; ++x) {
        double T = 1.0, col[3] = {0, 0, 0};
        for (int64_t k = 0; k < nf; ++k) {
          const flat_t* f = &flats[k];
          double d0 = x - f->mu2d[0], d1 = y - f->mu2d[1];
          double c0 = f->conic[0] * d0 + f->conic[1] * d1, c1 = f->conic[2] * d0 + f->conic[3] * d1;
          double g = d0 * c0 + d1 * c1;
          if (fabs(g - cutoff2) < margin_g) { ok = 0; break; }
          if (g > cutoff2) continue;
          double ar = f->opacity * exp(-0.5 * g);
          if (fabs(ar - cfg->alpha_clamp) < margin_alpha) { ok = 0; break; }
          double al = ar < cfg->alpha_clamp ? ar : cfg->alpha_clamp;
          for (int c = 0; c < 3; ++c) col[c] += f->color[c] * (al * T);
          T *= (1.0 - al);
          if (fabs(T - cfg->early_termination) < margin_term) { ok = 0; break; }
          if (T < cfg->early_termination) break;
        }
        for (int c = 0; c < 3 && ok; ++c) {
          double v = col[c] + bg[c] * T;
          if (fabs(v - 1.0) < margin_color) ok = 0;
        }
      }
    }
  }
  free(flats);
  return ok;
}

static double render_dot(const orc_cloud* cloud, const orc_camera* cam, const double bg[3],
                         const orc_raster_config* cfg, const double* d_image) {
  orc_render_out* out = orc_render(cloud, cam, bg, cfg);
  double loss = 0.0;
  const size_t n = (size_t)cam->width * cam->height * 3;
  for (size_t i = 0; i < n; ++i) loss += d_image[i] * out->image[i];
  orc_render_free(out);
  return loss;
}
static void gc_update(double* max_err, char* worst, int32_t* checked, double an, double fd, const char* label) {
  double den = fabs(fd) > 1e-3 ? fabs(fd) : 1e-3;
  double err = fabs(an - fd) / den;
  if (fabs(an - fd) < 1e-8) err = 0.0;
  if (err > *max_err) {
    *max_err = err;
    if (worst) snprintf(worst, 32, "%s", label);
  }
  ++*checked;
}
/* tests/gradcheck.hpp:201-254 */
double orc_gradcheck(const orc_cloud* cloud, const orc_camera* cam, const double bg[3], const orc_raster_config* cfg,
                     orc_rng* rng, double step, int32_t* checked, char* worst) {
  const size_t np = (size_t)cam->width * cam->height * 3;
  double* d_image = (double*)malloc(sizeof(double) * np);
  for (size_t i = 0; i < np; ++i) d_image[i] = orc_rng_uniform_range(rng, -1.0, 1.0);
  orc_render_out* out = orc_render(cloud, cam, bg, cfg);
  orc_grads g;
  orc_render_backward(cloud, cam, out, d_image, cam->width, cam->height, &g);
  orc_render_free(out);
  orc_cloud probe;
  orc_cloud_alloc(&probe, cloud->n, cloud->sh_degree);
  probe.active_sh_degree = cloud->active_sh_degree;
  const int basis = sh_count(cloud->sh_degree);
  memcpy(probe.means, cloud->means, sizeof(double) * 3 * cloud->n);
  memcpy(probe.rotations, cloud->rotations, sizeof(double) * 4 * cloud->n);
  memcpy(probe.log_scales, cloud->log_scales, sizeof(double) * 3 * cloud->n);
  memcpy(probe.opacity_logits, cloud->opacity_logits, sizeof(double) * cloud->n);
  memcpy(probe.sh, cloud->sh, sizeof(double) * 3 * basis * cloud->n);
  double max_err = 0.0;
  *checked = 0;
#define FD_AT(slot, out_fd) do { double saved = *(slot); *(slot) = saved + step; \
    double up = render_dot(&probe, cam, bg, cfg, d_image); *(slot) = saved - step; \
    double dn = render_dot(&probe, cam, bg, cfg, d_image); *(slot) = saved; (out_fd) = (up - dn) / (2.0 * step); } while (0)
  char label[32];
  for (int64_t i = 0; i < cloud->n; ++i) {
    double fd;
    for (int k = 0; k < 3; ++k) { FD_AT(&probe.means[3 * i + k], fd); snprintf(label, 32, "mean/%lld", (long long)i); gc_update(&max_err, worst, checked, g.d_means[3 * i + k], fd, label); }
    for (int k = 0; k < 4; ++k) { FD_AT(&probe.rotations[4 * i + k], fd); snprintf(label, 32, "rot/%lld", (long long)i); gc_update(&max_err, worst, checked, g.d_rotations[4 * i + k], fd, label); }
    for (int k = 0; k < 3; ++k) { FD_AT(&probe.log_scales[3 * i + k], fd); snprintf(label, 32, "scale/%lld", (long long)i); gc_update(&max_err, worst, checked, g.d_log_scales[3 * i + k], fd, label); }
    FD_AT(&probe.opacity_logits[i], fd); snprintf(label, 32, "opacity/%lld", (long long)i); gc_update(&max_err, worst, checked, g.d_opacity_logits[i], fd, label);
    for (int k = 0; k < 3 * basis; ++k) { FD_AT(&probe.sh[(size_t)i * 3 * basis + k], fd); snprintf(label, 32, "sh/%lld", (long long)i); gc_update(&max_err, worst, checked, g.d_sh[(size_t)i * 3 * basis + k], fd, label); }
  }
#undef FD_AT
  for (int k = 0; k < 6; ++k) {
    double val[2];
    for (int sgn = 0; sgn < 2; ++sgn) {
      double tau[6] = {0, 0, 0, 0, 0, 0};
      tau[k] = sgn == 0 ? step : -step;
      double Re[9], te[3];
      orc_se3_exp(tau, Re, te);
      orc_camera moved = *cam;
      mat3_mul(Re, cam->R, moved.R);
      mat3_vec(Re, cam->t, moved.t);
      moved.t[0] += te[0]; moved.t[1] += te[1]; moved.t[2] += te[2];
      val[sgn] = render_dot(cloud, &moved, bg, cfg, d_image);
    }
    snprintf(label, 32, "pose/%d", k);
    gc_update(&max_err, worst, checked, g.d_pose[k], (val[0] - val[1]) / (2.0 * step), label);
  }
  orc_cloud_free(&probe);
  orc_grads_free(&g);
  free(d_image);
  return max_err;
}
