// k_optim.cu — K5a SE(3) pose step and K5b Adam on Gaussians.
//
// K5a restates pose_step (trainer.cpp:71-90): Adam on the 6-vector with bias
// correction (beta1 .9, beta2 .999, eps 1e-15, trainer.hpp:80-82), return
// the pose bit-for-bit when the update is exactly zero (86), otherwise
// se3_exp(delta) * pose (lie.cpp:117-129 with series_coeffs 26-43) followed
// by SVD re-orthonormalisation (lie.cpp:87-97; two-sided Jacobi SVD as in
// Eigen's JacobiSVD). Runs in FP64 on the device, batched over views, and
// fused with pose_descent's bookkeeping (pipelines.cpp:66-90: best-loss
// pose, loss < 1e-14 exit, cosine lr schedule, |applied| < eps exit) so the
// pose-estimation loop never returns to the host between iterations.
//
// K5b restates cloud_adam_step (pipelines.cpp:18-41) / adam_step
// (trainer.cpp:40-69) over the plane-major FP32 cloud: per-plane learning
// rate groups (means, rotations, log-scales, opacity, SH DC / rest by
// k % basis == 0) and renormalisation of exactly those quaternions whose
// bits changed.
#include "gsb_internal.cuh"

#include <algorithm>
#include <cmath>

namespace gsb {

constexpr double kB1 = 0.9, kB2 = 0.999, kEps = 1e-15;

struct PoseState {
  double R[9], t[3];
  double m[6], v[6];
  int64_t step;
  double best_R[9], best_t[3];
  double best_loss, final_loss;
  double applied[6];
  int32_t iter, steps_used, converged, stop;
  int32_t aborted;         // iterations discarded (entry capacity / per-tile sort overflow)
  uint32_t abort_k_max;    // largest K seen by a discarded iteration
  uint32_t abort_tile_ovf; // a discarded iteration had a tile beyond the per-tile sort
  int32_t pad;
};

struct PoseCtl {
  double lr_start, lr_end, eps;
  int32_t budget;
  int32_t fixed_lr;  // 1: use lr_start for every step (single pose_step calls)
};

__device__ void d_series(double theta, double* a, double* b, double* d) {
  const double t2 = theta * theta;
  if (theta < 1e-8) {
    *a = 1.0 - t2 / 6.0;
    *b = 0.5 - t2 / 24.0;
  } else {
    const double hs = sin(0.5 * theta);
    *a = sin(theta) / theta;
    *b = 2.0 * hs * hs / t2;
  }
  if (theta < 1e-2) *d = 1.0 / 6.0 - t2 / 120.0 + t2 * t2 / 5040.0;
  else *d = (theta - sin(theta)) / (t2 * theta);
}

__device__ void d_mat3_mul(const double* A, const double* B, double* C) {
  double r[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
  for (int k = 0; k < 9; ++k) C[k] = r[k];
}

// Two-sided Jacobi SVD of a 3x3 (Eigen JacobiSVD's sweep, 2x2 real SVD step,
// sign fix and descending sort), returning the polar factor U V^T with the
// det < 0 fix of Se3Pose::orthonormalize.
__device__ void d_orthonormalize(double* Rm) {
  const double eps = 2.220446049250313e-16, min_pos = 2.2250738585072014e-308;
  double M[9], U[9], V[9];
  double scale = 0.0;
  for (int k = 0; k < 9; ++k) scale = fmax(scale, fabs(Rm[k]));
  if (scale == 0.0) scale = 1.0;
  for (int k = 0; k < 9; ++k) {
    M[k] = Rm[k] / scale;
    U[k] = V[k] = (k % 4 == 0) ? 1.0 : 0.0;
  }
  double max_diag = fmax(fabs(M[0]), fmax(fabs(M[4]), fabs(M[8])));
  bool finished = false;
  for (int sweep = 0; sweep < 100 && !finished; ++sweep) {
    finished = true;
    for (int p = 1; p < 3; ++p) {
      for (int q = 0; q < p; ++q) {
        const double thr = fmax(min_pos, 2.0 * eps * max_diag);
        if (!(fabs(M[p * 3 + q]) > thr || fabs(M[q * 3 + p]) > thr)) continue;
        finished = false;
        const double m00 = M[p * 3 + p], m01 = M[p * 3 + q], m10 = M[q * 3 + p], m11 = M[q * 3 + q];
        double c1 = 1.0, s1 = 0.0;
        const double tt = m00 + m11, dd = m10 - m01;
        if (!(fabs(dd) < min_pos)) {
          const double u = tt / dd, tmp = sqrt(1.0 + u * u);
          s1 = 1.0 / tmp;
          c1 = u / tmp;
        }
        const double n00 = c1 * m00 + s1 * m10, n01 = c1 * m01 + s1 * m11, n11 = -s1 * m01 + c1 * m11;
        double cr = 1.0, sr = 0.0;
        const double deno = 2.0 * fabs(n01);
        if (!(deno < min_pos)) {
          const double tau = (n00 - n11) / deno, w = sqrt(tau * tau + 1.0);
          const double t = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
          const double sgn = t > 0.0 ? 1.0 : -1.0, nn = 1.0 / sqrt(t * t + 1.0);
          sr = -sgn * (n01 / fabs(n01)) * fabs(t) * nn;
          cr = nn;
        }
        // j_left = rot1 * j_right^T
        const double jlc = c1 * cr - s1 * (-sr), jls = c1 * (-sr) + s1 * cr;
        for (int i = 0; i < 3; ++i) {  // M.applyOnTheLeft(p,q,jl)
          const double x = M[p * 3 + i], y = M[q * 3 + i];
          M[p * 3 + i] = jlc * x + jls * y;
          M[q * 3 + i] = -jls * x + jlc * y;
        }
        for (int i = 0; i < 3; ++i) {  // U.applyOnTheRight(p,q,jl^T): uses (c, -s)^T = (c, s)
          const double x = U[i * 3 + p], y = U[i * 3 + q];
          U[i * 3 + p] = jlc * x + jls * y;
          U[i * 3 + q] = -jls * x + jlc * y;
        }
        for (int i = 0; i < 3; ++i) {  // M, V .applyOnTheRight(p,q,jr): rotation (c, -s)
          double x = M[i * 3 + p], y = M[i * 3 + q];
          M[i * 3 + p] = cr * x - sr * y;
          M[i * 3 + q] = sr * x + cr * y;
          x = V[i * 3 + p];
          y = V[i * 3 + q];
          V[i * 3 + p] = cr * x - sr * y;
          V[i * 3 + q] = sr * x + cr * y;
        }
        max_diag = fmax(max_diag, fmax(fabs(M[p * 3 + p]), fabs(M[q * 3 + q])));
      }
    }
  }
  double S[3];
  for (int i = 0; i < 3; ++i) {
    const double a = M[i * 3 + i];
    S[i] = fabs(a);
    if (a < 0.0)
      for (int r = 0; r < 3; ++r) U[r * 3 + i] = -U[r * 3 + i];
  }
  for (int i = 0; i < 3; ++i) {
    int best = i;
    for (int k = i + 1; k < 3; ++k)
      if (S[k] > S[best]) best = k;
    if (best != i) {
      const double ts = S[i];
      S[i] = S[best];
      S[best] = ts;
      for (int r = 0; r < 3; ++r) {
        double tu = U[r * 3 + i];
        U[r * 3 + i] = U[r * 3 + best];
        U[r * 3 + best] = tu;
        tu = V[r * 3 + i];
        V[r * 3 + i] = V[r * 3 + best];
        V[r * 3 + best] = tu;
      }
    }
  }
  double Vt[9], out[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Vt[i * 3 + j] = V[j * 3 + i];
  d_mat3_mul(U, Vt, out);
  const double det = out[0] * (out[4] * out[8] - out[5] * out[7]) - out[1] * (out[3] * out[8] - out[5] * out[6]) +
                     out[2] * (out[3] * out[7] - out[4] * out[6]);
  if (det < 0.0) {
    for (int r = 0; r < 3; ++r) U[r * 3 + 2] = -U[r * 3 + 2];
    d_mat3_mul(U, Vt, out);
  }
  for (int k = 0; k < 9; ++k) Rm[k] = out[k];
}

__device__ void d_pose_step(PoseState& s, const double* dpose, double lr) {
  ++s.step;
  const double bc1 = 1.0 - pow(kB1, (double)s.step), bc2 = 1.0 - pow(kB2, (double)s.step);
  double delta[6];
  bool zero = true;
  for (int k = 0; k < 6; ++k) {
    const double g = dpose[k];
    s.m[k] = kB1 * s.m[k] + (1.0 - kB1) * g;
    s.v[k] = kB2 * s.v[k] + (1.0 - kB2) * g * g;
    const double mh = s.m[k] / bc1, vh = s.v[k] / bc2;
    delta[k] = -lr * mh / (sqrt(vh) + kEps);
    s.applied[k] = delta[k];
    zero = zero && delta[k] == 0.0;
  }
  if (zero) return;
  // se3_exp(delta)
  const double* w = delta + 3;
  const double theta = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double a, b, d;
  d_series(theta, &a, &b, &d);
  const double W[9] = {0.0, -w[2], w[1], w[2], 0.0, -w[0], -w[1], w[0], 0.0};
  double W2[9], Re[9], Vm[9];
  d_mat3_mul(W, W, W2);
  for (int k = 0; k < 9; ++k) {
    const double I = (k % 4 == 0) ? 1.0 : 0.0;
    Re[k] = I + a * W[k] + b * W2[k];
    Vm[k] = I + b * W[k] + d * W2[k];
  }
  double te[3], tn[3], Rn[9];
  for (int i = 0; i < 3; ++i) te[i] = Vm[i * 3] * delta[0] + Vm[i * 3 + 1] * delta[1] + Vm[i * 3 + 2] * delta[2];
  d_mat3_mul(Re, s.R, Rn);
  for (int i = 0; i < 3; ++i) tn[i] = Re[i * 3] * s.t[0] + Re[i * 3 + 1] * s.t[1] + Re[i * 3 + 2] * s.t[2] + te[i];
  d_orthonormalize(Rn);
  for (int k = 0; k < 9; ++k) s.R[k] = Rn[k];
  for (int k = 0; k < 3; ++k) s.t[k] = tn[k];
}

__device__ void d_write_cam(const PoseState& s, CamDev* cam) {
  for (int k = 0; k < 9; ++k) cam->R[k] = s.R[k];
  for (int k = 0; k < 3; ++k) cam->t[k] = s.t[k];
  for (int i = 0; i < 3; ++i)  // center = -(R^T t)
    cam->center[i] = -(s.R[i] * s.t[0] + s.R[3 + i] * s.t[1] + s.R[6 + i] * s.t[2]);
}

// One pose_descent iteration tail (after render + loss + backward).
// One 256-thread block: the d_pose reduction of K4b's block partials
// (block_reduce_pose, the same fixed order as pose_reduce_kernel) fused in
// front of the pose step, which thread 0 runs. d_pose is also written to
// dpose_out for the session's readers.
__global__ void __launch_bounds__(256) pose_iter_kernel(PoseState* st, const double* __restrict__ pose_blocks,
                                                        int64_t nb, double* __restrict__ dpose_out,
                                                        const double* __restrict__ loss3, PoseCtl ctl, CamDev* cam,
                                                        double* trace_pose, double* trace_loss,
                                                        const uint32_t* __restrict__ k_dev, int64_t k_cap) {
  __shared__ double s_red[6][256];
  double dpose[6];
  block_reduce_pose(pose_blocks, nb, s_red, dpose);
  if (threadIdx.x != 0) return;
  for (int k = 0; k < 6; ++k) dpose_out[k] = dpose[k];
  PoseState s = *st;
  if (s.stop) return;
  // k_dev = {K, tile overflow flag}: the entry capacity or the per-tile sort
  // overflowed — discard the iteration; the host fixes the cause and re-runs it
  if ((int64_t)k_dev[0] > k_cap || k_dev[1] != 0u) {
    st->aborted = s.aborted + 1;
    st->abort_k_max = max(s.abort_k_max, k_dev[0]);
    st->abort_tile_ovf = s.abort_tile_ovf | k_dev[1];
    return;
  }
  const int it = s.iter;
  const double loss = loss3[2];
  if (trace_pose) {
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) trace_pose[12 * it + r * 4 + c] = s.R[r * 3 + c];
      trace_pose[12 * it + r * 4 + 3] = s.t[r];
    }
  }
  if (trace_loss) trace_loss[it] = loss;
  if (loss < s.best_loss) {
    s.best_loss = loss;
    for (int k = 0; k < 9; ++k) s.best_R[k] = s.R[k];
    for (int k = 0; k < 3; ++k) s.best_t[k] = s.t[k];
    s.final_loss = loss;
  }
  if (loss < 1e-14) {
    s.converged = 1;
    s.steps_used = it + 1;
    s.stop = 1;
    *st = s;
    return;
  }
  double lr = ctl.lr_start;
  if (!ctl.fixed_lr) {  // schedule(cosine, start, end, t, budget) (trainer.cpp:30-38)
    double f = ctl.budget > 0 ? (double)it / (double)ctl.budget : 1.0;
    f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
    lr = ctl.budget > 0 ? ctl.lr_end + (ctl.lr_start - ctl.lr_end) * 0.5 * (1.0 + cos(M_PI * f)) : ctl.lr_end;
  }
  d_pose_step(s, dpose, lr);
  s.steps_used = it + 1;
  s.iter = it + 1;
  double an = 0.0;
  for (int k = 0; k < 6; ++k) an += s.applied[k] * s.applied[k];
  if (sqrt(an) < ctl.eps) {
    s.converged = 1;
    s.stop = 1;
  }
  if (s.iter >= ctl.budget) s.stop = 1;
  *st = s;
  if (cam) d_write_cam(s, cam);
}

// Plain pose_step on a batch of poses (C-ABI gsb_pose_step).
__global__ void pose_step_kernel(PoseState* st, const double* __restrict__ dpose, double lr, int nb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  PoseState s = st[i];
  d_pose_step(s, dpose + 6 * i, lr);
  st[i] = s;
}

// adam_step (trainer.cpp:40-53) on a flat FP64 array.
// adam_step (trainer.cpp:40-69), both overloads: lrs == nullptr -> the scalar
// lr, else lr_of(i) = lrs[i]. Explicitly rounded FP64 in the reference's
// expression order (no FMA contraction), so the update is the reference's
// bit for bit.
__global__ void adam_f64_kernel(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                                double* __restrict__ v, int64_t n, double lr, const double* __restrict__ lrs,
                                double bc1, double bc2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double gi = g[i];
  const double mi = __dadd_rn(__dmul_rn(kB1, m[i]), __dmul_rn(1.0 - kB1, gi));
  const double vi = __dadd_rn(__dmul_rn(kB2, v[i]), __dmul_rn(__dmul_rn(1.0 - kB2, gi), gi));
  m[i] = mi;
  v[i] = vi;
  const double m_hat = __ddiv_rn(mi, bc1), v_hat = __ddiv_rn(vi, bc2);
  const double step = __ddiv_rn(__dmul_rn(lrs ? lrs[i] : lr, m_hat), __dadd_rn(__dsqrt_rn(v_hat), kEps));
  p[i] = __dsub_rn(p[i], step);
}

// CloudAdam's element update (pipelines.cpp:18-41) on an FP32 plane entry;
// one definition for every kernel that steps cloud planes. Every operation is
// an explicitly rounded intrinsic, so the result does not depend on how the
// compiler contracts the expression in a given unrolling. Returns the new
// parameter.
__device__ __forceinline__ float adam_f32(float& m, float& v, float p, float gi, float lr, float bc1, float bc2) {
  const float mi = __fmaf_rn(m, 0.9f, __fmul_rn(gi, 0.1f));                    // 0.9 m + 0.1 g
  const float vi = __fmaf_rn(v, 0.999f, __fmul_rn(gi, __fmul_rn(gi, 0.001f)));  // 0.999 v + 0.001 g g
  m = mi;
  v = vi;
  const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(vi, bc2)), 1e-15f);
  return __fsub_rn(p, __fdiv_rn(__fmul_rn(lr, __fdiv_rn(mi, bc1)), den));
}

struct AdamCoef {
  float lr[6];  // pos, rot, scale, opacity, sh_dc, sh_rest
  float bc1[5], bc2[5];
};

// cloud_adam_step over FP32 planes; one thread per Gaussian.
__global__ void __launch_bounds__(256) cloud_adam_kernel(float* __restrict__ params, const float* __restrict__ grads,
                                                         float* __restrict__ m, float* __restrict__ v, int64_t n,
                                                         int64_t n_pad, int nplanes, int basis, AdamCoef c) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool quat_moved = false;
  float q[4];
  auto step = [&](int p, int grp, float lr) {
    const int64_t k = (int64_t)p * n_pad + i;
    float mk = m[k], vk = v[k];
    const float old = params[k];
    const float nw = adam_f32(mk, vk, old, grads[k], lr, c.bc1[grp], c.bc2[grp]);
    m[k] = mk;
    v[k] = vk;
    params[k] = nw;
    if (grp == 1) {
      q[p - kQuatW] = nw;
      quat_moved = quat_moved || (nw != old);
    }
  };
  // geometry / opacity planes unrolled (constant group indices: no local memory)
#pragma unroll
  for (int p = 0; p < kShBase; ++p) {
    const int grp = p < kQuatW ? 0 : p < kScaleX ? 1 : p < kOpacity ? 2 : 3;
    step(p, grp, c.lr[grp]);
  }
  for (int p = kShBase; p < nplanes; ++p) step(p, 4, ((p - kShBase) % basis == 0) ? c.lr[4] : c.lr[5]);
  if (quat_moved) {  // pipelines.cpp:36-40
    const float nn = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) params[(int64_t)(kQuatW + k) * n_pad + i] = q[k] / nn;
  }
}

// ------------------------------------------------------------ joint loop
// joint_optimize (pipelines.cpp:96-216) as a device-resident step: `slots`
// training views per step (data parallel: `local` of them on this rank, the
// rest on the other ranks), the Adam gradient is the mean of the slots'
// render gradients plus the anisotropy / opacity-L1 regularisers evaluated
// once on the pre-step parameters (losses.cpp:217-257, pipelines.cpp:144-157),
// then the slots' pose steps in slot order (176-180). The step counter, the
// learning-rate schedules and Adam's bias corrections live on the device, so
// one CUDA graph replays every step. See DESIGN.md §7.

// Exchange slot (FP64, summed over ranks = gathered): d_pose, L1, SSIM,
// rgb loss, overflow flag, K seen, tile overflow.
constexpr int kXchgW = 12;
enum XchgField : int { kXPose = 0, kXL1 = 6, kXSsim = 7, kXRgb = 8, kXOvf = 9, kXK = 10, kXTile = 11 };

struct JointDev {
  int64_t t;          // steps completed
  int64_t adam_step;  // CloudAdam / AdamState step (== t unless steps were discarded)
  int32_t diverged;   // 1 + the step whose total loss was non-finite (0: none)
  int32_t aborted;    // steps discarded for capacity growth since the host last looked
  double abort_k_max;
  int32_t abort_tile;
  int32_t pad;
};

// schedule (trainer.cpp:30-38): kind 0 cosine, 1 exponential
__device__ double d_schedule(int kind, double start, double end, int64_t step, int64_t total) {
  if (total <= 0) return end;
  double s = (double)step / (double)total;
  s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
  if (kind == 0) return end + (start - end) * 0.5 * (1.0 + cos(M_PI * s));
  return start * pow(end / start, s);
}

// Slot b of this rank: camera of the scheduled view into the frame, target
// planes into the frame's target buffer (3 P floats).
__global__ void joint_slot_begin_kernel(const JointDev* __restrict__ js, const int32_t* __restrict__ seq, JointCtl ctl,
                                        int b, const CamDev* __restrict__ cams, CamDev* __restrict__ frame_cam,
                                        const float* const* __restrict__ targets, float* __restrict__ tbuf,
                                        int64_t n3p) {
  const int64_t t = js->t < ctl.iterations ? js->t : ctl.iterations - 1;
  const int v = seq[t * ctl.slots + ctl.slot0 + b];
  if (blockIdx.x == 0 && threadIdx.x == 0) *frame_cam = cams[v];
  const float4* src = reinterpret_cast<const float4*>(targets[v]);
  float4* dst = reinterpret_cast<float4*>(tbuf);
  const int64_t n4 = n3p >> 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  for (int64_t i = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n3p;
       i += (int64_t)gridDim.x * blockDim.x)
    tbuf[i] = targets[v][i];
}

// Slot b's results into the exchange buffer (zeroed at step start).
__global__ void joint_slot_end_kernel(JointCtl ctl, int b, const double* __restrict__ d_pose,
                                      const double* __restrict__ loss3, const uint32_t* __restrict__ counters,
                                      int64_t k_cap, double* __restrict__ xchg) {
  double* x = xchg + (int64_t)(ctl.slot0 + b) * kXchgW;
  for (int k = 0; k < 6; ++k) x[kXPose + k] = d_pose[k];
  x[kXL1] = loss3[0];
  x[kXSsim] = loss3[1];
  x[kXRgb] = loss3[2];
  const bool ovf = (int64_t)counters[1] > k_cap || counters[2] != 0u;
  x[kXOvf] = ovf ? 1.0 : 0.0;
  x[kXK] = (double)counters[1];
  x[kXTile] = counters[2] != 0u ? 1.0 : 0.0;
}

// grads[0] += grads[1..local-1] in slot order (local batches on one rank).
__global__ void joint_sum_kernel(float* __restrict__ g0, const float* __restrict__ rest, int64_t len, int nrest,
                                 int64_t stride) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  float acc = g0[i];
  for (int b = 0; b < nrest; ++b) acc += rest[(int64_t)b * stride + i];
  g0[i] = acc;
}

__device__ __forceinline__ bool joint_step_discarded(const double* xchg, int slots) {
  for (int s = 0; s < slots; ++s)
    if (xchg[(int64_t)s * kXchgW + kXOvf] != 0.0) return true;
  return false;
}

// A step's updates are skipped when it has run out of iterations, an earlier
// step diverged, some slot overflowed (the host re-runs the step), or a slot's
// loss is non-finite (pipelines.cpp:159-162 raises `diverged` before
// GradAccum::add, cloud_adam_step and the pose steps).
__device__ __forceinline__ bool joint_step_skipped(const JointDev* js, const JointCtl& ctl, const double* xchg) {
  if (js->t >= ctl.iterations || js->diverged || joint_step_discarded(xchg, ctl.slots)) return true;
  for (int s = 0; s < ctl.slots; ++s)
    if (!isfinite(xchg[(int64_t)s * kXchgW + kXRgb])) return true;
  return false;
}

// GradAccum::add (trainer.cpp:134-142), second half: the step's local slots'
// staged increments (grad_norm_kernel, -1 = not visible) added in slot order,
// only for a step that is kept — a discarded step adds nothing, its re-run
// adds its views once.
__global__ void grad_accum_commit_kernel(const double* __restrict__ stage, int local, int64_t stride, int64_t n,
                                         const JointDev* __restrict__ js, JointCtl ctl,
                                         const double* __restrict__ xchg, double* __restrict__ gsum,
                                         int32_t* __restrict__ gcnt) {
  __shared__ int s_skip;
  if (threadIdx.x == 0) s_skip = joint_step_skipped(js, ctl, xchg) ? 1 : 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s_skip || i >= n) return;
  double sum = gsum[i];
  int32_t cnt = gcnt[i];
  for (int b = 0; b < local; ++b) {
    const double v = stage[(int64_t)b * stride + i];
    if (v >= 0.0) {
      sum = __dadd_rn(sum, v);
      cnt += 1;
    }
  }
  gsum[i] = sum;
  gcnt[i] = cnt;
}

// cloud_adam_step (pipelines.cpp:18-41) on the averaged gradient plus the
// regularisers, one thread per Gaussian over the FP32 planes; block partial
// sums (aniso loss, opacity sum) for the step's total loss. Skipped when the
// step is discarded (some slot overflowed its entry capacity) or has already
// run out of iterations.
constexpr int kJointBlock = 256;
// The step's Adam coefficients, written by the geometry kernel's block 0 for
// the SH kernel (stored behind the block partials in the reduction buffer).
struct JointCoef {
  float lr_dc, lr_rest, bc1, bc2, inv_s;
  int skip;
};
__global__ void __launch_bounds__(kJointBlock) joint_adam_kernel(float* __restrict__ params,
                                                               const float* __restrict__ grads, float* __restrict__ m,
                                                               float* __restrict__ v, int64_t n, int64_t n_pad,
                                                               const JointDev* __restrict__ js, JointCtl ctl,
                                                               const double* __restrict__ xchg,
                                                               double* __restrict__ red_blocks,
                                                               JointCoef* __restrict__ coef) {
  __shared__ float s_lr[6], s_bc1, s_bc2;
  __shared__ int s_skip, s_opl1;
  __shared__ double s_red[kJointBlock / 32][2];
  if (threadIdx.x == 0) {
    const int64_t t = js->t;
    s_skip = joint_step_skipped(js, ctl, xchg) ? 1 : 0;
    s_opl1 = (t < ctl.opacity_l1_steps && ctl.opacity_l1_weight > 0.0) ? 1 : 0;
    const double st = (double)(js->adam_step + 1);
    s_bc1 = (float)(1.0 - pow(kB1, st));
    s_bc2 = (float)(1.0 - pow(kB2, st));
    s_lr[0] = (float)d_schedule(1, ctl.pos_lr_start, ctl.pos_lr_end, t, ctl.iterations);
    s_lr[1] = (float)ctl.rot_lr;
    s_lr[2] = (float)ctl.scale_lr;
    s_lr[3] = (float)ctl.opacity_lr;
    s_lr[4] = (float)ctl.sh_dc_lr;
    s_lr[5] = (float)ctl.sh_rest_lr;
    if (blockIdx.x == 0) *coef = JointCoef{s_lr[4], s_lr[5], s_bc1, s_bc2, (float)ctl.inv_slots, s_skip};
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double aniso = 0.0, opsum = 0.0;
  if (i < n) {
    const double inv_n = 1.0 / (double)n;
    // anisotropy_loss (losses.cpp:217-244) on the pre-step log-scales
    double sc[3];
    for (int k = 0; k < 3; ++k) sc[k] = exp((double)params[(int64_t)(kScaleX + k) * n_pad + i]);
    // first arg-max / arg-min, tracked in registers (no local memory)
    int amax = 0, amin = 0;
    double smax = sc[0], smin = sc[0];
#pragma unroll
    for (int k = 1; k < 3; ++k) {
      if (sc[k] > smax) { amax = k; smax = sc[k]; }
      if (sc[k] < smin) { amin = k; smin = sc[k]; }
    }
    const double r = smax / smin;
    double dls[3] = {0.0, 0.0, 0.0};
    if (r > ctl.aniso_ratio) {
      aniso = (r - ctl.aniso_ratio) * inv_n;
      const double dmax = inv_n / smin * smax, dmin = -inv_n * smax / (smin * smin) * smin;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (amax == k) dls[k] += dmax;
        if (amin == k) dls[k] += dmin;
      }
    }
    // opacity_l1 (losses.cpp:246-257) through the sigmoid (pipelines.cpp:148-157)
    const double o = 1.0 / (1.0 + exp(-(double)params[(int64_t)kOpacity * n_pad + i]));
    opsum = o * inv_n;
    const double dop = s_opl1 ? ctl.opacity_l1_weight * inv_n * o * (1.0 - o) : 0.0;
    if (!s_skip) {
      const float inv_s = (float)ctl.inv_slots;
      bool quat_moved = false;
      float q[4];
      auto step = [&](int p, float lr) {
        const int64_t k = (int64_t)p * n_pad + i;
        float gi = grads[k] * inv_s;
        if (p >= kScaleX && p < kOpacity) gi = (float)((double)gi + dls[p - kScaleX]);
        if (p == kOpacity) gi = (float)((double)gi + dop);
        float mk = m[k], vk = v[k];
        const float old = params[k];
        const float nw = adam_f32(mk, vk, old, gi, lr, s_bc1, s_bc2);
        m[k] = mk;
        v[k] = vk;
        params[k] = nw;
        if (p >= kQuatW && p < kScaleX) {
          q[p - kQuatW] = nw;
          quat_moved = quat_moved || (nw != old);
        }
      };
      // geometry / opacity planes (fixed count, unrolled); the SH planes are
      // joint_adam_sh_kernel's
#pragma unroll
      for (int p = 0; p < kShBase; ++p)
        step(p, p < kQuatW ? s_lr[0] : p < kScaleX ? s_lr[1] : p < kOpacity ? s_lr[2] : s_lr[3]);
      if (quat_moved) {  // pipelines.cpp:36-40
        const float nn = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        for (int k = 0; k < 4; ++k) params[(int64_t)(kQuatW + k) * n_pad + i] = q[k] / nn;
      }
    }
  }
  // fixed-order block reduction of (aniso, opacity sum)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    aniso += __shfl_xor_sync(0xffffffffu, aniso, o);
    opsum += __shfl_xor_sync(0xffffffffu, opsum, o);
  }
  if (lane == 0) {
    s_red[warp][0] = aniso;
    s_red[warp][1] = opsum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kJointBlock / 32; ++w) {
      a += s_red[w][0];
      b += s_red[w][1];
    }
    red_blocks[2 * blockIdx.x] = a;
    red_blocks[2 * blockIdx.x + 1] = b;
  }
}

// The SH planes' Adam update (same arithmetic as the geometry kernel's
// `step`): plain streaming over 3 * basis planes, blockIdx.y picks
// kShPlanesPerThread of them, so that every thread has 4 × that many
// independent loads in flight. Plane c * basis + b is the DC band at b == 0
// (pipelines.cpp:33).
#ifndef GSB_SH_PPT
#define GSB_SH_PPT 1
#endif
#ifndef GSB_SH_VEC
#define GSB_SH_VEC 1
#endif
constexpr int kShPlanesPerThread = GSB_SH_PPT;
constexpr int kShVec = GSB_SH_VEC ? 4 : 1;  // consecutive Gaussians per thread (float4 accesses)
__global__ void __launch_bounds__(kJointBlock) joint_adam_sh_kernel(float* __restrict__ params,
                                                                  const float* __restrict__ grads,
                                                                  float* __restrict__ m, float* __restrict__ v,
                                                                  int64_t n, int64_t n_pad, int basis,
                                                                  const JointCoef* __restrict__ coef) {
  const JointCoef c = *coef;
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kShVec;
  if (c.skip || i0 >= n) return;
  const int q0 = blockIdx.y * kShPlanesPerThread, nsh = 3 * basis;
  if (kShVec == 4 && i0 + 4 <= n) {  // n_pad % 32 == 0: every plane row is 16-B aligned
    float4 g[kShPlanesPerThread], mo[kShPlanesPerThread], vo[kShPlanesPerThread], po[kShPlanesPerThread];
#pragma unroll
    for (int u = 0; u < kShPlanesPerThread; ++u) {
      if (q0 + u < nsh) {
        const int64_t k = (int64_t)(kShBase + q0 + u) * n_pad + i0;
        g[u] = __ldcs(reinterpret_cast<const float4*>(grads + k));
        mo[u] = __ldcs(reinterpret_cast<const float4*>(m + k));
        vo[u] = __ldcs(reinterpret_cast<const float4*>(v + k));
        po[u] = *reinterpret_cast<const float4*>(params + k);
      }
    }
#pragma unroll
    for (int u = 0; u < kShPlanesPerThread; ++u) {
      if (q0 + u < nsh) {
        const int64_t k = (int64_t)(kShBase + q0 + u) * n_pad + i0;
        const float lr = ((q0 + u) % basis == 0) ? c.lr_dc : c.lr_rest;
        float4 np;
        np.x = adam_f32(mo[u].x, vo[u].x, po[u].x, g[u].x * c.inv_s, lr, c.bc1, c.bc2);
        np.y = adam_f32(mo[u].y, vo[u].y, po[u].y, g[u].y * c.inv_s, lr, c.bc1, c.bc2);
        np.z = adam_f32(mo[u].z, vo[u].z, po[u].z, g[u].z * c.inv_s, lr, c.bc1, c.bc2);
        np.w = adam_f32(mo[u].w, vo[u].w, po[u].w, g[u].w * c.inv_s, lr, c.bc1, c.bc2);
        *reinterpret_cast<float4*>(params + k) = np;
        __stcs(reinterpret_cast<float4*>(m + k), mo[u]);
        __stcs(reinterpret_cast<float4*>(v + k), vo[u]);
      }
    }
    return;
  }
  for (int64_t i = i0; i < i0 + kShVec && i < n; ++i) {
    float g[kShPlanesPerThread], mo[kShPlanesPerThread], vo[kShPlanesPerThread], po[kShPlanesPerThread];
#pragma unroll
    for (int u = 0; u < kShPlanesPerThread; ++u) {
      if (q0 + u < nsh) {
        const int64_t k = (int64_t)(kShBase + q0 + u) * n_pad + i;
        g[u] = grads[k];
        mo[u] = m[k];
        vo[u] = v[k];
        po[u] = params[k];
      }
    }
#pragma unroll
    for (int u = 0; u < kShPlanesPerThread; ++u) {
      if (q0 + u < nsh) {
        const int64_t k = (int64_t)(kShBase + q0 + u) * n_pad + i;
        const float lr = ((q0 + u) % basis == 0) ? c.lr_dc : c.lr_rest;
        params[k] = adam_f32(mo[u], vo[u], po[u], g[u] * c.inv_s, lr, c.bc1, c.bc2);
        m[k] = mo[u];
        v[k] = vo[u];
      }
    }
  }
}

// Step tail: total loss trace and divergence check (pipelines.cpp:159-162),
// the slots' pose steps in slot order with each view's PoseAdam and the
// cosine camera schedule (176-180), step counters. One block.
__global__ void joint_finalize_kernel(JointDev* __restrict__ js, const int32_t* __restrict__ seq, JointCtl ctl,
                                      const double* __restrict__ xchg, const double* __restrict__ red_blocks,
                                      int64_t nblocks, PoseState* __restrict__ poses, CamDev* __restrict__ cams,
                                      double* __restrict__ trace_total, double* __restrict__ trace_l1) {
  __shared__ double s_a[256], s_b[256];
  double a = 0.0, b = 0.0;
  for (int64_t k = threadIdx.x; k < nblocks; k += 256) {
    a += red_blocks[2 * k];
    b += red_blocks[2 * k + 1];
  }
  s_a[threadIdx.x] = a;
  s_b[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x != 0) return;
  JointDev j = *js;
  if (j.t >= ctl.iterations || j.diverged) return;
  if (joint_step_discarded(xchg, ctl.slots)) {  // the host grows the capacity and replays this step
    j.aborted += 1;
    for (int s = 0; s < ctl.slots; ++s) {
      j.abort_k_max = fmax(j.abort_k_max, xchg[(int64_t)s * kXchgW + kXK]);
      if (xchg[(int64_t)s * kXchgW + kXTile] != 0.0) j.abort_tile = 1;
    }
    *js = j;
    return;
  }
  double aniso = 0.0, opsum = 0.0;
  for (int k = 0; k < 256; ++k) {
    aniso += s_a[k];
    opsum += s_b[k];
  }
  double rgb = 0.0, l1 = 0.0;
  for (int s = 0; s < ctl.slots; ++s) {
    rgb += xchg[(int64_t)s * kXchgW + kXRgb];
    l1 += xchg[(int64_t)s * kXchgW + kXL1];
  }
  const bool opl1 = j.t < ctl.opacity_l1_steps && ctl.opacity_l1_weight > 0.0;
  const double total = rgb * ctl.inv_slots + aniso + ctl.opacity_l1_weight * (opl1 ? opsum : 0.0);
  if (trace_total) trace_total[j.t] = total;
  if (trace_l1) trace_l1[j.t] = l1 * ctl.inv_slots;
  if (!isfinite(total)) {  // pipelines.cpp:159-162: throw before the cloud and pose updates
    j.diverged = (int32_t)(j.t + 1);
    *js = j;
    return;
  }
  if (ctl.optimize_poses) {
    const double lr = d_schedule(0, ctl.cam_lr_start, ctl.cam_lr_end, j.t, ctl.iterations);
    for (int s = 0; s < ctl.slots; ++s) {
      const int v = seq[j.t * ctl.slots + s];
      PoseState p = poses[v];
      d_pose_step(p, xchg + (int64_t)s * kXchgW + kXPose, lr);
      poses[v] = p;
      d_write_cam(p, &cams[v]);
    }
  }
  j.t += 1;
  j.adam_step += 1;
  *js = j;
}

int launch_joint_slot_begin(cudaStream_t st, const void* js, const int32_t* seq, const JointCtl& ctl, int b,
                            const CamDev* cams, CamDev* frame_cam, const float* const* targets, float* tbuf,
                            int64_t n3p) {
  const int64_t blocks = std::min<int64_t>((n3p / 4 + 255) / 256 + 1, 4 * 148);
  joint_slot_begin_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const JointDev*>(js), seq, ctl, b, cams,
                                                            frame_cam, targets, tbuf, n3p);
  GSB_CHECK_LAUNCH("joint_slot_begin_kernel");
  return GSB_OK;
}
int launch_joint_slot_end(cudaStream_t st, const JointCtl& ctl, int b, const double* d_pose, const double* loss3,
                          const uint32_t* counters, int64_t k_cap, double* xchg) {
  joint_slot_end_kernel<<<1, 1, 0, st>>>(ctl, b, d_pose, loss3, counters, k_cap, xchg);
  GSB_CHECK_LAUNCH("joint_slot_end_kernel");
  return GSB_OK;
}
int launch_joint_sum(cudaStream_t st, float* g0, const float* rest, int64_t len, int nrest, int64_t stride) {
  if (nrest > 0 && len > 0)
    joint_sum_kernel<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(g0, rest, len, nrest, stride);
  GSB_CHECK_LAUNCH("joint_sum_kernel");
  return GSB_OK;
}
int launch_grad_accum_commit(cudaStream_t st, const double* stage, int local, int64_t stride, int64_t n,
                             const void* js, const JointCtl& ctl, const double* xchg, double* gsum, int32_t* gcnt) {
  if (n > 0)
    grad_accum_commit_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        stage, local, stride, n, static_cast<const JointDev*>(js), ctl, xchg, gsum, gcnt);
  GSB_CHECK_LAUNCH("grad_accum_commit_kernel");
  return GSB_OK;
}
int64_t joint_adam_blocks(int64_t n) { return (n + kJointBlock - 1) / kJointBlock; }
int64_t joint_red_doubles(int64_t n) { return 2 * joint_adam_blocks(n) + 4; }

int launch_joint_adam(cudaStream_t st, float* params, const float* grads, float* m, float* v, int64_t n,
                      int64_t n_pad, const void* js, const JointCtl& ctl, const double* xchg, double* red_blocks) {
  const int64_t nb = joint_adam_blocks(n);
  if (nb <= 0) return GSB_OK;
  static_assert(sizeof(JointCoef) <= 4 * sizeof(double), "joint_red_doubles");
  JointCoef* coef = reinterpret_cast<JointCoef*>(red_blocks + 2 * nb);
  joint_adam_kernel<<<(unsigned)nb, kJointBlock, 0, st>>>(params, grads, m, v, n, n_pad,
                                                          static_cast<const JointDev*>(js), ctl, xchg, red_blocks, coef);
  GSB_CHECK_LAUNCH("joint_adam_kernel");
  const dim3 grid((unsigned)((n + (int64_t)kJointBlock * kShVec - 1) / ((int64_t)kJointBlock * kShVec)),
                  (unsigned)((3 * ctl.basis + kShPlanesPerThread - 1) / kShPlanesPerThread));
  joint_adam_sh_kernel<<<grid, kJointBlock, 0, st>>>(params, grads, m, v, n, n_pad, ctl.basis, coef);
  GSB_CHECK_LAUNCH("joint_adam_sh_kernel");
  return GSB_OK;
}
int launch_joint_finalize(cudaStream_t st, void* js, const int32_t* seq, const JointCtl& ctl, const double* xchg,
                          const double* red_blocks, int64_t nblocks, void* poses, CamDev* cams, double* trace_total,
                          double* trace_l1) {
  joint_finalize_kernel<<<1, 256, 0, st>>>(static_cast<JointDev*>(js), seq, ctl, xchg, red_blocks, nblocks,
                                           static_cast<PoseState*>(poses), cams, trace_total, trace_l1);
  GSB_CHECK_LAUNCH("joint_finalize_kernel");
  return GSB_OK;
}
size_t joint_state_bytes() { return sizeof(JointDev); }
size_t joint_xchg_doubles() { return kXchgW; }
void joint_state_read(const void* host, int64_t* t, int32_t* diverged, int32_t* aborted, double* k_max,
                      int32_t* tile) {
  const JointDev* j = static_cast<const JointDev*>(host);
  if (t) *t = j->t;
  if (diverged) *diverged = j->diverged;
  if (aborted) *aborted = j->aborted;
  if (k_max) *k_max = j->abort_k_max;
  if (tile) *tile = j->abort_tile;
}
void joint_state_clear_abort(void* host) {
  JointDev* j = static_cast<JointDev*>(host);
  j->aborted = 0;
  j->abort_k_max = 0.0;
  j->abort_tile = 0;
}

// ------------------------------------------------------------- host glue
int launch_pose_iter(cudaStream_t st, void* state, const double* pose_blocks, int64_t nb, double* dpose_out,
                     const double* loss3, double lr_start, double lr_end, double eps, int budget, CamDev* cam,
                     double* trace_pose, double* trace_loss, const uint32_t* k_dev, int64_t k_cap) {
  PoseCtl ctl{lr_start, lr_end, eps, budget, 0};
  pose_iter_kernel<<<1, 256, 0, st>>>(static_cast<PoseState*>(state), pose_blocks, nb, dpose_out, loss3, ctl, cam,
                                      trace_pose, trace_loss, k_dev, k_cap);
  GSB_CHECK_LAUNCH("pose_iter_kernel");
  return GSB_OK;
}
size_t pose_state_bytes() { return sizeof(PoseState); }
int pose_state_init(void* host_state, const double pose[12]) {
  PoseState* s = static_cast<PoseState*>(host_state);
  *s = PoseState{};
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) s->R[r * 3 + c] = pose[r * 4 + c];
    s->t[r] = pose[r * 4 + 3];
  }
  for (int k = 0; k < 9; ++k) s->best_R[k] = s->R[k];
  for (int k = 0; k < 3; ++k) s->best_t[k] = s->t[k];
  s->best_loss = INFINITY;
  return GSB_OK;
}
void pose_state_read(const void* host_state, double best_pose[12], double cur_pose[12], double* final_loss,
                     int32_t* steps_used, int32_t* converged, int32_t* stop, double applied[6], double m[6],
                     double v[6], int64_t* step) {
  const PoseState* s = static_cast<const PoseState*>(host_state);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) {
      if (best_pose) best_pose[r * 4 + c] = s->best_R[r * 3 + c];
      if (cur_pose) cur_pose[r * 4 + c] = s->R[r * 3 + c];
    }
    if (best_pose) best_pose[r * 4 + 3] = s->best_t[r];
    if (cur_pose) cur_pose[r * 4 + 3] = s->t[r];
  }
  if (final_loss) *final_loss = s->final_loss;
  if (steps_used) *steps_used = s->steps_used;
  if (converged) *converged = s->converged;
  if (stop) *stop = s->stop;
  for (int k = 0; k < 6; ++k) {
    if (applied) applied[k] = s->applied[k];
    if (m) m[k] = s->m[k];
    if (v) v[k] = s->v[k];
  }
  if (step) *step = s->step;
}
int32_t pose_state_aborted(const void* host_state) { return static_cast<const PoseState*>(host_state)->aborted; }
int32_t pose_state_take_aborted(void* host_state, uint32_t* k_max, uint32_t* tile_ovf) {
  PoseState* s = static_cast<PoseState*>(host_state);
  const int32_t a = s->aborted;
  *k_max = s->abort_k_max;
  *tile_ovf = s->abort_tile_ovf;
  s->aborted = 0;
  s->abort_k_max = 0;
  s->abort_tile_ovf = 0;
  return a;
}
void pose_state_set_adam(void* host_state, const double m[6], const double v[6], int64_t step) {
  PoseState* s = static_cast<PoseState*>(host_state);
  for (int k = 0; k < 6; ++k) {
    s->m[k] = m[k];
    s->v[k] = v[k];
  }
  s->step = step;
}
int launch_pose_step(cudaStream_t st, void* states, const double* dpose, double lr, int nb) {
  pose_step_kernel<<<(nb + 63) / 64, 64, 0, st>>>(static_cast<PoseState*>(states), dpose, lr, nb);
  GSB_CHECK_LAUNCH("pose_step_kernel");
  return GSB_OK;
}
int launch_adam_f64(cudaStream_t st, double* p, const double* g, double* m, double* v, int64_t n, double lr,
                    const double* lrs, int64_t step) {
  const double bc1 = 1.0 - pow(kB1, (double)step), bc2 = 1.0 - pow(kB2, (double)step);
  if (n > 0) adam_f64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, g, m, v, n, lr, lrs, bc1, bc2);
  GSB_CHECK_LAUNCH("adam_f64_kernel");
  return GSB_OK;
}
int launch_cloud_adam(cudaStream_t st, float* params, const float* grads, float* m, float* v, int64_t n,
                      int64_t n_pad, int sh_degree, const double lrs[6], const int64_t steps[5]) {
  AdamCoef c;
  for (int k = 0; k < 6; ++k) c.lr[k] = (float)lrs[k];
  for (int k = 0; k < 5; ++k) {
    c.bc1[k] = (float)(1.0 - pow(kB1, (double)steps[k]));
    c.bc2[k] = (float)(1.0 - pow(kB2, (double)steps[k]));
  }
  const int basis = (sh_degree + 1) * (sh_degree + 1);
  if (n > 0)
    cloud_adam_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(params, grads, m, v, n, n_pad,
                                                                   num_planes(sh_degree), basis, c);
  GSB_CHECK_LAUNCH("cloud_adam_kernel");
  return GSB_OK;
}

}  // namespace gsb
