// k_densify.cu — densify_and_prune (trainer.cpp:144-239) and GradAccum::add
// (trainer.cpp:134-142) on the plane-major device cloud.
//
// The population is rebuilt with prefix sums instead of push_back, in the
// reference's order: kept originals (split parents are consumed), then in
// index order each clone / the two children of each split. Decisions are
// taken in FP64 from the FP32-stored parameters (exactly the doubles the
// reference would hold for the same cloud); split children are
// mean + R(q) (scale .* n) with n drawn by the host from the run's Rng in the
// reference's draw order, and log-scale - ln 1.6. Pruning keeps opacity >
// max(prune_opacity, (n_target+1)-th largest opacity); the rank is taken on
// the FP32 logits (sigmoid is monotone), the comparison on the FP64 sigmoid.
// CloudAdam::remap (trainer.cpp:101-132) gathers the moments of survivors and
// zeroes fresh Gaussians. All explicit-rounding FP64 (no contraction), so the
// new parameters are the reference's doubles rounded to FP32.
#include "gsb_internal.cuh"

namespace gsb {

constexpr int kDenBlock = 256;

__device__ __forceinline__ double m_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double s_(double a, double b) { return __dsub_rn(a, b); }

// GradAccum::add for one rendered view, first half: the view's per-Gaussian
// increment |d_mu2d| * 0.5 max(W, H) for visible splats (tile count > 0), -1
// for the others, into a staging row. The joint step commits the rows in slot
// order only once it knows the step is kept (grad_accum_commit_kernel,
// k_optim.cu), so a step discarded for entry-capacity growth and re-run adds
// its views exactly once.
__global__ void grad_norm_kernel(const float* __restrict__ grads, int nplanes, int64_t n_pad, int64_t n,
                                 const uint32_t* __restrict__ cnt_g, double scale, double* __restrict__ stage) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if ((cnt_g[i] & kCntMask) == 0u) {
    stage[i] = -1.0;
    return;
  }
  const double x = grads[(int64_t)nplanes * n_pad + i], y = grads[(int64_t)(nplanes + 1) * n_pad + i];
  stage[i] = m_(sqrt(a_(m_(x, x), m_(y, y))), scale);
}

// Per-block min / max of the means (exact in any order).
__global__ void __launch_bounds__(kDenBlock) densify_bbox_kernel(const float* __restrict__ params, int64_t n,
                                                                 int64_t n_pad, float* __restrict__ out) {
  __shared__ float s[6][kDenBlock];
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = (int64_t)blockIdx.x * kDenBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDenBlock)
    for (int k = 0; k < 3; ++k) {
      const float v = params[(int64_t)(kMeanX + k) * n_pad + i];
      lo[k] = fminf(lo[k], v);
      hi[k] = fmaxf(hi[k], v);
    }
  for (int k = 0; k < 3; ++k) {
    s[k][threadIdx.x] = lo[k];
    s[3 + k][threadIdx.x] = hi[k];
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    float r = s[threadIdx.x][0];
    for (int t = 1; t < kDenBlock; ++t) r = threadIdx.x < 3 ? fminf(r, s[threadIdx.x][t]) : fmaxf(r, s[threadIdx.x][t]);
    out[blockIdx.x * 6 + threadIdx.x] = r;
  }
}

// Actions (trainer.cpp:162-169): keep flag, extra Gaussians (clone 1, split 2)
// and split flag per Gaussian.
__global__ void densify_action_kernel(const float* __restrict__ params, int64_t n, int64_t n_pad,
                                      const double* __restrict__ gsum, const int32_t* __restrict__ gcnt,
                                      double grad_threshold, double size_threshold, uint32_t* __restrict__ keep,
                                      uint32_t* __restrict__ extra, uint32_t* __restrict__ split) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int act = 0;  // keep
  if (gcnt[i] > 0) {
    const double avg = gsum[i] / (double)gcnt[i];
    if (!(avg < grad_threshold)) {
      double mx = exp((double)params[(int64_t)kScaleX * n_pad + i]);
      mx = fmax(mx, exp((double)params[(int64_t)kScaleY * n_pad + i]));
      mx = fmax(mx, exp((double)params[(int64_t)kScaleZ * n_pad + i]));
      act = mx <= size_threshold ? 1 : 2;
    }
  }
  keep[i] = act != 2 ? 1u : 0u;
  extra[i] = act == 1 ? 1u : (act == 2 ? 2u : 0u);
  split[i] = act == 2 ? 1u : 0u;
}

// Post-densify population (before pruning), plane-major with stride n_pad_o.
__global__ void densify_build_kernel(const float* __restrict__ params, int64_t n, int64_t n_pad, int nplanes,
                                     const uint32_t* __restrict__ keep, const uint32_t* __restrict__ keep_pos,
                                     const uint32_t* __restrict__ extra, const uint32_t* __restrict__ extra_pos,
                                     const uint32_t* __restrict__ split_rank, const double* __restrict__ normals,
                                     uint32_t n_keep, float* __restrict__ out, int64_t n_pad_o,
                                     int32_t* __restrict__ src_o) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  auto copy_to = [&](int64_t j) {
    for (int p = 0; p < nplanes; ++p) out[(int64_t)p * n_pad_o + j] = params[(int64_t)p * n_pad + i];
  };
  if (keep[i]) {
    const int64_t j = keep_pos[i];
    copy_to(j);
    src_o[j] = (int32_t)i;
  }
  const uint32_t e = extra[i];
  if (e == 1u) {  // clone: same parameters, fresh moments
    const int64_t j = (int64_t)n_keep + extra_pos[i];
    copy_to(j);
    src_o[j] = -1;
  } else if (e == 2u) {  // split: two children from the parent's distribution
    const double qw = params[(int64_t)kQuatW * n_pad + i], qx = params[(int64_t)kQuatX * n_pad + i],
                 qy = params[(int64_t)kQuatY * n_pad + i], qz = params[(int64_t)kQuatZ * n_pad + i];
    const double qn = sqrt(a_(a_(a_(m_(qw, qw), m_(qx, qx)), m_(qy, qy)), m_(qz, qz)));
    const double w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
    double R[9];  // quat_to_rotation (scene.cpp:46-54)
    R[0] = s_(1.0, m_(2.0, a_(m_(y, y), m_(z, z))));
    R[1] = m_(2.0, s_(m_(x, y), m_(w, z)));
    R[2] = m_(2.0, a_(m_(x, z), m_(w, y)));
    R[3] = m_(2.0, a_(m_(x, y), m_(w, z)));
    R[4] = s_(1.0, m_(2.0, a_(m_(x, x), m_(z, z))));
    R[5] = m_(2.0, s_(m_(y, z), m_(w, x)));
    R[6] = m_(2.0, s_(m_(x, z), m_(w, y)));
    R[7] = m_(2.0, a_(m_(y, z), m_(w, x)));
    R[8] = s_(1.0, m_(2.0, a_(m_(x, x), m_(y, y))));
    double ls[3], sc[3], mu[3];
    for (int k = 0; k < 3; ++k) {
      ls[k] = params[(int64_t)(kScaleX + k) * n_pad + i];
      sc[k] = exp(ls[k]);
      mu[k] = params[(int64_t)(kMeanX + k) * n_pad + i];
    }
    const double ln16 = log(1.6);
    const int64_t r = split_rank[i];
    for (int c = 0; c < 2; ++c) {
      const int64_t j = (int64_t)n_keep + extra_pos[i] + c;
      copy_to(j);
      const double* nv = normals + 6 * r + 3 * c;
      const double v[3] = {m_(sc[0], nv[0]), m_(sc[1], nv[1]), m_(sc[2], nv[2])};
      for (int k = 0; k < 3; ++k) {
        const double smp = a_(a_(m_(R[k * 3], v[0]), m_(R[k * 3 + 1], v[1])), m_(R[k * 3 + 2], v[2]));
        out[(int64_t)(kMeanX + k) * n_pad_o + j] = (float)a_(mu[k], smp);
        out[(int64_t)(kScaleX + k) * n_pad_o + j] = (float)s_(ls[k], ln16);
      }
      src_o[j] = -1;
    }
  }
}

// Order-preserving uint32 key of an FP32 logit (ascending sort).
__global__ void densify_logit_keys_kernel(const float* __restrict__ params, int64_t n, int64_t n_pad,
                                          uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = __float_as_uint(params[(int64_t)kOpacity * n_pad + i]);
  keys[i] = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  vals[i] = (uint32_t)i;
}

__global__ void densify_prune_flag_kernel(const float* __restrict__ params, int64_t n, int64_t n_pad,
                                          double threshold, uint32_t* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double op = 1.0 / (1.0 + exp(-(double)params[(int64_t)kOpacity * n_pad + i]));  // core.hpp:112
  flag[i] = op > threshold ? 1u : 0u;
}

__global__ void densify_gather_kernel(const float* __restrict__ in, int64_t n, int64_t n_pad_i, int nplanes,
                                      const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                      const int32_t* __restrict__ src_i, float* __restrict__ out, int64_t n_pad_o,
                                      int32_t* __restrict__ src_o) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const int64_t j = pos[i];
  for (int p = 0; p < nplanes; ++p) out[(int64_t)p * n_pad_o + j] = in[(int64_t)p * n_pad_i + i];
  src_o[j] = src_i[i];
}

// CloudAdam::remap: moments of survivors, zeros for fresh Gaussians.
__global__ void densify_adam_remap_kernel(const float* __restrict__ m, const float* __restrict__ v, int64_t n_pad_i,
                                          int nplanes, const int32_t* __restrict__ src, int64_t n_o, int64_t n_pad_o,
                                          float* __restrict__ m_o, float* __restrict__ v_o) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_o) return;
  const int32_t s = src[j];
  for (int p = 0; p < nplanes; ++p) {
    m_o[(int64_t)p * n_pad_o + j] = s >= 0 ? m[(int64_t)p * n_pad_i + s] : 0.f;
    v_o[(int64_t)p * n_pad_o + j] = s >= 0 ? v[(int64_t)p * n_pad_i + s] : 0.f;
  }
}

// mean_knn_distance (scene.cpp:115-180) for k = 3, brute force over shared
// memory tiles (the exact k nearest distances, like the reference's grid
// search), FP64 with explicit rounding: sqrt(dx^2 + dy^2 + dz^2).
constexpr int kKnnTile = 256;
__global__ void __launch_bounds__(kKnnTile) knn3_mean_kernel(const double* __restrict__ pts, int64_t n,
                                                             double* __restrict__ out) {
  __shared__ double s[3][kKnnTile];
  const int64_t i = (int64_t)blockIdx.x * kKnnTile + threadIdx.x;
  double px = 0, py = 0, pz = 0;
  if (i < n) {
    px = pts[3 * i];
    py = pts[3 * i + 1];
    pz = pts[3 * i + 2];
  }
  double b0 = INFINITY, b1 = INFINITY, b2 = INFINITY;
  for (int64_t t0 = 0; t0 < n; t0 += kKnnTile) {
    const int64_t j = t0 + threadIdx.x;
    __syncthreads();
    for (int k = 0; k < 3; ++k) s[k][threadIdx.x] = j < n ? pts[3 * j + k] : 0.0;
    __syncthreads();
    const int m = (int)min((int64_t)kKnnTile, n - t0);
    for (int q = 0; q < m; ++q) {
      if (t0 + q == i) continue;
      const double dx = s_(s[0][q], px), dy = s_(s[1][q], py), dz = s_(s[2][q], pz);
      const double d = sqrt(a_(a_(m_(dx, dx), m_(dy, dy)), m_(dz, dz)));
      if (d < b2) {  // insertion into the sorted best three
        if (d < b1) {
          b2 = b1;
          if (d < b0) {
            b1 = b0;
            b0 = d;
          } else {
            b1 = d;
          }
        } else {
          b2 = d;
        }
      }
    }
  }
  if (i < n) out[i] = a_(a_(b0, b1), b2) / 3.0;
}

static unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>((n + kDenBlock - 1) / kDenBlock, 1); }

int launch_grad_norm(cudaStream_t st, const float* grads, int nplanes, int64_t n_pad, int64_t n,
                     const uint32_t* cnt_g, double scale, double* stage) {
  if (n > 0) grad_norm_kernel<<<grid_of(n), kDenBlock, 0, st>>>(grads, nplanes, n_pad, n, cnt_g, scale, stage);
  GSB_CHECK_LAUNCH("grad_norm_kernel");
  return GSB_OK;
}
int launch_knn3_mean(cudaStream_t st, const double* pts, int64_t n, double* out) {
  if (n > 0) knn3_mean_kernel<<<(unsigned)((n + kKnnTile - 1) / kKnnTile), kKnnTile, 0, st>>>(pts, n, out);
  GSB_CHECK_LAUNCH("knn3_mean_kernel");
  return GSB_OK;
}
int densify_bbox_blocks() { return 148; }
int launch_densify_bbox(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, float* out) {
  densify_bbox_kernel<<<densify_bbox_blocks(), kDenBlock, 0, st>>>(params, n, n_pad, out);
  GSB_CHECK_LAUNCH("densify_bbox_kernel");
  return GSB_OK;
}
int launch_densify_action(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, const double* gsum,
                          const int32_t* gcnt, double grad_threshold, double size_threshold, uint32_t* keep,
                          uint32_t* extra, uint32_t* split) {
  if (n > 0)
    densify_action_kernel<<<grid_of(n), kDenBlock, 0, st>>>(params, n, n_pad, gsum, gcnt, grad_threshold,
                                                             size_threshold, keep, extra, split);
  GSB_CHECK_LAUNCH("densify_action_kernel");
  return GSB_OK;
}
int launch_densify_build(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, int nplanes,
                         const uint32_t* keep, const uint32_t* keep_pos, const uint32_t* extra,
                         const uint32_t* extra_pos, const uint32_t* split_rank, const double* normals,
                         uint32_t n_keep, float* out, int64_t n_pad_o, int32_t* src_o) {
  if (n > 0)
    densify_build_kernel<<<grid_of(n), kDenBlock, 0, st>>>(params, n, n_pad, nplanes, keep, keep_pos, extra,
                                                            extra_pos, split_rank, normals, n_keep, out, n_pad_o,
                                                            src_o);
  GSB_CHECK_LAUNCH("densify_build_kernel");
  return GSB_OK;
}
int launch_densify_logit_keys(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, uint32_t* keys,
                              uint32_t* vals) {
  if (n > 0) densify_logit_keys_kernel<<<grid_of(n), kDenBlock, 0, st>>>(params, n, n_pad, keys, vals);
  GSB_CHECK_LAUNCH("densify_logit_keys_kernel");
  return GSB_OK;
}
int launch_densify_prune_flag(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, double threshold,
                              uint32_t* flag) {
  if (n > 0) densify_prune_flag_kernel<<<grid_of(n), kDenBlock, 0, st>>>(params, n, n_pad, threshold, flag);
  GSB_CHECK_LAUNCH("densify_prune_flag_kernel");
  return GSB_OK;
}
int launch_densify_gather(cudaStream_t st, const float* in, int64_t n, int64_t n_pad_i, int nplanes,
                          const uint32_t* flag, const uint32_t* pos, const int32_t* src_i, float* out,
                          int64_t n_pad_o, int32_t* src_o) {
  if (n > 0)
    densify_gather_kernel<<<grid_of(n), kDenBlock, 0, st>>>(in, n, n_pad_i, nplanes, flag, pos, src_i, out, n_pad_o,
                                                             src_o);
  GSB_CHECK_LAUNCH("densify_gather_kernel");
  return GSB_OK;
}
int launch_densify_adam_remap(cudaStream_t st, const float* m, const float* v, int64_t n_pad_i, int nplanes,
                              const int32_t* src, int64_t n_o, int64_t n_pad_o, float* m_o, float* v_o) {
  if (n_o > 0)
    densify_adam_remap_kernel<<<grid_of(n_o), kDenBlock, 0, st>>>(m, v, n_pad_i, nplanes, src, n_o, n_pad_o, m_o,
                                                                   v_o);
  GSB_CHECK_LAUNCH("densify_adam_remap_kernel");
  return GSB_OK;
}

}  // namespace gsb
