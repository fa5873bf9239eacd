// k_preprocess.cu — K1: per-Gaussian cull / project / EWA conic / SH colour /
// tile rect. One thread per Gaussian over plane-major FP32 parameters (every
// plane load is a fully coalesced 128 B warp transaction).
//
// Reference: rasterizer.cpp:95-125 (prepare's parallel stage) with
// project (185-190), covariance2d (192-199), projection_jacobian (31-39),
// max_eigenvalue_2x2 (24-28), invert_spd2 (17-22), covariance3d
// (scene.cpp:90-94), quat_to_rotation (scene.cpp:46-54), sh_eval
// (sh.cpp:66-84, incl. the (d_active+1)^2 channel stride), sigmoid
// (core.hpp:112) and the tile span (rasterizer.cpp:138-146).
//
// Geometry is evaluated in FP64 with explicitly rounded (non-fused)
// multiply/add in the reference's expression order, so mu2d and depth are
// bit-identical to an FP64 evaluation of the reference expressions on the
// same (FP32-stored) parameters; the depth sort and tile spans — the
// discrete decisions — therefore match the reference. The per-splat record
// is then rounded to FP32 for compositing (except mu2d, kept FP64).
#include "gsb_internal.cuh"

namespace gsb {

__device__ __forceinline__ double m_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double s_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double d_(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
  return a_(a_(m_(a0, b0), m_(a1, b1)), m_(a2, b2));
}

// sh.cpp:9-14
__constant__ double kC1 = 0.4886025119029199;
__constant__ double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                              0.5462742152960396};
__constant__ double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                              -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
constexpr double kSh0 = 0.28209479177387814;

// sh.cpp:18-40
__device__ __forceinline__ void sh_basis(double x, double y, double z, int degree, double* out) {
  out[0] = kSh0;
  if (degree < 1) return;
  out[1] = m_(-kC1, y);
  out[2] = m_(kC1, z);
  out[3] = m_(-kC1, x);
  if (degree < 2) return;
  const double xx = m_(x, x), yy = m_(y, y), zz = m_(z, z);
  out[4] = m_(m_(kC2[0], x), y);
  out[5] = m_(m_(kC2[1], y), z);
  out[6] = m_(kC2[2], s_(s_(m_(2.0, zz), xx), yy));
  out[7] = m_(m_(kC2[3], x), z);
  out[8] = m_(kC2[4], s_(xx, yy));
  if (degree < 3) return;
  out[9] = m_(m_(kC3[0], y), s_(m_(3.0, xx), yy));
  out[10] = m_(m_(m_(kC3[1], x), y), z);
  out[11] = m_(m_(kC3[2], y), s_(s_(m_(4.0, zz), xx), yy));
  out[12] = m_(m_(kC3[3], z), s_(s_(m_(2.0, zz), m_(3.0, xx)), m_(3.0, yy)));
  out[13] = m_(m_(kC3[4], x), s_(s_(m_(4.0, zz), xx), yy));
  out[14] = m_(m_(kC3[5], z), s_(xx, yy));
  out[15] = m_(m_(kC3[6], x), s_(xx, m_(3.0, yy)));
}

__device__ __forceinline__ int clamp_tile(double v, int n_tiles) {  // rasterizer.cpp:140-143
  const double hi = n_tiles - 1.0;
  const double c = v < 0.0 ? 0.0 : (v > hi ? hi : v);
  return (int)c;
}

__global__ void __launch_bounds__(256) preprocess_kernel(
    const float* __restrict__ params, int64_t n, int64_t n_pad, int sh_cap, int sh_active,
    const CamDev* __restrict__ cam_p, RasterDev rc, SplatRec* __restrict__ rec_g, uint2* __restrict__ rect_g,
    uint32_t* __restrict__ cnt_g, double* __restrict__ depth_g, double* __restrict__ radius_g,
    int32_t* __restrict__ rank_of_g) {
  __shared__ CamDev cam;
  if (threadIdx.x == 0) cam = *cam_p;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  rank_of_g[i] = -1;
  const float* P = params + i;
  const double mx = P[kMeanX * n_pad], my = P[kMeanY * n_pad], mz = P[kMeanZ * n_pad];
  // Se3Pose::act: rotation * p + translation (lie.hpp:38)
  const double cx = a_(dot3(cam.R[0], cam.R[1], cam.R[2], mx, my, mz), cam.t[0]);
  const double cy = a_(dot3(cam.R[3], cam.R[4], cam.R[5], mx, my, mz), cam.t[1]);
  const double cz = a_(dot3(cam.R[6], cam.R[7], cam.R[8], mx, my, mz), cam.t[2]);
  uint32_t cnt = 0;
  if (cz > rc.z_near) {
    // project (rasterizer.cpp:185-190)
    const double u = a_(d_(m_(cam.fx, cx), cz), cam.cx);
    const double v = a_(d_(m_(cam.fy, cy), cz), cam.cy);
    if (isfinite(u) && isfinite(v)) {
      // covariance3d: R(q) diag(s) (R(q) diag(s))^T
      const double qw = P[kQuatW * n_pad], qx = P[kQuatX * n_pad], qy = P[kQuatY * n_pad], qz = P[kQuatZ * n_pad];
      const double qn = __dsqrt_rn(a_(a_(a_(m_(qw, qw), m_(qx, qx)), m_(qy, qy)), m_(qz, qz)));
      const double w = d_(qw, qn), x = d_(qx, qn), y = d_(qy, qn), z = d_(qz, qn);
      double Rg[9];
      Rg[0] = s_(1.0, m_(2.0, a_(m_(y, y), m_(z, z))));
      Rg[1] = m_(2.0, s_(m_(x, y), m_(w, z)));
      Rg[2] = m_(2.0, a_(m_(x, z), m_(w, y)));
      Rg[3] = m_(2.0, a_(m_(x, y), m_(w, z)));
      Rg[4] = s_(1.0, m_(2.0, a_(m_(x, x), m_(z, z))));
      Rg[5] = m_(2.0, s_(m_(y, z), m_(w, x)));
      Rg[6] = m_(2.0, s_(m_(x, z), m_(w, y)));
      Rg[7] = m_(2.0, a_(m_(y, z), m_(w, x)));
      Rg[8] = s_(1.0, m_(2.0, a_(m_(x, x), m_(y, y))));
      const double sx = exp((double)P[kScaleX * n_pad]), sy = exp((double)P[kScaleY * n_pad]),
                   sz = exp((double)P[kScaleZ * n_pad]);
      double M[9];
      for (int r = 0; r < 3; ++r) {
        M[r * 3 + 0] = m_(Rg[r * 3 + 0], sx);
        M[r * 3 + 1] = m_(Rg[r * 3 + 1], sy);
        M[r * 3 + 2] = m_(Rg[r * 3 + 2], sz);
      }
      double S[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) S[r * 3 + c] = dot3(M[r * 3], M[r * 3 + 1], M[r * 3 + 2], M[c * 3], M[c * 3 + 1], M[c * 3 + 2]);
      // projection_jacobian (rasterizer.cpp:31-39)
      const double iz = d_(1.0, cz);
      const double iz2 = m_(iz, iz);
      const double J00 = m_(cam.fx, iz), J02 = m_(m_(-cam.fx, cx), iz2);
      const double J11 = m_(cam.fy, iz), J12 = m_(m_(-cam.fy, cy), iz2);
      // m = J R (2x3); row0 = J00*R0 + 0*R1 + J02*R2
      double m[6];
      for (int c = 0; c < 3; ++c) {
        m[c] = a_(a_(m_(J00, cam.R[c]), m_(0.0, cam.R[3 + c])), m_(J02, cam.R[6 + c]));
        m[3 + c] = a_(a_(m_(0.0, cam.R[c]), m_(J11, cam.R[3 + c])), m_(J12, cam.R[6 + c]));
      }
      double ms[6];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) ms[r * 3 + c] = dot3(m[r * 3], m[r * 3 + 1], m[r * 3 + 2], S[c], S[3 + c], S[6 + c]);
      double cov[4];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) cov[r * 2 + c] = dot3(ms[r * 3], ms[r * 3 + 1], ms[r * 3 + 2], m[c * 3], m[c * 3 + 1], m[c * 3 + 2]);
      cov[0] = a_(cov[0], rc.dilation);
      cov[3] = a_(cov[3], rc.dilation);
      // max_eigenvalue_2x2 + radius
      const double mid = m_(0.5, a_(cov[0], cov[3]));
      const double diff = m_(0.5, s_(cov[0], cov[3]));
      const double lmax = a_(mid, __dsqrt_rn(a_(m_(diff, diff), m_(cov[1], cov[2]))));
      const double radius = m_(rc.cutoff_sigma, __dsqrt_rn(lmax));
      if (radius > 0.0 && isfinite(radius) && !(a_(u, radius) < 0.0) && !(s_(u, radius) > cam.width - 1) &&
          !(a_(v, radius) < 0.0) && !(s_(v, radius) > cam.height - 1)) {
        // invert_spd2
        const double det = s_(m_(cov[0], cov[3]), m_(cov[1], cov[2]));
        const double ca = d_(cov[3], det), cb = d_(-cov[1], det), cc2 = d_(-cov[2], det), cd = d_(cov[0], det);
        // colour: sh_eval at dir = normalize(mean - center)
        double dx = s_(mx, cam.center[0]), dy = s_(my, cam.center[1]), dz = s_(mz, cam.center[2]);
        const double dn = __dsqrt_rn(a_(a_(m_(dx, dx), m_(dy, dy)), m_(dz, dz)));
        dx = d_(dx, dn);
        dy = d_(dy, dn);
        dz = d_(dz, dn);
        const int deg = sh_active < sh_cap ? sh_active : sh_cap;
        const int nb = (deg + 1) * (deg + 1);
        double basis[kMaxShCoeffs];
        sh_basis(dx, dy, dz, deg, basis);
        float col[3];
        uint32_t clamp = 0;
        for (int c = 0; c < 3; ++c) {
          double acc = 0.5;
          // quirk kept: channel stride (d_active+1)^2 inside the capacity-strided block (sh.cpp:74)
          for (int b = 0; b < nb; ++b) acc = a_(acc, m_((double)P[(kShBase + c * nb + b) * n_pad], basis[b]));
          if (acc < 0.0) {
            clamp |= 1u << c;
            acc = 0.0;
          }
          col[c] = (float)acc;
        }
        const double op = d_(1.0, a_(1.0, exp(-(double)P[kOpacity * n_pad])));
        // tile span (rasterizer.cpp:138-146)
        const double tile = (double)kTile;
        const int tx0 = clamp_tile(floor(d_(s_(u, radius), tile)), cam.tiles_x);
        const int tx1 = clamp_tile(floor(d_(a_(u, radius), tile)), cam.tiles_x);
        const int ty0 = clamp_tile(floor(d_(s_(v, radius), tile)), cam.tiles_y);
        const int ty1 = clamp_tile(floor(d_(a_(v, radius), tile)), cam.tiles_y);
        cnt = (uint32_t)(tx1 - tx0 + 1) * (uint32_t)(ty1 - ty0 + 1);
        SplatRec rec;
        rec.mu_x = u;
        rec.mu_y = v;
        rec.conic_a = (float)ca;
        rec.conic_b = (float)(0.5 * (cb + cc2));
        rec.conic_c = (float)cd;
        rec.opacity = (float)op;
        rec.col_r = col[0];
        rec.col_g = col[1];
        rec.col_b = col[2];
        rec.clamp_bits = clamp;
        rec_g[i] = rec;
        rect_g[i] = make_uint2((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16));
        depth_g[i] = cz;
        radius_g[i] = radius;
      }
    }
  }
  cnt_g[i] = cnt;
}

int launch_preprocess(cudaStream_t st, const gsb_cloud* cloud, const CamDev* cam, const RasterDev& rc,
                      gsb_frame* f) {
  const int64_t n = cloud->n;
  if (n > 0)
    preprocess_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        cloud->params.as<float>(), n, cloud->n_pad, cloud->sh_degree, cloud->active_sh_degree, cam, rc,
        f->rec_g.as<SplatRec>(), f->rect_g.as<uint2>(), f->cnt_g.as<uint32_t>(), f->depth_g.as<double>(),
        f->radius_g.as<double>(), f->rank_of_g.as<int32_t>());
  GSB_CHECK_LAUNCH("preprocess_kernel");
  return GSB_OK;
}

}  // namespace gsb
