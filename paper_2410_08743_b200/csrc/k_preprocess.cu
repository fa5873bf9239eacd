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
#include <algorithm>

#include "gsb_internal.cuh"

namespace gsb {

__device__ __forceinline__ double m_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double s_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double d_(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
  return a_(a_(m_(a0, b0), m_(a1, b1)), m_(a2, b2));
}


__device__ __forceinline__ int clamp_tile(double v, int n_tiles) {  // rasterizer.cpp:140-143
  const double hi = n_tiles - 1.0;
  const double c = v < 0.0 ? 0.0 : (v > hi ? hi : v);
  return (int)c;
}

// sh_eval (sh.cpp:66-84) in FP32 — the colour is stored FP32 anyway — plus
// the colour/direction Jacobian G[c][k] = sum_b coeff[c*cap+b] dY_b/d dir_k
// with clamped rows zeroed: the d_dir chain of render_backward
// (rasterizer.cpp:496-511, sh.cpp:42-64, capacity stride as there),
// precomputed while the SH planes are streamed so the backward never re-reads
// them. kQuirk: active degree < capacity, where the forward indexes channel c
// at c*(DEG+1)^2 (sh.cpp:74) but storage / backward use c*(cap+1)^2.
template <int DEG, bool kQuirk>
__device__ __forceinline__ void sh_colour(const float* __restrict__ P, int64_t n_pad, int sh_cap, float x, float y,
                                          float z, float col[3], uint32_t* clamp, float G[9]) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  const int bcap = (sh_cap + 1) * (sh_cap + 1);
  const float C1 = 0.4886025119029199f;
  const float C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f, -1.0925484305920792f,
                       0.5462742152960396f};
  const float C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f, 0.3731763325901154f,
                       -0.4570457994644658f, 1.445305721320277f, -0.5900435899266435f};
  float B[16], gx[16], gy[16], gz[16];
  B[0] = 0.28209479177387814f;
  gx[0] = gy[0] = gz[0] = 0.f;
  if (DEG >= 1) {
    B[1] = -C1 * y; B[2] = C1 * z; B[3] = -C1 * x;
    gx[1] = 0; gy[1] = -C1; gz[1] = 0;
    gx[2] = 0; gy[2] = 0; gz[2] = C1;
    gx[3] = -C1; gy[3] = 0; gz[3] = 0;
  }
  const float xx = x * x, yy = y * y, zz = z * z;
  if (DEG >= 2) {
    B[4] = C2[0] * x * y; B[5] = C2[1] * y * z; B[6] = C2[2] * (2.f * zz - xx - yy);
    B[7] = C2[3] * x * z; B[8] = C2[4] * (xx - yy);
    gx[4] = C2[0] * y; gy[4] = C2[0] * x; gz[4] = 0;
    gx[5] = 0; gy[5] = C2[1] * z; gz[5] = C2[1] * y;
    gx[6] = C2[2] * (-2.f * x); gy[6] = C2[2] * (-2.f * y); gz[6] = C2[2] * (4.f * z);
    gx[7] = C2[3] * z; gy[7] = 0; gz[7] = C2[3] * x;
    gx[8] = C2[4] * (2.f * x); gy[8] = C2[4] * (-2.f * y); gz[8] = 0;
  }
  if (DEG >= 3) {
    B[9] = C3[0] * y * (3.f * xx - yy); B[10] = C3[1] * x * y * z; B[11] = C3[2] * y * (4.f * zz - xx - yy);
    B[12] = C3[3] * z * (2.f * zz - 3.f * xx - 3.f * yy); B[13] = C3[4] * x * (4.f * zz - xx - yy);
    B[14] = C3[5] * z * (xx - yy); B[15] = C3[6] * x * (xx - 3.f * yy);
    gx[9] = C3[0] * (6.f * x * y); gy[9] = C3[0] * (3.f * xx - 3.f * yy); gz[9] = 0;
    gx[10] = C3[1] * (y * z); gy[10] = C3[1] * (x * z); gz[10] = C3[1] * (x * y);
    gx[11] = C3[2] * (-2.f * x * y); gy[11] = C3[2] * (4.f * zz - xx - 3.f * yy); gz[11] = C3[2] * (8.f * y * z);
    gx[12] = C3[3] * (-6.f * x * z); gy[12] = C3[3] * (-6.f * y * z); gz[12] = C3[3] * (6.f * zz - 3.f * xx - 3.f * yy);
    gx[13] = C3[4] * (4.f * zz - 3.f * xx - yy); gy[13] = C3[4] * (-2.f * x * y); gz[13] = C3[4] * (8.f * x * z);
    gx[14] = C3[5] * (2.f * x * z); gy[14] = C3[5] * (-2.f * y * z); gz[14] = C3[5] * (xx - yy);
    gx[15] = C3[6] * (3.f * xx - 3.f * yy); gy[15] = C3[6] * (-6.f * x * y); gz[15] = 0;
  }
  uint32_t cl = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float v = 0.5f, g0 = 0.f, g1 = 0.f, g2 = 0.f;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const float co = P[(int64_t)(kShBase + c * (kQuirk ? NB : bcap) + b) * n_pad];
      v = fmaf(co, B[b], v);
      if (!kQuirk) {
        g0 = fmaf(co, gx[b], g0);
        g1 = fmaf(co, gy[b], g1);
        g2 = fmaf(co, gz[b], g2);
      }
    }
    if (kQuirk) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const float co = P[(int64_t)(kShBase + c * bcap + b) * n_pad];
        g0 = fmaf(co, gx[b], g0);
        g1 = fmaf(co, gy[b], g1);
        g2 = fmaf(co, gz[b], g2);
      }
    }
    if (v < 0.f) {
      cl |= 1u << c;
      v = 0.f;
      g0 = g1 = g2 = 0.f;
    }
    col[c] = v;
    G[3 * c] = g0;
    G[3 * c + 1] = g1;
    G[3 * c + 2] = g2;
  }
  *clamp = cl;
}

// The CTA's kPreBlock-Gaussian segment of every parameter plane is staged into
// shared memory with one TMA bulk copy per plane (issued by one thread,
// completing on an mbarrier), so all ~59 KB are in flight at once; the
// per-thread reads below then come from shared memory (stride kPreBlock).
#ifndef GSB_PRE_BLOCK
#define GSB_PRE_BLOCK 128
#endif
constexpr int kPreBlock = GSB_PRE_BLOCK;
// (an explicit minBlocks of 1 lets ptxas spend 138 registers -> 1 CTA/SM;
// the default form keeps 124 and 2 CTAs/SM of 256 threads; measured best:
// 128-thread CTAs at 5 CTAs/SM — K1 0.107 (256 x 2) -> 0.101 (256 x 3) ->
// 0.094 ms (128 x 5), pose batch +1.2 % over 256 x 2)
#ifndef GSB_PRE_MIN_BLOCKS
#define GSB_PRE_MIN_BLOCKS 5
#endif
#if GSB_PRE_MIN_BLOCKS > 1
#define GSB_PRE_BOUNDS __launch_bounds__(kPreBlock, GSB_PRE_MIN_BLOCKS)
#else
#define GSB_PRE_BOUNDS __launch_bounds__(kPreBlock)
#endif

// Per-view outputs of K1 (one forward state).
struct PreOut {
  const CamDev* cam_src;  // camera of this iteration (device resident)
  CamDev* cam_dst;        // copied into the forward state by block 0 (multi-view launch only)
  SplatRec* rec_g;
  uint2* rect_g;
  uint32_t* cnt_g;
  double* depth_g;
  double* radius_g;
  int32_t* rank_of_g;
  float* colj;
  uint32_t* counters;
  SplatAux* aux_g;
  uint32_t* off_g;
  int64_t n_pad_out;  // plane stride of colj
  int32_t tile_local;
  int32_t write_rect;    // tile rect (global binning / export)
  int32_t write_export;  // radius, rank_of_g = -1 (RenderOutput export only)
  int32_t pad;
};
constexpr int kMaxPreViews = 16;
struct PreViews {
  PreOut v[kMaxPreViews];
};

// View-independent per-Gaussian geometry: mean, the 3D covariance
// R(q) diag(s)^2 R(q)^T (scene.cpp:90-94, symmetric: 6 entries) and the
// opacity sigmoid — evaluated once and reused by every view of a launch.
struct GaussGeom {
  double mx, my, mz;
  double S00, S01, S02, S11, S12, S22;
  double op;
};

__device__ __forceinline__ GaussGeom gauss_geom(const float* P, int64_t n_pad) {
  GaussGeom g;
  g.mx = P[kMeanX * n_pad];
  g.my = P[kMeanY * n_pad];
  g.mz = P[kMeanZ * n_pad];
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
  // S[r][c] = <M_r, M_c>; exactly symmetric (the products commute)
  g.S00 = dot3(M[0], M[1], M[2], M[0], M[1], M[2]);
  g.S01 = dot3(M[0], M[1], M[2], M[3], M[4], M[5]);
  g.S02 = dot3(M[0], M[1], M[2], M[6], M[7], M[8]);
  g.S11 = dot3(M[3], M[4], M[5], M[3], M[4], M[5]);
  g.S12 = dot3(M[3], M[4], M[5], M[6], M[7], M[8]);
  g.S22 = dot3(M[6], M[7], M[8], M[6], M[7], M[8]);
  g.op = d_(1.0, a_(1.0, exp(-(double)P[kOpacity * n_pad])));
  return g;
}

// One Gaussian seen from one camera: rasterizer.cpp:95-125 + 138-146.
// Returns the packed tile count | clamp bits (0 = culled) and the tile rect.
template <int DEG, bool kQuirk>
__device__ __forceinline__ uint32_t project_one(const float* P, int64_t n_pad, int sh_cap, const GaussGeom& g,
                                                const CamDev& cam, const RasterDev& rc, int64_t i,
                                                const PreOut& o, uint32_t* rect_x, uint32_t* rect_y) {
  // Se3Pose::act: rotation * p + translation (lie.hpp:38)
  const double cx = a_(dot3(cam.R[0], cam.R[1], cam.R[2], g.mx, g.my, g.mz), cam.t[0]);
  const double cy = a_(dot3(cam.R[3], cam.R[4], cam.R[5], g.mx, g.my, g.mz), cam.t[1]);
  const double cz = a_(dot3(cam.R[6], cam.R[7], cam.R[8], g.mx, g.my, g.mz), cam.t[2]);
  if (!(cz > rc.z_near)) return 0u;
  // project (rasterizer.cpp:185-190)
  const double u = a_(d_(m_(cam.fx, cx), cz), cam.cx);
  const double v = a_(d_(m_(cam.fy, cy), cz), cam.cy);
  if (!(isfinite(u) && isfinite(v))) return 0u;
  const double S[9] = {g.S00, g.S01, g.S02, g.S01, g.S11, g.S12, g.S02, g.S12, g.S22};
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
  if (!(radius > 0.0 && isfinite(radius) && !(a_(u, radius) < 0.0) && !(s_(u, radius) > cam.width - 1) &&
        !(a_(v, radius) < 0.0) && !(s_(v, radius) > cam.height - 1)))
    return 0u;
  // invert_spd2 (one reciprocal: the conic is stored in FP32, so the FP64
  // quotient's last bit never matters; 3 DP divisions fewer per view)
  const double det = s_(m_(cov[0], cov[3]), m_(cov[1], cov[2]));
  const double idet = d_(1.0, det);
  const double ca = m_(cov[3], idet), cb = m_(-cov[1], idet), cc2 = m_(-cov[2], idet), cd = m_(cov[0], idet);
  // colour: sh_eval at dir = normalize(mean - center)
  double dx = s_(g.mx, cam.center[0]), dy = s_(g.my, cam.center[1]), dz = s_(g.mz, cam.center[2]);
  const double dn = __dsqrt_rn(a_(a_(m_(dx, dx), m_(dy, dy)), m_(dz, dz)));
  const double idn = d_(1.0, dn);  // the direction feeds the FP32 SH evaluation
  dx = m_(dx, idn);
  dy = m_(dy, idn);
  dz = m_(dz, idn);
  float col[3], G[9];
  uint32_t clamp = 0;
  sh_colour<DEG, kQuirk>(P, n_pad, sh_cap, (float)dx, (float)dy, (float)dz, col, &clamp, G);
  for (int k = 0; k < 9; ++k) o.colj[(int64_t)k * o.n_pad_out + i] = G[k];
  // tile span (rasterizer.cpp:138-146); x / 16 == x * (1/16) exactly (power of two)
  static_assert((kTile & (kTile - 1)) == 0, "tile size must be a power of two");
  const double itile = 1.0 / (double)kTile;
  const int tx0 = clamp_tile(floor(m_(s_(u, radius), itile)), cam.tiles_x);
  const int tx1 = clamp_tile(floor(m_(a_(u, radius), itile)), cam.tiles_x);
  const int ty0 = clamp_tile(floor(m_(s_(v, radius), itile)), cam.tiles_y);
  const int ty1 = clamp_tile(floor(m_(a_(v, radius), itile)), cam.tiles_y);
  SplatRec rec;
  rec.mu_x = u;
  rec.mu_y = v;
  rec.conic_a = (float)ca;
  rec.conic_b = (float)(0.5 * (cb + cc2));
  rec.conic_c = (float)cd;
  rec.opacity = (float)g.op;
  rec.col_r = col[0];
  rec.col_g = col[1];
  rec.col_b = col[2];
  rec.clamp_bits = clamp;
  o.rec_g[i] = rec;
  *rect_x = (uint32_t)tx0 | ((uint32_t)tx1 << 16);
  *rect_y = (uint32_t)ty0 | ((uint32_t)ty1 << 16);
  if (o.write_rect) o.rect_g[i] = make_uint2(*rect_x, *rect_y);
  o.depth_g[i] = cz;
  if (o.write_export) o.radius_g[i] = radius;
  return ((uint32_t)(tx1 - tx0 + 1) * (uint32_t)(ty1 - ty0 + 1)) | (clamp << kClampShift);
}

// Tile-local binning (k_bin.cu): reserve the splat's entry slots with one
// atomic per warp (slot order is free — every consumer indexes them by
// (gid, tile) — so the result stays deterministic) and count V.
__device__ __forceinline__ void reserve_slots(const PreOut& o, int64_t i, uint32_t cnt, uint32_t rect_x,
                                              uint32_t rect_y) {
  const uint32_t c = cnt & kCntMask, lane = threadIdx.x & 31u;
  uint32_t x = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= (uint32_t)off) x += y;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
  const uint32_t vis = __popc(__ballot_sync(0xffffffffu, c > 0u));
  uint32_t base = 0;
  if (lane == 0 && tot) {
    base = atomicAdd(o.counters + 1, tot);
    atomicAdd(o.counters + 0, vis);
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (c) {
    const uint32_t off = base + x - c;
    const uint32_t tx0 = rect_x & 0xffffu, tx1 = rect_x >> 16, ty0 = rect_y & 0xffffu, ty1 = rect_y >> 16;
    SplatAux a;
    a.off = off;
    a.tx0_ty0 = tx0 | (ty0 << 16);
    a.nx_ny = (tx1 - tx0 + 1u) | ((ty1 - ty0 + 1u) << 16);
    a.gid = (int32_t)i;
    o.aux_g[i] = a;
    o.off_g[i] = off;
  }
}

// K1 over `nviews` cameras at once: the CTA's kPreBlock-Gaussian segment of every
// parameter plane is staged into shared memory with one TMA bulk copy per
// plane (issued by one thread, completing on an mbarrier), the
// view-independent geometry is evaluated once, and each view's projection,
// colour and tile rect follow from the same staged parameters — the cloud is
// read from HBM once per launch instead of once per view.
template <int DEG, bool kQuirk>
__global__ void GSB_PRE_BOUNDS preprocess_kernel(const float* __restrict__ params, int64_t n,
                                                               int64_t n_pad_g, int sh_cap, RasterDev rc,
                                                               int nviews, const __grid_constant__ PreViews views) {
  extern __shared__ __align__(128) float s_par[];  // [planes][kPreBlock]
  __shared__ CamDev s_cam[kMaxPreViews];
  __shared__ __align__(8) uint64_t bar;
  const int nplanes = kShBase + 3 * (sh_cap + 1) * (sh_cap + 1);
  const int64_t i0 = (int64_t)blockIdx.x * kPreBlock;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    const int64_t cnt_here = n - i0 < kPreBlock ? n - i0 : kPreBlock;
    const uint32_t bytes = (uint32_t)(((cnt_here * 4) + 15) & ~(int64_t)15);  // n_pad covers the round-up
    mbar_arrive_expect_tx(&bar, bytes * (uint32_t)nplanes);
    for (int p = 0; p < nplanes; ++p) tma_load_1d(s_par + p * kPreBlock, params + p * n_pad_g + i0, bytes, &bar);
  }
  for (int v = threadIdx.x; v < nviews; v += kPreBlock) {
    s_cam[v] = *views.v[v].cam_src;
    if (blockIdx.x == 0 && views.v[v].cam_dst) *views.v[v].cam_dst = s_cam[v];
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int64_t i = i0 + threadIdx.x;
  const float* P = s_par + threadIdx.x;
  constexpr int64_t n_pad = kPreBlock;  // plane stride of the staged copy
  GaussGeom g{};
  if (i < n) g = gauss_geom(P, n_pad);
  for (int v = 0; v < nviews; ++v) {
    const PreOut& o = views.v[v];
    uint32_t cnt = 0, rect_x = 0, rect_y = 0;
    if (i < n) {
      if (o.write_export) o.rank_of_g[i] = -1;
      cnt = project_one<DEG, kQuirk>(P, n_pad, sh_cap, g, s_cam[v], rc, i, o, &rect_x, &rect_y);
      o.cnt_g[i] = cnt;
    }
    if (o.tile_local) reserve_slots(o, i, cnt, rect_x, rect_y);
  }
}

static PreOut pre_out(const CamDev* cam_src, CamDev* cam_dst, gsb_frame* f, int64_t n_pad) {
  PreOut o{};
  o.cam_src = cam_src;
  o.cam_dst = cam_dst;
  o.rec_g = f->rec_g.as<SplatRec>();
  o.rect_g = f->rect_g.as<uint2>();
  o.cnt_g = f->cnt_g.as<uint32_t>();
  o.depth_g = f->depth_g.as<double>();
  o.radius_g = f->radius_g.as<double>();
  o.rank_of_g = f->rank_of_g.as<int32_t>();
  o.colj = f->colj.as<float>();
  o.counters = f->counters.as<uint32_t>();
  o.aux_g = f->aux_g.as<SplatAux>();
  o.off_g = f->off_g.as<uint32_t>();
  o.n_pad_out = n_pad;
  o.tile_local = f->binning == kBinTileLocal ? 1 : 0;
  o.write_export = f->lean ? 0 : 1;
  o.write_rect = (!f->lean || f->binning != kBinTileLocal) ? 1 : 0;
  return o;
}

static int launch_pre(cudaStream_t st, const gsb_cloud* cloud, const RasterDev& rc, int nviews, const PreViews& pv) {
  const int64_t n = cloud->n;
  const int deg = std::min(cloud->active_sh_degree, cloud->sh_degree);
  const bool quirk = deg < cloud->sh_degree;
  const size_t smem = sizeof(float) * kPreBlock * num_planes(cloud->sh_degree);
#define GSB_PRE(D, Q)                                                                             \
  preprocess_kernel<D, Q><<<(unsigned)((n + kPreBlock - 1) / kPreBlock), kPreBlock, smem, st>>>( \
      cloud->params.as<float>(), n, cloud->n_pad, cloud->sh_degree, rc, nviews, pv)
  if (n > 0) {
    switch (deg * 2 + (quirk ? 1 : 0)) {
      case 0: GSB_PRE(0, false); break;
      case 1: GSB_PRE(0, true); break;
      case 2: GSB_PRE(1, false); break;
      case 3: GSB_PRE(1, true); break;
      case 4: GSB_PRE(2, false); break;
      case 5: GSB_PRE(2, true); break;
      default: GSB_PRE(3, false); break;
    }
  }
#undef GSB_PRE
  GSB_CHECK_LAUNCH("preprocess_kernel");
  return GSB_OK;
}

int launch_preprocess(cudaStream_t st, const gsb_cloud* cloud, const CamDev* cam, const RasterDev& rc,
                      gsb_frame* f) {
  PreViews pv{};
  pv.v[0] = pre_out(cam, nullptr, f, cloud->n_pad);
  return launch_pre(st, cloud, rc, 1, pv);
}

// One launch for several forward states of the same cloud (pose batches):
// cams[k] is view k's camera, copied into frames[k]->cam by the kernel.
int launch_preprocess_multi(cudaStream_t st, const gsb_cloud* cloud, const RasterDev& rc, const CamDev* const* cams,
                            gsb_frame* const* frames, int nviews) {
  for (int v0 = 0; v0 < nviews; v0 += kMaxPreViews) {
    PreViews pv{};
    const int nv = std::min(kMaxPreViews, nviews - v0);
    for (int k = 0; k < nv; ++k)
      pv.v[k] = pre_out(cams[v0 + k], frames[v0 + k]->cam.as<CamDev>(), frames[v0 + k], cloud->n_pad);
    if (int r = launch_pre(st, cloud, rc, nv, pv)) return r;
  }
  return GSB_OK;
}

// Opt every instantiation into the dynamic shared memory its staging needs
// (59 KB at SH-3). Called once per context, outside any graph capture.
int init_preprocess_attributes() {
  const int smem = (int)(sizeof(float) * kPreBlock * num_planes(3));
#define GSB_ATTR(D, Q) \
  GSB_CUDA(cudaFuncSetAttribute(preprocess_kernel<D, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
  GSB_ATTR(0, false);
  GSB_ATTR(0, true);
  GSB_ATTR(1, false);
  GSB_ATTR(1, true);
  GSB_ATTR(2, false);
  GSB_ATTR(2, true);
  GSB_ATTR(3, false);
#undef GSB_ATTR
  return GSB_OK;
}

}  // namespace gsb
