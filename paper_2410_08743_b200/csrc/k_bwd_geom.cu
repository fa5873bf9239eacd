// k_bwd_geom.cu — K4b: per-Gaussian geometry chain of the backward pass and
// the SE(3) pose gradient, with a deterministic (atomic-free) reduction of
// the 6-vector: warp butterfly -> fixed warp order -> per-block partials ->
// one fixed-order final block.
//
// Reference: render_backward phases 2-3 (rasterizer.cpp:407-538):
// per-splat sums of the entry partials in tile order (410-418), conic ->
// cov2d (460), cov2d = M Sigma M^T (462-463), M = J W (465-466), J -> mu_cam
// (469-477), mu2d -> mu_cam (479-482), Sigma = R D R^T -> log-scales and raw
// quaternion through quat_rotation_jacobian (485-494, scene.cpp:56-88), SH
// colour chain with clamp mask (496-513, sh.cpp:18-64), parameter grads
// (516-521) and the pose tangent: v = d_mu_cam + R_c d_to_gaussian,
// w = mu_cam x d_mu_cam + sum_k <d_R_c, [e_k]x R_c> (523-532,
// lie.cpp:173-181). Geometry is recomputed in FP64 from the FP32 parameters.
//
// One thread per Gaussian in index order. Everything it reads is plane-major
// and indexed by the Gaussian id (coalesced): tile count + clamp bits, the
// entry offset, 10 geometry planes and the 9-plane colour Jacobian that K1
// precomputed from the SH planes (so SH coefficients are never re-read);
// its partials are one contiguous run. Gradient planes are written coalesced.
#include "gsb_internal.cuh"

namespace gsb {

__constant__ double kBC1 = 0.4886025119029199;
__constant__ double kBC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                               0.5462742152960396};
__constant__ double kBC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                               -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

// sh.cpp:18-40
__device__ __forceinline__ void sh_basis_d(double x, double y, double z, int degree, double* B) {
  B[0] = 0.28209479177387814;
  if (degree < 1) return;
  B[1] = -kBC1 * y; B[2] = kBC1 * z; B[3] = -kBC1 * x;
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  B[4] = kBC2[0] * x * y; B[5] = kBC2[1] * y * z; B[6] = kBC2[2] * (2.0 * zz - xx - yy);
  B[7] = kBC2[3] * x * z; B[8] = kBC2[4] * (xx - yy);
  if (degree < 3) return;
  B[9] = kBC3[0] * y * (3.0 * xx - yy); B[10] = kBC3[1] * x * y * z;
  B[11] = kBC3[2] * y * (4.0 * zz - xx - yy); B[12] = kBC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  B[13] = kBC3[4] * x * (4.0 * zz - xx - yy); B[14] = kBC3[5] * z * (xx - yy);
  B[15] = kBC3[6] * x * (xx - 3.0 * yy);
}

// The CTA's 256-Gaussian segments of the 11 geometry/opacity planes, the 9
// colour-Jacobian planes, the tile counts and the entry offsets are staged
// into shared memory by TMA bulk copies (one elected thread, one mbarrier).
#ifndef GSB_GEOM_BLOCK
#define GSB_GEOM_BLOCK 256
#endif
constexpr int kGeomBlock = GSB_GEOM_BLOCK;
constexpr int kGeomWarps = kGeomBlock / 32;
#ifndef GSB_GEOM_POSE_MIN_BLOCKS
#define GSB_GEOM_POSE_MIN_BLOCKS 5  // 48 registers: occupancy over ~100 spilled bytes (measured: 4 -> 5 CTAs/SM, 0.087 -> 0.085 ms)
#endif
#ifndef GSB_GEOM_FULL_MIN_BLOCKS
#define GSB_GEOM_FULL_MIN_BLOCKS 2
#endif
#ifndef GSB_FULL_CHAIN_T
#define GSB_FULL_CHAIN_T double
#endif
#ifndef GSB_POSE_CHAIN_T
#define GSB_POSE_CHAIN_T float
#endif
constexpr int kGeomPlanes = kOpacity + 1;  // means, quat, log-scale, opacity

// Where K4b finds each splat's tile rect (tile-local binning: aux_g; global:
// rect_g) and the per-tile cut K4a wrote (k_raster.cu).
struct EntryCut {
  const double2* tile_cut;
  const double* depth_g;
  const SplatAux* aux_g;
  const uint2* rect_g;
  int32_t tiles_x;
};

// R: arithmetic type of the per-splat chain — double for the full gradient
// bundle (joint_optimize's parameter gradients), float for the pose-only
// path (the 6-vector itself is accumulated in FP64 either way).
template <bool kFull, typename R>
__global__ void __launch_bounds__(kGeomBlock, (kFull ? GSB_GEOM_FULL_MIN_BLOCKS : GSB_GEOM_POSE_MIN_BLOCKS)) backward_geom_kernel(
    const float* __restrict__ params, int64_t n, int64_t n_pad_g, int sh_cap, int sh_active,
    const CamDev* __restrict__ cam_p, RasterDev rc, const uint32_t* __restrict__ cnt_g,
    const uint32_t* __restrict__ off_g, const float* __restrict__ colj, const float* __restrict__ partials,
    int64_t k_cap, const EntryCut cutd, float* __restrict__ grads, double* __restrict__ pose_blocks) {
  __shared__ __align__(128) float s_par[kGeomPlanes * kGeomBlock];
  __shared__ __align__(128) float s_colj[9 * kGeomBlock];
  __shared__ __align__(128) uint32_t s_cnt[kGeomBlock], s_off[kGeomBlock];
  __shared__ __align__(128) uint4 s_rect[kGeomBlock];  // SplatAux (tile-local) or uint2 rect pairs (global)
  __shared__ __align__(128) double s_dep[kGeomBlock];
  __shared__ CamDev cam;
  __shared__ double s_pose[kGeomWarps][6];
  __shared__ __align__(8) uint64_t bar, bar2;
  const int64_t i0 = (int64_t)blockIdx.x * kGeomBlock;
  // Two transactions: the entry bookkeeping (counts, offsets, rects, depths)
  // lands first and the partial-sum loop starts on it while the parameter
  // and colour-Jacobian planes are still in flight.
  if (threadIdx.x == 0) {
    cam = *cam_p;
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    const int64_t here = n - i0 < kGeomBlock ? n - i0 : kGeomBlock;
    const uint32_t bytes = (uint32_t)(((here * 4) + 15) & ~(int64_t)15);
    const uint32_t b8 = (uint32_t)(((here * 8) + 15) & ~(int64_t)15);
    const uint32_t brect = cutd.aux_g ? (uint32_t)(here * 16) : b8;
    // cnt_g / off_g are sized to whole 256-blocks (frame_reserve), colj to n_pad
    mbar_arrive_expect_tx(&bar, bytes * 2 + b8 + brect);
    tma_load_1d(s_cnt, cnt_g + i0, bytes, &bar);
    tma_load_1d(s_off, off_g + i0, bytes, &bar);
    tma_load_1d(s_dep, cutd.depth_g + i0, b8, &bar);
    if (cutd.aux_g)
      tma_load_1d(s_rect, cutd.aux_g + i0, brect, &bar);
    else
      tma_load_1d(s_rect, cutd.rect_g + i0, brect, &bar);
    mbar_arrive_expect_tx(&bar2, bytes * (kGeomPlanes + 9));
    for (int p = 0; p < kGeomPlanes; ++p) tma_load_1d(s_par + p * kGeomBlock, params + p * n_pad_g + i0, bytes, &bar2);
    for (int p = 0; p < 9; ++p) tma_load_1d(s_colj + p * kGeomBlock, colj + p * n_pad_g + i0, bytes, &bar2);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int64_t i = i0 + threadIdx.x;
  const int bcap = (sh_cap + 1) * (sh_cap + 1);
  const int nplanes = kShBase + 3 * bcap;
  double pc0 = 0, pc1 = 0, pc2 = 0, pc3 = 0, pc4 = 0, pc5 = 0;
  const uint32_t craw = i < n ? s_cnt[threadIdx.x] : 0u;
  const uint32_t cnt = craw & kCntMask;
  if (kFull && i < n && cnt == 0u) {
    for (int p = 0; p < nplanes + 2; ++p) grads[(int64_t)p * n_pad_g + i] = 0.f;
  }
  // (off + cnt > k_cap only when the entry capacity overflowed: the iteration
  // is discarded by the pose step and re-run, so skip the splat.)
  const uint32_t off = s_off[threadIdx.x];
  if (i < n && cnt > 0u && (int64_t)off + cnt <= k_cap) {
    const uint32_t clamp = craw >> kClampShift;
    // phase 2: ordered sum of this splat's entry partials (tile order); the
    // pose-only backward stores 8 per entry (no opacity), two 16-B loads
    // Entries past their tile's cut were replayed by no pixel (zero partials,
    // never stored by K4a): skipping them leaves every sum bit-identical.
    double acc[kPartial];
#pragma unroll
    for (int c = 0; c < kPartial; ++c) acc[c] = 0.0;
    uint32_t tx0, ty0, nx;
    if (cutd.aux_g) {
      const uint4 A = s_rect[threadIdx.x];  // SplatAux {off, tx0_ty0, nx_ny, gid}
      tx0 = A.y & 0xffffu; ty0 = A.y >> 16; nx = A.z & 0xffffu;
    } else {
      const uint2 rc2 = reinterpret_cast<const uint2*>(s_rect)[threadIdx.x];
      tx0 = rc2.x & 0xffffu; ty0 = rc2.y & 0xffffu; nx = (rc2.x >> 16) - tx0 + 1u;
    }
    const double dep = s_dep[threadIdx.x], gidd = (double)i;
    const double2* cutrow = cutd.tile_cut + (int64_t)ty0 * cutd.tiles_x + tx0;
    uint32_t jx = 0;
    // 32 entries at a time: the cut loads are independent, then only the
    // live entries' partials are loaded (in tile order).
    for (uint32_t j0 = 0; j0 < cnt; j0 += 32) {
      const uint32_t m = cnt - j0 < 32u ? cnt - j0 : 32u;
      uint32_t live = 0;
      for (uint32_t u = 0; u < m; ++u) {
        const double2 ct = __ldg(cutrow + jx);
        if (dep < ct.x || (dep == ct.x && gidd <= ct.y)) live |= 1u << u;
        if (++jx == nx) { jx = 0; cutrow += cutd.tiles_x; }
      }
      while (live) {
        const uint32_t j = j0 + (uint32_t)(__ffs(live) - 1);
        live &= live - 1u;
        if (kFull) {
          const float* pp = partials + ((int64_t)off + j) * kPartial;
#pragma unroll
          for (int c = 0; c < kPartial; ++c) acc[c] += (double)pp[c];
        } else {
          const float4* pp = reinterpret_cast<const float4*>(partials) + ((int64_t)off + j) * 2;
          const float4 lo = pp[0], hi = pp[1];
          acc[0] += (double)lo.x; acc[1] += (double)lo.y; acc[2] += (double)lo.z; acc[3] += (double)lo.w;
          acc[4] += (double)hi.x; acc[5] += (double)hi.y; acc[6] += (double)hi.z; acc[7] += (double)hi.w;
        }
      }
    }
    mbar_wait(&bar2, 0);
    const float* P = s_par + threadIdx.x;
    constexpr int64_t n_pad = kGeomBlock;  // plane stride of the staged copy
    const R mean0 = P[kMeanX * n_pad], mean1 = P[kMeanY * n_pad], mean2 = P[kMeanZ * n_pad];
    R Rc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Rc[k] = (R)cam.R[k];
    R mc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) mc[a] = Rc[a * 3] * mean0 + Rc[a * 3 + 1] * mean1 + Rc[a * 3 + 2] * mean2 + (R)cam.t[a];
    const R iz = R(1.0) / mc[2], iz2 = iz * iz, iz3 = iz2 * iz;
    const R fx = (R)cam.fx, fy = (R)cam.fy;
    const R J00 = fx * iz, J02 = -fx * mc[0] * iz2, J11 = fy * iz, J12 = -fy * mc[1] * iz2;
    R m[6];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      m[b] = J00 * Rc[b] + J02 * Rc[6 + b];
      m[3 + b] = J11 * Rc[3 + b] + J12 * Rc[6 + b];
    }
    const R sc0 = exp((R)P[kScaleX * n_pad]), sc1 = exp((R)P[kScaleY * n_pad]),
                 sc2 = exp((R)P[kScaleZ * n_pad]);
    const R qr0 = P[kQuatW * n_pad], qr1 = P[kQuatX * n_pad], qr2 = P[kQuatY * n_pad], qr3 = P[kQuatZ * n_pad];
    const R qn = sqrt(qr0 * qr0 + qr1 * qr1 + qr2 * qr2 + qr3 * qr3);
    const R w = qr0 / qn, x = qr1 / qn, y = qr2 / qn, zq = qr3 / qn;
    const R Rg[9] = {1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y),
                          2 * (x * y + w * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x),
                          2 * (x * zq - w * y), 2 * (y * zq + w * x), 1 - 2 * (x * x + y * y)};
    const R s2[3] = {sc0 * sc0, sc1 * sc1, sc2 * sc2};
    R Sg[6];  // symmetric Sigma: 00 01 02 11 12 22
    Sg[0] = Rg[0] * Rg[0] * s2[0] + Rg[1] * Rg[1] * s2[1] + Rg[2] * Rg[2] * s2[2];
    Sg[1] = Rg[0] * Rg[3] * s2[0] + Rg[1] * Rg[4] * s2[1] + Rg[2] * Rg[5] * s2[2];
    Sg[2] = Rg[0] * Rg[6] * s2[0] + Rg[1] * Rg[7] * s2[1] + Rg[2] * Rg[8] * s2[2];
    Sg[3] = Rg[3] * Rg[3] * s2[0] + Rg[4] * Rg[4] * s2[1] + Rg[5] * Rg[5] * s2[2];
    Sg[4] = Rg[3] * Rg[6] * s2[0] + Rg[4] * Rg[7] * s2[1] + Rg[5] * Rg[8] * s2[2];
    Sg[5] = Rg[6] * Rg[6] * s2[0] + Rg[7] * Rg[7] * s2[1] + Rg[8] * Rg[8] * s2[2];
    auto S = [&](int r, int c) -> R {
      const int a = r < c ? r : c, b = r < c ? c : r;
      return Sg[a == 0 ? b : (a == 1 ? 2 + b : 5)];
    };
    // cov2d = m Sigma m^T + dilation; conic = cov2d^-1 (same expressions as K1)
    R ms[6];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) ms[a * 3 + b] = m[a * 3] * S(0, b) + m[a * 3 + 1] * S(1, b) + m[a * 3 + 2] * S(2, b);
    const R c00 = ms[0] * m[0] + ms[1] * m[1] + ms[2] * m[2] + (R)rc.dilation;
    const R c01 = ms[0] * m[3] + ms[1] * m[4] + ms[2] * m[5];
    const R c11 = ms[3] * m[3] + ms[4] * m[4] + ms[5] * m[5] + (R)rc.dilation;
    const R det = c00 * c11 - c01 * c01;
    const R C0 = c11 / det, C1 = -c01 / det, C3 = c00 / det;
    // d_cov2d = -(C D C), D symmetric = [[D00, D01], [D01, D11]]
    const R D00 = acc[2], D01 = acc[3], D11 = acc[4];
    const R E0 = C0 * D00 + C1 * D01, E1 = C0 * D01 + C1 * D11;  // (C D) row 0
    const R E2 = C1 * D00 + C3 * D01, E3 = C1 * D01 + C3 * D11;  // (C D) row 1
    const R dc00 = -(E0 * C0 + E1 * C1), dc01 = -(E0 * C1 + E1 * C3), dc11 = -(E2 * C1 + E3 * C3);
    // d_m = 2 dcov m Sigma (2x3)
    R t0[3], t1[3], dm[6];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      t0[b] = R(2.0) * (dc00 * m[b] + dc01 * m[3 + b]);
      t1[b] = R(2.0) * (dc01 * m[b] + dc11 * m[3 + b]);
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      dm[b] = t0[0] * S(0, b) + t0[1] * S(1, b) + t0[2] * S(2, b);
      dm[3 + b] = t1[0] * S(0, b) + t1[1] * S(1, b) + t1[2] * S(2, b);
    }
    // d_jac = d_m R^T (only columns 0 and 2 of row 0, 1 and 2 of row 1 matter)
    const R dj00 = dm[0] * Rc[0] + dm[1] * Rc[1] + dm[2] * Rc[2];
    const R dj02 = dm[0] * Rc[6] + dm[1] * Rc[7] + dm[2] * Rc[8];
    const R dj11 = dm[3] * Rc[3] + dm[4] * Rc[4] + dm[5] * Rc[5];
    const R dj12 = dm[3] * Rc[6] + dm[4] * Rc[7] + dm[5] * Rc[8];
    const R dmu2x = acc[0], dmu2y = acc[1];
    R dmc[3];
    dmc[0] = dj02 * (-fx * iz2) + dmu2x * fx * iz;
    dmc[1] = dj12 * (-fy * iz2) + dmu2y * fy * iz;
    dmc[2] = dj00 * (-fx * iz2) + dj11 * (-fy * iz2) + dj02 * (R(2.0) * fx * mc[0] * iz3) +
             dj12 * (R(2.0) * fy * mc[1] * iz3) - dmu2x * fx * mc[0] * iz2 - dmu2y * fy * mc[1] * iz2;
    // colour chain: d_dir = G^T d_colour, projected and scaled by 1/dist
    const R tg0 = mean0 - (R)cam.center[0], tg1 = mean1 - (R)cam.center[1], tg2 = mean2 - (R)cam.center[2];
    const R dist = sqrt(tg0 * tg0 + tg1 * tg1 + tg2 * tg2);
    const R dir0 = tg0 / dist, dir1 = tg1 / dist, dir2 = tg2 / dist;
    const R dcol[3] = {(R)acc[5], (R)acc[6], (R)acc[7]};
    R dd0 = 0, dd1 = 0, dd2 = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      dd0 += dcol[c] * (R)s_colj[(3 * c + 0) * kGeomBlock + threadIdx.x];
      dd1 += dcol[c] * (R)s_colj[(3 * c + 1) * kGeomBlock + threadIdx.x];
      dd2 += dcol[c] * (R)s_colj[(3 * c + 2) * kGeomBlock + threadIdx.x];
    }
    const R pd = dir0 * dd0 + dir1 * dd1 + dir2 * dd2;
    const R dtg0 = (dd0 - dir0 * pd) / dist, dtg1 = (dd1 - dir1 * pd) / dist, dtg2 = (dd2 - dir2 * pd) / dist;
    // pose tangent (rasterizer.cpp:523-533); d_R_c = J^T d_m has rows
    // J00 dm0, J11 dm1, J02 dm0 + J12 dm1.
    pc0 = dmc[0] + (Rc[0] * dtg0 + Rc[1] * dtg1 + Rc[2] * dtg2);
    pc1 = dmc[1] + (Rc[3] * dtg0 + Rc[4] * dtg1 + Rc[5] * dtg2);
    pc2 = dmc[2] + (Rc[6] * dtg0 + Rc[7] * dtg1 + Rc[8] * dtg2);
    pc3 = mc[1] * dmc[2] - mc[2] * dmc[1];
    pc4 = mc[2] * dmc[0] - mc[0] * dmc[2];
    pc5 = mc[0] * dmc[1] - mc[1] * dmc[0];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const R r0 = J00 * dm[b], r1 = J11 * dm[3 + b], r2 = J02 * dm[b] + J12 * dm[3 + b];
      pc3 += -r1 * Rc[6 + b] + r2 * Rc[3 + b];
      pc4 += r0 * Rc[6 + b] - r2 * Rc[b];
      pc5 += -r0 * Rc[3 + b] + r1 * Rc[b];
    }
    if (kFull) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double dtga = a == 0 ? dtg0 : (a == 1 ? dtg1 : dtg2);
        grads[(int64_t)(kMeanX + a) * n_pad_g + i] = (float)(Rc[a] * dmc[0] + Rc[3 + a] * dmc[1] + Rc[6 + a] * dmc[2] + dtga);
      }
      // d_Sigma = m^T dcov m (symmetric)
      double dS[9];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          dS[a * 3 + b] = (m[a] * dc00 + m[3 + a] * dc01) * m[b] + (m[a] * dc01 + m[3 + a] * dc11) * m[3 + b];
      // d_Rg = 2 dS Rg diag(s^2); d_log_scale_k = 2 s_k (Rg^T dS Rg)_kk s_k
      double dRg[9];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          dRg[a * 3 + b] = 2.0 * (dS[a * 3] * Rg[b] + dS[a * 3 + 1] * Rg[3 + b] + dS[a * 3 + 2] * Rg[6 + b]) * s2[b];
      const double scs[3] = {sc0, sc1, sc2};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double rtr = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
          rtr += Rg[a * 3 + k] * (dS[a * 3] * Rg[k] + dS[a * 3 + 1] * Rg[3 + k] + dS[a * 3 + 2] * Rg[6 + k]);
        grads[(int64_t)(kScaleX + k) * n_pad_g + i] = (float)(2.0 * scs[k] * rtr * scs[k]);
      }
      // quat_rotation_jacobian (scene.cpp:56-88): d_q_k = sum_j <dRg, 2 U_j> (delta_jk - q_j q_k)/|q|
      const double q[4] = {w, x, y, zq};
      const double U[4][9] = {{0, -zq, y, zq, 0, -x, -y, x, 0},
                              {0, y, zq, y, -2 * x, -w, zq, w, -2 * x},
                              {-2 * y, x, w, x, 0, zq, -w, zq, -2 * y},
                              {-2 * zq, -w, x, w, -2 * zq, y, x, y, 0}};
      double dU[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < 9; ++e) s += dRg[e] * (2.0 * U[j][e]);
        dU[j] = s;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) s += dU[j] * ((((j == k) ? 1.0 : 0.0) - q[j] * q[k]) / qn);
        grads[(int64_t)(kQuatW + k) * n_pad_g + i] = (float)s;
      }
      // SH coefficients: d_sh[c][b] = d_colour_c Y_b(dir) for active bands of unclamped channels
      const int deg = sh_active < sh_cap ? sh_active : sh_cap;
      const int nb = (deg + 1) * (deg + 1);
      double Bv[kMaxShCoeffs];
      sh_basis_d(dir0, dir1, dir2, deg, Bv);
      for (int c = 0; c < 3; ++c) {
        const bool clamped = (clamp >> c) & 1u;
        for (int b = 0; b < bcap; ++b)
          grads[(int64_t)(kShBase + c * bcap + b) * n_pad_g + i] = (!clamped && b < nb) ? (float)(dcol[c] * Bv[b]) : 0.f;
      }
      const double o = 1.0 / (1.0 + exp(-(double)P[kOpacity * n_pad]));
      grads[(int64_t)kOpacity * n_pad_g + i] = (float)(acc[8] * o * (1.0 - o));
      grads[(int64_t)nplanes * n_pad_g + i] = (float)dmu2x;
      grads[(int64_t)(nplanes + 1) * n_pad_g + i] = (float)dmu2y;
    }
  }
  mbar_wait(&bar2, 0);  // no thread leaves before every bulk copy into this CTA's shared memory has landed
  // deterministic block reduction of the pose contributions
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double pcs[6] = {pc0, pc1, pc2, pc3, pc4, pc5};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double v = pcs[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_pose[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double t = 0.0;
    for (int w2 = 0; w2 < kGeomWarps; ++w2) t += s_pose[w2][threadIdx.x];
    pose_blocks[(int64_t)blockIdx.x * 6 + threadIdx.x] = t;
  }
}

// Fixed-order reduction of the per-block pose partials: each thread sums a
// strided subset in order, then a fixed binary tree in shared memory (same
// association every launch: deterministic), 6 components at once.
__global__ void __launch_bounds__(256) pose_reduce_kernel(const double* __restrict__ blocks, int64_t nb,
                                                          double* __restrict__ out) {
  __shared__ double s[6][256];
  double r[6];
  block_reduce_pose(blocks, nb, s, r);
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) out[k] = r[k];
}

int64_t bwd_geom_blocks(int64_t n) { return (n + kGeomBlock - 1) / kGeomBlock; }

// reduce = false: the pose 6-vector stays as per-block partials in
// f->pose_blocks (a session's pose_iter_kernel sums them itself).
int launch_backward_geom(cudaStream_t st, const gsb_cloud* cloud, gsb_frame* f, const RasterDev& rc, bool full,
                         float* grads, int64_t* launches, bool reduce) {
  const int64_t n = cloud->n;
  EntryCut cutd;
  cutd.tile_cut = f->tile_cut.as<double2>();
  cutd.depth_g = f->depth_g.as<double>();
  cutd.aux_g = f->binning == kBinTileLocal ? f->aux_g.as<SplatAux>() : nullptr;
  cutd.rect_g = f->rect_g.as<uint2>();
  cutd.tiles_x = f->tiles_x;
  const int64_t nb = (n + kGeomBlock - 1) / kGeomBlock;
  if (nb > 0) {
    if (full)
      backward_geom_kernel<true, GSB_FULL_CHAIN_T><<<(unsigned)nb, kGeomBlock, 0, st>>>(
          cloud->params.as<float>(), n, cloud->n_pad, cloud->sh_degree, cloud->active_sh_degree, f->cam.as<CamDev>(),
          rc, f->cnt_g.as<uint32_t>(), f->off_g.as<uint32_t>(), f->colj.as<float>(), f->partials.as<float>(), f->k_cap, cutd, grads,
          f->pose_blocks.as<double>());
    else
      backward_geom_kernel<false, GSB_POSE_CHAIN_T><<<(unsigned)nb, kGeomBlock, 0, st>>>(
          cloud->params.as<float>(), n, cloud->n_pad, cloud->sh_degree, cloud->active_sh_degree, f->cam.as<CamDev>(),
          rc, f->cnt_g.as<uint32_t>(), f->off_g.as<uint32_t>(), f->colj.as<float>(), f->partials.as<float>(), f->k_cap, cutd, nullptr,
          f->pose_blocks.as<double>());
  }
  if (reduce) pose_reduce_kernel<<<1, 256, 0, st>>>(f->pose_blocks.as<double>(), nb, f->d_pose.as<double>());
  *launches += (nb > 0 ? 1 : 0) + (reduce ? 1 : 0);
  GSB_CHECK_LAUNCH("backward_geom_kernel");
  return GSB_OK;
}

}  // namespace gsb
