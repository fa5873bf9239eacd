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
// colour chain with clamp mask (496-513, sh.cpp:42-64), parameter grads
// (516-521) and the pose tangent: v = d_mu_cam + R_c d_to_gaussian,
// w = mu_cam x d_mu_cam + sum_k <d_R_c, [e_k]x R_c> (523-532,
// lie.cpp:173-181). Geometry is recomputed in FP64 from the FP32 parameters.
//
// One thread per Gaussian in index order: parameter planes are read and
// gradient planes written fully coalesced; each visible Gaussian reads its
// partials contiguously from its rank-major slot range.
#include "gsb_internal.cuh"

namespace gsb {

__constant__ double kBC1 = 0.4886025119029199;
__constant__ double kBC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                               0.5462742152960396};
__constant__ double kBC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                               -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

// sh.cpp:18-64: basis values and gradients w.r.t. the unit direction.
__device__ void sh_basis_and_grad(double x, double y, double z, int degree, double* B, double (*G)[3]) {
  B[0] = 0.28209479177387814;
  G[0][0] = G[0][1] = G[0][2] = 0.0;
  if (degree < 1) return;
  B[1] = -kBC1 * y; B[2] = kBC1 * z; B[3] = -kBC1 * x;
  G[1][0] = 0; G[1][1] = -kBC1; G[1][2] = 0;
  G[2][0] = 0; G[2][1] = 0; G[2][2] = kBC1;
  G[3][0] = -kBC1; G[3][1] = 0; G[3][2] = 0;
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  B[4] = kBC2[0] * x * y; B[5] = kBC2[1] * y * z; B[6] = kBC2[2] * (2.0 * zz - xx - yy);
  B[7] = kBC2[3] * x * z; B[8] = kBC2[4] * (xx - yy);
  G[4][0] = kBC2[0] * y; G[4][1] = kBC2[0] * x; G[4][2] = 0;
  G[5][0] = 0; G[5][1] = kBC2[1] * z; G[5][2] = kBC2[1] * y;
  G[6][0] = kBC2[2] * (-2.0 * x); G[6][1] = kBC2[2] * (-2.0 * y); G[6][2] = kBC2[2] * (4.0 * z);
  G[7][0] = kBC2[3] * z; G[7][1] = 0; G[7][2] = kBC2[3] * x;
  G[8][0] = kBC2[4] * (2.0 * x); G[8][1] = kBC2[4] * (-2.0 * y); G[8][2] = 0;
  if (degree < 3) return;
  B[9] = kBC3[0] * y * (3.0 * xx - yy); B[10] = kBC3[1] * x * y * z;
  B[11] = kBC3[2] * y * (4.0 * zz - xx - yy); B[12] = kBC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  B[13] = kBC3[4] * x * (4.0 * zz - xx - yy); B[14] = kBC3[5] * z * (xx - yy);
  B[15] = kBC3[6] * x * (xx - 3.0 * yy);
  G[9][0] = kBC3[0] * (6.0 * x * y); G[9][1] = kBC3[0] * (3.0 * xx - 3.0 * yy); G[9][2] = 0;
  G[10][0] = kBC3[1] * (y * z); G[10][1] = kBC3[1] * (x * z); G[10][2] = kBC3[1] * (x * y);
  G[11][0] = kBC3[2] * (-2.0 * x * y); G[11][1] = kBC3[2] * (4.0 * zz - xx - 3.0 * yy); G[11][2] = kBC3[2] * (8.0 * y * z);
  G[12][0] = kBC3[3] * (-6.0 * x * z); G[12][1] = kBC3[3] * (-6.0 * y * z); G[12][2] = kBC3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
  G[13][0] = kBC3[4] * (4.0 * zz - 3.0 * xx - yy); G[13][1] = kBC3[4] * (-2.0 * x * y); G[13][2] = kBC3[4] * (8.0 * x * z);
  G[14][0] = kBC3[5] * (2.0 * x * z); G[14][1] = kBC3[5] * (-2.0 * y * z); G[14][2] = kBC3[5] * (xx - yy);
  G[15][0] = kBC3[6] * (3.0 * xx - 3.0 * yy); G[15][1] = kBC3[6] * (-6.0 * x * y); G[15][2] = 0;
}

template <bool kFull>
__global__ void __launch_bounds__(256) backward_geom_kernel(
    const float* __restrict__ params, int64_t n, int64_t n_pad, int sh_cap, int sh_active,
    const CamDev* __restrict__ cam_p, RasterDev rc, const uint32_t* __restrict__ cnt_g,
    const int32_t* __restrict__ rank_of_g, const SplatRec* __restrict__ rec, const SplatAux* __restrict__ aux,
    const float* __restrict__ partials, float* __restrict__ grads, double* __restrict__ pose_blocks) {
  __shared__ CamDev cam;
  __shared__ double s_pose[8][6];
  if (threadIdx.x == 0) cam = *cam_p;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nplanes = kShBase + 3 * (sh_cap + 1) * (sh_cap + 1);
  const int bcap = (sh_cap + 1) * (sh_cap + 1);
  double pc[6] = {0, 0, 0, 0, 0, 0};
  const uint32_t cnt = i < n ? cnt_g[i] : 0u;
  if (i < n && cnt == 0u && kFull) {
    for (int p = 0; p < nplanes + 2; ++p) grads[(int64_t)p * n_pad + i] = 0.f;
  }
  if (i < n && cnt > 0u) {
    const int32_t r = rank_of_g[i];
    const SplatAux A = aux[r];
    const SplatRec S = rec[r];
    // phase 2: ordered sum of this splat's entry partials (tile order)
    double acc[kPartial];
#pragma unroll
    for (int c = 0; c < kPartial; ++c) acc[c] = 0.0;
    const float* pp = partials + (int64_t)A.off * kPartial;
    for (uint32_t j = 0; j < cnt; ++j) {
#pragma unroll
      for (int c = 0; c < kPartial; ++c) acc[c] += (double)pp[j * kPartial + c];
    }
    const double dmu2x = acc[0], dmu2y = acc[1];
    const double D00 = acc[2], D01 = acc[3], D11 = acc[4];
    const double dcol[3] = {acc[5], acc[6], acc[7]};
    const double dop = acc[8];
    const float* P = params + i;
    const double mean[3] = {P[kMeanX * n_pad], P[kMeanY * n_pad], P[kMeanZ * n_pad]};
    const double* Rc = cam.R;
    double mc[3];
    for (int a = 0; a < 3; ++a) mc[a] = Rc[a * 3] * mean[0] + Rc[a * 3 + 1] * mean[1] + Rc[a * 3 + 2] * mean[2] + cam.t[a];
    const double z = mc[2];
    const double iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
    const double fx = cam.fx, fy = cam.fy;
    const double J[6] = {fx * iz, 0.0, -fx * mc[0] * iz2, 0.0, fy * iz, -fy * mc[1] * iz2};
    double m[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) m[a * 3 + b] = J[a * 3] * Rc[b] + J[a * 3 + 1] * Rc[3 + b] + J[a * 3 + 2] * Rc[6 + b];
    const double sc[3] = {exp((double)P[kScaleX * n_pad]), exp((double)P[kScaleY * n_pad]), exp((double)P[kScaleZ * n_pad])};
    const double qr[4] = {P[kQuatW * n_pad], P[kQuatX * n_pad], P[kQuatY * n_pad], P[kQuatZ * n_pad]};
    const double qn = sqrt(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
    const double w = qr[0] / qn, x = qr[1] / qn, y = qr[2] / qn, zq = qr[3] / qn;
    double Rg[9] = {1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y),
                    2 * (x * y + w * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x),
                    2 * (x * zq - w * y), 2 * (y * zq + w * x), 1 - 2 * (x * x + y * y)};
    double Sg[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        Sg[a * 3 + b] = Rg[a * 3] * sc[0] * Rg[b * 3] * sc[0] + Rg[a * 3 + 1] * sc[1] * Rg[b * 3 + 1] * sc[1] +
                        Rg[a * 3 + 2] * sc[2] * Rg[b * 3 + 2] * sc[2];
    // conic from the FP64 cov2d (same expressions as the forward)
    double ms[6], cov[4];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) ms[a * 3 + b] = m[a * 3] * Sg[b] + m[a * 3 + 1] * Sg[3 + b] + m[a * 3 + 2] * Sg[6 + b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) cov[a * 2 + b] = ms[a * 3] * m[b * 3] + ms[a * 3 + 1] * m[b * 3 + 1] + ms[a * 3 + 2] * m[b * 3 + 2];
    cov[0] += rc.dilation;
    cov[3] += rc.dilation;
    const double det = cov[0] * cov[3] - cov[1] * cov[2];
    const double C[4] = {cov[3] / det, -cov[1] / det, -cov[2] / det, cov[0] / det};
    // d_cov2d = -(C D C), D symmetric (D01 = D10)
    const double D[4] = {D00, D01, D01, D11};
    double CD[4], dcov[4];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) CD[a * 2 + b] = C[a * 2] * D[b] + C[a * 2 + 1] * D[2 + b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) dcov[a * 2 + b] = -(CD[a * 2] * C[b] + CD[a * 2 + 1] * C[2 + b]);
    // d_m = 2 dcov m Sigma ; d_Sigma = m^T dcov m
    double t23[6], dm[6], dS[9];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) t23[a * 3 + b] = 2.0 * (dcov[a * 2] * m[b] + dcov[a * 2 + 1] * m[3 + b]);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) dm[a * 3 + b] = t23[a * 3] * Sg[b] + t23[a * 3 + 1] * Sg[3 + b] + t23[a * 3 + 2] * Sg[6 + b];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        dS[a * 3 + b] = (m[a] * dcov[0] + m[3 + a] * dcov[2]) * m[b] + (m[a] * dcov[1] + m[3 + a] * dcov[3]) * m[3 + b];
    // d_jac = dm R^T ; d_R_c = J^T dm
    double djac[6], dRc[9];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) djac[a * 3 + b] = dm[a * 3] * Rc[b * 3] + dm[a * 3 + 1] * Rc[b * 3 + 1] + dm[a * 3 + 2] * Rc[b * 3 + 2];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) dRc[a * 3 + b] = J[a] * dm[b] + J[3 + a] * dm[3 + b];
    double dmc[3];
    dmc[0] = djac[2] * (-fx * iz2) + dmu2x * fx * iz;
    dmc[1] = djac[5] * (-fy * iz2) + dmu2y * fy * iz;
    dmc[2] = djac[0] * (-fx * iz2) + djac[4] * (-fy * iz2) + djac[2] * (2.0 * fx * mc[0] * iz3) +
             djac[5] * (2.0 * fy * mc[1] * iz3) - dmu2x * fx * mc[0] * iz2 - dmu2y * fy * mc[1] * iz2;
    // SH colour chain
    double tg[3] = {mean[0] - cam.center[0], mean[1] - cam.center[1], mean[2] - cam.center[2]};
    const double dist = sqrt(tg[0] * tg[0] + tg[1] * tg[1] + tg[2] * tg[2]);
    const double dir[3] = {tg[0] / dist, tg[1] / dist, tg[2] / dist};
    const int deg = sh_active < sh_cap ? sh_active : sh_cap;
    const int nb = (deg + 1) * (deg + 1);
    double Bv[kMaxShCoeffs], Gv[kMaxShCoeffs][3];
    sh_basis_and_grad(dir[0], dir[1], dir[2], deg, Bv, Gv);
    double ddir[3] = {0, 0, 0};
    for (int c = 0; c < 3; ++c) {
      const bool clamped = (S.clamp_bits >> c) & 1u;
      for (int b = 0; b < bcap; ++b) {
        double g = 0.0;
        if (!clamped && b < nb) {
          g = dcol[c] * Bv[b];
          const double f = dcol[c] * (double)P[(kShBase + c * bcap + b) * n_pad];
          ddir[0] += f * Gv[b][0];
          ddir[1] += f * Gv[b][1];
          ddir[2] += f * Gv[b][2];
        }
        if (kFull) grads[(int64_t)(kShBase + c * bcap + b) * n_pad + i] = (float)g;
      }
    }
    const double pd = dir[0] * ddir[0] + dir[1] * ddir[1] + dir[2] * ddir[2];
    const double dtg[3] = {(ddir[0] - dir[0] * pd) / dist, (ddir[1] - dir[1] * pd) / dist, (ddir[2] - dir[2] * pd) / dist};
    if (kFull) {
      // d_means = R_c^T dmc + dtg
      for (int a = 0; a < 3; ++a)
        grads[(int64_t)(kMeanX + a) * n_pad + i] = (float)(Rc[a] * dmc[0] + Rc[3 + a] * dmc[1] + Rc[6 + a] * dmc[2] + dtg[a]);
      // Sigma = R D R^T: d_Rg = 2 dS Rg diag(s^2); rt = Rg^T dS Rg
      double dRg[9], RtdS[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          dRg[a * 3 + b] = 2.0 * (dS[a * 3] * Rg[b] + dS[a * 3 + 1] * Rg[3 + b] + dS[a * 3 + 2] * Rg[6 + b]) * (sc[b] * sc[b]);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) RtdS[a * 3 + b] = Rg[a] * dS[b] + Rg[3 + a] * dS[3 + b] + Rg[6 + a] * dS[6 + b];
      for (int k = 0; k < 3; ++k) {
        const double rtr = RtdS[k * 3] * Rg[k] + RtdS[k * 3 + 1] * Rg[3 + k] + RtdS[k * 3 + 2] * Rg[6 + k];
        grads[(int64_t)(kScaleX + k) * n_pad + i] = (float)(2.0 * sc[k] * rtr * sc[k]);
      }
      // quat_rotation_jacobian (scene.cpp:56-88)
      const double q[4] = {w, x, y, zq};
      const double U[4][9] = {{0, -zq, y, zq, 0, -x, -y, x, 0},
                              {0, y, zq, y, -2 * x, -w, zq, w, -2 * x},
                              {-2 * y, x, w, x, 0, zq, -w, zq, -2 * y},
                              {-2 * zq, -w, x, w, -2 * zq, y, x, y, 0}};
      double dU[4];  // <dRg, 2 U_j>
      for (int j = 0; j < 4; ++j) {
        double s = 0.0;
        for (int e = 0; e < 9; ++e) s += dRg[e] * (2.0 * U[j][e]);
        dU[j] = s;
      }
      for (int k = 0; k < 4; ++k) {
        double s = 0.0;
        for (int j = 0; j < 4; ++j) s += dU[j] * ((((j == k) ? 1.0 : 0.0) - q[j] * q[k]) / qn);
        grads[(int64_t)(kQuatW + k) * n_pad + i] = (float)s;
      }
      const double o = S.opacity;
      grads[(int64_t)kOpacity * n_pad + i] = (float)(dop * o * (1.0 - o));
      grads[(int64_t)nplanes * n_pad + i] = (float)dmu2x;
      grads[(int64_t)(nplanes + 1) * n_pad + i] = (float)dmu2y;
    }
    // pose tangent (rasterizer.cpp:523-533)
    for (int a = 0; a < 3; ++a) pc[a] = dmc[a] + (Rc[a * 3] * dtg[0] + Rc[a * 3 + 1] * dtg[1] + Rc[a * 3 + 2] * dtg[2]);
    pc[3] = mc[1] * dmc[2] - mc[2] * dmc[1];
    pc[4] = mc[2] * dmc[0] - mc[0] * dmc[2];
    pc[5] = mc[0] * dmc[1] - mc[1] * dmc[0];
    double f0 = 0, f1 = 0, f2 = 0;  // <dRc, [e_k]x Rc>
    for (int j = 0; j < 3; ++j) {
      f0 += -dRc[3 + j] * Rc[6 + j] + dRc[6 + j] * Rc[3 + j];
      f1 += dRc[j] * Rc[6 + j] - dRc[6 + j] * Rc[j];
      f2 += -dRc[j] * Rc[3 + j] + dRc[3 + j] * Rc[j];
    }
    pc[3] += f0;
    pc[4] += f1;
    pc[5] += f2;
  }
  // deterministic block reduction of the pose contributions
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double v = pc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_pose[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double t = 0.0;
    for (int w2 = 0; w2 < 8; ++w2) t += s_pose[w2][threadIdx.x];
    pose_blocks[(int64_t)blockIdx.x * 6 + threadIdx.x] = t;
  }
}

__global__ void pose_reduce_kernel(const double* __restrict__ blocks, int64_t nb, double* __restrict__ out) {
  __shared__ double s[6][256];
  for (int k = 0; k < 6; ++k) {
    double t = 0.0;
    for (int64_t b = threadIdx.x; b < nb; b += 256) t += blocks[b * 6 + k];
    s[k][threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double t = 0.0;
    for (int j = 0; j < 256; ++j) t += s[threadIdx.x][j];
    out[threadIdx.x] = t;
  }
}

int launch_backward_geom(cudaStream_t st, const gsb_cloud* cloud, gsb_frame* f, const RasterDev& rc, bool full,
                         float* grads, int64_t* launches) {
  const int64_t n = cloud->n;
  const int64_t nb = (n + 255) / 256;
  if (nb > 0) {
    if (full)
      backward_geom_kernel<true><<<(unsigned)nb, 256, 0, st>>>(
          cloud->params.as<float>(), n, cloud->n_pad, cloud->sh_degree, cloud->active_sh_degree, f->cam.as<CamDev>(),
          rc, f->cnt_g.as<uint32_t>(), f->rank_of_g.as<int32_t>(), f->rec.as<SplatRec>(), f->aux.as<SplatAux>(),
          f->partials.as<float>(), grads, f->pose_blocks.as<double>());
    else
      backward_geom_kernel<false><<<(unsigned)nb, 256, 0, st>>>(
          cloud->params.as<float>(), n, cloud->n_pad, cloud->sh_degree, cloud->active_sh_degree, f->cam.as<CamDev>(),
          rc, f->cnt_g.as<uint32_t>(), f->rank_of_g.as<int32_t>(), f->rec.as<SplatRec>(), f->aux.as<SplatAux>(),
          f->partials.as<float>(), nullptr, f->pose_blocks.as<double>());
  }
  pose_reduce_kernel<<<1, 256, 0, st>>>(f->pose_blocks.as<double>(), nb, f->d_pose.as<double>());
  *launches += nb > 0 ? 2 : 1;
  GSB_CHECK_LAUNCH("backward_geom_kernel");
  return GSB_OK;
}

}  // namespace gsb
