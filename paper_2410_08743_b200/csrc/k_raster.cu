// k_raster.cu — K3 front-to-back compositing and K4a back-to-front backward
// raster. One CTA per 16x16 tile, one thread per pixel (warp w owns tile
// rows 2w, 2w+1); splat records are staged through shared memory in batches
// of 256 (one record per thread per batch, gathered by rank), so each record
// is read from L2/HBM once per tile.
//
// K3 restates render's compositing loop (rasterizer.cpp:234-279):
// integer pixel centres (245), processed counter set before the cutoff test
// (251), hard g > cutoff^2 skip (254), alpha = min(clamp, o e^{-g/2}) (255),
// break after including the splat once T < early_termination (258), colour
// clamp at 1 with overflow bits (262-268).
//
// K4a restates phase 1 of render_backward (rasterizer.cpp:354-405): per
// pixel back-to-front replay from contrib_count-1 with t_before = T/(1-a),
// clamped channels zeroed, alpha-chain gradients only when a_raw < clamp.
// The per-(pixel, splat) partials are reduced over the tile's 256 pixels in
// a fixed order (warp recursive-halving reduce-scatter, then warps 0..7) and
// written — zero when untouched — to the entry's slot in the rank-major
// (pre-sort) stream, so K4b reads each splat's partials contiguously and in
// tile order (phase 2's per-splat order, rasterizer.cpp:410-418). No
// atomics: deterministic.
//
// Both kernels skip a staged splat warp-uniformly when its cutoff ellipse
// (|dy| <= cutoff * sqrt(Sigma_yy), Sigma = conic^-1, with a safety margin)
// misses the warp's two pixel rows: every pixel of such a warp would fail the
// g <= cutoff^2 test, so the result is unchanged.
#include "gsb_internal.cuh"

namespace gsb {

constexpr int kBatch = 256;
constexpr int kWarps = kTilePix / 32;
constexpr unsigned kFull = 0xffffffffu;

struct Staged {
  float4 geo;  // tile-local mean x, y; conic a, b
  float4 app;  // conic c, opacity, colour r, g
  float4 ext;  // colour b, ellipse half-height (with margin), -, -
};

__device__ __forceinline__ void stage_splat(const SplatRec& R, double ox, double oy, float cutoff2, float4* geo,
                                            float4* app, float4* ext) {
  const float a = R.conic_a, b = R.conic_b, c = R.conic_c;
  const float det = a * c - b * b;
  const float half_h = sqrtf(cutoff2 * a / det) * 1.001f + 1e-3f;  // |dy| bound of g <= cutoff2
  *geo = make_float4((float)(R.mu_x - ox), (float)(R.mu_y - oy), a, b);
  *app = make_float4(c, R.opacity, R.col_r, R.col_g);
  *ext = make_float4(R.col_b, half_h, 0.f, 0.f);
}

// Mahalanobis power g = d^T conic d. Forward and backward must take the
// identical cutoff / alpha decisions, so both call exactly this.
__device__ __forceinline__ float splat_power(float ca, float cb, float cc, float dx, float dy) {
  return fmaf(ca * dx, dx, fmaf(cc * dy, dy, 2.0f * cb * dx * dy));
}

// Warp-uniform: does the splat's ellipse reach rows [row0, row0+1]?
__device__ __forceinline__ bool rows_hit(float my, float half_h, float row_c) {
  return fabsf(row_c - my) <= half_h + 0.5f;
}

__global__ void __launch_bounds__(kTilePix) composite_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g, float bg_b, int64_t npix,
    float* __restrict__ image, float* __restrict__ final_t, uint32_t* __restrict__ pixstate) {
  __shared__ float4 s_geo[kBatch], s_app[kBatch], s_ext[kBatch];
  __shared__ int s_w, s_h, s_tx;
  if (threadIdx.x == 0) {
    s_w = cam_p->width;
    s_h = cam_p->height;
    s_tx = cam_p->tiles_x;
  }
  __syncthreads();
  const int W = s_w, H = s_h;
  const int tile = blockIdx.x;
  const int tx = tile % s_tx, ty = tile / s_tx;
  const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x / kTile;
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const bool inside = x < W && y < H;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const float px = (float)lx, py = (float)ly;
  const float row_c = (float)(2 * (threadIdx.x >> 5)) + 0.5f;
  const uint2 range = ranges[tile];
  float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
  uint32_t processed = 0;
  bool done = !inside;
  for (uint32_t base = range.x; base < range.y; base += kBatch) {
    if (__syncthreads_count(done) == kTilePix) break;
    const uint32_t e = base + threadIdx.x;
    if (e < range.y) stage_splat(rec[ranks[e]], ox, oy, rc.cutoff2_f, &s_geo[threadIdx.x], &s_app[threadIdx.x], &s_ext[threadIdx.x]);
    __syncthreads();
    const int cnt = min((uint32_t)kBatch, range.y - base);
    if (!__all_sync(kFull, done)) {
      int k = 0;
      for (; k < cnt; ++k) {
        const float4 ge = s_geo[k];
        const float4 ex = s_ext[k];
        if (!rows_hit(ge.y, ex.y, row_c)) continue;  // warp-uniform
        if (done) continue;
        const float dx = px - ge.x, dy = py - ge.y;
        const float4 ap = s_app[k];
        const float g = splat_power(ge.z, ge.w, ap.x, dx, dy);
        if (g > rc.cutoff2_f) continue;
        const float alpha = fminf(rc.alpha_clamp_f, ap.y * __expf(-0.5f * g));
        const float w = alpha * T;
        cr = fmaf(ap.z, w, cr);
        cg = fmaf(ap.w, w, cg);
        cb = fmaf(ex.x, w, cb);
        T *= (1.0f - alpha);
        if (T < rc.early_term_f) {
          done = true;
          processed = base - range.x + (uint32_t)k + 1u;
        }
      }
      if (!done) processed = base - range.x + (uint32_t)cnt;
    }
  }
  if (!inside) return;
  cr = fmaf(bg_r, T, cr);
  cg = fmaf(bg_g, T, cg);
  cb = fmaf(bg_b, T, cb);
  uint32_t of = 0;
  if (cr > 1.0f) { cr = 1.0f; of |= 1u; }
  if (cg > 1.0f) { cg = 1.0f; of |= 2u; }
  if (cb > 1.0f) { cb = 1.0f; of |= 4u; }
  const int64_t p = (int64_t)y * W + x;
  image[p] = cr;
  image[npix + p] = cg;
  image[2 * npix + p] = cb;
  final_t[p] = T;
  pixstate[p] = processed | (of << 29);
}

// Recursive-halving reduce-scatter of 9 values over a warp (12 shuffles
// instead of 45): returns the component index this lane ends up owning (or
// -1) and its warp total in *out. Fixed order, deterministic.
__device__ __forceinline__ int warp_reduce9(const float v[kPartial], float* out) {
  const int lane = threadIdx.x & 31;
  const bool h1 = lane & 16, h2 = lane & 8, h3 = lane & 4, h4 = lane & 2;
  float w[6];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const float lo = v[i], hi = (i < 4) ? v[5 + i] : 0.f;
    const float send = h1 ? lo : hi, keep = h1 ? hi : lo;
    w[i] = keep + __shfl_xor_sync(kFull, send, 16);
  }
  w[5] = 0.f;
  float x[4];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float lo = w[i], hi = w[3 + i];
    const float send = h2 ? lo : hi, keep = h2 ? hi : lo;
    x[i] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  x[3] = 0.f;
  float y[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float lo = x[i], hi = x[2 + i];
    const float send = h3 ? lo : hi, keep = h3 ? hi : lo;
    y[i] = keep + __shfl_xor_sync(kFull, send, 4);
  }
  float z;
  {
    const float send = h4 ? y[0] : y[1], keep = h4 ? y[1] : y[0];
    z = keep + __shfl_xor_sync(kFull, send, 2);
  }
  z += __shfl_xor_sync(kFull, z, 1);
  const int xi = (h3 ? 2 : 0) + (h4 ? 1 : 0);
  const int wi = (h2 ? 3 : 0) + xi;
  const int vi = (h1 ? 5 : 0) + wi;
  if ((lane & 1) || xi >= 3 || wi >= 5 || vi >= kPartial) return -1;
  *out = z;
  return vi;
}

__global__ void __launch_bounds__(kTilePix) backward_raster_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const SplatAux* __restrict__ aux, const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g,
    float bg_b, int64_t npix, const float* __restrict__ d_image, const float* __restrict__ final_t,
    const uint32_t* __restrict__ pixstate, float* __restrict__ partials, uint32_t k_cap) {
  __shared__ float4 s_geo[kBatch], s_app[kBatch], s_ext[kBatch];
  __shared__ uint32_t s_slot[kBatch];
  __shared__ float s_red[kWarps][32][kPartial];  // [warp][entry in sub-batch][component]
  __shared__ int s_w, s_h, s_tx;
  __shared__ uint32_t s_maxc[kWarps];
  if (threadIdx.x == 0) {
    s_w = cam_p->width;
    s_h = cam_p->height;
    s_tx = cam_p->tiles_x;
  }
  for (int i = threadIdx.x; i < kWarps * 32 * kPartial; i += kTilePix) (&s_red[0][0][0])[i] = 0.f;
  __syncthreads();
  const int W = s_w, H = s_h;
  const int tile = blockIdx.x;
  const int tx = tile % s_tx, ty = tile / s_tx;
  const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x / kTile;
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool inside = x < W && y < H;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const float px = (float)lx, py = (float)ly;
  const float row_c = (float)(2 * warp) + 0.5f;
  const uint2 range = ranges[tile];

  float dr = 0.f, dg = 0.f, db = 0.f, T = 0.f;
  uint32_t contrib = 0;
  if (inside) {
    const int64_t p = (int64_t)y * W + x;
    const uint32_t ps = pixstate[p];
    const uint32_t of = ps >> 29;
    dr = (of & 1u) ? 0.f : d_image[p];
    dg = (of & 2u) ? 0.f : d_image[npix + p];
    db = (of & 4u) ? 0.f : d_image[2 * npix + p];
    T = final_t[p];
    contrib = ps & 0x1fffffffu;
    if (dr == 0.f && dg == 0.f && db == 0.f) contrib = 0;  // rasterizer.cpp:372
  }
  float br = bg_r * T, bgg = bg_g * T, bb = bg_b * T;
  const uint32_t wmax = __reduce_max_sync(kFull, contrib);
  if (lane == 0) s_maxc[warp] = wmax;
  __syncthreads();
  uint32_t maxc = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) maxc = max(maxc, s_maxc[w]);
  const uint32_t len = range.y - range.x;

  // Batches walk the list from the back; entries past maxc only get zeros.
  const uint32_t nbatch = (len + kBatch - 1) / kBatch;
  for (int bi = (int)nbatch - 1; bi >= 0; --bi) {
    const uint32_t b0 = (uint32_t)bi * kBatch;  // list-local start
    const uint32_t cnt = min((uint32_t)kBatch, len - b0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const uint32_t e = range.x + b0 + threadIdx.x;
      const uint32_t r = ranks[e];
      const SplatAux A = aux[r];
      const uint32_t tx0 = A.tx0_ty0 & 0xffffu, ty0 = A.tx0_ty0 >> 16, nx = A.nx_ny & 0xffffu;
      s_slot[threadIdx.x] = A.off + ((uint32_t)ty - ty0) * nx + ((uint32_t)tx - tx0);
      if (b0 + threadIdx.x < maxc)
        stage_splat(rec[r], ox, oy, rc.cutoff2_f, &s_geo[threadIdx.x], &s_app[threadIdx.x], &s_ext[threadIdx.x]);
    }
    __syncthreads();
    // Sub-batches of 32 entries, back to front; each reduced into s_red, then
    // flushed (fixed warp order) to the entries' global slots.
    for (int sb = (int)((cnt + 31) / 32) - 1; sb >= 0; --sb) {
      const int k0 = sb * 32;
      const int k1 = min((int)cnt, k0 + 32);
      if (b0 + (uint32_t)k0 < wmax) {  // this warp has work in the sub-batch
        for (int k = k1 - 1; k >= k0; --k) {
          const uint32_t j = b0 + (uint32_t)k;
          if (j >= wmax) continue;  // warp-uniform
          const float4 ge = s_geo[k];
          const float4 ex = s_ext[k];
          if (!rows_hit(ge.y, ex.y, row_c)) continue;  // warp-uniform
          float v[kPartial];
#pragma unroll
          for (int c = 0; c < kPartial; ++c) v[c] = 0.f;
          bool hit = false;
          if (j < contrib) {
            const float dx = px - ge.x, dy = py - ge.y;
            const float4 ap = s_app[k];
            const float g = splat_power(ge.z, ge.w, ap.x, dx, dy);
            if (!(g > rc.cutoff2_f)) {
              hit = true;
              const float G = __expf(-0.5f * g);
              const float araw = ap.y * G;
              const float alpha = fminf(rc.alpha_clamp_f, araw);
              const float inv = 1.0f / (1.0f - alpha);
              const float tb = T * inv;
              const float wgt = alpha * tb;
              v[5] = wgt * dr;
              v[6] = wgt * dg;
              v[7] = wgt * db;
              const float dal =
                  dr * (ap.z * tb - br * inv) + dg * (ap.w * tb - bgg * inv) + db * (ex.x * tb - bb * inv);
              if (araw < rc.alpha_clamp_f) {
                const float cx_ = ge.z * dx + ge.w * dy, cy_ = ge.w * dx + ap.x * dy;
                v[8] = dal * G;
                const float dgg = dal * (-0.5f * araw);
                v[0] = -2.0f * dgg * cx_;
                v[1] = -2.0f * dgg * cy_;
                v[2] = dgg * dx * dx;
                v[3] = dgg * dx * dy;
                v[4] = dgg * dy * dy;
              }
              T = tb;
              br = fmaf(ap.z, wgt, br);
              bgg = fmaf(ap.w, wgt, bgg);
              bb = fmaf(ex.x, wgt, bb);
            }
          }
          if (__any_sync(kFull, hit)) {
            float tot;
            const int vi = warp_reduce9(v, &tot);
            if (vi >= 0) s_red[warp][k - k0][vi] = tot;
          }
        }
      }
      __syncthreads();
      // flush: 32 entries x 9 components, summed over warps 0..7 in order
      for (int idx = threadIdx.x; idx < 32 * kPartial; idx += kTilePix) {
        const int kk = idx / kPartial, c = idx - kk * kPartial;
        const int k = k0 + kk;
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          acc += s_red[w][kk][c];
          s_red[w][kk][c] = 0.f;
        }
        if (k < k1 && s_slot[k] < k_cap) partials[(int64_t)s_slot[k] * kPartial + c] = acc;
      }
      __syncthreads();
    }
  }
}

int launch_composite(cudaStream_t st, gsb_frame* f, const RasterDev& rc) {
  const int n_tiles = f->tiles_x * f->tiles_y;
  const int64_t npix = (int64_t)f->width * f->height;
  if (n_tiles > 0)
    composite_kernel<<<n_tiles, kTilePix, 0, st>>>(
        f->ranges.as<uint2>(), f->eval_[f->sorted_sel].as<uint32_t>(), f->rec.as<SplatRec>(), f->cam.as<CamDev>(), rc,
        (float)f->background[0], (float)f->background[1], (float)f->background[2], npix, f->image.as<float>(),
        f->final_t.as<float>(), f->pixstate.as<uint32_t>());
  GSB_CHECK_LAUNCH("composite_kernel");
  return GSB_OK;
}

int launch_backward_raster(cudaStream_t st, gsb_frame* f, const RasterDev& rc) {
  const int n_tiles = f->tiles_x * f->tiles_y;
  const int64_t npix = (int64_t)f->width * f->height;
  if (n_tiles > 0)
    backward_raster_kernel<<<n_tiles, kTilePix, 0, st>>>(
        f->ranges.as<uint2>(), f->eval_[f->sorted_sel].as<uint32_t>(), f->rec.as<SplatRec>(), f->aux.as<SplatAux>(),
        f->cam.as<CamDev>(), rc, (float)f->background[0], (float)f->background[1], (float)f->background[2], npix,
        f->d_image.as<float>(), f->final_t.as<float>(), f->pixstate.as<uint32_t>(), f->partials.as<float>(),
        (uint32_t)f->k_cap);
  GSB_CHECK_LAUNCH("backward_raster_kernel");
  return GSB_OK;
}

}  // namespace gsb
