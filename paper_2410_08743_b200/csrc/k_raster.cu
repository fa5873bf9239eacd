// k_raster.cu — K3 front-to-back compositing and K4a back-to-front backward
// raster. One CTA per 16x16 tile, one thread per pixel; splat records are
// staged through shared memory in batches of 256 (one record per thread per
// batch, gathered by rank), so each record is read from L2/HBM once per tile.
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
// a fixed order (warp butterfly, then warps 0..7) and written — zero when
// untouched — to the entry's slot in the rank-major (pre-sort) stream, so
// K4b reads each splat's partials contiguously and in tile order (phase 2's
// per-splat order, rasterizer.cpp:410-418). No atomics: deterministic.
#include "gsb_internal.cuh"

namespace gsb {

constexpr int kBatch = 256;

struct __align__(16) SmemSplat {
  float mx, my, ca, cb;   // tile-local mean, conic a, b
  float cc, op, r, g;     // conic c, opacity, colour r, g
  float b, pad0, pad1, pad2;
};

// Mahalanobis power g = d^T conic d. Forward and backward must take the
// identical cutoff / alpha decisions, so both call exactly this.
__device__ __forceinline__ float splat_power(const SmemSplat& q, float dx, float dy) {
  return fmaf(q.ca * dx, dx, fmaf(q.cc * dy, dy, 2.0f * q.cb * dx * dy));
}
__device__ __forceinline__ SmemSplat stage_splat(const SplatRec& R, double ox, double oy) {
  SmemSplat q;
  q.mx = (float)(R.mu_x - ox);
  q.my = (float)(R.mu_y - oy);
  q.ca = R.conic_a;
  q.cb = R.conic_b;
  q.cc = R.conic_c;
  q.op = R.opacity;
  q.r = R.col_r;
  q.g = R.col_g;
  q.b = R.col_b;
  q.pad0 = q.pad1 = q.pad2 = 0.f;
  return q;
}

__global__ void __launch_bounds__(kTilePix) composite_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g, float bg_b, int64_t npix,
    float* __restrict__ image, float* __restrict__ final_t, uint32_t* __restrict__ pixstate) {
  __shared__ SmemSplat s[kBatch];
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
  const uint2 range = ranges[tile];
  float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
  uint32_t processed = 0;
  bool done = !inside;
  for (uint32_t base = range.x; base < range.y; base += kBatch) {
    if (__syncthreads_count(done) == kTilePix) break;
    const uint32_t e = base + threadIdx.x;
    if (e < range.y) {
      s[threadIdx.x] = stage_splat(rec[ranks[e]], ox, oy);
    }
    __syncthreads();
    const int cnt = min((uint32_t)kBatch, range.y - base);
    if (!done) {
      int k = 0;
      for (; k < cnt; ++k) {
        const SmemSplat& q = s[k];
        const float dx = px - q.mx, dy = py - q.my;
        const float g = splat_power(q, dx, dy);
        if (g > rc.cutoff2_f) continue;
        const float alpha = fminf(rc.alpha_clamp_f, q.op * __expf(-0.5f * g));
        const float w = alpha * T;
        cr = fmaf(q.r, w, cr);
        cg = fmaf(q.g, w, cg);
        cb = fmaf(q.b, w, cb);
        T *= (1.0f - alpha);
        if (T < rc.early_term_f) {
          done = true;
          break;
        }
      }
      processed = base - range.x + (done ? (uint32_t)k + 1u : (uint32_t)cnt);
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

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kTilePix) backward_raster_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const SplatAux* __restrict__ aux, const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g,
    float bg_b, int64_t npix, const float* __restrict__ d_image, const float* __restrict__ final_t,
    const uint32_t* __restrict__ pixstate, float* __restrict__ partials) {
  constexpr int kWarps = kTilePix / 32;
  __shared__ SmemSplat s[kBatch];
  __shared__ uint32_t s_slot[kBatch];
  __shared__ float s_red[kWarps][kPartial][kBatch / 8 + 1];  // reduced per sub-batch of 32 entries
  __shared__ int s_w, s_h, s_tx;
  __shared__ uint32_t s_maxc[kWarps];
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool inside = x < W && y < H;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const float px = (float)lx, py = (float)ly;
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
  const uint32_t wmax = __reduce_max_sync(0xffffffffu, contrib);
  if (lane == 0) s_maxc[warp] = wmax;
  __syncthreads();
  uint32_t maxc = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) maxc = max(maxc, s_maxc[w]);
  const uint32_t len = range.y - range.x;

  // Batches walk the list from the back; entries past maxc only get zeros.
  const uint32_t nbatch = (len + kBatch - 1) / kBatch;
  for (int bi = (int)nbatch - 1; bi >= 0; --bi) {
    const uint32_t b0 = (uint32_t)bi * kBatch;                // list-local start
    const uint32_t cnt = min((uint32_t)kBatch, len - b0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const uint32_t e = range.x + b0 + threadIdx.x;
      const uint32_t r = ranks[e];
      const SplatAux A = aux[r];
      const uint32_t tx0 = A.tx0_ty0 & 0xffffu, ty0 = A.tx0_ty0 >> 16, nx = A.nx_ny & 0xffffu;
      s_slot[threadIdx.x] = A.off + ((uint32_t)ty - ty0) * nx + ((uint32_t)tx - tx0);
      if (b0 + threadIdx.x < maxc) {
        s[threadIdx.x] = stage_splat(rec[r], ox, oy);
      }
    }
    __syncthreads();
    const uint32_t active_cnt = b0 < maxc ? min(cnt, maxc - b0) : 0u;
    // Process entries in sub-batches of 32 (back to front), reducing each
    // sub-batch's partials into s_red, then flushing them to global.
    for (int sb = (int)((cnt + 31) / 32) - 1; sb >= 0; --sb) {
      const int k0 = sb * 32;
      const int k1 = min((int)cnt, k0 + 32);
      for (int k = k1 - 1; k >= k0; --k) {
        float v[kPartial];
#pragma unroll
        for (int c = 0; c < kPartial; ++c) v[c] = 0.f;
        bool hit = false;
        if ((uint32_t)k < active_cnt && b0 + (uint32_t)k < contrib) {
          const SmemSplat& q = s[k];
          const float dx = px - q.mx, dy = py - q.my;
          const float g = splat_power(q, dx, dy);
          if (!(g > rc.cutoff2_f)) {
            const float cx_ = q.ca * dx + q.cb * dy, cy_ = q.cb * dx + q.cc * dy;
            hit = true;
            const float G = __expf(-0.5f * g);
            const float araw = q.op * G;
            const float alpha = fminf(rc.alpha_clamp_f, araw);
            const float inv = 1.0f / (1.0f - alpha);
            const float tb = T * inv;
            const float wgt = alpha * tb;
            v[5] = wgt * dr;
            v[6] = wgt * dg;
            v[7] = wgt * db;
            const float dal = dr * (q.r * tb - br * inv) + dg * (q.g * tb - bgg * inv) + db * (q.b * tb - bb * inv);
            if (araw < rc.alpha_clamp_f) {
              v[8] = dal * G;
              const float dgg = dal * (-0.5f * araw);
              v[0] = -2.0f * dgg * cx_;
              v[1] = -2.0f * dgg * cy_;
              v[2] = dgg * dx * dx;
              v[3] = dgg * dx * dy;
              v[4] = dgg * dy * dy;
            }
            T = tb;
            br = fmaf(q.r, wgt, br);
            bgg = fmaf(q.g, wgt, bgg);
            bb = fmaf(q.b, wgt, bb);
          }
        }
        const int kk = k - k0;
        if (__any_sync(0xffffffffu, hit)) {
#pragma unroll
          for (int c = 0; c < kPartial; ++c) v[c] = warp_sum(v[c]);
          if (lane == 0) {
#pragma unroll
            for (int c = 0; c < kPartial; ++c) s_red[warp][c][kk] = v[c];
          }
        } else if (lane == 0) {
#pragma unroll
          for (int c = 0; c < kPartial; ++c) s_red[warp][c][kk] = 0.f;
        }
      }
      __syncthreads();
      // flush: thread t handles (entry kk = t / 9 ... ) -> 32 entries x 9 comps = 288 values
      for (int idx = threadIdx.x; idx < 32 * kPartial; idx += kTilePix) {
        const int kk = idx / kPartial, c = idx % kPartial;
        const int k = k0 + kk;
        if (k < k1) {
          float acc = 0.f;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) acc += s_red[w][c][kk];
          partials[(int64_t)s_slot[k] * kPartial + c] = acc;
        }
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
        f->d_image.as<float>(), f->final_t.as<float>(), f->pixstate.as<uint32_t>(), f->partials.as<float>());
  GSB_CHECK_LAUNCH("backward_raster_kernel");
  return GSB_OK;
}

}  // namespace gsb
