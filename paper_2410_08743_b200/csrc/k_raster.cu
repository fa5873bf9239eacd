// k_raster.cu — K3 front-to-back compositing and K4a back-to-front backward
// raster. One 128-thread CTA per 16x16 tile. The tile is cut into sixteen
// 4x4-pixel regions; each warp owns one 8x8 quadrant and runs it as four
// independent 8-lane sub-warps, one per region, every lane owning two
// vertically adjacent pixels.
//
// Splat records are staged through shared memory in batches of 128 (one
// record per thread, gathered by id), so each record is read from L2/HBM once
// per tile. Staging also computes a 16-bit mask of the regions the bounding
// box of the splat's cutoff ellipse touches; each warp then compacts the
// batch into four per-region lists (ballot + popc). In the inner loop the
// four sub-warps walk their own lists in lockstep, i.e. one warp instruction
// serves four different splats, and a splat costs a region nothing unless its
// footprint reaches it. For the ~2-5 px footprints of a 1M-Gaussian scene
// this culls ~2x more (pixel, splat) pairs than 8x8-quadrant lists at the
// same SIMT width.
//
// K3 restates render's compositing loop (rasterizer.cpp:234-279):
// integer pixel centres (245), processed counter set before the cutoff test
// (251), hard g > cutoff^2 skip (254), alpha = min(clamp, o e^{-g/2}) (255),
// break after including the splat once T < early_termination (258), colour
// clamp at 1 with overflow bits (262-268). Region culling is exact: every
// pixel outside the bounding box of {g <= cutoff^2} fails the test anyway.
//
// K4a restates phase 1 of render_backward (rasterizer.cpp:354-405): per
// pixel back-to-front replay from contrib_count-1 with t_before = T/(1-a),
// clamped channels zeroed, alpha-chain gradients only when a_raw < clamp.
// Each warp owns an 8x8 quadrant (two pixels per lane). Per-(pixel, splat)
// partials are reduced in a fixed order: the lane's two pixels, a warp (full
// gradient) or 16-lane half (pose-only: each half walks its own 8x4 list)
// recursive-halving reduce-scatter, ordered adds per warp, then warps 0..3 —
// and written to the entry's slot in the splat-major entry stream, so K4b
// reads each splat's partials contiguously and in tile order (phase 2's
// per-splat order, rasterizer.cpp:410-418). Entries at list positions no
// pixel replays are not written; K4b skips them through the per-tile cut.
// No atomics: deterministic.
#include "gsb_internal.cuh"

namespace gsb {

constexpr int kThreads = 128;          // 2 pixels per thread
constexpr int kBatch = kThreads;       // records staged per batch (backward)
// Composite steps: every lane runs the (no-op when inactive) pair update and
// only a step no lane of the warp hits is skipped (warp-uniform), instead of
// per-lane branches around exhausted sub-lists and missing lanes: 0.107 ->
// 0.103 ms.
#ifndef GSB_COMP_UNIFORM_SKIP
#define GSB_COMP_UNIFORM_SKIP 1
#endif
#ifndef GSB_COMP_BATCH
#define GSB_COMP_BATCH 128
#endif
constexpr int kCompBatch = GSB_COMP_BATCH;  // records staged per composite batch (multiple of 128, <= 256)
constexpr int kWarps = kThreads / 32;  // 4 warps = 4 quadrants of 8x8
constexpr int kSubs = 4;               // 8-lane sub-warps per warp = 4x4 regions
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t lanemask_lt_() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Bits [lo, hi] of a 4-bit row/column range (empty if lo > hi).
__device__ __forceinline__ uint32_t span4(int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, 3);
  return lo > hi ? 0u : ((2u << hi) - (1u << lo));
}

// Stages one record (tile-local mean, conic, opacity, colour) and returns the
// 16-bit mask of 4x4 regions (bit 4*by + bx) meeting the bounding box of the
// cutoff ellipse: |dx| <= sqrt(cutoff2 Sigma_xx), |dy| <= sqrt(cutoff2
// Sigma_yy), Sigma = conic^-1, with a safety margin against FP32 rounding of g.
__device__ __forceinline__ uint32_t stage_splat(const SplatRec& R, double ox, double oy, float cutoff2, float4* geo,
                                                float4* app, float* col_b) {
  const float a = R.conic_a, b = R.conic_b, c = R.conic_c;
  const float det = a * c - b * b;
  const float hw = sqrtf(cutoff2 * c / det) * 1.001f + 1e-2f;
  const float hh = sqrtf(cutoff2 * a / det) * 1.001f + 1e-2f;
  const float mx = (float)(R.mu_x - ox), my = (float)(R.mu_y - oy);
  *geo = make_float4(mx, my, a, b);
  *app = make_float4(c, R.opacity, R.col_r, R.col_g);
  *col_b = R.col_b;
  if (!(det > 0.f) || !(hw < 1e30f) || !(hh < 1e30f)) return 0xffffu;  // degenerate in FP32: test every pixel
  const float x0 = mx - hw, x1 = mx + hw, y0 = my - hh, y1 = my + hh;
  if (!(x1 >= 0.0f && x0 <= 15.0f && y1 >= 0.0f && y0 <= 15.0f)) return 0u;
  // region bx holds pixel columns 4bx..4bx+3: it meets [x0, x1] iff x1 >= 4bx and x0 <= 4bx + 3
  const uint32_t cols = span4((int)ceilf((x0 - 3.0f) * 0.25f), (int)floorf(x1 * 0.25f));
  const uint32_t rows = span4((int)ceilf((y0 - 3.0f) * 0.25f), (int)floorf(y1 * 0.25f));
  // spread the row bits to 0x1, 0x10, 0x100, 0x1000 and replicate the column bits into each
  const uint32_t spread = (rows & 1u) | ((rows & 2u) << 3) | ((rows & 4u) << 6) | ((rows & 8u) << 9);
  return cols * spread;
}

// exp(-g/2) and 1/x via the MUFU approximations with flush-to-zero: the
// arguments never reach the denormal range here (g <= cutoff^2, 1 - alpha >=
// 1 - alpha_clamp), so the non-FTZ fix-up code around MUFU is dead weight.
// Forward and backward use the same helper, so their decisions agree.
__device__ __forceinline__ float exp_neg_half(float g) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(g * -0.7213475204444817f));
  return y;
}
__device__ __forceinline__ float rcp_fast(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Mahalanobis power g = d^T conic d. Forward and backward must take the
// identical cutoff / alpha decisions, so both call exactly this.
__device__ __forceinline__ float splat_power(float ca, float cb, float cc, float dx, float dy) {
  return fmaf(ca * dx, dx, fmaf(cc * dy, dy, 2.0f * cb * dx * dy));
}

// Pixel layout. Warp w -> quadrant (w & 1, w >> 1); sub-warp s = lane >> 3 ->
// 4x4 region (s & 1, s >> 1) of it; lane l8 = lane & 7 -> column l8 & 3,
// rows 2 (l8 >> 2) and +1 of the region.
__device__ __forceinline__ void pixel_coords(int warp, int lane, int* lx, int* ly) {
  const int s = lane >> 3, l8 = lane & 7;
  *lx = (warp & 1) * 8 + (s & 1) * 4 + (l8 & 3);
  *ly = (warp >> 1) * 8 + (s >> 1) * 4 + 2 * (l8 >> 2);
}
// region index (bit of the staging mask) of sub-warp s of warp w
__device__ __forceinline__ int region_of(int warp, int s) {
  return ((warp >> 1) * 2 + (s >> 1)) * 4 + (warp & 1) * 2 + (s & 1);
}

// Compacts the batch entries whose mask has sub-warp s's region bit (and
// whose list position is below lim[s]) into list[s][...] in ascending order,
// for the four sub-warps of this warp at once; returns this lane's
// sub-warp count in *mine and the warp's largest count.
template <int CB>
__device__ __forceinline__ int build_lists(const uint16_t* s_mask, int cnt, int warp, const uint32_t lim[kSubs],
                                           uint32_t b0, uint8_t (*list)[CB], int* mine) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt_();
  int r[kSubs], n[kSubs];
#pragma unroll
  for (int s = 0; s < kSubs; ++s) {
    r[s] = region_of(warp, s);
    n[s] = 0;
  }
#pragma unroll
  for (int c = 0; c < CB / 32; ++c) {
    const int e = c * 32 + lane;
    const uint32_t m = e < cnt ? s_mask[e] : 0u;
#pragma unroll
    for (int s = 0; s < kSubs; ++s) {
      const bool take = ((m >> r[s]) & 1u) && (b0 + (uint32_t)e < lim[s]);
      const uint32_t bits = __ballot_sync(kFull, take);
      if (take) list[s][n[s] + __popc(bits & lt)] = (uint8_t)e;
      n[s] += __popc(bits);
    }
  }
  __syncwarp();
  const int sub = lane >> 3;
  *mine = sub == 0 ? n[0] : sub == 1 ? n[1] : sub == 2 ? n[2] : n[3];
  return max(max(n[0], n[1]), max(n[2], n[3]));
}

// A splat record as the raster loops read it from shared memory: one base
// address per entry (tile-local mean, conic, opacity, colour; entry slot).
struct __align__(16) StagedSplat {
  float4 geo;  // mx, my, conic a, conic b
  float4 app;  // conic c, opacity, colour r, g
  float col_b;
  uint32_t slot;
  uint32_t pad[2];
};

// Shared-window loads from a 32-bit shared address computed once per kernel
// (otherwise the generic->shared conversion is rematerialised in the inner
// loops under register pressure: S2R SR_CgaCtaId + LEA per entry).
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f1(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

// Pixel state of the forward pass; bit 31 of `processed` = done (the pixel
// terminated, or lies outside the image and is never written).
constexpr uint32_t kDone = 0x80000000u;
struct PixFwd {
  float T, r, g, b;
  uint32_t processed;
};
__device__ __forceinline__ bool pix_done(const PixFwd& p, const RasterDev&) { return (int32_t)p.processed < 0; }

// Both pixels of a lane for one splat, branch free (alpha = 0 is an exact
// no-op for a pixel that is done or outside the cutoff).
// hrow (kHits): the batch entry's 16 region masks in shared memory; the
// sub-warp's 8 lanes' pixel-pair hits go to slot `region` (pixel a of lane
// l8 -> bit l8, pixel b -> bit 8 + l8), the exact set of (pixel, entry) pairs
// the replay of render_backward visits (rasterizer.cpp:378-383).
// kHitMode 2: the first lane of each sub-warp whose pixels hit sets the
// entry's byte flag for its 4x4 region (rbyte = &s_rb[k][region]; one
// predicated shared store per step, every flag has a single writer); the
// batch's flags are packed to 16-bit region words at its end.
template <int kHitMode>
__device__ __forceinline__ void composite_pair(PixFwd& a, PixFwd& b, const float4& ge, const float4& ap, float col_b,
                                               float dx, float dy, const RasterDev& rc, uint32_t idx1,
                                               bool act = true, uint16_t* hrow = nullptr, int region = 0,
                                               uint8_t* rbyte = nullptr) {
  const float ga = splat_power(ge.z, ge.w, ap.x, dx, dy);
  const float gb = splat_power(ge.z, ge.w, ap.x, dx, dy + 1.0f);
  const bool ha = act && !pix_done(a, rc) && ga <= rc.cutoff2_f;
  const bool hb = act && !pix_done(b, rc) && gb <= rc.cutoff2_f;
  if (kHitMode == 1) {  // the two ballots double as the warp-uniform skip test
    const uint32_t ba = __ballot_sync(kFull, ha), bb = __ballot_sync(kFull, hb);
    if (!(ba | bb)) return;
    const int lane = threadIdx.x & 31, sh = lane & 24;
    if ((lane & 7) == 0 && act) hrow[region] = (uint16_t)(__byte_perm(ba >> sh, bb >> sh, 0x0040));
  } else if (kHitMode == 2) {  // the ballot doubles as the warp-uniform skip test
    const uint32_t bal = __ballot_sync(kFull, ha || hb);
    if (!bal) return;  // (the step's slot was zeroed at staging)
    const int lane = threadIdx.x & 31;
    if ((lane & 7) == 0 && act && ((bal >> (lane & 24)) & 0xffu)) *rbyte = 1;
  } else {
#if GSB_COMP_UNIFORM_SKIP
    if (!__any_sync(kFull, ha || hb)) return;  // warp-uniform: lanes without a hit run the no-op update
#else
    if (!(ha || hb)) return;
#endif
  }
  const float al_a = ha ? fminf(rc.alpha_clamp_f, ap.y * exp_neg_half(ga)) : 0.f;
  const float al_b = hb ? fminf(rc.alpha_clamp_f, ap.y * exp_neg_half(gb)) : 0.f;
  const float wa = al_a * a.T, wb = al_b * b.T;
  a.r = fmaf(ap.z, wa, a.r);
  a.g = fmaf(ap.w, wa, a.g);
  a.b = fmaf(col_b, wa, a.b);
  b.r = fmaf(ap.z, wb, b.r);
  b.g = fmaf(ap.w, wb, b.g);
  b.b = fmaf(col_b, wb, b.b);
  a.T *= (1.0f - al_a);
  b.T *= (1.0f - al_b);
  if (ha && a.T < rc.early_term_f) a.processed = idx1 | kDone;
  if (hb && b.T < rc.early_term_f) b.processed = idx1 | kDone;
}

__device__ __forceinline__ void write_pixel(const PixFwd& p, int x, int y, int W, int H, float bg_r, float bg_g,
                                            float bg_b, int64_t npix, float* image, float* final_t,
                                            uint32_t* pixstate) {
  if (x >= W || y >= H) return;
  float cr = fmaf(bg_r, p.T, p.r), cg = fmaf(bg_g, p.T, p.g), cb = fmaf(bg_b, p.T, p.b);
  uint32_t of = 0;
  if (cr > 1.0f) { cr = 1.0f; of |= 1u; }
  if (cg > 1.0f) { cg = 1.0f; of |= 2u; }
  if (cb > 1.0f) { cb = 1.0f; of |= 4u; }
  const int64_t q = (int64_t)y * W + x;
  image[q] = cr;
  image[npix + q] = cg;
  image[2 * npix + q] = cb;
  final_t[q] = p.T;
  pixstate[q] = (p.processed & ~kDone) | (of << 29);
}

#ifdef GSB_COMP_MIN_BLOCKS  // (an explicit minimum of 1 changes ptxas's register choice: leave it unset)
#define GSB_COMP_BOUNDS __launch_bounds__(kThreads, GSB_COMP_MIN_BLOCKS)
#else
#define GSB_COMP_BOUNDS __launch_bounds__(kThreads)
#endif
template <int kHitMode>
__global__ void GSB_COMP_BOUNDS composite_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g, float bg_b, int64_t npix,
    float* __restrict__ image, float* __restrict__ final_t, uint32_t* __restrict__ pixstate,
    uint16_t* __restrict__ hits, uint32_t k_cap) {
  constexpr int CB = kCompBatch;
  __shared__ StagedSplat s_sp[CB];
  __shared__ uint16_t s_mask[CB];
  __shared__ uint8_t s_list[kWarps][kSubs][CB];
  constexpr bool kHits = kHitMode == 1;
  __shared__ __align__(16) uint16_t s_hits[kHits ? CB : 1][16];
  constexpr bool kBits = kHitMode == 2;
  __shared__ __align__(16) uint8_t s_rb[kBits ? CB : 1][16];  // per batch entry: a flag per 4x4 region it touched
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sub = lane >> 3;
  const unsigned sub_mask = 0xffu << (8 * sub);
  int lx, ly;
  pixel_coords(warp, lane, &lx, &ly);
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const float px = (float)lx, py = (float)ly;
  const int region = region_of(warp, sub);
  const uint2 range = ranges[tile];
  PixFwd a{1.f, 0.f, 0.f, 0.f, (x < W && y < H) ? 0u : kDone};
  PixFwd b{1.f, 0.f, 0.f, 0.f, (x < W && y + 1 < H) ? 0u : kDone};
  for (uint32_t base = range.x; base < range.y; base += CB) {
    if (__syncthreads_count(pix_done(a, rc) && pix_done(b, rc)) == kThreads) break;
    const int cnt = min((uint32_t)CB, range.y - base);
#pragma unroll
    for (int u = 0; u < CB / kThreads; ++u) {
      const int t = u * kThreads + threadIdx.x;
      if (t < cnt)
        s_mask[t] = (uint16_t)stage_splat(rec[ranks[base + t]], ox, oy, rc.cutoff2_f, &s_sp[t].geo, &s_sp[t].app,
                                          &s_sp[t].col_b);
      if (kHits) {
        uint4* hz = reinterpret_cast<uint4*>(s_hits[t]);
        hz[0] = make_uint4(0u, 0u, 0u, 0u);
        hz[1] = make_uint4(0u, 0u, 0u, 0u);
      }
      if (kBits) *reinterpret_cast<uint4*>(s_rb[t]) = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    const uint32_t list0 = base - range.x;
    // a finished sub-warp lists nothing (its region's pixels are all terminated)
    uint32_t lim[kSubs];
    const uint32_t live = __ballot_sync(kFull, !(pix_done(a, rc) && pix_done(b, rc)));
#pragma unroll
    for (int s = 0; s < kSubs; ++s) lim[s] = ((live >> (8 * s)) & 0xffu) ? 0xffffffffu : 0u;
    int mine = 0;
    const int nmax = build_lists<CB>(s_mask, cnt, warp, lim, 0u, s_list[warp], &mine);
    for (int it = 0; it < nmax; ++it) {
#if GSB_COMP_UNIFORM_SKIP
      {
        const bool act = it < mine;
        const int k = act ? s_list[warp][sub][it] : 0;
        const StagedSplat& S = s_sp[k];
        const float4 ge = S.geo;
        const float4 ap = S.app;
        const float cb = S.col_b;
        const float dx = px - ge.x, dy = py - ge.y;
        composite_pair<kHitMode>(a, b, ge, ap, cb, dx, dy, rc, list0 + k + 1u, act, kHits ? s_hits[k] : nullptr,
                                 region, kBits ? &s_rb[k][region] : nullptr);
      }
#else
      if (it < mine) {
        const int k = s_list[warp][sub][it];
        const StagedSplat& S = s_sp[k];
        const float4 ge = S.geo;
        const float4 ap = S.app;
        const float cb = S.col_b;
        const float dx = px - ge.x, dy = py - ge.y;
        composite_pair<0>(a, b, ge, ap, cb, dx, dy, rc, list0 + k + 1u);
      }
#endif
      // a sub-warp whose 16 pixels have all terminated stops early
      if (__all_sync(kFull, (pix_done(a, rc) && pix_done(b, rc)) || it + 1 >= mine)) break;
    }
    (void)sub_mask;
    if (!pix_done(a, rc)) a.processed = list0 + (uint32_t)cnt;
    if (!pix_done(b, rc)) b.processed = list0 + (uint32_t)cnt;
    if (kBits) {  // the batch's region bits, 2 B per entry, coalesced
      __syncthreads();
#pragma unroll
      for (int u = 0; u < CB / kThreads; ++u) {
        const int t = u * kThreads + threadIdx.x;
        if (t < cnt && base + t < k_cap) {  // 16 flag bytes (0 / 1) -> bit r = region r
          const uint4 f = *reinterpret_cast<const uint4*>(s_rb[t]);
          const uint32_t w = ((f.x * 0x01020408u) >> 24) | (((f.y * 0x01020408u) >> 24) << 4) |
                             (((f.z * 0x01020408u) >> 24) << 8) | (((f.w * 0x01020408u) >> 24) << 12);
          hits[base + t] = (uint16_t)w;
        }
      }
    }
    if (kHits) {  // the batch's masks, 32 B per entry, coalesced
      __syncthreads();
#pragma unroll
      for (int u = 0; u < CB / kThreads; ++u) {
        const int t = u * kThreads + threadIdx.x;
        if (t < cnt && base + t < k_cap) {
          const uint4* src = reinterpret_cast<const uint4*>(s_hits[t]);
          uint4* dst = reinterpret_cast<uint4*>(hits + (size_t)(base + t) * 16);
          dst[0] = src[0];
          dst[1] = src[1];
        }
      }
    }
  }
  write_pixel(a, x, y, W, H, bg_r, bg_g, bg_b, npix, image, final_t, pixstate);
  write_pixel(b, x, y + 1, W, H, bg_r, bg_g, bg_b, npix, image, final_t, pixstate);
}


// ---- K4a helpers: 8x8-quadrant lists (one warp = one quadrant, 2 px/lane)
__device__ __forceinline__ void quad_pixel_coords(int warp, int lane, int* lx, int* ly) {
  *lx = (warp & 1) * 8 + (lane & 7);
  *ly = (warp >> 1) * 8 + (lane >> 3) * 2;
}
// quadrant bits of a 16-bit region mask: quadrant q = (qx, qy) holds regions (2qx..2qx+1, 2qy..2qy+1)
__device__ __forceinline__ uint32_t quad_mask(uint32_t m16) {
  uint32_t q = 0;
  if (m16 & 0x0033u) q |= 1u;
  if (m16 & 0x00ccu) q |= 2u;
  if (m16 & 0x3300u) q |= 4u;
  if (m16 & 0xcc00u) q |= 8u;
  return q;
}
__device__ __forceinline__ int build_list(const uint8_t* s_mask, int cnt, int warp, uint8_t* list) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt_();
  int n = 0;
#pragma unroll
  for (int c = 0; c < kBatch / 32; ++c) {
    const int e = c * 32 + lane;
    const bool mine = e < cnt && ((s_mask[e] >> warp) & 1u);
    const uint32_t bits = __ballot_sync(kFull, mine);
    if (mine) list[n + __popc(bits & lt)] = (uint8_t)e;
    n += __popc(bits);
  }
  __syncwarp();
  return n;
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

// Pose-only backward: 8 components (the opacity partial has no consumer),
// reduce-scatter xor 16 / 8 / 4 (4 + 2 + 1 shuffles) then a plain xor 2 / 1
// sum: 9 shuffles. Lanes with (lane & 3) == 0 end owning component
// 4 b4 + 2 b3 + b2 (b_k = bit k of lane).
__device__ __forceinline__ int warp_reduce8(const float v[8], float* out) {
  const int lane = threadIdx.x & 31;
  const bool h1 = lane & 16, h2 = lane & 8, h3 = lane & 4;
  float w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = h1 ? v[i] : v[4 + i], keep = h1 ? v[4 + i] : v[i];
    w[i] = keep + __shfl_xor_sync(kFull, send, 16);
  }
  float x[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = h2 ? w[i] : w[2 + i], keep = h2 ? w[2 + i] : w[i];
    x[i] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  float z;
  {
    const float send = h3 ? x[0] : x[1], keep = h3 ? x[1] : x[0];
    z = keep + __shfl_xor_sync(kFull, send, 4);
  }
  z += __shfl_xor_sync(kFull, z, 2);
  z += __shfl_xor_sync(kFull, z, 1);
  *out = z;
  return (lane & 3) ? -1 : (h1 ? 4 : 0) + (h2 ? 2 : 0) + (h3 ? 1 : 0);
}

// Backward pixel state. Bd = sum_c d_pix[c] * behind[c]: the replay only
// ever needs the behind colour dotted with the pixel's upstream gradient
// (rasterizer.cpp:386-390), so one scalar replaces the three channels.
struct PixBwd {
  float dr, dg, db, T, Bd;
  uint32_t contrib;
};

__device__ __forceinline__ void load_pixel_bwd(PixBwd& p, int x, int y, int W, int H, int64_t npix, float bg_r,
                                               float bg_g, float bg_b, const float* d_image, const float* final_t,
                                               const uint32_t* pixstate) {
  p.dr = p.dg = p.db = p.T = 0.f;
  p.contrib = 0;
  if (x < W && y < H) {
    const int64_t q = (int64_t)y * W + x;
    const uint32_t ps = pixstate[q];
    const uint32_t of = ps >> 29;
    p.dr = (of & 1u) ? 0.f : d_image[q];
    p.dg = (of & 2u) ? 0.f : d_image[npix + q];
    p.db = (of & 4u) ? 0.f : d_image[2 * npix + q];
    p.T = final_t[q];
    p.contrib = ps & 0x1fffffffu;
    if (p.dr == 0.f && p.dg == 0.f && p.db == 0.f) p.contrib = 0;  // rasterizer.cpp:372
  }
  p.Bd = p.T * (p.dr * bg_r + p.dg * bg_g + p.db * bg_b);
}

// Both pixels of a lane for one splat (one replay step of phase 1), branch
// free: a pixel that is past its contrib count or outside the cutoff (ha/hb
// false) gets alpha_raw = 0, which makes every update below an exact no-op
// (inv = 1, weight 0, d_alpha chain times 0), so the two chains interleave
// and lanes without a hit need no separate path. Writes v (NC = 8: no
// opacity partial).
template <int NC>
__device__ __forceinline__ void backward_pair(PixBwd& a, PixBwd& b, const float4& ge, const float4& ap, float col_b,
                                              float dx, float dy, float ga, float gb, bool ha, bool hb,
                                              const RasterDev& rc, float v[NC]) {
  const float Ga = exp_neg_half(ga), Gb = exp_neg_half(gb);
  const float ra = ha ? ap.y * Ga : 0.f, rb = hb ? ap.y * Gb : 0.f;  // alpha_raw
  const float al_a = fminf(rc.alpha_clamp_f, ra), al_b = fminf(rc.alpha_clamp_f, rb);
  const float ia = rcp_fast(1.0f - al_a), ib = rcp_fast(1.0f - al_b);
  const float ta = a.T * ia, tb = b.T * ib;  // t_before
  const float wa = al_a * ta, wb = al_b * tb;
  v[5] = fmaf(wa, a.dr, wb * b.dr);
  v[6] = fmaf(wa, a.dg, wb * b.dg);
  v[7] = fmaf(wa, a.db, wb * b.db);
  const float dca = fmaf(a.dr, ap.z, fmaf(a.dg, ap.w, a.db * col_b));
  const float dcb = fmaf(b.dr, ap.z, fmaf(b.dg, ap.w, b.db * col_b));
  const float dala = fmaf(ta, dca, -ia * a.Bd), dalb = fmaf(tb, dcb, -ib * b.Bd);
  // alpha-chain gradients only where alpha_raw < clamp (rasterizer.cpp:392)
  const float ka = ra < rc.alpha_clamp_f ? dala * (-0.5f * ra) : 0.f;
  const float kb = rb < rc.alpha_clamp_f ? dalb * (-0.5f * rb) : 0.f;
  if (NC > 8) {
    v[NC - 1] = fmaf(ra < rc.alpha_clamp_f ? dala : 0.f, Ga * (ha ? 1.f : 0.f),
                     (rb < rc.alpha_clamp_f ? dalb : 0.f) * (Gb * (hb ? 1.f : 0.f)));
  }
  // pixel b sits at dy + 1: with s = ka + kb the pair's sums factor as
  // conic.d_a s + conic.(0, 1) kb, dx^2 s, dx (dy s + kb), dy^2 s + (2 dy + 1) kb;
  // components 0 and 1 leave out the factor -2 (applied exactly at the flush)
  const float sk = ka + kb;
  const float cxa = fmaf(ge.z, dx, ge.w * dy), cya = fmaf(ge.w, dx, ap.x * dy);
  v[0] = fmaf(sk, cxa, kb * ge.w);
  v[1] = fmaf(sk, cya, kb * ap.x);
  v[2] = (sk * dx) * dx;
  v[3] = dx * fmaf(sk, dy, kb);
  v[4] = fmaf(sk * dy, dy, kb * (dy + dy + 1.0f));
  a.T = ta;
  b.T = tb;
  a.Bd = fmaf(wa, dca, a.Bd);
  b.Bd = fmaf(wb, dcb, b.Bd);
}

#ifndef GSB_LDS_ASM
#define GSB_LDS_ASM 1
#endif
// K4a occupancy: a minimum of 6 CTAs/SM lets ptxas keep its natural 72
// registers (7 CTAs/SM resident); forcing 8 CTAs/SM caps it at 64 and it
// rematerialises addresses in the step loop. Measured: 0.232 -> 0.217 ms per
// launch alone, pose batch unchanged within noise.
#ifndef GSB_BWD_MIN_BLOCKS
#define GSB_BWD_MIN_BLOCKS 6
#endif
template <int NC>
__global__ void __launch_bounds__(kThreads, GSB_BWD_MIN_BLOCKS) backward_raster_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const SplatAux* __restrict__ aux, const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g,
    float bg_b, int64_t npix, const float* __restrict__ d_image, const float* __restrict__ final_t,
    const uint32_t* __restrict__ pixstate, const double* __restrict__ depth_g, double2* __restrict__ tile_cut,
    float* __restrict__ partials, uint32_t k_cap) {
  __shared__ StagedSplat s_sp[kBatch];
  __shared__ uint8_t s_mask[kBatch];
  __shared__ uint8_t s_list[kWarps][kBatch];
  __shared__ float s_red[kWarps][kBatch][NC];  // [warp][entry in batch][component]
  __shared__ int s_w, s_h, s_tx;
  __shared__ uint32_t s_maxc[kWarps];
  if (threadIdx.x == 0) {
    s_w = cam_p->width;
    s_h = cam_p->height;
    s_tx = cam_p->tiles_x;
  }
  for (int i = threadIdx.x; i < kWarps * kBatch * NC; i += kThreads) (&s_red[0][0][0])[i] = 0.f;
  __syncthreads();
  const int W = s_w, H = s_h;
  const int tile = blockIdx.x;
  const int tx = tile % s_tx, ty = tile / s_tx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int lx, ly;
  quad_pixel_coords(warp, lane, &lx, &ly);
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const float px = (float)lx, py = (float)ly;
  const uint2 range = ranges[tile];
  const uint32_t sp_base = (uint32_t)__cvta_generic_to_shared(s_sp);

  PixBwd a, b;
  load_pixel_bwd(a, x, y, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  load_pixel_bwd(b, x, y + 1, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  const uint32_t wmax = __reduce_max_sync(kFull, max(a.contrib, b.contrib));
  if (lane == 0) s_maxc[warp] = wmax;
  __syncthreads();
  uint32_t maxc = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) maxc = max(maxc, s_maxc[w]);
  // Entries at list positions >= maxc are replayed by no pixel: their
  // partials are zero and are neither computed nor stored. K4b skips them by
  // comparing its (FP64 depth, gid) with the tile's cut — the key of entry
  // maxc - 1 (tile lists are sorted by exactly that key).
  if (threadIdx.x == 0) {
    double2 cut = make_double2(-1.0, 0.0);
    if (maxc > 0) {
      const int32_t gid = aux[ranks[range.x + maxc - 1]].gid;
      cut = make_double2(depth_g[gid], (double)gid);
    }
    tile_cut[tile] = cut;
  }
  const uint32_t len = min(range.y - range.x, maxc);

  // Batches walk the live part of the list from the back.
  const uint32_t nbatch = (len + kBatch - 1) / kBatch;
  for (int bi = (int)nbatch - 1; bi >= 0; --bi) {
    const uint32_t b0 = (uint32_t)bi * kBatch;  // list-local start
    const int cnt = (int)min((uint32_t)kBatch, len - b0);
    if (threadIdx.x < cnt) {
      const uint32_t e = range.x + b0 + threadIdx.x;
      const uint32_t r = ranks[e];
      const SplatAux A = aux[r];
      const uint32_t tx0 = A.tx0_ty0 & 0xffffu, ty0 = A.tx0_ty0 >> 16, nx = A.nx_ny & 0xffffu;
      StagedSplat& S = s_sp[threadIdx.x];
      S.slot = A.off + ((uint32_t)ty - ty0) * nx + ((uint32_t)tx - tx0);
      s_mask[threadIdx.x] = (uint8_t)quad_mask(stage_splat(rec[r], ox, oy, rc.cutoff2_f, &S.geo, &S.app, &S.col_b));
    }
    __syncthreads();
    if (b0 < wmax) {  // this warp has pixels that replay entries of this batch
      const int n = build_list(s_mask, cnt, warp, s_list[warp]);
      for (int i = n - 1; i >= 0; --i) {  // back to front
        const int k = s_list[warp][i];
        const uint32_t j = b0 + (uint32_t)k;
        if (j >= wmax) continue;  // warp-uniform
#if GSB_LDS_ASM
        const uint32_t sa = sp_base + (uint32_t)k * (uint32_t)sizeof(StagedSplat);
        const float4 ge = lds_f4(sa);
        const float4 ap = lds_f4(sa + 16u);
        const float cb = lds_f1(sa + 32u);
#else
        const float4 ge = s_sp[k].geo;
        const float4 ap = s_sp[k].app;
        const float cb = s_sp[k].col_b;
        (void)sp_base;
#endif
        const float dx = px - ge.x, dy = py - ge.y;
        const float ga = splat_power(ge.z, ge.w, ap.x, dx, dy);
        const float gb = splat_power(ge.z, ge.w, ap.x, dx, dy + 1.0f);
        const bool ha = j < a.contrib && ga <= rc.cutoff2_f;
        const bool hb = j < b.contrib && gb <= rc.cutoff2_f;
        if (!__any_sync(kFull, ha || hb)) continue;  // s_red stays zero for this entry
        float v[NC];
        backward_pair<NC>(a, b, ge, ap, cb, dx, dy, ga, gb, ha, hb, rc, v);
        float tot;
        const int vi = NC == 8 ? warp_reduce8(v, &tot) : warp_reduce9(v, &tot);
        if (vi >= 0) s_red[warp][k][vi] = tot;
      }
    }
    __syncthreads();
    // flush: batch entries x 9 components, summed over warps 0..3 in order
    for (int idx = threadIdx.x; idx < cnt * NC; idx += kThreads) {
      const int k = idx / NC, c = idx - k * NC;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        acc += s_red[w][k][c];
        s_red[w][k][c] = 0.f;
      }
      if (c < 2) acc *= -2.0f;  // d_mu2d = -2 dg (conic d) (rasterizer.cpp:396)
      const uint32_t slot = s_sp[k].slot;
      if (slot < k_cap) partials[(int64_t)slot * NC + c] = acc;
    }
    __syncthreads();
  }
}

// ---- K4a, pose-only variant on half-quadrant lists: each warp still owns
// an 8x8 quadrant (same pixel layout as above), but its two 16-lane halves
// (rows 0-3 and 4-7 of the quadrant) walk their own lists of the batch
// entries whose cutoff-ellipse box reaches their 8x4 half, so one warp step
// serves two entries and a splat costs a half nothing unless it reaches it.
// Per-entry partials: a 16-lane reduce-scatter (8 shuffles serve both halves'
// entries) and a fixed-order add into the warp's shared slot (half 0 before
// half 1 within a step; steps in list order) — deterministic.
__device__ __forceinline__ uint32_t half_mask(uint32_t m16) {
  uint32_t r = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int by = 2 * (q >> 1) + h, bx = 2 * (q & 1);
      if ((m16 >> (4 * by + bx)) & 3u) r |= 1u << (2 * q + h);
    }
  return r;
}

// Lists of batch entries (list-local position < lim0 / lim1) reaching half 0 / 1
// of warp w's quadrant, ascending; returns both counts.
__device__ __forceinline__ void build_half_lists(const uint8_t* s_mask, int cnt, int warp, uint32_t lim0,
                                                 uint32_t lim1, uint8_t (*list)[kBatch], int* n0, int* n1) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt_();
  int c0 = 0, c1 = 0;
#pragma unroll
  for (int c = 0; c < kBatch / 32; ++c) {
    const int e = c * 32 + lane;
    const uint32_t m = e < cnt ? (s_mask[e] >> (2 * warp)) : 0u;
    const bool t0 = (m & 1u) && (uint32_t)e < lim0, t1 = (m & 2u) && (uint32_t)e < lim1;
    const uint32_t b0 = __ballot_sync(kFull, t0), b1 = __ballot_sync(kFull, t1);
    if (t0) list[0][c0 + __popc(b0 & lt)] = (uint8_t)e;
    if (t1) list[1][c1 + __popc(b1 & lt)] = (uint8_t)e;
    c0 += __popc(b0);
    c1 += __popc(b1);
  }
  __syncwarp();
  *n0 = c0;
  *n1 = c1;
}

// Exact culling of (entry, half) pairs (GSB_BWD_EXACT_CULL): the minimum of
// the splat's power g = d^T conic d over the half's 8x4 rectangle of pixel
// centres (tile-local [x0, x0 + 7] x [y0, y0 + 3]) — 0 if the mean is inside,
// else the least of the four edge minima, each a clamped 1-D quadratic in
// completed-square form (c (v - v*)^2 + (det / c) u^2: two non-negative terms,
// no cancellation). A half whose minimum exceeds the cutoff by a margin far
// above the FP32 rounding of the in-step g has no pixel the entry can touch:
// its list skips the entry, whose contribution there is an exact zero.
// Splats too elongated for that error bound (det < 1e-3 a c) keep the box test.
// Measured on the bench: K4a 0.2162 -> 0.2209 ms (the staging cost exceeds the
// steps it saves) — off.
#ifndef GSB_BWD_EXACT_CULL
#define GSB_BWD_EXACT_CULL 0
#endif
__device__ __forceinline__ float rect_min_power(float mx, float my, float a, float b, float c, float det, float x0,
                                                float y0) {
  const float u0 = x0 - mx, u1 = x0 + 7.0f - mx, v0 = y0 - my, v1 = y0 + 3.0f - my;
  if (u0 <= 0.0f && u1 >= 0.0f && v0 <= 0.0f && v1 >= 0.0f) return 0.0f;
  const float ia = 1.0f / a, ic = 1.0f / c, dc = det * ic, da = det * ia;
  auto edge_x = [&](float u) {  // dx = u fixed, dy in [v0, v1]; minimiser v* = -b u / c
    const float vs = -b * u * ic, w = fminf(fmaxf(vs, v0), v1) - vs;
    return c * w * w + dc * u * u;
  };
  auto edge_y = [&](float v) {  // dy = v fixed, dx in [u0, u1]; minimiser u* = -b v / a
    const float us = -b * v * ia, w = fminf(fmaxf(us, u0), u1) - us;
    return a * w * w + da * v * v;
  };
  return fminf(fminf(edge_x(u0), edge_x(u1)), fminf(edge_y(v0), edge_y(v1)));
}
__device__ __forceinline__ uint32_t exact_half_mask(uint32_t m, const float4& ge, float c, float cutoff2) {
  const float a = ge.z, b = ge.w, det = fmaf(a, c, -b * b);
  if (!(a > 0.f && c > 0.f && det >= 1e-3f * a * c) || !(a * c < 1e30f)) return m;
  const float thr = cutoff2 * 1.001f + 1e-3f;
  uint32_t keep = 0u;
  for (uint32_t r = m; r; r &= r - 1u) {
    const int hb = __ffs(r) - 1, q = hb >> 1, h = hb & 1;
    if (rect_min_power(ge.x, ge.y, a, b, c, det, (float)((q & 1) * 8), (float)((q >> 1) * 8 + 4 * h)) <= thr)
      keep |= 1u << hb;
  }
  return keep;
}

// 8 values over each 16-lane half: xor 8 / 4 / 2 reduce-scatter (4 + 2 + 1
// shuffles) and a plain xor-1 sum; even lanes end owning component
// 4 b3 + 2 b2 + b1 (b_k = bit k of the lane) of their half's sum.
__device__ __forceinline__ int half_reduce8(const float v[8], float* out) {
  const int lane = threadIdx.x & 31;
  const bool h1 = lane & 8, h2 = lane & 4, h3 = lane & 2;
  float w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = h1 ? v[i] : v[4 + i], keep = h1 ? v[4 + i] : v[i];
    w[i] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  float x[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = h2 ? w[i] : w[2 + i], keep = h2 ? w[2 + i] : w[i];
    x[i] = keep + __shfl_xor_sync(kFull, send, 4);
  }
  float z;
  {
    const float send = h3 ? x[0] : x[1], keep = h3 ? x[1] : x[0];
    z = keep + __shfl_xor_sync(kFull, send, 2);
  }
  z += __shfl_xor_sync(kFull, z, 1);
  *out = z;
  return (lane & 1) ? -1 : (h1 ? 4 : 0) + (h2 ? 2 : 0) + (h3 ? 1 : 0);
}

// 9 values (full gradient: + the opacity partial) over each 16-lane half:
// uneven reduce-scatter 9 -> 5 -> 3 -> 2 -> 1 (5 + 3 + 2 + 1 shuffles); the
// lane with bits (b3 b2 b1 b0) ends owning component 5 b3 + 3 b2 + 2 b1 + b0
// when that index chain stays in range (each component exactly once).
__device__ __forceinline__ int half_reduce9(const float v[9], float* out) {
  const int lane = threadIdx.x & 31;
  const bool h8 = lane & 8, h4 = lane & 4, h2 = lane & 2, h1 = lane & 1;
  float w[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const float lo = v[i], hi = i < 4 ? v[5 + i] : 0.f;
    const float send = h8 ? lo : hi, keep = h8 ? hi : lo;
    w[i] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  float x[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float lo = w[i], hi = i < 2 ? w[3 + i] : 0.f;
    const float send = h4 ? lo : hi, keep = h4 ? hi : lo;
    x[i] = keep + __shfl_xor_sync(kFull, send, 4);
  }
  float y[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float lo = x[i], hi = i < 1 ? x[2] : 0.f;
    const float send = h2 ? lo : hi, keep = h2 ? hi : lo;
    y[i] = keep + __shfl_xor_sync(kFull, send, 2);
  }
  float z;
  {
    const float send = h1 ? y[0] : y[1], keep = h1 ? y[1] : y[0];
    z = keep + __shfl_xor_sync(kFull, send, 1);
  }
  const int xi = (h2 ? 2 : 0) + (h1 ? 1 : 0), wi = (h4 ? 3 : 0) + xi, vi = (h8 ? 5 : 0) + wi;
  *out = z;
  return (xi < 3 && wi < 5 && vi < 9) ? vi : -1;
}

// cp.async (LDGSTS) staging for K4a (GSB_BWD_CPASYNC=1, off by default — see
// profiles/README.md for the A/B): the next batch's raw records (48 B
// SplatRec + 16 B SplatAux per entry, gathered by rank) are copied into a
// second shared buffer while the current batch is replayed.
#ifndef GSB_BWD_CPASYNC
#define GSB_BWD_CPASYNC 0
#endif
#ifndef GSB_HALF_LDS_ASM
#define GSB_HALF_LDS_ASM 0
#endif
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

#ifndef GSB_BWD_HITS_MIN_BLOCKS
#define GSB_BWD_HITS_MIN_BLOCKS 6  // (7: 70 registers, 0.2168 ms; 6: 78 registers, 0.202 ms)
#endif
template <int NC, int kHitMode>
__global__ void __launch_bounds__(kThreads, kHitMode == 1 ? GSB_BWD_HITS_MIN_BLOCKS : GSB_BWD_MIN_BLOCKS) backward_raster_half_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const SplatAux* __restrict__ aux, const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g,
    float bg_b, int64_t npix, const float* __restrict__ d_image, const float* __restrict__ final_t,
    const uint32_t* __restrict__ pixstate, const double* __restrict__ depth_g, double2* __restrict__ tile_cut,
    float* __restrict__ partials, uint32_t k_cap, const uint16_t* __restrict__ hits) {
  __shared__ StagedSplat s_sp[kBatch];
  constexpr bool kHits = kHitMode == 1;
  // kHitMode 2: the composite's region bits (one uint16 per list position)
  // narrow each entry's half mask to the halves it touched.
  // kHits: the composite's hit masks of the batch entries, one 32-bit word per
  // (quadrant, half) = its two 4x4 regions' 16-bit masks
  __shared__ uint32_t s_hm[kHits ? kBatch : 1][8];
  __shared__ uint8_t s_mask[kBatch];
  __shared__ uint8_t s_list[kWarps][2][kBatch];
  __shared__ float s_red[kWarps][kBatch][NC];  // [warp][entry in batch][component]
  __shared__ int s_w, s_h, s_tx;
  __shared__ uint32_t s_maxc[kWarps];
  if (threadIdx.x == 0) {
    s_w = cam_p->width;
    s_h = cam_p->height;
    s_tx = cam_p->tiles_x;
  }
  for (int i = threadIdx.x; i < kWarps * kBatch * NC; i += kThreads) (&s_red[0][0][0])[i] = 0.f;
  __syncthreads();
  const int W = s_w, H = s_h;
  const int tile = blockIdx.x;
  const int tx = tile % s_tx, ty = tile / s_tx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4;
  int lx, ly;
  quad_pixel_coords(warp, lane, &lx, &ly);
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const float px = (float)lx, py = (float)ly;
  const uint2 range = ranges[tile];
  const uint32_t sp_base = (uint32_t)__cvta_generic_to_shared(s_sp);

  PixBwd a, b;
  load_pixel_bwd(a, x, y, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  load_pixel_bwd(b, x, y + 1, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  const uint32_t pmax = max(a.contrib, b.contrib);
  const uint32_t wmax = __reduce_max_sync(kFull, pmax);
  // per-half replay depth: an entry at or past it is replayed by no pixel of the half
  const uint32_t hmax0 = __reduce_max_sync(kFull, half ? 0u : pmax), hmax1 = __reduce_max_sync(kFull, half ? pmax : 0u);
  if (lane == 0) s_maxc[warp] = wmax;
  __syncthreads();
  uint32_t maxc = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) maxc = max(maxc, s_maxc[w]);
  // entries at list positions >= maxc: see backward_raster_kernel
  if (threadIdx.x == 0) {
    double2 cut = make_double2(-1.0, 0.0);
    if (maxc > 0) {
      const int32_t gid = aux[ranks[range.x + maxc - 1]].gid;
      cut = make_double2(depth_g[gid], (double)gid);
    }
    tile_cut[tile] = cut;
  }
  // this lane's bit in its half's hit word: region column (lane & 7) >> 2,
  // composite lane l8 = column % 4 + 4 (row % 4) / 2 (pixel a; b at + 8)
  const int hbit = (((lane & 7) >> 2) << 4) + ((lane & 3) | (((lane >> 3) & 1) << 2));
  const uint32_t len = min(range.y - range.x, maxc);
  const uint32_t nbatch = (len + kBatch - 1) / kBatch;
#if GSB_BWD_CPASYNC
  __shared__ __align__(16) SplatRec s_raw[2][kBatch];
  __shared__ __align__(16) SplatAux s_rawx[2][kBatch];
  auto issue = [&](int bj, int buf, uint32_t r) {
    const uint32_t bb = (uint32_t)bj * kBatch;
    if (threadIdx.x < min((uint32_t)kBatch, len - bb)) {
      const char* src = reinterpret_cast<const char*>(rec + r);
      char* dst = reinterpret_cast<char*>(&s_raw[buf][threadIdx.x]);
      cp_async16(dst, src);
      cp_async16(dst + 16, src + 16);
      cp_async16(dst + 32, src + 32);
      cp_async16(&s_rawx[buf][threadIdx.x], aux + r);
    }
    cp_async_commit();
  };
  auto rank_of = [&](int bj) -> uint32_t {
    const uint32_t bb = (uint32_t)bj * kBatch;
    return (bj >= 0 && threadIdx.x < min((uint32_t)kBatch, len - bb)) ? ranks[range.x + bb + threadIdx.x] : 0u;
  };
  if (nbatch > 0) issue((int)nbatch - 1, 0, rank_of((int)nbatch - 1));
#endif
  for (int bi = (int)nbatch - 1; bi >= 0; --bi) {
    const uint32_t b0 = (uint32_t)bi * kBatch;  // list-local start
    const int cnt = (int)min((uint32_t)kBatch, len - b0);
#if GSB_BWD_CPASYNC
    const int buf = ((int)nbatch - 1 - bi) & 1;
    const uint32_t r_next = rank_of(bi - 1);  // issued now, used after this batch's staging
    cp_async_wait_all();
    __syncthreads();
    if (threadIdx.x < cnt) {
      const SplatAux A = s_rawx[buf][threadIdx.x];
      const uint32_t tx0 = A.tx0_ty0 & 0xffffu, ty0 = A.tx0_ty0 >> 16, nx = A.nx_ny & 0xffffu;
      StagedSplat& S = s_sp[threadIdx.x];
      S.slot = A.off + ((uint32_t)ty - ty0) * nx + ((uint32_t)tx - tx0);
      s_mask[threadIdx.x] =
          (uint8_t)half_mask(stage_splat(s_raw[buf][threadIdx.x], ox, oy, rc.cutoff2_f, &S.geo, &S.app, &S.col_b));
    }
    if (bi > 0) issue(bi - 1, buf ^ 1, r_next);
#else
    if (threadIdx.x < cnt) {
      const uint32_t e = range.x + b0 + threadIdx.x;
      const uint32_t r = ranks[e];
      const SplatAux A = aux[r];
      const uint32_t tx0 = A.tx0_ty0 & 0xffffu, ty0 = A.tx0_ty0 >> 16, nx = A.nx_ny & 0xffffu;
      StagedSplat& S = s_sp[threadIdx.x];
      S.slot = A.off + ((uint32_t)ty - ty0) * nx + ((uint32_t)tx - tx0);
      uint32_t bbox = half_mask(stage_splat(rec[r], ox, oy, rc.cutoff2_f, &S.geo, &S.app, &S.col_b));
      if (GSB_BWD_EXACT_CULL && !kHits && bbox) bbox = exact_half_mask(bbox, S.geo, S.app.x, rc.cutoff2_f);
      if (kHits) {
        // region r = 4 ry + rx; (quadrant q = qx + 2 qy, half h) holds regions
        // 4 (2 qy + h) + 2 qx and + 1
        const uint4* hp = reinterpret_cast<const uint4*>(hits + (size_t)e * 16);
        const uint4 h0 = __ldg(hp), h1 = __ldg(hp + 1);
        const uint32_t w[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};  // w[i] = regions 2i, 2i+1
        uint32_t m = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int rg = 4 * (2 * (q >> 1) + h) + 2 * (q & 1);  // even: regions rg, rg + 1 = word rg / 2
            const uint32_t word = w[rg >> 1];
            s_hm[threadIdx.x][2 * q + h] = word;
            if (word) m |= 1u << (2 * q + h);
          }
        s_mask[threadIdx.x] = (uint8_t)(m & bbox);
      } else if (kHitMode == 2) {
        s_mask[threadIdx.x] = (uint8_t)(bbox & half_mask(__ldg(hits + e)));
      } else {
        s_mask[threadIdx.x] = (uint8_t)bbox;
      }
    }
#endif
    __syncthreads();
    if (b0 < wmax) {  // this warp has pixels that replay entries of this batch
      int n0, n1;
      build_half_lists(s_mask, cnt, warp, hmax0 > b0 ? hmax0 - b0 : 0u, hmax1 > b0 ? hmax1 - b0 : 0u,
                       s_list[warp], &n0, &n1);
      const int mine = half ? n1 : n0;
      const int nmax = max(n0, n1);
      const uint8_t* my_list = s_list[warp][half];
      for (int it = 0; it < nmax; ++it) {  // each half back to front
        const bool act = it < mine;
        const int k = act ? my_list[mine - 1 - it] : 0;
        const uint32_t j = b0 + (uint32_t)k;
#if GSB_HALF_LDS_ASM
        const uint32_t sa = sp_base + (uint32_t)k * (uint32_t)sizeof(StagedSplat);
        const float4 ge = lds_f4(sa);
        const float4 ap = lds_f4(sa + 16u);
#else
        // plain shared-array loads: LDS offsets in the CTA's window need no
        // generic->shared base (the asm form rematerialised S2R SR_CgaCtaId +
        // LEA in the step loop)
        const float4 ge = s_sp[k].geo;
        const float4 ap = s_sp[k].app;
#endif
        const float dx = px - ge.x, dy = py - ge.y;
        const float ga = splat_power(ge.z, ge.w, ap.x, dx, dy);
        const float gb = splat_power(ge.z, ge.w, ap.x, dx, dy + 1.0f);
        bool ha, hb;
        if (kHits) {  // the composite's decisions (bits hb_sh, hb_sh + 8) gated by a non-zero upstream gradient
          const uint32_t word = s_hm[k][2 * warp + half];
          ha = act && a.contrib != 0u && ((word >> hbit) & 1u);
          hb = act && b.contrib != 0u && ((word >> (hbit + 8)) & 1u);
        } else {
          ha = act && j < a.contrib && ga <= rc.cutoff2_f;
          hb = act && j < b.contrib && gb <= rc.cutoff2_f;
        }
        if (!__any_sync(kFull, ha || hb)) continue;  // neither half's entry touched: zero partials
#if GSB_HALF_LDS_ASM
        const float cb = lds_f1(sa + 32u);
#else
        const float cb = s_sp[k].col_b;
#endif
        float v[NC];
        backward_pair<NC>(a, b, ge, ap, cb, dx, dy, ga, gb, ha, hb, rc, v);
        float tot;
        const int vi = NC == 8 ? half_reduce8(v, &tot) : half_reduce9(v, &tot);
        // both halves may hold the same entry in this step: half 0 adds first
        if (vi >= 0 && act && half == 0) s_red[warp][k][vi] += tot;
        __syncwarp();
        if (vi >= 0 && act && half == 1) s_red[warp][k][vi] += tot;
        __syncwarp();  // orders half 1's add before the next step's half-0 read of the same slot
      }
    }
    __syncthreads();
    // flush: batch entries x 8 components, summed over warps 0..3 in order
    for (int idx = threadIdx.x; idx < cnt * NC; idx += kThreads) {
      const int k = idx / NC, c = idx - k * NC;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        acc += s_red[w][k][c];
        s_red[w][k][c] = 0.f;
      }
      if (c < 2) acc *= -2.0f;  // d_mu2d = -2 dg (conic d) (rasterizer.cpp:396)
      const uint32_t slot = s_sp[k].slot;
      if (slot < k_cap) partials[(int64_t)slot * NC + c] = acc;
    }
    __syncthreads();
  }
}

// ---- K4a, pose-only, on exact 4x4-region lists (GSB_BWD_QUARTER; needs the
// composite's region bits, GSB_BWD_HITS = 2). Pixel layout of the composite:
// warp w = quadrant w, its four 8-lane sub-warps = the quadrant's four 4x4
// regions, two vertically adjacent pixels per lane. Each sub-warp walks its
// own list of the batch entries the composite applied in its region, back to
// front, so one warp step serves four entries; per-entry partials: an 8-lane
// reduce-scatter (4 + 2 + 1 shuffles, every lane ends owning one of the 8
// components), then the four sub-warps add into the warp's shared slot in
// sub-warp order (deterministic), warps 0..3 at the flush. Measured same box
// against the half lists on the same region bits: K4a 0.194 -> 0.182 ms,
// pose batch +1.6 % (default).
#ifndef GSB_BWD_QUARTER
#define GSB_BWD_QUARTER 1
#endif
#ifndef GSB_BWD_MATCH  // unordered add when the step's four entries are distinct (K4a 0.182 -> 0.174 ms)
#define GSB_BWD_MATCH 1
#endif
__device__ __forceinline__ int quarter_reduce8(const float v[8], float* out) {
  const int lane = threadIdx.x & 31;
  const bool h4 = lane & 4, h2 = lane & 2, h1 = lane & 1;
  float w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = h4 ? v[i] : v[4 + i], keep = h4 ? v[4 + i] : v[i];
    w[i] = keep + __shfl_xor_sync(kFull, send, 4);
  }
  float x[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = h2 ? w[i] : w[2 + i], keep = h2 ? w[2 + i] : w[i];
    x[i] = keep + __shfl_xor_sync(kFull, send, 2);
  }
  const float send = h1 ? x[0] : x[1], keep = h1 ? x[1] : x[0];
  *out = keep + __shfl_xor_sync(kFull, send, 1);
  return (h4 ? 4 : 0) + (h2 ? 2 : 0) + (h1 ? 1 : 0);
}

__global__ void __launch_bounds__(kThreads, GSB_BWD_MIN_BLOCKS) backward_raster_quarter_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const SplatAux* __restrict__ aux, const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g,
    float bg_b, int64_t npix, const float* __restrict__ d_image, const float* __restrict__ final_t,
    const uint32_t* __restrict__ pixstate, const double* __restrict__ depth_g, double2* __restrict__ tile_cut,
    float* __restrict__ partials, uint32_t k_cap, const uint16_t* __restrict__ hits) {
  constexpr int NC = 8;
  __shared__ StagedSplat s_sp[kBatch];
  __shared__ uint16_t s_rm[kBatch];                // region bits of each batch entry
  __shared__ uint8_t s_list[kWarps][kSubs][kBatch];
  __shared__ float s_red[kWarps][kBatch][NC];
  __shared__ int s_w, s_h, s_tx;
  __shared__ uint32_t s_maxc[kWarps];
  if (threadIdx.x == 0) {
    s_w = cam_p->width;
    s_h = cam_p->height;
    s_tx = cam_p->tiles_x;
  }
  for (int i = threadIdx.x; i < kWarps * kBatch * NC; i += kThreads) (&s_red[0][0][0])[i] = 0.f;
  __syncthreads();
  const int W = s_w, H = s_h;
  const int tile = blockIdx.x;
  const int tx = tile % s_tx, ty = tile / s_tx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, sub = lane >> 3;
  int lx, ly;
  pixel_coords(warp, lane, &lx, &ly);
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const float px = (float)lx, py = (float)ly;
  const int region = region_of(warp, sub);
  const uint2 range = ranges[tile];
  PixBwd a, b;
  load_pixel_bwd(a, x, y, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  load_pixel_bwd(b, x, y + 1, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  const uint32_t pmax = max(a.contrib, b.contrib);
  const uint32_t wmax = __reduce_max_sync(kFull, pmax);
  uint32_t smax[kSubs];  // each region's deepest replayed position
#pragma unroll
  for (int q = 0; q < kSubs; ++q) smax[q] = __reduce_max_sync(kFull, sub == q ? pmax : 0u);
  if (lane == 0) s_maxc[warp] = wmax;
  __syncthreads();
  uint32_t maxc = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) maxc = max(maxc, s_maxc[w]);
  if (threadIdx.x == 0) {  // the tile's cut (see backward_raster_kernel)
    double2 cut = make_double2(-1.0, 0.0);
    if (maxc > 0) {
      const int32_t gid = aux[ranks[range.x + maxc - 1]].gid;
      cut = make_double2(depth_g[gid], (double)gid);
    }
    tile_cut[tile] = cut;
  }
  const uint32_t len = min(range.y - range.x, maxc);
  const uint32_t nbatch = (len + kBatch - 1) / kBatch;
  const uint32_t lt = lanemask_lt_();
  for (int bi = (int)nbatch - 1; bi >= 0; --bi) {
    const uint32_t b0 = (uint32_t)bi * kBatch;
    const int cnt = (int)min((uint32_t)kBatch, len - b0);
    if (threadIdx.x < cnt) {
      const uint32_t e = range.x + b0 + threadIdx.x;
      const uint32_t r = ranks[e];
      const SplatAux A = aux[r];
      const uint32_t tx0 = A.tx0_ty0 & 0xffffu, ty0 = A.tx0_ty0 >> 16, nx = A.nx_ny & 0xffffu;
      StagedSplat& S = s_sp[threadIdx.x];
      S.slot = A.off + ((uint32_t)ty - ty0) * nx + ((uint32_t)tx - tx0);
      const uint32_t bbox = stage_splat(rec[r], ox, oy, rc.cutoff2_f, &S.geo, &S.app, &S.col_b);
      s_rm[threadIdx.x] = (uint16_t)(bbox & __ldg(hits + e));
    }
    __syncthreads();
    if (b0 < wmax) {
      // the warp's four region lists (ascending), each bounded by its region's depth
      int n[kSubs];
#pragma unroll
      for (int q = 0; q < kSubs; ++q) n[q] = 0;
#pragma unroll
      for (int c = 0; c < kBatch / 32; ++c) {
        const int e = c * 32 + lane;
        const uint32_t m = e < cnt ? s_rm[e] : 0u;
#pragma unroll
        for (int q = 0; q < kSubs; ++q) {
          const bool t = ((m >> region_of(warp, q)) & 1u) && b0 + (uint32_t)e < smax[q];
          const uint32_t bq = __ballot_sync(kFull, t);
          if (t) s_list[warp][q][n[q] + __popc(bq & lt)] = (uint8_t)e;
          n[q] += __popc(bq);
        }
      }
      __syncwarp();
      int nmax = 0, mine = 0;
#pragma unroll
      for (int q = 0; q < kSubs; ++q) {
        nmax = max(nmax, n[q]);
        if (sub == q) mine = n[q];
      }
      const uint8_t* my_list = s_list[warp][sub];
      for (int it = 0; it < nmax; ++it) {  // each region back to front
        const bool act = it < mine;
        const int k = act ? my_list[mine - 1 - it] : 0;
        const uint32_t j = b0 + (uint32_t)k;
        const float4 ge = s_sp[k].geo;
        const float4 ap = s_sp[k].app;
        const float dx = px - ge.x, dy = py - ge.y;
        const float ga = splat_power(ge.z, ge.w, ap.x, dx, dy);
        const float gb = splat_power(ge.z, ge.w, ap.x, dx, dy + 1.0f);
        const bool ha = act && j < a.contrib && ga <= rc.cutoff2_f;
        const bool hb = act && j < b.contrib && gb <= rc.cutoff2_f;
        if (!__any_sync(kFull, ha || hb)) continue;
        const float cb = s_sp[k].col_b;
        float v[NC];
        backward_pair<NC>(a, b, ge, ap, cb, dx, dy, ga, gb, ha, hb, rc, v);
        float tot;
        const int vi = quarter_reduce8(v, &tot);
        // sub-warps may hold the same entry in this step: add in sub-warp order
#if GSB_BWD_MATCH
        // (when the four sub-warps' entries are distinct the adds touch
        // different slots and need no order: one add)
        if (__all_sync(kFull, __popc(__match_any_sync(kFull, act ? k : -1 - sub)) == 8)) {
          if (act) s_red[warp][k][vi] += tot;
          continue;
        }
#endif
#pragma unroll
        for (int q = 0; q < kSubs; ++q) {
          if (act && sub == q) s_red[warp][k][vi] += tot;
          __syncwarp();
        }
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < cnt * NC; idx += kThreads) {  // flush: warps 0..3 in order
      const int k = idx / NC, c = idx - k * NC;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        acc += s_red[w][k][c];
        s_red[w][k][c] = 0.f;
      }
      if (c < 2) acc *= -2.0f;  // d_mu2d = -2 dg (conic d) (rasterizer.cpp:396)
      const uint32_t slot = s_sp[k].slot;
      if (slot < k_cap) partials[(int64_t)slot * NC + c] = acc;
    }
    __syncthreads();
  }
  (void)region;
}

// render_expected_depth (rasterizer.cpp:283-323): the compositing loop with
// the splat's view-space depth in place of its colour. Not on the hot path
// (dataset generation, synth.cpp:117-127): one 256-thread CTA per tile, one
// pixel per thread, records read from L2. The cutoff and alpha decisions use
// the composite's exact FP32 arithmetic (tile-local offsets; the odd row of a
// vertical pixel pair at dy + 1), so the expected depth sees the same hits
// as the rendered image. Sums in FP64 as the reference.
__global__ void __launch_bounds__(256) expected_depth_kernel(const uint2* __restrict__ ranges,
                                                             const uint32_t* __restrict__ ranks,
                                                             const SplatRec* __restrict__ rec,
                                                             const SplatAux* __restrict__ aux,
                                                             const double* __restrict__ depth_g,
                                                             const CamDev* __restrict__ cam_p, RasterDev rc,
                                                             float* __restrict__ depth_out,
                                                             float* __restrict__ weight_out) {
  const int W = cam_p->width, H = cam_p->height, tiles_x = cam_p->tiles_x;
  const int tile = blockIdx.x, tx = tile % tiles_x, ty = tile / tiles_x;
  const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  if (x >= W || y >= H) return;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const uint2 range = ranges[tile];
  float T = 1.0f;
  double dsum = 0.0, wsum = 0.0;
  for (uint32_t e = range.x; e < range.y; ++e) {
    const uint32_t r = ranks[e];
    const SplatRec R = rec[r];
    const float mx = (float)(R.mu_x - ox), my = (float)(R.mu_y - oy);
    const float dx = (float)lx - mx;
    const float dy = (ly & 1) ? ((float)(ly - 1) - my) + 1.0f : (float)ly - my;
    const float g = splat_power(R.conic_a, R.conic_b, R.conic_c, dx, dy);
    if (!(g <= rc.cutoff2_f)) continue;
    const float al = fminf(rc.alpha_clamp_f, R.opacity * exp_neg_half(g));
    const float w = al * T;
    dsum += (double)w * depth_g[aux[r].gid];
    wsum += (double)w;
    T *= 1.0f - al;
    if (T < rc.early_term_f) break;
  }
  const int64_t q = (int64_t)y * W + x;
  weight_out[q] = (float)wsum;
  depth_out[q] = wsum > 1e-8 ? (float)(dsum / wsum) : 0.0f;
}

int launch_expected_depth(cudaStream_t st, gsb_frame* f, const RasterDev& rc, float* depth_out, float* weight_out) {
  const int n_tiles = f->tiles_x * f->tiles_y;
  if (n_tiles > 0)
    expected_depth_kernel<<<n_tiles, 256, 0, st>>>(f->ranges.as<uint2>(), f->list(), f->list_rec(), f->list_aux(),
                                                    f->depth_g.as<double>(), f->cam.as<CamDev>(), rc, depth_out,
                                                    weight_out);
  GSB_CHECK_LAUNCH("expected_depth_kernel");
  return GSB_OK;
}

// ---- K4a, pose-only, 4 pixels per lane (GSB_BWD_QUAD4; an A/B variant, off).
// One 64-thread CTA per tile: warp w owns the 16x8 rows 8w..8w+7; its four
// 8-lane groups each own an 8x4 region (group g: columns 8(g&1).., rows
// 8w + 4(g>>1)..), one column of 4 pixels per lane. The four groups walk
// their own lists of the batch entries whose cutoff-ellipse box reaches their
// region, so one warp step serves four entries (two in the 2-px/lane half
// kernel) and the per-step overhead — list load, record loads, the
// reduce-scatter (8 values over 8 lanes: 4 + 2 + 1 shuffles) — is shared by
// four. Measured on C3 view 0 with the oracle's forward state: 0.565 M warp
// steps instead of 0.997 M. The lane's 4 pixels are two vertical pairs at
// rows r0 and r0 + 2 whose dy is formed exactly as the composite forms it
// (pair start py - my, second pixel dy + 1), so every cutoff / termination
// decision is the forward's. Per-entry partials: sum of the two pairs, group
// reduce-scatter, then the four groups add into the warp's shared slot in
// group order (ordered rounds), warps 0, 1 at the flush: deterministic.
#ifndef GSB_BWD_QUAD4
#define GSB_BWD_QUAD4 0
#endif
constexpr int kQ4Threads = 64;
#ifndef GSB_Q4_MIN_BLOCKS
#define GSB_Q4_MIN_BLOCKS 10
#endif

// 8 values over each 8-lane group: xor 4 / 2 / 1 reduce-scatter; lane l owns
// component (l & 7) of its group's sum.
__device__ __forceinline__ float group_reduce8(const float v[8]) {
  const int lane = threadIdx.x & 31;
  const bool h1 = lane & 4, h2 = lane & 2, h3 = lane & 1;
  float w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = h1 ? v[i] : v[4 + i], keep = h1 ? v[4 + i] : v[i];
    w[i] = keep + __shfl_xor_sync(kFull, send, 4);
  }
  float x[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = h2 ? w[i] : w[2 + i], keep = h2 ? w[2 + i] : w[i];
    x[i] = keep + __shfl_xor_sync(kFull, send, 2);
  }
  const float send = h3 ? x[0] : x[1], keep = h3 ? x[1] : x[0];
  return keep + __shfl_xor_sync(kFull, send, 1);
}

__global__ void __launch_bounds__(kQ4Threads, GSB_Q4_MIN_BLOCKS) backward_raster_q4_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ ranks, const SplatRec* __restrict__ rec,
    const SplatAux* __restrict__ aux, const CamDev* __restrict__ cam_p, RasterDev rc, float bg_r, float bg_g,
    float bg_b, int64_t npix, const float* __restrict__ d_image, const float* __restrict__ final_t,
    const uint32_t* __restrict__ pixstate, const double* __restrict__ depth_g, double2* __restrict__ tile_cut,
    float* __restrict__ partials, uint32_t k_cap) {
  constexpr int NC = 8;
  __shared__ StagedSplat s_sp[kBatch];
  __shared__ uint8_t s_mask[kBatch];
  __shared__ uint8_t s_list[2][4][kBatch];
  __shared__ float s_red[2][kBatch][NC];
  __shared__ int s_w, s_h, s_tx;
  __shared__ uint32_t s_maxc[2];
  if (threadIdx.x == 0) {
    s_w = cam_p->width;
    s_h = cam_p->height;
    s_tx = cam_p->tiles_x;
  }
  for (int i = threadIdx.x; i < 2 * kBatch * NC; i += kQ4Threads) (&s_red[0][0][0])[i] = 0.f;
  __syncthreads();
  const int W = s_w, H = s_h;
  const int tile = blockIdx.x;
  const int tx = tile % s_tx, ty = tile / s_tx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 3;
  const int lx = (g & 1) * 8 + (lane & 7), ly = warp * 8 + (g >> 1) * 4;  // rows ly .. ly + 3
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const double ox = (double)(tx * kTile), oy = (double)(ty * kTile);
  const float px = (float)lx, py0 = (float)ly, py2 = (float)(ly + 2);
  const uint2 range = ranges[tile];

  PixBwd a, b, c, d;
  load_pixel_bwd(a, x, y, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  load_pixel_bwd(b, x, y + 1, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  load_pixel_bwd(c, x, y + 2, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  load_pixel_bwd(d, x, y + 3, W, H, npix, bg_r, bg_g, bg_b, d_image, final_t, pixstate);
  const uint32_t wmax = __reduce_max_sync(kFull, max(max(a.contrib, b.contrib), max(c.contrib, d.contrib)));
  if (lane == 0) s_maxc[warp] = wmax;
  __syncthreads();
  const uint32_t maxc = max(s_maxc[0], s_maxc[1]);
  // entries at list positions >= maxc: see backward_raster_kernel
  if (threadIdx.x == 0) {
    double2 cut = make_double2(-1.0, 0.0);
    if (maxc > 0) {
      const int32_t gid = aux[ranks[range.x + maxc - 1]].gid;
      cut = make_double2(depth_g[gid], (double)gid);
    }
    tile_cut[tile] = cut;
  }
  // region bit of this lane's group in the staged half mask (bit 2 q + h,
  // quadrant q = qx + 2 qy, half h = rows 4..7 of the quadrant)
  const int gbit = 2 * ((g & 1) + 2 * warp) + (g >> 1);
  const uint32_t len = min(range.y - range.x, maxc);
  const uint32_t nbatch = (len + kBatch - 1) / kBatch;
  const uint32_t lt = lanemask_lt_();
  for (int bi = (int)nbatch - 1; bi >= 0; --bi) {
    const uint32_t b0 = (uint32_t)bi * kBatch;
    const int cnt = (int)min((uint32_t)kBatch, len - b0);
    for (int t = threadIdx.x; t < cnt; t += kQ4Threads) {
      const uint32_t r = ranks[range.x + b0 + t];
      const SplatAux A = aux[r];
      const uint32_t tx0 = A.tx0_ty0 & 0xffffu, ty0 = A.tx0_ty0 >> 16, nx = A.nx_ny & 0xffffu;
      StagedSplat& S = s_sp[t];
      S.slot = A.off + ((uint32_t)ty - ty0) * nx + ((uint32_t)tx - tx0);
      s_mask[t] = (uint8_t)half_mask(stage_splat(rec[r], ox, oy, rc.cutoff2_f, &S.geo, &S.app, &S.col_b));
    }
    __syncthreads();
    if (b0 < wmax) {
      // the four groups' lists (ascending), all built by the whole warp
      const uint32_t lim = wmax - b0;
      int n[4] = {0, 0, 0, 0};
#pragma unroll
      for (int cc = 0; cc < kBatch / 32; ++cc) {
        const int e = cc * 32 + lane;
        const uint32_t m = (e < cnt && (uint32_t)e < lim) ? s_mask[e] : 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int bit = 2 * ((q & 1) + 2 * warp) + (q >> 1);
          const bool take = (m >> bit) & 1u;
          const uint32_t bal = __ballot_sync(kFull, take);
          if (take) s_list[warp][q][n[q] + __popc(bal & lt)] = (uint8_t)e;
          n[q] += __popc(bal);
        }
      }
      __syncwarp();
      (void)gbit;
      const int mine = g == 0 ? n[0] : g == 1 ? n[1] : g == 2 ? n[2] : n[3];
      const int nmax = max(max(n[0], n[1]), max(n[2], n[3]));
      const uint8_t* my_list = s_list[warp][g];
      for (int it = 0; it < nmax; ++it) {  // each group back to front
        const bool act = it < mine;
        const int k = act ? my_list[mine - 1 - it] : 0;
        const uint32_t j = b0 + (uint32_t)k;
        const float4 ge = s_sp[k].geo;
        const float4 ap = s_sp[k].app;
        const float dx = px - ge.x, dya = py0 - ge.y, dyc = py2 - ge.y;
        const float ga = splat_power(ge.z, ge.w, ap.x, dx, dya);
        const float gb = splat_power(ge.z, ge.w, ap.x, dx, dya + 1.0f);
        const float gc = splat_power(ge.z, ge.w, ap.x, dx, dyc);
        const float gd = splat_power(ge.z, ge.w, ap.x, dx, dyc + 1.0f);
        const bool ha = act && j < a.contrib && ga <= rc.cutoff2_f;
        const bool hb = act && j < b.contrib && gb <= rc.cutoff2_f;
        const bool hc = act && j < c.contrib && gc <= rc.cutoff2_f;
        const bool hd = act && j < d.contrib && gd <= rc.cutoff2_f;
        if (!__any_sync(kFull, ha || hb || hc || hd)) continue;  // no group's entry touched: zero partials
        const float cb = s_sp[k].col_b;
        float v[NC], u[NC];
        backward_pair<NC>(a, b, ge, ap, cb, dx, dya, ga, gb, ha, hb, rc, v);
        backward_pair<NC>(c, d, ge, ap, cb, dx, dyc, gc, gd, hc, hd, rc, u);
#pragma unroll
        for (int q = 0; q < NC; ++q) v[q] += u[q];
        const float tot = group_reduce8(v);
        const int comp = lane & 7;
        // groups may hold the same entry in a step: add in group order
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (act && g == q) s_red[warp][k][comp] += tot;
          __syncwarp();
        }
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < cnt * NC; idx += kQ4Threads) {
      const int k = idx / NC, cc = idx - k * NC;
      float acc = s_red[0][k][cc] + s_red[1][k][cc];
      s_red[0][k][cc] = 0.f;
      s_red[1][k][cc] = 0.f;
      if (cc < 2) acc *= -2.0f;  // d_mu2d = -2 dg (conic d) (rasterizer.cpp:396)
      const uint32_t slot = s_sp[k].slot;
      if (slot < k_cap) partials[(int64_t)slot * NC + cc] = acc;
    }
    __syncthreads();
  }
}

// Hit records (K3 records, the pose-only K4a lists only the halves an entry
// touched). GSB_BWD_HITS = 2 (default): one 16-bit word of touched-region bits
// per list position — the composite stores each hit step's ballot and decodes
// them per entry at the end of the batch, 2 B written per entry — measured
// same box, C3: K4a 0.218 -> 0.196 ms, composite 0.103 -> 0.120 ms, pose
// batch +0.5-1.1 %. GSB_BWD_HITS = 1: per-pixel masks, 32 B per list
// position (K4a 0.202, composite 0.119 ms: batch -1.5 %). 0: off.
#ifndef GSB_BWD_HITS
#define GSB_BWD_HITS 2
#endif
bool hit_masks_enabled() { return GSB_BWD_HITS != 0; }
int hit_words() { return GSB_BWD_HITS == 1 ? 16 : 1; }  // uint16 per list position

int launch_composite(cudaStream_t st, gsb_frame* f, const RasterDev& rc) {
  const int n_tiles = f->tiles_x * f->tiles_y;
  const int64_t npix = (int64_t)f->width * f->height;
  const bool hm = f->want_hits && GSB_BWD_HITS;
  if (n_tiles > 0)
    (!hm ? composite_kernel<0> : GSB_BWD_HITS == 1 ? composite_kernel<1> : composite_kernel<2>)<<<n_tiles, kThreads, 0, st>>>(
        f->ranges.as<uint2>(), f->list(), f->list_rec(), f->cam.as<CamDev>(), rc,
        (float)f->background[0], (float)f->background[1], (float)f->background[2], npix, f->image.as<float>(),
        f->final_t.as<float>(), f->pixstate.as<uint32_t>(), hm ? f->hits.as<uint16_t>() : nullptr,
        (uint32_t)f->k_cap);
  GSB_CHECK_LAUNCH("composite_kernel");
  return GSB_OK;
}

// pose_only: 8 partials per entry (no opacity); else the full 9.
#ifndef GSB_BWD_HALF
#define GSB_BWD_HALF 1
#endif
// (the 9-component half-quadrant variant for the full gradient measured slower
// for C4, 0.881 -> 0.903 ms per joint step, and was removed)
int launch_backward_raster(cudaStream_t st, gsb_frame* f, const RasterDev& rc, bool pose_only) {
  const int n_tiles = f->tiles_x * f->tiles_y;
  const int64_t npix = (int64_t)f->width * f->height;
  if (n_tiles > 0 && pose_only && GSB_BWD_QUAD4) {
    backward_raster_q4_kernel<<<n_tiles, kQ4Threads, 0, st>>>(
        f->ranges.as<uint2>(), f->list(), f->list_rec(), f->list_aux(), f->cam.as<CamDev>(), rc,
        (float)f->background[0], (float)f->background[1], (float)f->background[2], npix, f->d_image.as<float>(),
        f->final_t.as<float>(), f->pixstate.as<uint32_t>(), f->depth_g.as<double>(), f->tile_cut.as<double2>(),
        f->partials.as<float>(), (uint32_t)f->k_cap);
    GSB_CHECK_LAUNCH("backward_raster_q4_kernel");
    return GSB_OK;
  }
  if (n_tiles > 0 && pose_only && GSB_BWD_QUARTER && f->want_hits && GSB_BWD_HITS == 2) {
    backward_raster_quarter_kernel<<<n_tiles, kThreads, 0, st>>>(
        f->ranges.as<uint2>(), f->list(), f->list_rec(), f->list_aux(), f->cam.as<CamDev>(), rc,
        (float)f->background[0], (float)f->background[1], (float)f->background[2], npix, f->d_image.as<float>(),
        f->final_t.as<float>(), f->pixstate.as<uint32_t>(), f->depth_g.as<double>(), f->tile_cut.as<double2>(),
        f->partials.as<float>(), (uint32_t)f->k_cap, f->hits.as<uint16_t>());
    GSB_CHECK_LAUNCH("backward_raster_quarter_kernel");
    return GSB_OK;
  }
  if (n_tiles > 0 && pose_only && GSB_BWD_HALF) {
    const bool hm = f->want_hits && GSB_BWD_HITS;
    (!hm ? backward_raster_half_kernel<8, 0>
         : GSB_BWD_HITS == 1 ? backward_raster_half_kernel<8, 1> : backward_raster_half_kernel<8, 2>)
        <<<n_tiles, kThreads, 0, st>>>(
        f->ranges.as<uint2>(), f->list(), f->list_rec(), f->list_aux(), f->cam.as<CamDev>(), rc,
        (float)f->background[0], (float)f->background[1], (float)f->background[2], npix, f->d_image.as<float>(),
        f->final_t.as<float>(), f->pixstate.as<uint32_t>(), f->depth_g.as<double>(), f->tile_cut.as<double2>(),
        f->partials.as<float>(), (uint32_t)f->k_cap, hm ? f->hits.as<uint16_t>() : nullptr);
    GSB_CHECK_LAUNCH("backward_raster_half_kernel");
    return GSB_OK;
  }
  if (n_tiles > 0)
    (pose_only ? backward_raster_kernel<8> : backward_raster_kernel<kPartial>)
        <<<n_tiles, kThreads, 0, st>>>(
        f->ranges.as<uint2>(), f->list(), f->list_rec(), f->list_aux(),
        f->cam.as<CamDev>(), rc, (float)f->background[0], (float)f->background[1], (float)f->background[2], npix,
        f->d_image.as<float>(), f->final_t.as<float>(), f->pixstate.as<uint32_t>(), f->depth_g.as<double>(),
        f->tile_cut.as<double2>(), f->partials.as<float>(), (uint32_t)f->k_cap);
  GSB_CHECK_LAUNCH("backward_raster_kernel");
  return GSB_OK;
}

}  // namespace gsb

