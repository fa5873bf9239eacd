// k_loss.cu — K6: fused photometric loss (1-beta) L1 + beta (1 - SSIM) with
// its analytic image gradient, on planar FP32 images, FP64 accumulation.
//
// Reference: rgb_loss (losses.cpp:201-215) <- l1_core (158-192),
// ssim_core (74-155), conv_window (37-63), gaussian_window (19-32).
// SSIM uses the 11x11 sigma 1.5 separable window with zero padding, C1 =
// 1e-4, C2 = 9e-4, averaged over pixels where the window fits, x,y in
// [5, dim-5) (losses.cpp:78-79); its gradient back-convolves the three
// per-pixel maps g_mu, g_eaa, g_eab (144-151). The factored gradient
// expressions of the reference are kept so identical images give exactly
// zero loss and gradient.
//
// Two tiled kernels (32x32 outputs + 5 px halo staged in shared memory,
// register-blocked separable passes: each thread computes 4 consecutive
// outputs from 14 inputs held in registers):
//   loss_maps:  5 forward convolutions -> SSIM map sum, L1 sum, g maps;
//   loss_grad:  3 back-convolutions + L1 sign term -> d_image.
// The separable convolutions run in FP32 (the images are FP32; the window is
// the reference's FP64 window rounded once), the pointwise SSIM terms, the
// L1 terms and every sum in FP64. Per-block partial sums are reduced in a
// fixed order (deterministic). FP32 convolutions keep the identical-image
// identities exact: equal inputs give bitwise-equal statistics, and
// conv(-x) = -conv(x), conv(2x) = 2 conv(x) hold exactly in any precision.
#include <cstring>
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point; no libcuda link)

#include "gsb_internal.cuh"

namespace gsb {

constexpr int kHalf = 5;
constexpr int kWin = 11;
// Register-blocked tiles: 32x32 outputs per 256-thread CTA, every thread
// producing R = 4 consecutive outputs per pass (the 14 inputs they share are
// loaded once into registers), 42x42 staged inputs.
constexpr int kTW = 32, kTH = 32, kR = 4;
constexpr int kSW = kTW + 2 * kHalf, kSH = kTH + 2 * kHalf;  // 42 x 42
constexpr int kThr = 256;
__constant__ float c_win[kWin];

// Transmittance mask of masked_rgb_loss (losses.cpp:259-289): pixel p takes
// part iff accum = 1 - final_T > thr; norms (device) = {L1 norm, SSIM scale,
// masked count, masked valid-window count} from mask_count / mask_norms.
struct MaskArgs {
  const float* final_t;  // nullptr: unmasked rgb_loss (host norms)
  double thr;
  const double* norms;
};
__device__ __forceinline__ bool mask_at(const MaskArgs& m, int64_t p) {
  return !m.final_t || (1.0 - (double)m.final_t[p]) > m.thr;
}

__device__ __forceinline__ double m_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double s_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double d_(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ double blk_reduce_sum(double v, double* s_tmp) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s_tmp[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_tmp[w];
  __syncthreads();
  return t;  // valid in thread 0
}

// Stages a (kSH x kSW) window of NM FP32 planes starting at (gx0, gy0),
// zero outside the image (conv_window's zero padding, losses.cpp:37-63).
// All of a thread's loads are issued before its first shared store, so the
// ~7 x NM global loads per thread are in flight together.
template <int NM>
__device__ __forceinline__ void stage_planes(float (*dst)[kSH][kSW + 1], const float* const* src, int W, int H,
                                             int gx0, int gy0) {
  constexpr int kIt = (kSH * kSW + kThr - 1) / kThr;
  float v[kIt][NM];
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int idx = it * kThr + threadIdx.x;
    const int r = idx / kSW, q = idx - r * kSW;
    const int gx = gx0 + q, gy = gy0 + r;
    const bool ok = idx < kSH * kSW && gx >= 0 && gx < W && gy >= 0 && gy < H;
    const int64_t p = ok ? (int64_t)gy * W + gx : 0;
#pragma unroll
    for (int m = 0; m < NM; ++m) v[it][m] = ok ? __ldg(src[m] + p) : 0.f;
  }
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int idx = it * kThr + threadIdx.x;
    if (idx < kSH * kSW) {
      const int r = idx / kSW, q = idx - r * kSW;
#pragma unroll
      for (int m = 0; m < NM; ++m) dst[m][r][q] = v[it][m];
    }
  }
}

// Horizontal pass of the five SSIM statistics (a, b, a^2, b^2, ab) over the
// staged rows: task = (row, HR-column group). Every output sums its 11 taps in
// the same order whatever HR is (bit-identical); HR = 2 gives 42 x 16 = 672
// tasks = 2.6 rounds of 256 threads instead of 336 = 1.3 rounds at HR = 4.
#ifndef GSB_LOSS_HR
#define GSB_LOSS_HR 4
#endif
constexpr int kHR = GSB_LOSS_HR;
template <int PITCH, int XOFF>
__device__ __forceinline__ void hpass5(const float* __restrict__ st0, const float* __restrict__ st1,
                                       float (*hq)[kSH][kTW + 1]) {
  for (int task = threadIdx.x; task < kSH * (kTW / kHR); task += kThr) {
    const int r = task / (kTW / kHR), q0 = (task - r * (kTW / kHR)) * kHR;
    float x[kHR + kWin - 1], y[kHR + kWin - 1];
#pragma unroll
    for (int k = 0; k < kHR + kWin - 1; ++k) {
      x[k] = st0[r * PITCH + XOFF + q0 + k];
      y[k] = st1[r * PITCH + XOFF + q0 + k];
    }
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      float acc[kHR];
#pragma unroll
      for (int j = 0; j < kHR; ++j) acc[j] = 0.f;
#pragma unroll
      for (int k = 0; k < kHR + kWin - 1; ++k) {
        const float f = m == 0 ? x[k] : m == 1 ? y[k] : m == 2 ? x[k] * x[k] : m == 3 ? y[k] * y[k] : x[k] * y[k];
#pragma unroll
        for (int j = 0; j < kHR; ++j)
          if (k - j >= 0 && k - j < kWin) acc[j] = fmaf(c_win[k - j], f, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < kHR; ++j) hq[m][r][q0 + j] = acc[j];
    }
  }
}

#ifndef GSB_LOSS_RCP
#define GSB_LOSS_RCP 1
#endif
#ifdef GSB_LOSS_MIN_BLOCKS
#define GSB_LOSS_BOUNDS __launch_bounds__(kThr, GSB_LOSS_MIN_BLOCKS)
#else
#define GSB_LOSS_BOUNDS __launch_bounds__(kThr)
#endif
// TMA staging (kTma): the windows of channel c + 1 are loaded by the tensor
// memory accelerator (3-D tensor maps over the planar images, box 44 x 42 x
// 1, out-of-bounds elements zero-filled = conv_window's zero padding) into a
// second buffer while channel c is convolved; one mbarrier per buffer.
// The box starts 8 columns left of the tile (a 16-byte aligned inner
// coordinate, as the tensor unit requires; measured: a start at -5 columns
// faults) and is 48 wide, so the 5-px halo window sits at column offset 3.
constexpr int kTP = 48;                        // TMA window pitch (floats; 192 B rows)
constexpr int kTX = 3;                         // column of the halo window inside the box
constexpr uint32_t kTWinBytes = kSH * kTP * 4u;  // bytes one TMA window load delivers (8064)
constexpr int kTWin = (kSH * kTP + 31) / 32 * 32;  // window stride in shared memory: 128-byte aligned destinations
// TMA window buffers per kernel: 2 = the next channel's windows load into the
// other buffer while this one is convolved; 1 = one buffer, reloaded as soon
// as the horizontal pass has consumed it (less shared memory: one more CTA
// per SM)
#ifndef GSB_LOSS_TMA_BUFS
#define GSB_LOSS_TMA_BUFS 1  // (2: same K6 time, 16 KB more shared memory per CTA)
#endif
constexpr int kBufs = GSB_LOSS_TMA_BUFS;
// GSB_LOSS_CH_SPLIT: one CTA per (tile, channel) (grid z = channel) instead of
// one per tile looping over the channels: 3x the CTAs, so the last wave is a
// small fraction of the launch (768 tile CTAs on 3-4 resident per SM leave
// the second wave ~70 % empty). Measured: K6 alone 0.061 -> 0.057 ms, but the
// pose batch, whose other branches already fill the tail, loses 0.7 % — off.
#ifndef GSB_LOSS_CH_SPLIT
#define GSB_LOSS_CH_SPLIT 0
#endif
constexpr bool kChSplit = GSB_LOSS_CH_SPLIT != 0;

__device__ __forceinline__ void tma_load_3d(float* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct LossMaps {  // tensor maps of the TMA path (unused otherwise)
  CUtensorMap ren, tgt, gm;
};

template <bool kTma>
__global__ void GSB_LOSS_BOUNDS loss_maps_kernel(const float* __restrict__ ren, const float* __restrict__ tgt,
                                                 int W, int H, double scale, float* __restrict__ gmaps,
                                                 double* __restrict__ block_sums, MaskArgs mk,
                                                 const __grid_constant__ LossMaps tm) {
  if (mk.final_t) scale = mk.norms[1];
  constexpr int PITCH = kTma ? kTP : kSW + 1;
  constexpr int WIN = kTma ? kTWin : kSH * (kSW + 1);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* win = reinterpret_cast<float*>(smem_raw);  // [buffers][2 planes][WIN]
  float(*hq)[kSH][kTW + 1] =
      reinterpret_cast<float(*)[kSH][kTW + 1]>(smem_raw + sizeof(float) * (kTma ? 2 * kBufs : 2) * WIN);
  __shared__ double s_tmp[kThr / 32];
  __shared__ __align__(8) uint64_t bar[2];
  const int64_t P = (int64_t)W * H;
  const int bx = blockIdx.x * kTW, by = blockIdx.y * kTH;
  const int ch0 = kChSplit ? (int)blockIdx.z : 0, ch_end = kChSplit ? ch0 + 1 : 3;
  if (kTma && threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_expect_tx(&bar[0], 2 * kTWinBytes);
    tma_load_3d(win, &tm.ren, bx - kHalf - kTX, by - kHalf, ch0, &bar[0]);
    tma_load_3d(win + kTWin, &tm.tgt, bx - kHalf - kTX, by - kHalf, ch0, &bar[0]);
  }
  if (kTma) __syncthreads();  // barrier initialisation visible to every waiting thread
  // vertical task: column c, rows 4 rg .. 4 rg + 3
  const int c = threadIdx.x & (kTW - 1), rg = threadIdx.x / kTW;
  const int x = bx + c;
  double l1 = 0.0, ss = 0.0;
  for (int ch = ch0; ch < ch_end; ++ch) {
    const int it = ch - ch0;  // channel iteration of this CTA (buffer / phase index)
    const float* st0;
    if (kTma && kBufs == 1) {
      mbar_wait(&bar[0], (uint32_t)(it & 1));
      st0 = win;
    } else if (kTma) {
      if (threadIdx.x == 0 && ch + 1 < ch_end) {  // next channel into the other buffer
        float* nb = win + ((it + 1) & 1) * 2 * kTWin;
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[(it + 1) & 1], 2 * kTWinBytes);
        tma_load_3d(nb, &tm.ren, bx - kHalf - kTX, by - kHalf, ch + 1, &bar[(it + 1) & 1]);
        tma_load_3d(nb + kTWin, &tm.tgt, bx - kHalf - kTX, by - kHalf, ch + 1, &bar[(it + 1) & 1]);
      }
      mbar_wait(&bar[it & 1], (uint32_t)(it >> 1));
      st0 = win + (it & 1) * 2 * kTWin;
    } else {
      const float* src[2] = {ren + ch * P, tgt + ch * P};
      stage_planes<2>(reinterpret_cast<float(*)[kSH][kSW + 1]>(win), src, W, H, bx - kHalf, by - kHalf);
      __syncthreads();
      st0 = win;
    }
    const float* st1 = st0 + WIN;
    hpass5<PITCH, kTma ? kTX : 0>(st0, st1, hq);
    float av[kR], bv[kR];  // this thread's output pixels of both images
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int o = (rg * kR + j + kHalf) * PITCH + (kTma ? kTX : 0) + c + kHalf;
      av[j] = st0[o];
      bv[j] = st1[o];
    }
    __syncthreads();
    if (kTma && kBufs == 1 && threadIdx.x == 0 && ch + 1 < ch_end) {  // window consumed: next channel into it
      fence_proxy_async();
      mbar_arrive_expect_tx(&bar[0], 2 * kTWinBytes);
      tma_load_3d(win, &tm.ren, bx - kHalf - kTX, by - kHalf, ch + 1, &bar[0]);
      tma_load_3d(win + kTWin, &tm.tgt, bx - kHalf - kTX, by - kHalf, ch + 1, &bar[0]);
    }
    float mv[5][kR];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      float acc[kR];
#pragma unroll
      for (int j = 0; j < kR; ++j) acc[j] = 0.f;
#pragma unroll
      for (int k = 0; k < kR + kWin - 1; ++k) {
        const float f = hq[m][rg * kR + k][c];
#pragma unroll
        for (int j = 0; j < kR; ++j)
          if (k - j >= 0 && k - j < kWin) acc[j] = fmaf(c_win[k - j], f, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < kR; ++j) mv[m][j] = acc[j];
    }
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int y = by + rg * kR + j;
      if (x >= W || y >= H) continue;
      const double a = av[j], b = bv[j];
      const int64_t p = (int64_t)y * W + x;
      const bool in_mask = mask_at(mk, p);
      if (in_mask) l1 += fabs(a - b);
      if (in_mask && x >= kHalf && x < W - kHalf && y >= kHalf && y < H - kHalf) {
        const double ma = mv[0][j], mb = mv[1][j], eaa = mv[2][j], ebb = mv[3][j], eab = mv[4][j];
        // Pointwise SSIM terms with explicitly rounded (unfused) arithmetic in
        // the reference's expression order, so identical inputs cancel exactly
        // (a1 == b1, a2 == b2, s == 1 and a zero gradient; losses.cpp:112-131).
        const double C1 = 1e-4, C2 = 9e-4;
        const double va = s_(eaa, m_(ma, ma)), vb = s_(ebb, m_(mb, mb)), vab = s_(eab, m_(ma, mb));
        const double a1 = a_(m_(m_(2.0, ma), mb), C1), a2 = a_(m_(2.0, vab), C2);
        const double b1 = a_(a_(m_(ma, ma), m_(mb, mb)), C1), b2 = a_(a_(va, vb), C2);
        const double b12 = m_(b1, b2);
#if GSB_LOSS_RCP
        // one correctly rounded reciprocal instead of four divisions: the
        // quotients move by an ulp or two (against FP32 statistics), and the
        // two ratios identical inputs make exactly 1 (a1 a2 / b12, a2 / b2)
        // are pinned to 1 on equality, so they still cancel exactly
        const double r12 = __drcp_rn(b12), n12 = m_(a1, a2);
        const double s = n12 == b12 ? 1.0 : m_(n12, r12);
        ss += s;
        const double gmu = m_(m_(scale, a_(m_(m_(2.0, mb), s_(a2, a1)), m_(m_(m_(2.0, ma), s), s_(b1, b2)))), r12);
        const double qv = m_(a1, r12);
        const double a2b2 = a2 == b2 ? 1.0 : m_(m_(a2, b1), r12);
#else
        const double s = d_(m_(a1, a2), b12);
        ss += s;
        const double gmu = d_(m_(scale, a_(m_(m_(2.0, mb), s_(a2, a1)), m_(m_(m_(2.0, ma), s), s_(b1, b2)))), b12);
        const double qv = d_(a1, b12);
        const double a2b2 = d_(a2, b2);
#endif
        gmaps[(3 * ch + 0) * P + p] = (float)gmu;
        gmaps[(3 * ch + 1) * P + p] = (float)m_(-m_(scale, qv), a2b2);
        gmaps[(3 * ch + 2) * P + p] = (float)m_(2.0, m_(scale, qv));
      } else {
        gmaps[(3 * ch + 0) * P + p] = 0.f;
        gmaps[(3 * ch + 1) * P + p] = 0.f;
        gmaps[(3 * ch + 2) * P + p] = 0.f;
      }
    }
    __syncthreads();
  }
  const double t1 = blk_reduce_sum(l1, s_tmp);
  const double t2 = blk_reduce_sum(ss, s_tmp);
  if (threadIdx.x == 0) {
    const int bidx = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    block_sums[2 * bidx] = t1;
    block_sums[2 * bidx + 1] = t2;
  }
}

// Horizontal pass of the three gradient maps (back-convolution, losses.cpp:144-151).
template <int PITCH, int XOFF>
__device__ __forceinline__ void hpass3(const float* __restrict__ st, int plane_stride, float (*hq)[kSH][kTW + 1]) {
  for (int task = threadIdx.x; task < kSH * (kTW / kHR); task += kThr) {
    const int r = task / (kTW / kHR), q0 = (task - r * (kTW / kHR)) * kHR;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      float acc[kHR];
#pragma unroll
      for (int j = 0; j < kHR; ++j) acc[j] = 0.f;
#pragma unroll
      for (int k = 0; k < kHR + kWin - 1; ++k) {
        const float f = st[m * plane_stride + r * PITCH + XOFF + q0 + k];
#pragma unroll
        for (int j = 0; j < kHR; ++j)
          if (k - j >= 0 && k - j < kWin) acc[j] = fmaf(c_win[k - j], f, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < kHR; ++j) hq[m][r][q0 + j] = acc[j];
    }
  }
}

// 4 CTAs/SM (64 registers, 48 B of spills; 55 KB shared each): the kernel is
// load-latency bound, and in a pose batch the extra resident CTAs of the
// other branches fill in (measured: batch +3.8 % over the default 2 CTAs/SM)
#ifndef GSB_LOSS_GRAD_MIN_BLOCKS
#define GSB_LOSS_GRAD_MIN_BLOCKS 4
#endif
#define GSB_LOSS_GRAD_BOUNDS __launch_bounds__(kThr, GSB_LOSS_GRAD_MIN_BLOCKS)
template <bool kTma>
__global__ void GSB_LOSS_GRAD_BOUNDS loss_grad_kernel(const float* __restrict__ ren, const float* __restrict__ tgt,
                                                     const float* __restrict__ gmaps, int W, int H, double beta,
                                                     double l1_norm, int has_ssim, float* __restrict__ d_image,
                                                     MaskArgs mk, const __grid_constant__ LossMaps tm) {
  if (mk.final_t) {
    l1_norm = mk.norms[0];
    has_ssim = mk.norms[3] > 0.0 ? has_ssim : 0;
  }
  constexpr int PITCH = kTma ? kTP : kSW + 1;
  constexpr int WIN = kTma ? kTWin : kSH * (kSW + 1);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* win = reinterpret_cast<float*>(smem_raw);  // [buffers][3 maps][WIN]
  float(*hq)[kSH][kTW + 1] =
      reinterpret_cast<float(*)[kSH][kTW + 1]>(smem_raw + sizeof(float) * (kTma ? 3 * kBufs : 3) * WIN);
  __shared__ __align__(8) uint64_t bar[2];
  const int64_t P = (int64_t)W * H;
  const int bx = blockIdx.x * kTW, by = blockIdx.y * kTH;
  const int ch0 = kChSplit ? (int)blockIdx.z : 0, ch_end = kChSplit ? ch0 + 1 : 3;
  const int c = threadIdx.x & (kTW - 1), rg = threadIdx.x / kTW;
  const int x = bx + c;
  if (kTma && has_ssim && threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_expect_tx(&bar[0], 3 * kTWinBytes);
    for (int m = 0; m < 3; ++m)
      tma_load_3d(win + m * kTWin, &tm.gm, bx - kHalf - kTX, by - kHalf, 3 * ch0 + m, &bar[0]);
  }
  if (kTma) __syncthreads();  // barrier initialisation visible to every waiting thread
  for (int ch = ch0; ch < ch_end; ++ch) {
    const int it = ch - ch0;  // channel iteration of this CTA (buffer / phase index)
    // this channel's output pixels of both images, loaded before the
    // convolutions so their latency overlaps them (they were the kernel's
    // long-scoreboard stall)
    float av[kR], bv[kR];
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int y = by + rg * kR + j;
      const bool in = x < W && y < H;
      const int64_t p = in ? (int64_t)y * W + x : 0;
      av[j] = in ? __ldg(ren + ch * P + p) : 0.f;
      bv[j] = in ? __ldg(tgt + ch * P + p) : 0.f;
    }
    float cv[3][kR];
    if (has_ssim) {
      const float* st;
      if (kTma && kBufs == 1) {
        mbar_wait(&bar[0], (uint32_t)(it & 1));
        st = win;
      } else if (kTma) {
        if (threadIdx.x == 0 && ch + 1 < ch_end) {
          float* nb = win + ((it + 1) & 1) * 3 * kTWin;
          fence_proxy_async();
          mbar_arrive_expect_tx(&bar[(it + 1) & 1], 3 * kTWinBytes);
          for (int m = 0; m < 3; ++m)
            tma_load_3d(nb + m * kTWin, &tm.gm, bx - kHalf - kTX, by - kHalf, 3 * (ch + 1) + m, &bar[(it + 1) & 1]);
        }
        mbar_wait(&bar[it & 1], (uint32_t)(it >> 1));
        st = win + (it & 1) * 3 * kTWin;
      } else {
        const float* src[3] = {gmaps + (3 * ch + 0) * P, gmaps + (3 * ch + 1) * P, gmaps + (3 * ch + 2) * P};
        stage_planes<3>(reinterpret_cast<float(*)[kSH][kSW + 1]>(win), src, W, H, bx - kHalf, by - kHalf);
        __syncthreads();
        st = win;
      }
      hpass3<PITCH, kTma ? kTX : 0>(st, WIN, hq);
      __syncthreads();
      if (kTma && kBufs == 1 && threadIdx.x == 0 && ch + 1 < ch_end) {  // window consumed: next channel into it
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[0], 3 * kTWinBytes);
        for (int m = 0; m < 3; ++m)
          tma_load_3d(win + m * kTWin, &tm.gm, bx - kHalf - kTX, by - kHalf, 3 * (ch + 1) + m, &bar[0]);
      }
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        float acc[kR];
#pragma unroll
        for (int j = 0; j < kR; ++j) acc[j] = 0.f;
#pragma unroll
        for (int k = 0; k < kR + kWin - 1; ++k) {
          const float f = hq[m][rg * kR + k][c];
#pragma unroll
          for (int j = 0; j < kR; ++j)
            if (k - j >= 0 && k - j < kWin) acc[j] = fmaf(c_win[k - j], f, acc[j]);
        }
#pragma unroll
        for (int j = 0; j < kR; ++j) cv[m][j] = acc[j];
      }
    }
#pragma unroll
    for (int j = 0; j < kR; ++j) {
      const int y = by + rg * kR + j;
      if (x >= W || y >= H) continue;
      const int64_t p = (int64_t)y * W + x;
      const double a = av[j], b = bv[j];
      const double diff = a - b;
      const double dl1 = (diff == 0.0 || !mask_at(mk, p)) ? 0.0 : (diff > 0.0 ? l1_norm : -l1_norm);
      const double dss =
          has_ssim ? a_(a_((double)cv[0][j], m_(m_(2.0, a), (double)cv[1][j])), m_(b, (double)cv[2][j])) : 0.0;
      d_image[ch * P + p] = (float)s_(m_(1.0 - beta, dl1), m_(beta, dss));
    }
    if (has_ssim) __syncthreads();
  }
}

// Fixed-order reduction of the block partials; out = {l1_mean, ssim_mean, loss}.
__global__ void __launch_bounds__(256) loss_finalize_kernel(const double* __restrict__ block_sums, int nb,
                                                            double l1_norm, double scale, int has_ssim, double beta,
                                                            double* __restrict__ out, MaskArgs mk) {
  if (mk.final_t) {
    l1_norm = mk.norms[0];
    scale = mk.norms[1];
    has_ssim = mk.norms[3] > 0.0 ? has_ssim : 0;
  }
  __shared__ double s1[256], s2[256];
  double a = 0.0, b = 0.0;
  // four blocks' sums loaded per round (independent loads in flight), added
  // in block order: fixed association, deterministic
  for (int i0 = threadIdx.x; i0 < nb; i0 += 4 * 256) {
    double u[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q * 256;
      u[q][0] = i < nb ? block_sums[2 * i] : 0.0;
      u[q][1] = i < nb ? block_sums[2 * i + 1] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a += u[q][0];
      b += u[q][1];
    }
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {  // fixed binary tree: deterministic
    if (threadIdx.x < h) {
      s1[threadIdx.x] += s1[threadIdx.x + h];
      s2[threadIdx.x] += s2[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double l1 = s1[0] * l1_norm;
    const double ssim = has_ssim ? s2[0] * scale : 1.0;
    out[0] = l1;
    out[1] = ssim;
    out[2] = (1.0 - beta) * l1 + beta * (1.0 - ssim);
  }
}

// Masked pixel counts (integer atomics: exact) for masked_rgb_loss.
__global__ void mask_count_kernel(const float* __restrict__ final_t, int W, int H, double thr,
                                  unsigned long long* __restrict__ counts) {
  unsigned long long c1 = 0, c2 = 0;
  const int64_t P = (int64_t)W * H;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    if (!((1.0 - (double)final_t[p]) > thr)) continue;
    const int x = (int)(p % W), y = (int)(p / W);
    ++c1;
    if (x >= kHalf && x < W - kHalf && y >= kHalf && y < H - kHalf) ++c2;
  }
  for (int o = 16; o > 0; o >>= 1) {
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(counts, c1);
    atomicAdd(counts + 1, c2);
  }
}
__global__ void mask_norms_kernel(const unsigned long long* __restrict__ counts, double* __restrict__ norms) {
  const double c1 = (double)counts[0], c2 = (double)counts[1];
  norms[0] = c1 > 0.0 ? 1.0 / (3.0 * c1) : 0.0;
  norms[1] = c2 > 0.0 ? 1.0 / (3.0 * c2) : 0.0;
  norms[2] = c1;
  norms[3] = c2;
}

// gaussian_window (losses.cpp:19-32), FP64 on host, into constant memory of
// the current device. Called once per context (never inside graph capture).
int init_loss_constants() {
  double w[kWin], sum = 0.0;
  for (int i = 0; i < kWin; ++i) {
    const double d = i - kHalf;
    w[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
    sum += w[i];
  }
  float wf[kWin];
  for (int i = 0; i < kWin; ++i) wf[i] = (float)(w[i] / sum);
  GSB_CUDA(cudaMemcpyToSymbol(c_win, wf, sizeof wf));
  return GSB_OK;
}

constexpr size_t kMapsSmem = sizeof(float) * 2 * kSH * (kSW + 1) + sizeof(float) * 5 * kSH * (kTW + 1);
constexpr size_t kGradSmem = sizeof(float) * 3 * kSH * (kSW + 1) + sizeof(float) * 3 * kSH * (kTW + 1);
constexpr size_t kMapsSmemT = sizeof(float) * 2 * kBufs * kTWin + sizeof(float) * 5 * kSH * (kTW + 1);
constexpr size_t kGradSmemT = sizeof(float) * 3 * kBufs * kTWin + sizeof(float) * 3 * kSH * (kTW + 1);

int init_loss_attributes() {
  GSB_CUDA(cudaFuncSetAttribute(loss_maps_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMapsSmem));
  GSB_CUDA(cudaFuncSetAttribute(loss_grad_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGradSmem));
  GSB_CUDA(cudaFuncSetAttribute(loss_maps_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMapsSmemT));
  GSB_CUDA(cudaFuncSetAttribute(loss_grad_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGradSmemT));
  return GSB_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library links only the CUDA runtime).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 3-D map over `planes` FP32 planes of W x H, box 44 x 42 x 1, zero fill.
static bool encode_planes(CUtensorMap* m, const float* base, int W, int H, int planes) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)planes};
  const cuuint64_t strides[2] = {(cuuint64_t)W * 4u, (cuuint64_t)W * (cuuint64_t)H * 4u};
  const cuuint32_t box[3] = {(cuuint32_t)kTP, (cuuint32_t)kSH, 1u};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifndef GSB_LOSS_TMA
#define GSB_LOSS_TMA 1
#endif

// mask_t (nullable): final transmittance of the rendered frame; then the loss
// is masked_rgb_loss with accum = 1 - T > mask_thr, and mask_ws (>= 48 bytes of
// device scratch) receives the counts and norms ({l1 norm, ssim scale, count,
// valid count} as doubles at offset 16). TMA staging needs 16-byte aligned
// plane bases and rows (W % 4 == 0); otherwise the loads go through registers.
int launch_rgb_loss(cudaStream_t st, const float* ren, const float* tgt, int W, int H, double beta, float* gmaps,
                    double* block_sums, double* out3, float* d_image, int64_t* launches, const float* mask_t,
                    double mask_thr, void* mask_ws) {
  MaskArgs mk{mask_t, mask_thr, nullptr};
  if (mask_t) {
    unsigned long long* cnt = static_cast<unsigned long long*>(mask_ws);
    mk.norms = reinterpret_cast<const double*>(cnt + 2);
    GSB_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), st));
    mask_count_kernel<<<148, 256, 0, st>>>(mask_t, W, H, mask_thr, cnt);
    mask_norms_kernel<<<1, 1, 0, st>>>(cnt, reinterpret_cast<double*>(cnt + 2));
    *launches += 2;
  }
  const int64_t cnt_valid = (W > 2 * kHalf && H > 2 * kHalf) ? (int64_t)(W - 2 * kHalf) * (H - 2 * kHalf) : 0;
  const int has_ssim = cnt_valid > 0 ? 1 : 0;
  const double scale = has_ssim ? 1.0 / (3.0 * (double)cnt_valid) : 0.0;
  const double l1_norm = 1.0 / (3.0 * (double)W * (double)H);
  dim3 grid((W + kTW - 1) / kTW, (H + kTH - 1) / kTH, kChSplit ? 3 : 1);
  const auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  LossMaps tm;
  std::memset(&tm, 0, sizeof tm);
  bool tma = GSB_LOSS_TMA && W % 4 == 0 && aligned(ren) && aligned(tgt) && aligned(gmaps) &&
             encode_planes(&tm.ren, ren, W, H, 3) && encode_planes(&tm.tgt, tgt, W, H, 3) &&
             encode_planes(&tm.gm, gmaps, W, H, 9);
  if (tma) {
    loss_maps_kernel<true><<<grid, kThr, kMapsSmemT, st>>>(ren, tgt, W, H, scale, gmaps, block_sums, mk, tm);
    if (d_image)
      loss_grad_kernel<true><<<grid, kThr, kGradSmemT, st>>>(ren, tgt, gmaps, W, H, beta, l1_norm, has_ssim,
                                                             d_image, mk, tm);
  } else {
    loss_maps_kernel<false><<<grid, kThr, kMapsSmem, st>>>(ren, tgt, W, H, scale, gmaps, block_sums, mk, tm);
    if (d_image)
      loss_grad_kernel<false><<<grid, kThr, kGradSmem, st>>>(ren, tgt, gmaps, W, H, beta, l1_norm, has_ssim,
                                                              d_image, mk, tm);
  }
  loss_finalize_kernel<<<1, 256, 0, st>>>(block_sums, (int)(grid.x * grid.y * grid.z), l1_norm, scale, has_ssim, beta, out3,
                                          mk);
  *launches += d_image ? 3 : 2;
  GSB_CHECK_LAUNCH("rgb_loss kernels");
  return GSB_OK;
}

size_t loss_block_count(int W, int H) {
  return (size_t)((W + kTW - 1) / kTW) * ((H + kTH - 1) / kTH) * (kChSplit ? 3 : 1);
}

}  // namespace gsb
