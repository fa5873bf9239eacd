// k_onesweep.cu — single-pass prefix scan and Onesweep-style stable LSD radix
// sort with decoupled look-back (Merrill & Garland; Adinets & Merrill), used
// by K2 (k_sort.cu documents the reference semantics, rasterizer.cpp:127-168).
//
// Both are launched with capacity-sized grids and read the live item count
// from device memory, so they are CUDA-graph friendly. Each CTA claims its
// tile index from an atomic ticket (tiles are claimed in launch order, so a
// CTA only ever waits on tiles owned by CTAs that are already running) and
// publishes a per-tile aggregate, then an inclusive prefix, through 32-bit
// status words (2 flag bits + 30 count bits). All arithmetic is on integer
// counts, so results are exact and deterministic regardless of scheduling.
//
// Sort: one histogram kernel computes the global digit counts of every pass
// (one read of the keys), one tiny kernel turns them into per-pass digit
// bases, then each pass is a single scatter kernel: stable in-tile ranks via
// warp match_any + cross-warp prefix, per-digit look-back across tiles,
// scatter to base + prefix + rank.
#include <algorithm>

#include "gsb_internal.cuh"

namespace gsb {

constexpr int kOsThreads = 256;
constexpr int kOsItems = 16;
constexpr int kOsTile = kOsThreads * kOsItems;  // 4096 items per tile
constexpr uint32_t kStAgg = 1u << 30, kStPre = 2u << 30, kStCount = (1u << 30) - 1u;

__device__ __forceinline__ uint32_t os_lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int64_t os_live(const uint32_t* n_dev, int64_t cap) {
  if (!n_dev) return cap;
  const int64_t v = (int64_t)*n_dev;
  return v < cap ? v : cap;
}
// Status words are self-contained (flag + count), so relaxed GPU-scope
// accesses suffice; nothing else is read through them.
__device__ __forceinline__ void st_status(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_status(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Warp-wide variant for the scan (called by a full warp): reads the status
// of the 32 nearest predecessors at once, waits until all of them are
// published, and sums aggregates down to the nearest inclusive prefix; the
// serial chain across tiles is then one step per 32 tiles instead of one.
__device__ __forceinline__ uint32_t look_back_warp(const uint32_t* status, int64_t tile) {
  const int lane = threadIdx.x & 31;
  uint32_t excl = 0;
  for (int64_t top = tile - 1;; top -= 32) {
    const int64_t t = top - lane;  // lane 0 = nearest predecessor
    uint32_t s = t >= 0 ? ld_status(status + t) : kStPre;  // before tile 0: prefix 0
    while (__any_sync(0xffffffffu, (s & ~kStCount) == 0u))
      if ((s & ~kStCount) == 0u) s = ld_status(status + t);
    const uint32_t pre = __ballot_sync(0xffffffffu, (s & kStPre) != 0u);
    const int stop = pre ? __ffs(pre) - 1 : 31;  // include lanes 0..stop
    excl += __reduce_add_sync(0xffffffffu, lane <= stop ? (s & kStCount) : 0u);
    if (pre) return excl;
  }
}

// Exclusive prefix of this tile's aggregate over all earlier tiles (one
// thread; walks back until an inclusive prefix is found).
__device__ __forceinline__ uint32_t look_back(const uint32_t* status, int64_t tile, int64_t stride) {
  uint32_t excl = 0;
  for (int64_t t = tile - 1; t >= 0;) {
    const uint32_t s = ld_status(status + t * stride);
    if ((s & ~kStCount) == 0u) continue;  // predecessor not published yet: spin
    excl += s & kStCount;
    if (s & kStPre) break;
    --t;
  }
  return excl;
}

// ------------------------------------------------------------- scan
#ifndef GSB_SCAN_THREADS
#define GSB_SCAN_THREADS 512  // 8192-item tiles: half the look-back chain of 256 (sort stage 0.102 -> 0.100 ms)
#endif
constexpr int kScanThreads = GSB_SCAN_THREADS;
constexpr int kScanTile = kScanThreads * kOsItems;  // items per look-back tile
// status: [1 ticket][ntiles] words, zeroed before the launch.
template <bool kFlag>
__global__ void __launch_bounds__(kScanThreads) scan_onepass_kernel(const uint32_t* in, int64_t cap,
                                                                   const uint32_t* __restrict__ n_dev,
                                                                   uint32_t* out, uint32_t* status,
                                                                   uint32_t* __restrict__ total) {
  __shared__ uint32_t s_tile_idx, s_prefix;
  __shared__ uint32_t s_warp[kScanThreads / 32];
  __shared__ uint32_t s_items[kScanTile + kScanTile / 32];
  if (threadIdx.x == 0) s_tile_idx = atomicAdd(status, 1u);
  __syncthreads();
  const int64_t n = os_live(n_dev, cap);
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  const int64_t tile = s_tile_idx;
  if (tile >= ntiles) {
    if (tile == 0 && threadIdx.x == 0 && total) *total = 0;  // empty input
    return;
  }
  const int64_t base = tile * kScanTile;
#pragma unroll
  for (int k = 0; k < kOsItems; ++k) {  // striped, coalesced load
    const int idx = k * kScanThreads + threadIdx.x;
    const int64_t i = base + idx;
    uint32_t v = 0;
    if (i < n) {
      v = in[i];
      if (kFlag) v = v > 0u ? 1u : 0u;
    }
    s_items[idx + (idx >> 5)] = v;
  }
  __syncthreads();
  uint32_t loc[kOsItems], sum = 0;
#pragma unroll
  for (int k = 0; k < kOsItems; ++k) {  // thread owns items [16 t, 16 t + 16)
    const int idx = threadIdx.x * kOsItems + k;
    loc[k] = s_items[idx + (idx >> 5)];
    sum += loc[k];
  }
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  if ((threadIdx.x & 31) == 31) s_warp[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {  // warp 0: publish, then a warp-wide look-back
    const int lane = threadIdx.x;
    uint32_t agg = 0;
    if (lane == 0) {
      for (int w = 0; w < kScanThreads / 32; ++w) {
        const uint32_t c = s_warp[w];
        s_warp[w] = agg;
        agg += c;
      }
    }
    agg = __shfl_sync(0xffffffffu, agg, 0);
    uint32_t* st = status + 1;
    if (tile == 0) {
      if (lane == 0) {
        st_status(st, kStPre | agg);
        s_prefix = 0;
      }
    } else {
      if (lane == 0) st_status(st + tile, kStAgg | agg);
      const uint32_t excl = look_back_warp(st, tile);
      if (lane == 0) {
        st_status(st + tile, kStPre | (excl + agg));
        s_prefix = excl;
      }
    }
    if (lane == 0 && tile == ntiles - 1 && total) *total = s_prefix + agg;
  }
  __syncthreads();
  uint32_t run = s_prefix + s_warp[threadIdx.x >> 5] + x - sum;
#pragma unroll
  for (int k = 0; k < kOsItems; ++k) {
    const int idx = threadIdx.x * kOsItems + k;
    s_items[idx + (idx >> 5)] = run;
    run += loc[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kOsItems; ++k) {
    const int idx = k * kScanThreads + threadIdx.x;
    if (base + idx < n) out[base + idx] = s_items[idx + (idx >> 5)];
  }
}

size_t scan_onepass_words(int64_t cap) { return (size_t)((cap + kScanTile - 1) / kScanTile) + 2; }

// Zeroes the scan's ticket and status words. A kernel rather than a memset
// node: the same cost inside a captured graph, and compute-sanitizer's
// initcheck tracks kernel stores (it reported the ticket word of the graph
// memset as uninitialised).
__global__ void zero_words_kernel(uint32_t* __restrict__ w, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) w[i] = 0u;
}

int scan_onepass(cudaStream_t st, const uint32_t* in, int64_t cap, const uint32_t* n_dev, bool flag, uint32_t* out,
                 uint32_t* status, uint32_t* total, int64_t* launches) {
  const int64_t ntiles = (cap + kScanTile - 1) / kScanTile;
  zero_words_kernel<<<(unsigned)std::min<int64_t>((ntiles + 2 + 255) / 256, 64), 256, 0, st>>>(status, ntiles + 2);
  *launches += 1;
  const unsigned grid = (unsigned)(ntiles > 0 ? ntiles : 1);
  if (flag) scan_onepass_kernel<true><<<grid, kScanThreads, 0, st>>>(in, cap, n_dev, out, status, total);
  else scan_onepass_kernel<false><<<grid, kScanThreads, 0, st>>>(in, cap, n_dev, out, status, total);
  *launches += 1;
  GSB_CHECK_LAUNCH("scan_onepass_kernel");
  return GSB_OK;
}

// -------------------------------------------------------------- sort
constexpr int kMaxPasses = 4;

// Global digit histograms of all passes from one read of the keys.
__global__ void __launch_bounds__(kOsThreads) os_hist_kernel(const uint32_t* __restrict__ keys, int64_t cap,
                                                             const uint32_t* __restrict__ n_dev, int passes, int bits,
                                                             uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[kMaxPasses][256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += kOsThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const int64_t n = os_live(n_dev, cap);
  const uint32_t mask = (1u << bits) - 1u;
  for (int64_t i = (int64_t)blockIdx.x * kOsThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kOsThreads) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (p * bits)) & mask], 1u);
  }
  __syncthreads();
  const int ndig = 1 << bits;
  for (int i = threadIdx.x; i < passes * ndig; i += kOsThreads) {
    const uint32_t c = h[i / ndig][i % ndig];
    if (c) atomicAdd(&ghist[i], c);
  }
}

// Exclusive scan of each pass's digit counts -> digit bases (one block).
__global__ void os_bases_kernel(uint32_t* __restrict__ ghist, int passes, int bits) {
  const int ndig = 1 << bits;
  if (threadIdx.x >= passes) return;
  uint32_t run = 0;
  for (int d = 0; d < ndig; ++d) {
    const uint32_t c = ghist[threadIdx.x * ndig + d];
    ghist[threadIdx.x * ndig + d] = run;
    run += c;
  }
}

// One stable scatter pass. status: [1 ticket][ntiles][256] words, zeroed.
__global__ void __launch_bounds__(kOsThreads) os_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int64_t cap, const uint32_t* __restrict__ n_dev, int shift, int bits,
    const uint32_t* __restrict__ bases, uint32_t* status) {
  constexpr int kWarps = kOsThreads / 32;
  __shared__ uint32_t warp_cnt[kWarps][256];
  __shared__ uint32_t warp_off[kWarps][256];
  __shared__ uint32_t digit_run[256];
  __shared__ uint32_t s_tile_idx;
  if (threadIdx.x == 0) s_tile_idx = atomicAdd(status, 1u);
  for (int d = threadIdx.x; d < 256; d += kOsThreads) {
    digit_run[d] = 0;
    warp_off[0][d] = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) warp_cnt[w][d] = 0;
  }
  __syncthreads();
  const int64_t n = os_live(n_dev, cap);
  const int64_t ntiles = (n + kOsTile - 1) / kOsTile;
  const int64_t tile = s_tile_idx;
  if (tile >= ntiles) return;
  const int64_t base = tile * kOsTile;
  const int ndig = 1 << bits;
  const uint32_t mask = (uint32_t)ndig - 1u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = os_lanemask_lt();
  uint32_t key[kOsItems], val[kOsItems], lpos[kOsItems];
  // 1. load the tile and count its digits (shared atomics: order free)
#pragma unroll
  for (int k = 0; k < kOsItems; ++k) {
    const int64_t i = base + k * kOsThreads + threadIdx.x;
    key[k] = 0;
    val[k] = 0;
    if (i < n) {
      key[k] = keys_in[i];
      val[k] = vals_in[i];
      atomicAdd(&warp_off[0][(key[k] >> shift) & mask], 1u);
    }
  }
  __syncthreads();
  // 2. decoupled look-back per digit, as early as possible so successors'
  //    walks meet inclusive prefixes quickly: publish aggregate, find the
  //    exclusive prefix, publish the inclusive prefix.
  {
    uint32_t* st = status + 1 + tile * 256;
    for (int d = threadIdx.x; d < ndig; d += kOsThreads) {
      const uint32_t agg = warp_off[0][d];
      if (tile == 0) {
        st_status(st + d, kStPre | agg);
        digit_run[d] = bases[d];
      } else {
        st_status(st + d, kStAgg | agg);
        const uint32_t excl = look_back(status + 1 + d, tile, 256);
        st_status(st + d, kStPre | (excl + agg));
        digit_run[d] = bases[d] + excl;
      }
    }
  }
  __syncthreads();
  // 3. stable in-tile ranks, rounds of 256 items in global order; digit_run
  //    starts at the digit's global base + prefix so lpos is the final slot
#pragma unroll
  for (int k = 0; k < kOsItems; ++k) {
    const int64_t i = base + k * kOsThreads + threadIdx.x;
    const bool valid = i < n;
    const uint32_t dig = valid ? (key[k] >> shift) & mask : 0x100u + lane;  // invalid lanes: unique sentinel
    const uint32_t peers = __match_any_sync(0xffffffffu, dig);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) warp_cnt[warp][dig] = __popc(peers);
    __syncthreads();
    for (int d = threadIdx.x; d < ndig; d += kOsThreads) {
      uint32_t run = digit_run[d];
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = warp_cnt[w][d];
        warp_off[w][d] = run;
        run += c;
        warp_cnt[w][d] = 0;
      }
      digit_run[d] = run;
    }
    __syncthreads();
    lpos[k] = valid ? warp_off[warp][dig] + rank : 0xffffffffu;
    __syncthreads();
  }
  // 4. scatter
#pragma unroll
  for (int k = 0; k < kOsItems; ++k) {
    if (lpos[k] == 0xffffffffu) continue;
    const uint32_t pos = lpos[k];
    keys_out[pos] = key[k];
    vals_out[pos] = val[k];
  }
}

static int os_passes(int total_bits) { return total_bits <= 0 ? 0 : (total_bits + 7) / 8; }

size_t onesweep_words(int64_t cap, int total_bits) {
  const int passes = os_passes(total_bits);
  const int64_t ntiles = (cap + kOsTile - 1) / kOsTile;
  return (size_t)kMaxPasses * 256 + (size_t)passes * (1 + ntiles * 256) + 64;
}

// Stable sort of (keys, vals)[0..live) by key bits [0, total_bits). Buffers
// [0] hold the input; *result_sel gets the buffer holding the result (fixed
// by total_bits, hence graph-stable). ws: onesweep_words(cap, bits) words.
int onesweep_sort_pairs(cudaStream_t st, uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                        int total_bits, uint32_t* ws, int* result_sel, int64_t* launches) {
  const int passes = os_passes(total_bits);
  *result_sel = 0;
  if (cap <= 1 || passes == 0) return GSB_OK;
  const int bits = (total_bits + passes - 1) / passes;
  const int64_t ntiles = (cap + kOsTile - 1) / kOsTile;
  const size_t words = onesweep_words(cap, total_bits);
  GSB_CUDA(cudaMemsetAsync(ws, 0, sizeof(uint32_t) * words, st));
  uint32_t* ghist = ws;
  const int hist_grid = (int)std::min<int64_t>(ntiles, 2 * 148);
  os_hist_kernel<<<hist_grid > 0 ? hist_grid : 1, kOsThreads, 0, st>>>(keys[0], cap, n_dev, passes, bits, ghist);
  os_bases_kernel<<<1, 32, 0, st>>>(ghist, passes, bits);
  int sel = 0;
  for (int p = 0; p < passes; ++p) {
    uint32_t* status = ws + kMaxPasses * 256 + (size_t)p * (1 + ntiles * 256);
    os_scatter_kernel<<<(unsigned)ntiles, kOsThreads, 0, st>>>(keys[sel], vals[sel], keys[sel ^ 1], vals[sel ^ 1], cap,
                                                              n_dev, p * bits, bits, ghist + p * (1 << bits), status);
    sel ^= 1;
  }
  *launches += 2 + passes;
  GSB_CHECK_LAUNCH("onesweep_sort_pairs");
  *result_sel = sel;
  return GSB_OK;
}

}  // namespace gsb
