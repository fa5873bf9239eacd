// k_sort.cu — K2: device-wide scans, visible compaction, stable LSD radix
// sort (depth keys, then tile keys) and tile-range identification.
//
// Reference: rasterizer.cpp:127-168. The reference compacts visible splats
// in Gaussian-index order (127-130), std::stable_sort's them by double depth
// (131-132), then bins them with a count / prefix / fill pass in depth order
// (134-168) so every tile list is depth sorted and ties keep the lower
// Gaussian index. Here:
//   1. compaction in index order (scan of cnt_g > 0),
//   2. stable LSD radix sort of FP32 depth bits (4 x 8-bit passes) plus an
//      exact fix-up of FP32 ties by the FP64 depth -> the reference order,
//   3. rank-major duplication of (tile, rank) entries, tiles row-major inside
//      each splat rect (the reference fill order),
//   4. stable LSD radix sort of the entries by tile id (ceil(log2 T) bits),
//   5. ranges = [lower_bound(t), lower_bound(t+1)) for every tile.
// All passes are stable and order preserving, so the tile lists equal the
// reference's count/prefix/fill output bit for bit on the same FP64 records.
//
// Every kernel has a data-independent launch shape (sized by capacities) and
// reads the live counts (visible splats V, entries K) from device memory, so
// a whole iteration runs without a host round trip and can be captured in a
// CUDA graph. Entries beyond the entry capacity are dropped and flagged
// (K > cap); the pose step then discards the iteration and the host re-runs
// it with a larger capacity.
#include "gsb_internal.cuh"
#include <cstdlib>

namespace gsb {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ int64_t live_count(const uint32_t* n_dev, int64_t cap) {
  if (!n_dev) return cap;
  const int64_t v = (int64_t)*n_dev;
  return v < cap ? v : cap;
}

template <bool kFlag>
__device__ __forceinline__ uint32_t scan_load(const uint32_t* in, int64_t i, int64_t n) {
  if (i >= n) return 0u;
  uint32_t v = in[i];
  return kFlag ? (v > 0u ? 1u : 0u) : v;
}

// Block sums of 4096-element tiles.
template <bool kFlag>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in, int64_t cap,
                                                                    const uint32_t* __restrict__ n_dev,
                                                                    uint32_t* __restrict__ block_sums) {
  const int64_t n = live_count(n_dev, cap);
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
  if (base < n) {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s += scan_load<kFlag>(in, base + k * kScanThreads + threadIdx.x, n);
  }
  s = __reduce_add_sync(0xffffffffu, s);
  __shared__ uint32_t ws[kScanThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
    block_sums[blockIdx.x] = t;
  }
}

// Exclusive scan of nb block sums in one block; total -> sums[nb] and *total_out.
__global__ void __launch_bounds__(1024) scan_blocks_kernel(uint32_t* __restrict__ sums, int64_t nb,
                                                           uint32_t* __restrict__ total_out) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    uint32_t v = i < nb ? sums[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t w = wsum[threadIdx.x];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      wsum[threadIdx.x] = w;
    }
    __syncthreads();
    const uint32_t warp_excl = (threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : 0u;
    const uint32_t excl = carry + warp_excl + x - v;
    if (i < nb) sums[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sums[nb] = carry;
    if (total_out) *total_out = carry;
  }
}

// Block-local exclusive scan plus block offset. Items are striped
// (k*256 + tid) for coalescing; the scan order is the global index order.
template <bool kFlag>
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const uint32_t* in, int64_t cap,
                                                                   const uint32_t* __restrict__ n_dev,
                                                                   const uint32_t* __restrict__ block_offs,
                                                                   uint32_t* __restrict__ out) {
  const int64_t n = live_count(n_dev, cap);
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  if (base >= n) return;
  __shared__ uint32_t tile[kScanTile + kScanTile / 32];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int idx = k * kScanThreads + threadIdx.x;
    tile[idx + (idx >> 5)] = scan_load<kFlag>(in, base + idx, n);
  }
  __syncthreads();
  uint32_t local[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int idx = threadIdx.x * kScanItems + k;
    local[k] = tile[idx + (idx >> 5)];
    s += local[k];
  }
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  __shared__ uint32_t ws[kScanThreads / 32];
  if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
  __syncthreads();
  uint32_t woff = 0;
  for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) woff += ws[w];
  uint32_t run = block_offs[blockIdx.x] + woff + x - s;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int idx = threadIdx.x * kScanItems + k;
    tile[idx + (idx >> 5)] = run;
    run += local[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int idx = k * kScanThreads + threadIdx.x;
    if (base + idx < n) out[base + idx] = tile[idx + (idx >> 5)];
  }
}

static int64_t scan_blocks_for(int64_t cap) { return (cap + kScanTile - 1) / kScanTile; }
size_t scan_words(int64_t cap) { return (size_t)scan_blocks_for(cap) + 2; }

// Exclusive scan of the live prefix (n_dev, capped at cap; n_dev may be
// NULL = cap) of u32 values — or of the flags v > 0 — into out. *total
// (device) receives the sum. Launch shape depends on cap only.
int scan_exclusive(cudaStream_t st, const uint32_t* in, int64_t cap, const uint32_t* n_dev, bool flag, uint32_t* out,
                   uint32_t* scratch, uint32_t* total, int64_t* launches) {
  const int64_t nb = scan_blocks_for(cap);
  if (nb > 0) {
    if (flag) scan_reduce_kernel<true><<<(unsigned)nb, kScanThreads, 0, st>>>(in, cap, n_dev, scratch);
    else scan_reduce_kernel<false><<<(unsigned)nb, kScanThreads, 0, st>>>(in, cap, n_dev, scratch);
  }
  scan_blocks_kernel<<<1, 1024, 0, st>>>(scratch, nb, total);
  if (nb > 0) {
    if (flag) scan_apply_kernel<true><<<(unsigned)nb, kScanThreads, 0, st>>>(in, cap, n_dev, scratch, out);
    else scan_apply_kernel<false><<<(unsigned)nb, kScanThreads, 0, st>>>(in, cap, n_dev, scratch, out);
  }
  *launches += nb > 0 ? 3 : 1;
  GSB_CHECK_LAUNCH("scan_exclusive");
  return GSB_OK;
}

// ------------------------------------------------------------ radix sort
constexpr int kRadixThreads = 256;
constexpr int kRadixRounds = 16;
constexpr int kRadixTile = kRadixThreads * kRadixRounds;  // 4096 items per block

__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t cap,
                                                                   const uint32_t* __restrict__ n_dev, int shift,
                                                                   int bits, uint32_t* __restrict__ hist,
                                                                   int64_t nblocks) {
  __shared__ uint32_t h[256];
  const int64_t n = live_count(n_dev, cap);
  const int ndig = 1 << bits;
  if (threadIdx.x < ndig) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  const uint32_t mask = (uint32_t)ndig - 1u;
  const uint32_t lane = threadIdx.x & 31;
  if (base < n) {
#pragma unroll 4
    for (int k = 0; k < kRadixRounds; ++k) {
      // warp-aggregated: one shared atomic per distinct digit per warp (tile
      // keys arrive in long runs of equal digits)
      const int64_t i = base + k * kRadixThreads + threadIdx.x;
      const bool valid = i < n;
      const uint32_t dig = valid ? (keys[i] >> shift) & mask : 0x100u + lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, dig);
      if (valid && (peers & ((1u << lane) - 1u)) == 0u) atomicAdd(&h[dig], (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  if (threadIdx.x < ndig) hist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// Exclusive scan of a small array (radix histograms, <= ~1M words) in one
// CTA: each thread scans a contiguous chunk, chunk totals are scanned across
// the block. One launch instead of reduce / scan / apply.
__global__ void __launch_bounds__(1024) scan_small_kernel(uint32_t* __restrict__ a, int64_t n) {
  __shared__ uint32_t s_tot[1024];
  __shared__ uint32_t s_w[32];
  const int64_t chunk = (n + 1023) / 1024;
  const int64_t b = (int64_t)threadIdx.x * chunk, e = b + chunk < n ? b + chunk : n;
  uint32_t t = 0;
  for (int64_t i = b; i < e; ++i) t += a[i];
  uint32_t x = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t w = s_w[threadIdx.x];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (threadIdx.x >= o) w += y;
    }
    s_w[threadIdx.x] = w;
  }
  __syncthreads();
  uint32_t run = ((threadIdx.x >> 5) ? s_w[(threadIdx.x >> 5) - 1] : 0u) + x - t;
  for (int64_t i = b; i < e; ++i) {
    const uint32_t v = a[i];
    a[i] = run;
    run += v;
  }
  (void)s_tot;
}

// Stable scatter: items are processed in rounds of 512 in global order (two
// items per thread: sub-round s covers items s*256 + tid); ranks come from
// warp match_any, then a cross-(sub-round, warp) prefix per digit — 16
// virtual warps, two barriers per 512 items.
__global__ void __launch_bounds__(kRadixThreads) radix_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int64_t cap, const uint32_t* __restrict__ n_dev, int shift, int bits,
    const uint32_t* __restrict__ offs, int64_t nblocks) {
  constexpr int kWarps = kRadixThreads / 32;
  constexpr int kSubs = 2;
  constexpr int kV = kWarps * kSubs;  // virtual warps per round
  __shared__ uint32_t warp_cnt[kV][256];
  __shared__ uint32_t warp_off[kV][256];
  __shared__ uint32_t digit_run[256];
  const int64_t n = live_count(n_dev, cap);
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  if (base >= n) return;
  const int ndig = 1 << bits;
  const uint32_t mask = (uint32_t)ndig - 1u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int d = threadIdx.x; d < 256; d += kRadixThreads) {
    digit_run[d] = d < ndig ? offs[(int64_t)d * nblocks + blockIdx.x] : 0u;
    for (int w = 0; w < kV; ++w) warp_cnt[w][d] = 0;
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  for (int k = 0; k < kRadixRounds / kSubs; ++k) {
    const int64_t r0 = base + (int64_t)k * kSubs * kRadixThreads;
    if (r0 >= n) break;  // uniform across the block
    uint32_t key[kSubs], val[kSubs], dig[kSubs], rank[kSubs];
    bool valid[kSubs];
#pragma unroll
    for (int s = 0; s < kSubs; ++s) {
      const int64_t i = r0 + s * kRadixThreads + threadIdx.x;
      valid[s] = i < n;
      key[s] = valid[s] ? keys_in[i] : 0u;
      val[s] = valid[s] ? vals_in[i] : 0u;
      dig[s] = valid[s] ? (key[s] >> shift) & mask : 0x100u + lane;  // invalid lanes: unique sentinels
    }
#pragma unroll
    for (int s = 0; s < kSubs; ++s) {
      const uint32_t peers = __match_any_sync(0xffffffffu, dig[s]);
      rank[s] = __popc(peers & lt);
      if (valid[s] && rank[s] == 0) warp_cnt[s * kWarps + warp][dig[s]] = __popc(peers);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < ndig; d += kRadixThreads) {
      uint32_t run = digit_run[d];
#pragma unroll
      for (int w = 0; w < kV; ++w) {
        const uint32_t c = warp_cnt[w][d];
        warp_off[w][d] = run;
        run += c;
        warp_cnt[w][d] = 0;
      }
      digit_run[d] = run;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kSubs; ++s) {
      if (!valid[s]) continue;
      const uint32_t pos = warp_off[s * kWarps + warp][dig[s]] + rank[s];
      keys_out[pos] = key[s];
      vals_out[pos] = val[s];
    }
  }
}

static int radix_passes(int total_bits) { return total_bits <= 0 ? 0 : (total_bits + 7) / 8; }
int scan_onepass(cudaStream_t st, const uint32_t* in, int64_t cap, const uint32_t* n_dev, bool flag, uint32_t* out,
                 uint32_t* status, uint32_t* total, int64_t* launches);

// Sorts (keys, vals)[0..live) by key bits [0, total_bits) stably. Buffers [0]
// hold the input; *result_sel receives the buffer index holding the result
// (fixed by total_bits, hence graph-stable).
int radix_sort_pairs(cudaStream_t st, uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                     int total_bits, uint32_t* hist, int* result_sel, int64_t* launches) {
  int sel = 0;
  const int passes = radix_passes(total_bits);
  if (cap <= 1 || passes == 0) {
    *result_sel = 0;
    return GSB_OK;
  }
  const int bits = (total_bits + passes - 1) / passes;
  const int64_t nblocks = (cap + kRadixTile - 1) / kRadixTile;
  const int64_t nh = (int64_t)(1 << bits) * nblocks;
  for (int p = 0; p < passes; ++p) {
    const int shift = p * bits;
    radix_hist_kernel<<<(unsigned)nblocks, kRadixThreads, 0, st>>>(keys[sel], cap, n_dev, shift, bits, hist, nblocks);
    // few tiles -> short look-back: the single-pass scan wins for histograms
    static const bool legacy = [] { const char* e = std::getenv("GSB_HIST_SCAN"); return e && e[0] == 'l'; }();
    int rc = legacy ? scan_exclusive(st, hist, nh, nullptr, false, hist, hist + nh, nullptr, launches)
                    : scan_onepass(st, hist, nh, nullptr, false, hist, hist + nh, nullptr, launches);
    if (rc) return rc;
    radix_scatter_kernel<<<(unsigned)nblocks, kRadixThreads, 0, st>>>(keys[sel], vals[sel], keys[sel ^ 1],
                                                                      vals[sel ^ 1], cap, n_dev, shift, bits, hist,
                                                                      nblocks);
    *launches += 2;
    sel ^= 1;
  }
  GSB_CHECK_LAUNCH("radix_sort_pairs");
  *result_sel = sel;
  return GSB_OK;
}

size_t radix_hist_words(int64_t cap, int total_bits) {
  const int passes = radix_passes(total_bits);
  if (passes == 0) return 16;
  const int bits = (total_bits + passes - 1) / passes;
  const int64_t nblocks = (cap + kRadixTile - 1) / kRadixTile;
  const int64_t nh = (int64_t)(1 << bits) * nblocks;
  return (size_t)nh + scan_words(nh) + 16;
}

// ---------------------------------------------------- compaction + ranks
// vis_pos = exclusive scan of (cnt_g > 0). Emits visible slot v -> gid and
// the FP32 depth key (positive floats compare as their bit patterns).
__global__ void compact_kernel(const uint32_t* __restrict__ cnt_g, const uint32_t* __restrict__ vis_pos,
                               const double* __restrict__ depth_g, int64_t n, uint32_t* __restrict__ vis_idx,
                               uint32_t* __restrict__ dkey, uint32_t* __restrict__ dval) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || cnt_g[i] == 0u) return;
  const uint32_t v = vis_pos[i];
  vis_idx[v] = (uint32_t)i;
  dkey[v] = __float_as_uint((float)depth_g[i]);
  dval[v] = v;
}

// Restores the exact FP64 order inside runs of equal FP32 keys (stable:
// equal doubles keep visible-slot order = Gaussian index order).
__global__ void depth_tie_fix_kernel(const uint32_t* __restrict__ key, uint32_t* __restrict__ val,
                                     const uint32_t* __restrict__ vis_idx, const double* __restrict__ depth_g,
                                     int64_t cap, const uint32_t* __restrict__ nv_dev) {
  const int64_t n = live_count(nv_dev, cap);
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t k = key[r];
  if (r > 0 && key[r - 1] == k) return;       // not a run start
  if (r + 1 >= n || key[r + 1] != k) return;  // singleton
  int64_t end = r + 1;
  while (end < n && key[end] == k) ++end;
  for (int64_t a = r + 1; a < end; ++a) {     // insertion sort by FP64 depth
    const uint32_t v = val[a];
    const double d = depth_g[vis_idx[v]];
    int64_t b = a - 1;
    while (b >= r && depth_g[vis_idx[val[b]]] > d) {
      val[b + 1] = val[b];
      --b;
    }
    val[b + 1] = v;
  }
}

// Rank-order records: rank r holds visible slot sorted_v[r].
__global__ void gather_ranks_kernel(const uint32_t* __restrict__ sorted_v, const uint32_t* __restrict__ vis_idx,
                                    const SplatRec* __restrict__ rec_g, const uint2* __restrict__ rect_g,
                                    const uint32_t* __restrict__ cnt_g, int64_t cap, const uint32_t* __restrict__ nv_dev,
                                    SplatRec* __restrict__ rec, SplatAux* __restrict__ aux, uint32_t* __restrict__ cnt_r,
                                    int32_t* __restrict__ rank_of_g) {
  const int64_t nv = live_count(nv_dev, cap);
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nv) return;
  const uint32_t gid = vis_idx[sorted_v[r]];
  rec[r] = rec_g[gid];
  const uint2 rc = rect_g[gid];
  const uint32_t tx0 = rc.x & 0xffffu, tx1 = rc.x >> 16, ty0 = rc.y & 0xffffu, ty1 = rc.y >> 16;
  SplatAux a;
  a.off = 0;
  a.tx0_ty0 = tx0 | (ty0 << 16);
  a.nx_ny = (tx1 - tx0 + 1u) | ((ty1 - ty0 + 1u) << 16);
  a.gid = (int32_t)gid;
  aux[r] = a;
  cnt_r[r] = cnt_g[gid] & kCntMask;
  rank_of_g[gid] = (int32_t)r;
}

// Emits (tile, rank) for every tile of every splat, rank-major and row-major
// inside the rect — the reference fill order (rasterizer.cpp:163-167).
// Entries at or beyond k_cap are dropped (the iteration is then discarded).
__global__ void duplicate_kernel(const uint32_t* __restrict__ offs, SplatAux* __restrict__ aux, int64_t cap,
                                 const uint32_t* __restrict__ nv_dev, int tiles_x, int64_t k_cap,
                                 uint32_t* __restrict__ ekey, uint32_t* __restrict__ eval,
                                 uint32_t* __restrict__ off_g) {
  const int64_t nv = live_count(nv_dev, cap);
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nv) return;
  const uint32_t off = offs[r];
  const SplatAux a = aux[r];
  aux[r].off = off;
  off_g[a.gid] = off;
  const uint32_t tx0 = a.tx0_ty0 & 0xffffu, ty0 = a.tx0_ty0 >> 16;
  const uint32_t nx = a.nx_ny & 0xffffu, ny = a.nx_ny >> 16;
  int64_t j = off;
  for (uint32_t y = 0; y < ny; ++y) {
    const uint32_t row = (ty0 + y) * (uint32_t)tiles_x + tx0;
    for (uint32_t x = 0; x < nx; ++x, ++j) {
      if (j >= k_cap) return;
      ekey[j] = row + x;
      eval[j] = (uint32_t)r;
    }
  }
}

__global__ void tile_ranges_kernel(const uint32_t* __restrict__ ekey, int64_t k_cap, const uint32_t* __restrict__ k_dev,
                                   int n_tiles, uint2* __restrict__ ranges) {
  const int64_t k = live_count(k_dev, k_cap);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  auto lower = [&](uint32_t v) {
    int64_t lo = 0, hi = k;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ekey[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    return (uint32_t)lo;
  };
  ranges[t] = make_uint2(lower((uint32_t)t), lower((uint32_t)t + 1u));
}

// ------------------------------------------------------------ host glue
int launch_compact(cudaStream_t st, const uint32_t* cnt_g, const uint32_t* vis_pos, const double* depth_g, int64_t n,
                   uint32_t* vis_idx, uint32_t* dkey, uint32_t* dval) {
  if (n > 0) compact_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(cnt_g, vis_pos, depth_g, n, vis_idx, dkey, dval);
  GSB_CHECK_LAUNCH("compact_kernel");
  return GSB_OK;
}
int launch_depth_tie_fix(cudaStream_t st, const uint32_t* key, uint32_t* val, const uint32_t* vis_idx,
                         const double* depth_g, int64_t cap, const uint32_t* nv_dev) {
  if (cap > 1)
    depth_tie_fix_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, st>>>(key, val, vis_idx, depth_g, cap, nv_dev);
  GSB_CHECK_LAUNCH("depth_tie_fix_kernel");
  return GSB_OK;
}
int launch_gather_ranks(cudaStream_t st, const uint32_t* sorted_v, const uint32_t* vis_idx, const SplatRec* rec_g,
                        const uint2* rect_g, const uint32_t* cnt_g, int64_t cap, const uint32_t* nv_dev, SplatRec* rec,
                        SplatAux* aux, uint32_t* cnt_r, int32_t* rank_of_g) {
  if (cap > 0)
    gather_ranks_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, st>>>(sorted_v, vis_idx, rec_g, rect_g, cnt_g, cap,
                                                                       nv_dev, rec, aux, cnt_r, rank_of_g);
  GSB_CHECK_LAUNCH("gather_ranks_kernel");
  return GSB_OK;
}
int launch_duplicate(cudaStream_t st, const uint32_t* offs, SplatAux* aux, int64_t cap, const uint32_t* nv_dev,
                     int tiles_x, int64_t k_cap, uint32_t* ekey, uint32_t* eval, uint32_t* off_g) {
  if (cap > 0)
    duplicate_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, st>>>(offs, aux, cap, nv_dev, tiles_x, k_cap, ekey, eval,
                                                                    off_g);
  GSB_CHECK_LAUNCH("duplicate_kernel");
  return GSB_OK;
}
int launch_tile_ranges(cudaStream_t st, const uint32_t* ekey, int64_t k_cap, const uint32_t* k_dev, int n_tiles,
                       uint2* ranges) {
  if (n_tiles > 0) tile_ranges_kernel<<<(n_tiles + 255) / 256, 256, 0, st>>>(ekey, k_cap, k_dev, n_tiles, ranges);
  GSB_CHECK_LAUNCH("tile_ranges_kernel");
  return GSB_OK;
}

}  // namespace gsb
