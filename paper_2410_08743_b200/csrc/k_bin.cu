// k_bin.cu — K2, tile-local binning: a one-pass counting sort of the entries
// by tile, then a shared-memory sort of every tile list by (FP64 depth, gid).
//
// Reference: rasterizer.cpp:127-168 builds the tile lists by compacting the
// visible splats in Gaussian-index order, std::stable_sort'ing them by double
// depth and filling each tile in that rank order. Every tile list is
// therefore ordered by (depth, gid) — a stable sort of an index-ordered list —
// which is a total order on the tile's entries. Sorting each tile's entries by
// that key directly gives the same lists bit for bit without a global sort,
// and the order in which entries land in their tile range is irrelevant.
//
//   1. tile_count: CTA b counts the entries of Gaussians [b*G, (b+1)*G) per
//      tile in shared memory -> hist[tile][b] (tile-major).
//   2. exclusive scan of hist (single-pass look-back scan) -> for every
//      (tile, CTA) the start of that CTA's run inside the tile's range.
//   3. tile_ranges_from_scan: ranges, the list of tiles for the large per-tile
//      sort, the overflow flag for tiles beyond any per-tile sort.
//   4. tile_scatter: CTA b re-walks its Gaussians and appends (depth high
//      word, gid) with shared-memory cursors.
//   5. tile_sort_{small,large}: per-tile stable radix sort on a quantised
//      depth key, then exact (FP64 depth, gid) order inside key ties (see
//      the per-tile sort section).
//
// Launch shapes are data independent (grid = tiles / Gaussian chunks): a
// graph replay reads live counts from the device. Tiles with more than
// kTileSortLarge entries raise counters[2]; the host then switches the frame
// to the global binning path (k_sort.cu) and re-runs the iteration.
#include <algorithm>

#include "gsb_internal.cuh"

namespace gsb {

int scan_onepass(cudaStream_t st, const uint32_t* in, int64_t cap, const uint32_t* n_dev, bool flag, uint32_t* out,
                 uint32_t* status, uint32_t* total, int64_t* launches);

#ifndef GSB_BIN_THREADS
#define GSB_BIN_THREADS 1024  // (512: sort stage 0.109 -> 0.102 ms at 1024; 256 slower)
#endif
constexpr int kBinThreads = GSB_BIN_THREADS;
#ifndef GSB_BIN_CHUNK
#define GSB_BIN_CHUNK 4096
#endif
constexpr int kBinChunk = GSB_BIN_CHUNK;  // Gaussians per counting CTA

int64_t bin_chunks(int64_t n) { return std::max<int64_t>((n + kBinChunk - 1) / kBinChunk, 1); }

// 1. Per-(tile, chunk) entry counts.
__global__ void __launch_bounds__(kBinThreads) tile_count_kernel(const uint32_t* __restrict__ cnt_g,
                                                                 const SplatAux* __restrict__ aux_g, int64_t n,
                                                                 int n_tiles, int tiles_x, int64_t nchunks,
                                                                 uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t s_cnt[];
  for (int t = threadIdx.x; t < n_tiles; t += kBinThreads) s_cnt[t] = 0;
  __syncthreads();
  const int64_t g0 = (int64_t)blockIdx.x * kBinChunk;
  constexpr int kPer = kBinChunk / kBinThreads;  // Gaussians per thread: loads issued together
  uint32_t c[kPer];
  SplatAux a[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int64_t i = g0 + u * kBinThreads + threadIdx.x;
    c[u] = i < n ? (cnt_g[i] & kCntMask) : 0u;
    if (c[u]) a[u] = aux_g[i];
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    if (!c[u]) continue;
    const uint32_t tx0 = a[u].tx0_ty0 & 0xffffu, ty0 = a[u].tx0_ty0 >> 16;
    const uint32_t nx = a[u].nx_ny & 0xffffu, ny = a[u].nx_ny >> 16;
    for (uint32_t y = 0; y < ny; ++y) {
      const uint32_t row = (ty0 + y) * (uint32_t)tiles_x + tx0;
      for (uint32_t x = 0; x < nx; ++x) atomicAdd(s_cnt + row + x, 1u);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += kBinThreads) hist[(int64_t)t * nchunks + blockIdx.x] = s_cnt[t];
}

// 3. Tile ranges (clamped to the entry capacity so an overflowed iteration
// still reads in bounds), large-sort list, overflow flag.
__global__ void tile_ranges_from_scan_kernel(const uint32_t* __restrict__ offs, int n_tiles, int64_t nchunks,
                                             int64_t k_cap, uint2* __restrict__ ranges, uint32_t* __restrict__ big,
                                             uint32_t* __restrict__ counters) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  const uint32_t b = offs[(int64_t)t * nchunks];
  const uint32_t e = offs[(int64_t)(t + 1) * nchunks];  // offs[T * nchunks] = total (scan writes it)
  const uint32_t cap = (uint32_t)(k_cap < 0xffffffffll ? k_cap : 0xffffffffll);
  ranges[t] = make_uint2(min(b, cap), min(e, cap));
  const uint32_t c = e - b;
  if (c > (uint32_t)kTileSortSmall) big[atomicAdd(counters + 3, 1u)] = (uint32_t)t;
  if (c > (uint32_t)kTileSortLarge) counters[2] = 1u;
}

// 4. Scatter (depth high word, gid) — one 8-byte store per entry — into the
// CTA's run of every tile.
#ifdef GSB_SCATTER_MIN_BLOCKS
#define GSB_SCATTER_BOUNDS __launch_bounds__(kBinThreads, GSB_SCATTER_MIN_BLOCKS)
#else
#define GSB_SCATTER_BOUNDS __launch_bounds__(kBinThreads)
#endif
__global__ void GSB_SCATTER_BOUNDS tile_scatter_kernel(const uint32_t* __restrict__ cnt_g,
                                                                   const SplatAux* __restrict__ aux_g,
                                                                   const double* __restrict__ depth_g, int64_t n,
                                                                   int n_tiles, int tiles_x, int64_t nchunks,
                                                                   const uint32_t* __restrict__ offs, int64_t k_cap,
                                                                   unsigned long long* __restrict__ ent_key) {
  extern __shared__ uint32_t s_cur[];
  for (int t = threadIdx.x; t < n_tiles; t += kBinThreads) s_cur[t] = offs[(int64_t)t * nchunks + blockIdx.x];
  __syncthreads();
  const int64_t g0 = (int64_t)blockIdx.x * kBinChunk;
  constexpr int kPer = kBinChunk / kBinThreads;  // Gaussians per thread: loads issued together
  uint32_t c[kPer];
  SplatAux a[kPer];
  uint32_t dh[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int64_t i = g0 + u * kBinThreads + threadIdx.x;
    c[u] = i < n ? (cnt_g[i] & kCntMask) : 0u;
    if (c[u]) {
      a[u] = aux_g[i];
      dh[u] = (uint32_t)__double2hiint(depth_g[i]);  // depth > z_near > 0: bits order like the value
    }
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    if (!c[u]) continue;
    const int64_t i = g0 + u * kBinThreads + threadIdx.x;
    const unsigned long long key = ((unsigned long long)dh[u] << 32) | (unsigned long long)(uint32_t)i;
    const uint32_t tx0 = a[u].tx0_ty0 & 0xffffu, ty0 = a[u].tx0_ty0 >> 16;
    const uint32_t nx = a[u].nx_ny & 0xffffu, ny = a[u].nx_ny >> 16;
    for (uint32_t y = 0; y < ny; ++y) {
      const uint32_t row = (ty0 + y) * (uint32_t)tiles_x + tx0;
      for (uint32_t x = 0; x < nx; ++x) {
        const uint32_t pos = atomicAdd(s_cur + row + x, 1u);
        if ((int64_t)pos < k_cap) ent_key[pos] = key;
      }
    }
  }
}

// ------------------------------------------------------ per-tile sort
// Bucket sort in shared memory: the tile's entries are counted into NB
// buckets of a quantised key q = (hi - min_hi) >> s (hi = high word of the
// FP64 depth; s makes the tile's span fit NB buckets), the bucket counts are
// scanned and every entry is placed with a shared-memory cursor (order inside
// a bucket arbitrary). Each bucket — a few entries at most for real depth
// distributions — is then ordered by the exact key (FP64 depth, gid) by
// insertion. A bucket of more than 32 entries (mass depth ties) makes the CTA
// re-sort the whole tile with stable LSD radix passes on (gid, depth low
// word, depth high word).
__device__ __forceinline__ uint32_t bin_lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

constexpr int kRxWarps = 4;  // warps that run the (fallback) radix passes

template <int CAP, int NT, int NB>
struct TileSortSmem {
  static constexpr int kWarps = NT / 32;
  uint32_t hi[CAP], gid[CAP];  // by arrival position
  uint16_t perm[2][CAP];
  union {
    uint32_t bucket[NB];
    struct {
      uint32_t wcnt[kRxWarps][256], woff[kRxWarps][256], run[256];
    } rx;
  } u;
  uint32_t hmin, hmax, vary_or, vary_and, long_run;
};

// One stable LSD pass over digit(o) (o = arrival position) of permutation in
// -> out, ranked by the first kRxWarps warps in rounds of kRxWarps * 32 items
// (fallback path only; every thread takes part in the barriers).
template <class SM, typename DigitF>
__device__ __forceinline__ void tile_radix_pass(SM& S, DigitF digit, int n, const uint16_t* in, uint16_t* out) {
  constexpr int kW = kRxWarps, NT = SM::kWarps * 32, kRound = kRxWarps * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool ranker = warp < kRxWarps;
  auto& R = S.u.rx;
  for (int d = threadIdx.x; d < 256; d += NT) {
    R.run[d] = 0;
    for (int w = 0; w < kW; ++w) R.wcnt[w][d] = 0;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += NT) atomicAdd(&R.run[digit(p)], 1u);
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the 256 digit counts (8 per lane)
    uint32_t v[8], s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = R.run[lane * 8 + k];
      s += v[k];
    }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t r = x - s;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      R.run[lane * 8 + k] = r;
      r += v[k];
    }
  }
  __syncthreads();
  const uint32_t lt = bin_lanemask_lt();
  for (int r0 = 0; r0 < n; r0 += kRound) {  // rounds of kRound items in current order
    const int p = r0 + threadIdx.x;
    const bool valid = ranker && p < n;
    uint32_t o = 0, dig = 0, rank = 0;
    if (ranker) {
      o = valid ? in[p] : 0u;
      dig = valid ? digit(o) : 256u + lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, dig);
      rank = __popc(peers & lt);
      if (valid && rank == 0) R.wcnt[warp][dig] = __popc(peers);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += NT) {
      uint32_t run = R.run[d];
#pragma unroll
      for (int w = 0; w < kW; ++w) {
        const uint32_t c = R.wcnt[w][d];
        R.woff[w][d] = run;
        run += c;
        R.wcnt[w][d] = 0;
      }
      R.run[d] = run;
    }
    __syncthreads();
    if (valid) out[R.woff[warp][dig] + rank] = (uint16_t)o;
    __syncthreads();
  }
}

// LSD passes over the bytes of a 32-bit key that vary inside the tile.
template <class SM, typename KeyF>
__device__ __forceinline__ int tile_radix_full(SM& S, KeyF key, int n, int sel) {
  constexpr int NT = SM::kWarps * 32;
  if (threadIdx.x == 0) {
    S.vary_or = 0u;
    S.vary_and = ~0u;
  }
  __syncthreads();
  uint32_t vo = 0u, va = ~0u;
  for (int p = threadIdx.x; p < n; p += NT) {
    const uint32_t k = key(p);
    vo |= k;
    va &= k;
  }
  vo = __reduce_or_sync(0xffffffffu, vo);
  va = __reduce_and_sync(0xffffffffu, va);
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&S.vary_or, vo);
    atomicAnd(&S.vary_and, va);
  }
  __syncthreads();
  const uint32_t vary = S.vary_or ^ S.vary_and;
  for (int b = 0; b < 4; ++b) {
    if (((vary >> (8 * b)) & 255u) == 0u) continue;
    const int sh = 8 * b;
    tile_radix_pass(S, [&](uint32_t o) { return (key(o) >> sh) & 255u; }, n, S.perm[sel], S.perm[sel ^ 1]);
    sel ^= 1;
  }
  return sel;
}

template <int CAP, int NT, int NB>
__device__ void sort_tile(TileSortSmem<CAP, NT, NB>& S, uint2 r, const unsigned long long* __restrict__ ent_key,
                          const double* __restrict__ depth_g, uint32_t* __restrict__ ent_gid) {
  constexpr int kNbBits = __builtin_ctz(NB);
  const int n = (int)(r.y - r.x);
  if (n < 1) return;
  if (threadIdx.x == 0) {
    S.hmin = ~0u;
    S.hmax = 0u;
    S.long_run = 0u;
  }
  for (int b = threadIdx.x; b < NB; b += NT) S.u.bucket[b] = 0;
  __syncthreads();
  uint32_t mn = ~0u, mx = 0u;
#pragma unroll 4
  for (int p = threadIdx.x; p < n; p += NT) {
    const unsigned long long k = ent_key[r.x + p];
    const uint32_t h = (uint32_t)(k >> 32);
    mn = min(mn, h);
    mx = max(mx, h);
    S.hi[p] = h;
    S.gid[p] = (uint32_t)k;
  }
  mn = __reduce_min_sync(0xffffffffu, mn);  // (loads above: independent, issued back to back)
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&S.hmin, mn);
    atomicMax(&S.hmax, mx);
  }
  __syncthreads();
  const uint32_t h0 = S.hmin, span = S.hmax - S.hmin;
  const int span_bits = span ? 32 - __clz((int)span) : 0;
  const int shift = span_bits > kNbBits ? span_bits - kNbBits : 0;  // ((hi - h0) >> shift) < NB
  auto qkey = [&](uint32_t o) { return (S.hi[o] - h0) >> shift; };
  // count, scan, place
  for (int p = threadIdx.x; p < n; p += NT) atomicAdd(&S.u.bucket[qkey(p)], 1u);
  __syncthreads();
  {
    constexpr int kPer = NB / NT;  // buckets per thread (contiguous)
    uint32_t v[kPer], sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      v[k] = S.u.bucket[threadIdx.x * kPer + k];
      sum += v[k];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= (unsigned)o) x += y;
    }
    __shared__ uint32_t s_warp[NT / 32];
    if ((threadIdx.x & 31) == 31) s_warp[threadIdx.x >> 5] = x;
    __syncthreads();
    uint32_t run = x - sum;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) run += s_warp[w];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      S.u.bucket[threadIdx.x * kPer + k] = run;
      run += v[k];
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += NT) S.perm[0][atomicAdd(&S.u.bucket[qkey(p)], 1u)] = (uint16_t)p;
  __syncthreads();
  // exact (FP64 depth, gid) order inside every bucket
  auto greater = [&](uint32_t a, uint32_t b) {
    const uint32_t ha = S.hi[a], hb = S.hi[b];
    if (ha != hb) return ha > hb;
    const uint32_t la = (uint32_t)__double2loint(depth_g[S.gid[a]]);
    const uint32_t lb = (uint32_t)__double2loint(depth_g[S.gid[b]]);
    if (la != lb) return la > lb;
    return S.gid[a] > S.gid[b];
  };
  uint16_t* ord = S.perm[0];
  // after the placement pass bucket[k] holds the end of bucket k in ord, so
  // each thread sorts whole buckets it owns without reading its neighbours'
  // (a thread never touches entries another thread is permuting)
  for (int k = threadIdx.x; k < NB; k += NT) {
    const int p = k ? (int)S.u.bucket[k - 1] : 0, e = (int)S.u.bucket[k];
    if (e - p < 2) continue;
    if (e - p > 32) {
      S.long_run = 1u;
      continue;
    }
    for (int a = p + 1; a < e; ++a) {  // insertion; bucket size <= 32
      const uint16_t v = ord[a];
      int b = a - 1;
      while (b >= p && greater(ord[b], v)) {
        ord[b + 1] = ord[b];
        --b;
      }
      ord[b + 1] = v;
    }
  }
  __syncthreads();
  int sel = 0;
  if (S.long_run) {
    for (int p = threadIdx.x; p < n; p += NT) S.perm[0][p] = (uint16_t)p;
    __syncthreads();
    const uint32_t* gid = S.gid;
    const uint32_t* hi = S.hi;
    sel = tile_radix_full(S, [&](uint32_t o) { return gid[o]; }, n, 0);
    sel = tile_radix_full(S, [&](uint32_t o) { return (uint32_t)__double2loint(depth_g[gid[o]]); }, n, sel);
    sel = tile_radix_full(S, [&](uint32_t o) { return hi[o]; }, n, sel);
  }
  const uint16_t* fin = S.perm[sel];
  for (int p = threadIdx.x; p < n; p += NT) ent_gid[r.x + p] = S.gid[fin[p]];
  __syncthreads();
}

#ifndef GSB_SORT_SMALL_THREADS
#define GSB_SORT_SMALL_THREADS 512
#endif
constexpr int kSortThreads = GSB_SORT_SMALL_THREADS, kSortLargeThreads = 1024;
using SmallSmem = TileSortSmem<kTileSortSmall, kSortThreads, (kTileSortSmall > 2048 ? kTileSortSmall : 2048)>;
using LargeSmem = TileSortSmem<kTileSortLarge, kSortLargeThreads, 4096>;
static_assert(2 * (sizeof(LargeSmem) + 128 + 1024) <= 228 * 1024, "two large-sort CTAs per SM");

// One CTA per tile with count <= kTileSortSmall.
__global__ void __launch_bounds__(kSortThreads) tile_sort_small_kernel(
    const uint2* __restrict__ ranges, const unsigned long long* __restrict__ ent_key,
    const double* __restrict__ depth_g, uint32_t* __restrict__ ent_gid, const uint32_t* __restrict__ counters,
    int64_t k_cap) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  SmallSmem& S = *reinterpret_cast<SmallSmem*>(s_raw);
  const uint2 r = ranges[blockIdx.x];
  const uint32_t cnt = r.y - r.x;
  if (cnt == 0u || cnt > (uint32_t)kTileSortSmall) return;
  if ((int64_t)counters[1] > k_cap || counters[2] != 0u) return;  // discarded iteration
  sort_tile(S, r, ent_key, depth_g, ent_gid);
}

// Persistent CTAs (two per SM) over the list of larger tiles.
__global__ void __launch_bounds__(kSortLargeThreads) tile_sort_large_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ big,
    const unsigned long long* __restrict__ ent_key, const double* __restrict__ depth_g,
    uint32_t* __restrict__ ent_gid, const uint32_t* __restrict__ counters, int64_t k_cap) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  LargeSmem& S = *reinterpret_cast<LargeSmem*>(s_raw);
  if ((int64_t)counters[1] > k_cap || counters[2] != 0u) return;
  const uint32_t nbig = counters[3];
  for (uint32_t b = blockIdx.x; b < nbig; b += gridDim.x) sort_tile(S, ranges[big[b]], ent_key, depth_g, ent_gid);
}

int init_bin_attributes() {
  GSB_CUDA(cudaFuncSetAttribute(tile_sort_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(SmallSmem)));
  GSB_CUDA(cudaFuncSetAttribute(tile_sort_large_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(LargeSmem)));
  const int tiles_smem = (int)(sizeof(uint32_t) * kBinMaxTiles);
  GSB_CUDA(cudaFuncSetAttribute(tile_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tiles_smem));
  GSB_CUDA(cudaFuncSetAttribute(tile_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tiles_smem));
  return GSB_OK;
}

size_t bin_hist_words(int64_t n, int n_tiles) { return (size_t)n_tiles * (size_t)bin_chunks(n) + 1; }

int launch_tile_bin(cudaStream_t st, gsb_frame* f, int64_t n, int64_t* launches) {
  const int n_tiles = f->tiles_x * f->tiles_y;
  if (n_tiles <= 0) return GSB_OK;
  uint32_t* counters = f->counters.as<uint32_t>();
  const int64_t nchunks = bin_chunks(n);
  const int64_t nh = (int64_t)n_tiles * nchunks;
  uint32_t* hist = f->tile_hist.as<uint32_t>();
  const size_t tiles_smem = sizeof(uint32_t) * n_tiles;
  if (n > 0) {
    tile_count_kernel<<<(unsigned)nchunks, kBinThreads, tiles_smem, st>>>(
        f->cnt_g.as<uint32_t>(), f->aux_g.as<SplatAux>(), n, n_tiles, f->tiles_x, nchunks, hist);
    *launches += 1;
  } else {
    GSB_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * nh, st));
  }
  if (int rc = scan_onepass(st, hist, nh, nullptr, false, hist, f->tile_scan.as<uint32_t>(), hist + nh, launches))
    return rc;
  tile_ranges_from_scan_kernel<<<(n_tiles + 255) / 256, 256, 0, st>>>(hist, n_tiles, nchunks, f->k_cap,
                                                                      f->ranges.as<uint2>(),
                                                                      f->tile_big.as<uint32_t>(), counters);
  *launches += 1;
  if (n > 0) {
    tile_scatter_kernel<<<(unsigned)nchunks, kBinThreads, tiles_smem, st>>>(
        f->cnt_g.as<uint32_t>(), f->aux_g.as<SplatAux>(), f->depth_g.as<double>(), n, n_tiles, f->tiles_x, nchunks,
        hist, f->k_cap, f->ent_key.as<unsigned long long>());
    tile_sort_small_kernel<<<n_tiles, kSortThreads, sizeof(SmallSmem), st>>>(
        f->ranges.as<uint2>(), f->ent_key.as<unsigned long long>(), f->depth_g.as<double>(),
        f->ent_gid.as<uint32_t>(), counters, f->k_cap);
    const int grid = std::min(n_tiles, 2 * f->ctx->num_sms);
    tile_sort_large_kernel<<<grid, kSortLargeThreads, sizeof(LargeSmem), st>>>(
        f->ranges.as<uint2>(), f->tile_big.as<uint32_t>(), f->ent_key.as<unsigned long long>(),
        f->depth_g.as<double>(), f->ent_gid.as<uint32_t>(), counters, f->k_cap);
    *launches += 3;
  }
  GSB_CHECK_LAUNCH("tile binning");
  return GSB_OK;
}

}  // namespace gsb
