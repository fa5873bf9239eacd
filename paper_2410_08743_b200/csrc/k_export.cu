// k_export.cu — RenderOutput export for RasterConfig::tile_size != 16.
//
// The raster kernels always bin and composite 16x16 tiles. The tile size only
// changes which (pixel, splat) pairs the reference *examines*, not which ones
// contribute: a splat whose tile rect misses a pixel's 16-tile lies more than
// its radius 3 sqrt(lambda_max) from the pixel centre in x or y, so its
// Mahalanobis power there exceeds cutoff_sigma^2 and rasterizer.cpp:254 skips
// it. Image, transmittance, overflow bits and every gradient are therefore
// the same for any tile size; what differs are the exported tile lists /
// ranges and contrib_count (entries examined, counting skipped ones,
// rasterizer.cpp:251). Those are rebuilt here on the device for tile size S:
//
//   1. rect + count per splat (rank = depth order), exactly tile_span
//      (rasterizer.cpp:138-146) with S;
//   2. exclusive scan of the counts -> entry offsets; entries (tile, rank)
//      emitted splat by splat in row-major tile order;
//   3. stable LSD radix sort by tile -> per-tile lists in rank (= depth) order,
//      which is the reference's count / prefix / fill result; ranges from a
//      per-tile histogram (integer atomics, exact) and its exclusive scan, so
//      empty tiles get (offset, offset) as in rasterizer.cpp:151-156;
//   4. contrib_count for S: a pixel that terminated (final T below the early
//      termination threshold) stopped at the same splat in any tile order;
//      its position in the S-tile's list + 1 is found by binary search over
//      ranks; a pixel that never terminated examined its whole S-list.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gsb_internal.cuh"

namespace gsb {

__global__ void export_rect_kernel(const SplatRec* __restrict__ rec, const SplatAux* __restrict__ aux,
                                   const double* __restrict__ radius_g, int64_t V, int S, int tiles_x, int tiles_y,
                                   uint2* __restrict__ rect, uint32_t* __restrict__ count) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= V) return;
  const double u = rec[r].mu_x, v = rec[r].mu_y, rad = radius_g[aux[r].gid], s = (double)S;
  auto span = [s](double lo_v, double hi_v, int n, int* lo, int* hi) {
    const double top = n - 1.0;
    double a = floor(__ddiv_rn(lo_v, s)), b = floor(__ddiv_rn(hi_v, s));
    a = a < 0.0 ? 0.0 : (a > top ? top : a);
    b = b < 0.0 ? 0.0 : (b > top ? top : b);
    *lo = (int)a;
    *hi = (int)b;
  };
  int tx0, tx1, ty0, ty1;
  span(__dsub_rn(u, rad), __dadd_rn(u, rad), tiles_x, &tx0, &tx1);
  span(__dsub_rn(v, rad), __dadd_rn(v, rad), tiles_y, &ty0, &ty1);
  rect[r] = make_uint2((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16));
  count[r] = (uint32_t)(tx1 - tx0 + 1) * (uint32_t)(ty1 - ty0 + 1);
}

__global__ void export_fill_kernel(const uint2* __restrict__ rect, const uint32_t* __restrict__ offset, int64_t V,
                                   int tiles_x, uint32_t* __restrict__ key, uint32_t* __restrict__ val,
                                   uint32_t* __restrict__ tile_count) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= V) return;
  const uint2 q = rect[r];
  const uint32_t tx0 = q.x & 0xffffu, tx1 = q.x >> 16, ty0 = q.y & 0xffffu, ty1 = q.y >> 16;
  uint32_t o = offset[r];
  for (uint32_t ty = ty0; ty <= ty1; ++ty)
    for (uint32_t tx = tx0; tx <= tx1; ++tx) {
      const uint32_t t = ty * (uint32_t)tiles_x + tx;
      key[o] = t;
      val[o] = (uint32_t)r;
      ++o;
      atomicAdd(tile_count + t, 1u);
    }
}

__global__ void export_ranges_kernel(const uint32_t* __restrict__ begin, const uint32_t* __restrict__ count, int T,
                                     int2* __restrict__ ranges) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) ranges[t] = make_int2((int)begin[t], (int)(begin[t] + count[t]));
}

// list16: the 16-tile lists the raster ran on (gids when tile-local, ranks
// when global: rank_of maps gids; NULL for ranks).
__global__ void export_contrib_kernel(const uint32_t* __restrict__ pixstate, const float* __restrict__ final_t,
                                      const uint2* __restrict__ ranges16, const uint32_t* __restrict__ list16,
                                      const int32_t* __restrict__ rank_of, int W, int H, int tiles16_x, int S,
                                      int tilesS_x, float early_term, const int2* __restrict__ rangesS,
                                      const uint32_t* __restrict__ listS, int32_t* __restrict__ contrib_out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)W * H) return;
  const int x = (int)(p % W), y = (int)(p / W);
  const int2 rs = rangesS[(y / S) * tilesS_x + x / S];
  const uint32_t c16 = pixstate[p] & 0x1fffffffu;
  int32_t out = rs.y - rs.x;  // never terminated: the whole S-list was examined
  if (c16 > 0 && final_t[p] < early_term) {
    const uint2 r16 = ranges16[(y / kTile) * tiles16_x + x / kTile];
    const uint32_t id = list16[r16.x + c16 - 1];
    const uint32_t rank = rank_of ? (uint32_t)rank_of[id] : id;
    int lo = rs.x, hi = rs.y;  // S-list ascending in rank
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (listS[mid] < rank) lo = mid + 1;
      else hi = mid;
    }
    out = lo - rs.x + 1;
  }
  contrib_out[p] = out;
}

static int grid1(int64_t n) { return (int)((n + 255) / 256); }

// Fills f->exp_* for tile size S (f holds a valid forward state with the
// global rank order materialised and radius_g written).
int build_export_tiles(cudaStream_t st, gsb_frame* f, int S) {
  const int64_t V = f->n_splats;
  const int tx = (f->width + S - 1) / S, ty = (f->height + S - 1) / S, T = tx * ty;
  const int64_t P = (int64_t)f->width * f->height;
  DevBuf rect, cnt, off, key[2], val[2], tcount, tbegin, tmp;
  GSB_CUDA(rect.reserve(sizeof(uint2) * std::max<int64_t>(V, 1)));
  GSB_CUDA(cnt.reserve(sizeof(uint32_t) * (V + 1)));
  GSB_CUDA(off.reserve(sizeof(uint32_t) * (V + 1)));
  GSB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t) * (V + 1), st));
  if (V > 0)
    export_rect_kernel<<<grid1(V), 256, 0, st>>>(f->rec.as<SplatRec>(), f->aux.as<SplatAux>(),
                                                 f->radius_g.as<double>(), V, S, tx, ty, rect.as<uint2>(),
                                                 cnt.as<uint32_t>());
  GSB_CHECK_LAUNCH("export_rect_kernel");
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<uint32_t>(), off.as<uint32_t>(), (int)(V + 1), st);
  GSB_CUDA(tmp.reserve(std::max<size_t>(tb, 16)));
  GSB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.as<uint32_t>(), off.as<uint32_t>(), (int)(V + 1), st));
  uint32_t K = 0;
  GSB_CUDA(cudaMemcpyAsync(&K, off.as<uint32_t>() + V, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  GSB_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < 2; ++b) {
    GSB_CUDA(key[b].reserve(sizeof(uint32_t) * std::max<uint32_t>(K, 1)));
    GSB_CUDA(val[b].reserve(sizeof(uint32_t) * std::max<uint32_t>(K, 1)));
  }
  GSB_CUDA(tcount.reserve(sizeof(uint32_t) * (T + 1)));
  GSB_CUDA(tbegin.reserve(sizeof(uint32_t) * (T + 1)));
  GSB_CUDA(cudaMemsetAsync(tcount.p, 0, sizeof(uint32_t) * (T + 1), st));
  if (V > 0)
    export_fill_kernel<<<grid1(V), 256, 0, st>>>(rect.as<uint2>(), off.as<uint32_t>(), V, tx, key[0].as<uint32_t>(),
                                                 val[0].as<uint32_t>(), tcount.as<uint32_t>());
  GSB_CHECK_LAUNCH("export_fill_kernel");
  int bits = 1;
  while ((1ll << bits) < T) ++bits;
  cub::DoubleBuffer<uint32_t> dk(key[0].as<uint32_t>(), key[1].as<uint32_t>()),
      dv(val[0].as<uint32_t>(), val[1].as<uint32_t>());
  tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)K, 0, bits, st);
  GSB_CUDA(tmp.reserve(std::max<size_t>(tb, 16)));
  if (K > 0) GSB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, (int)K, 0, bits, st));
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, tcount.as<uint32_t>(), tbegin.as<uint32_t>(), T + 1, st);
  GSB_CUDA(tmp.reserve(std::max<size_t>(tb, 16)));
  GSB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, tcount.as<uint32_t>(), tbegin.as<uint32_t>(), T + 1, st));
  GSB_CUDA(f->exp_ranges.reserve(sizeof(int2) * std::max(T, 1)));
  export_ranges_kernel<<<grid1(T), 256, 0, st>>>(tbegin.as<uint32_t>(), tcount.as<uint32_t>(), T,
                                                 f->exp_ranges.as<int2>());
  GSB_CHECK_LAUNCH("export_ranges_kernel");
  GSB_CUDA(f->exp_lists.reserve(sizeof(uint32_t) * std::max<uint32_t>(K, 1)));
  if (K > 0)
    GSB_CUDA(cudaMemcpyAsync(f->exp_lists.p, dv.Current(), sizeof(uint32_t) * K, cudaMemcpyDeviceToDevice, st));
  GSB_CUDA(f->exp_contrib.reserve(sizeof(int32_t) * std::max<int64_t>(P, 1)));
  const bool tile_local = f->binning == kBinTileLocal;
  if (P > 0)
    export_contrib_kernel<<<grid1(P), 256, 0, st>>>(
        f->pixstate.as<uint32_t>(), f->final_t.as<float>(), f->ranges.as<uint2>(), f->list(),
        tile_local ? f->rank_of_g.as<int32_t>() : nullptr, f->width, f->height, f->tiles_x, S, tx,
        (float)f->config.early_termination, f->exp_ranges.as<int2>(), f->exp_lists.as<uint32_t>(),
        f->exp_contrib.as<int32_t>());
  GSB_CHECK_LAUNCH("export_contrib_kernel");
  GSB_CUDA(cudaStreamSynchronize(st));
  for (DevBuf* b : {&rect, &cnt, &off, &key[0], &key[1], &val[0], &val[1], &tcount, &tbegin, &tmp}) b->release();
  f->exp_tiles_x = tx;
  f->exp_tiles_y = ty;
  f->exp_k = K;
  f->exp_valid = true;
  return GSB_OK;
}

}  // namespace gsb
