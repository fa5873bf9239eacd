// gsb_internal.cuh — shared types, device layouts and launch helpers for
// libgsb200 (B200 / sm_100a). See DESIGN.md for the HBM layout rationale.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/gsb200.h"
#include <nvtx3/nvToolsExt.h>

namespace gsb {

// NVTX range over a C-ABI entry point (header-only NVTX v3: no link
// dependency; a profiler such as nsys / ncu --nvtx attaches through its
// injection library, otherwise the calls are no-ops).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define GSB_NVTX(name) ::gsb::NvtxRange gsb_nvtx_range_(name)

constexpr int kTile = 16;         // rasterizer tile (RasterConfig::tile_size, rasterizer.hpp:31)
constexpr int kTilePix = kTile * kTile;
constexpr int kMaxShCoeffs = 16;  // sh.hpp:10

// Camera as the kernels read it (device resident so the pose step can update
// it without a host round trip). R row-major world_to_cam, center = -R^T t.
struct CamDev {
  double fx, fy, cx, cy;
  double R[9];
  double t[3];
  double center[3];
  int32_t width, height, tiles_x, tiles_y;
};

struct RasterDev {
  float cutoff2_f, alpha_clamp_f, early_term_f, pad;
  double cutoff_sigma, alpha_clamp, dilation, early_termination, z_near;
};

// Per-splat record read by composite and the backward raster (rank order).
// mu2d stays FP64 so the tile-local offset (mu - tile origin) is formed
// without the ~3e-5 px FP32 rounding of absolute pixel coordinates.
struct __align__(16) SplatRec {
  double mu_x, mu_y;
  float conic_a, conic_b, conic_c, opacity;  // conic_b = symmetric off-diagonal
  float col_r, col_g, col_b;
  uint32_t clamp_bits;
};
static_assert(sizeof(SplatRec) == 48, "SplatRec layout");

// Per-splat bookkeeping (rank order): entry offset in the rank-major
// (pre-sort) entry stream, tile rect origin and width, Gaussian id.
struct __align__(16) SplatAux {
  uint32_t off;
  uint32_t tx0_ty0;  // tx0 | ty0 << 16
  uint32_t nx_ny;    // nx  | ny  << 16
  int32_t gid;
};

// Per-entry backward partial (PixelPartial, rasterizer.cpp:327-332) with the
// symmetric d_conic folded to 3 values: (D00, D01 (=D10), D11).
constexpr int kPartial = 9;  // d_mu2d(2) d_conic(3) d_color(3) d_opacity(1)

// cnt_g packs the tile count (low 28 bits) and the SH clamp bits (28..30).
constexpr uint32_t kCntMask = 0x0fffffffu;
constexpr int kClampShift = 28;

// Parameter planes of a cloud: plane-major [P][n_pad] FP32.
enum Plane : int {
  kMeanX = 0, kMeanY, kMeanZ, kQuatW, kQuatX, kQuatY, kQuatZ, kScaleX, kScaleY, kScaleZ, kOpacity,
  kShBase = 11
};
inline int num_planes(int sh_degree) { return kShBase + 3 * (sh_degree + 1) * (sh_degree + 1); }

// ------------------------------------------------ TMA bulk copies (sm_90+)
// 1-D bulk global->shared copies completing on an mbarrier (SASS UBLKCP):
// one elected thread stages whole parameter-plane segments of a CTA with no
// register cost and full memory-level parallelism.
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// Fixed-order sum of K4b's per-block pose partials (blocks[nb][6]) by a
// 256-thread block: four blocks' partials per round in block order, then a
// fixed binary tree — deterministic. Shared by pose_reduce_kernel and the
// session's fused pose_iter_kernel, so both give the same bits. out (shared,
// valid in thread 0): the 6-vector.
__device__ __forceinline__ void block_reduce_pose(const double* __restrict__ blocks, int64_t nb,
                                                  double (*s)[256], double out[6]) {
  double t[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t b0 = threadIdx.x; b0 < nb; b0 += 4 * 256) {
    double u[4][6];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t b = b0 + (int64_t)q * 256;
#pragma unroll
      for (int k = 0; k < 6; ++k) u[q][k] = b < nb ? blocks[b * 6 + k] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int k = 0; k < 6; ++k) t[k] += u[q][k];
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) s[k][threadIdx.x] = t[k];
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
#pragma unroll
      for (int k = 0; k < 6; ++k) s[k][threadIdx.x] += s[k][threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) out[k] = s[k][0];
}

// bytes: multiple of 16; src / dst 16-byte aligned.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
#endif  // __CUDACC__

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define GSB_CUDA(call)                                        \
  do {                                                        \
    cudaError_t e__ = (call);                                 \
    if (e__ != cudaSuccess) return ::gsb::cuda_fail(e__, #call); \
  } while (0)

#define GSB_CHECK_LAUNCH(what)                                \
  do {                                                        \
    cudaError_t e__ = cudaGetLastError();                     \
    if (e__ != cudaSuccess) return ::gsb::cuda_fail(e__, what); \
  } while (0)

// ---------------------------------------------------------------- buffers
// Grow-only device buffer; contents are not preserved across growth.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t want, bool* grew = nullptr) {
    if (want <= bytes) return cudaSuccess;
    if (grew) *grew = true;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t cap = want + want / 4 + 256;
    cudaError_t e = cudaMalloc(&p, cap);
    if (e == cudaSuccess) bytes = cap;
    return e;
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// K2 binning modes. Tile-local (default): per-tile entry counts and entry
// slots come out of preprocess, entries are scattered into their tile's
// range, and each tile's list is sorted by (FP64 depth, gid) in shared memory
// (k_bin.cu). Global: compaction + global stable depth sort + rank-major
// duplication + stable tile sort (k_sort.cu) — used when some tile holds more
// entries than the per-tile sort's capacity, and to materialise the
// reference's rank order for the splat-list export.
enum Binning : int { kBinTileLocal = 0, kBinGlobal = 1 };
#ifndef GSB_TILE_SORT_SMALL
#define GSB_TILE_SORT_SMALL 4096  // (2048 with 256 threads: sort stage 0.124 -> 0.108 ms at 4096 / 512)
#endif
constexpr int kTileSortSmall = GSB_TILE_SORT_SMALL;  // entries per tile sorted by one small-sort CTA
constexpr int kTileSortLarge = 8192;  // ... by the 512-thread persistent CTA (161 KB shared)
constexpr int kBinMaxTiles = 16384;   // per-tile counters held in shared memory (else global binning)

// Stage ids for the per-stage device timers (bench roofline attribution).
enum Stage : int {
  kStPreprocess = 0, kStSort, kStComposite, kStLoss, kStBwdRaster, kStBwdGeom, kStOptim, kStOther, kNumStages
};

struct StageTimer;  // defined in api.cu

// Joint-loop constants passed by value to the joint kernels (k_optim.cu).
struct JointCtl {
  int32_t iterations, slots, slot0, local, n_views, opacity_l1_steps, optimize_poses, nplanes, basis;
  double pos_lr_start, pos_lr_end, rot_lr, scale_lr, opacity_lr, sh_dc_lr, sh_rest_lr, cam_lr_start, cam_lr_end;
  double aniso_ratio, opacity_l1_weight, inv_slots;
};

}  // namespace gsb

// ------------------------------------------------------------- C structs
struct gsb_ctx {
  int device = 0;
  // objects created on this context (clouds, frames, images, ...) hold a
  // reference: gsb_ctx_destroy with live objects only marks the context
  // closing, and the last object's destroy frees it (any destruction order
  // of a caller's objects is safe)
  int64_t refs = 0;
  bool closing = false;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  gsb::DevBuf scratch_small;   // pinned-size device scratch (counters, partial sums)
  void* host_pinned = nullptr; // small pinned staging buffer
  size_t host_pinned_bytes = 0;
  int64_t launches = 0;
  bool profiling = false;
  gsb::StageTimer* timer = nullptr;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  gsb_frame* work = nullptr;   // scratch forward state shared by sessions
  cudaEvent_t (*stage_events)[2] = nullptr;  // set while capturing a profiled session graph
  int binning = 0;             // gsb::Binning preference (gsb_ctx_set_binning)
  std::vector<gsb_frame*> frame_pool;  // sized forward states returned by pose batches, reused
  std::vector<gsb::DevBuf> image_pool;  // target-image planes of destroyed gsb_images, reused by size
  std::vector<std::pair<void*, size_t>> pinned_pool;  // pinned session status blocks, reused
  void* up_buf[2] = {nullptr, nullptr};  // pinned image-upload staging slots (alternating)
  size_t up_bytes[2] = {0, 0};
  cudaEvent_t up_ev[2] = {nullptr, nullptr};  // last copy out of each slot
  int up_next = 0;
};

struct gsb_cloud {
  gsb_ctx* ctx = nullptr;
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  int64_t n = 0;
  int64_t n_pad = 0;
  int32_t sh_degree = 0, active_sh_degree = 0;
  gsb::DevBuf params;            // FP32 planes [num_planes][n_pad]
  uint64_t host_fingerprint = 0; // FNV-1a sample hash of the last uploaded FP64 arrays
  uint64_t version = 0;          // bumped by device-side updates (Adam)
  // The reference's fingerprint samples (rasterizer.cpp:62-71: 64 strided
  // Gaussians' FP64 parameters, in hash order) of the last host upload, valid
  // while version == fp_version (no device-side change since).
  std::vector<unsigned char> fp_samples;
  uint64_t fp_version = ~0ull;
};

struct gsb_image {
  gsb_ctx* ctx = nullptr;
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  int32_t width = 0, height = 0;
  gsb::DevBuf planes;  // FP32 [3][H*W]
};

struct gsb_grads {
  gsb_ctx* ctx = nullptr;
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  int64_t n = 0, n_pad = 0;
  int32_t sh_degree = 0;
  gsb::DevBuf planes;  // FP32 [num_planes + 2 (d_mu2d)][n_pad]
  gsb::DevBuf pose;    // double[6]
  bool valid = false;
};

struct gsb_adam {
  gsb_ctx* ctx = nullptr;
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  int64_t n = 0, n_pad = 0;
  int32_t sh_degree = 0;
  gsb::DevBuf m, v;    // FP32 planes like the cloud
  int64_t step[5] = {0, 0, 0, 0, 0};
};

struct gsb_frame {
  gsb_ctx* ctx = nullptr;
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  // bookkeeping
  int64_t n_gaussians = 0, n_splats = 0, n_entries = 0;
  int32_t width = 0, height = 0, tiles_x = 0, tiles_y = 0;
  uint64_t fingerprint = 0;
  uint64_t cloud_version = 0;
  int64_t k_cap = 0;      // entry capacity of the K-sized buffers
  uint64_t gen = 0;       // bumped whenever a buffer is reallocated (invalidates graphs)
  const gsb_cloud* cloud = nullptr;
  gsb_camera camera{};
  gsb_raster_config config{};
  double background[3] = {0, 0, 0};
  bool valid = false;
  bool has_dimage = false;
  bool lean = false;      // internal state (sessions, joint): skip the export-only K1 outputs
  // Hit masks (K3 -> pose-only K4a): per tile-list position, 16 regions x 16
  // bits of the pixels the composite applied the entry to (uint16 [k_cap][16]),
  // or (GSB_BWD_HITS = 2) one uint16 of touched-region bits per list position.
  bool want_hits = false;
  // device camera / config
  gsb::DevBuf cam;        // CamDev
  // per Gaussian (n)
  gsb::DevBuf rec_g;      // SplatRec
  gsb::DevBuf rect_g;     // uint2 (tx0|tx1<<16, ty0|ty1<<16)
  gsb::DevBuf cnt_g;      // uint32 tiles touched (0 = culled)
  gsb::DevBuf depth_g;    // double
  gsb::DevBuf radius_g;   // double (export only)
  gsb::DevBuf rank_of_g;  // int32 rank or -1
  gsb::DevBuf colj;       // FP32 [9][n_pad] colour/direction Jacobian (clamped rows zero)
  gsb::DevBuf off_g;      // uint32 entry offset of each visible Gaussian (rank-major stream)
  // visible (V)
  gsb::DevBuf vis_idx;    // uint32 gid, index order
  gsb::DevBuf dkey[2];    // uint32 depth keys (ping-pong)
  gsb::DevBuf dval[2];    // uint32 visible slot (ping-pong)
  gsb::DevBuf rec;        // SplatRec, rank order
  gsb::DevBuf aux;        // SplatAux, rank order
  gsb::DevBuf cnt_r;      // uint32 tiles per rank (scan input)
  // entries (K)
  gsb::DevBuf ekey[2];    // uint32 tile ids
  gsb::DevBuf eval_[2];   // uint32 ranks
  int sorted_sel = 0;     // which ekey/eval buffer holds the sorted result
  gsb::DevBuf ranges;     // uint2 per tile
  // per pixel
  gsb::DevBuf image;      // FP32 planes [3][P]
  gsb::DevBuf final_t;    // FP32 [P]
  gsb::DevBuf pixstate;   // uint32 contrib | overflow << 29
  gsb::DevBuf d_image;    // FP32 planes [3][P]
  // backward
  gsb::DevBuf partials;   // float [K][9] at pre-sort positions (live entries only)
  gsb::DevBuf hits;       // uint16 [k_cap][hit_words()] hit records by list position (want_hits frames)
  gsb::DevBuf tile_cut;   // double2 per tile: (FP64 depth, gid) of the last replayed entry, depth -1 if none
  gsb::DevBuf pose_blocks;// double [blocks][6]
  gsb::DevBuf d_pose;     // double[6]
  // loss
  gsb::DevBuf loss_blocks;// double [blocks][2]
  gsb::DevBuf loss_val;   // double[2] (l1, ssim)
  gsb::DevBuf mask_ws;    // masked_rgb_loss counts + norms (2 u64 + 4 doubles)
  gsb::DevBuf gmaps;      // FP32 [9][P] ssim gradient maps
  // scan / sort scratch
  gsb::DevBuf scan_tmp;
  gsb::DevBuf sort_hist;
  gsb::DevBuf counters;   // uint32 device counters: V, K, tile overflow flag
  // tile-local binning
  int binning = gsb::kBinTileLocal;
  bool fallback_global = false;  // a tile overflowed the per-tile sort: stay global
  gsb::DevBuf aux_g;      // SplatAux per Gaussian (slot base, tile rect)
  gsb::DevBuf tile_hist;  // uint32 [tiles][chunks] entry counts -> run offsets (+ total)
  gsb::DevBuf tile_scan;  // look-back scan status words
  gsb::DevBuf tile_big;   // uint32 tiles for the large per-tile sort (count in counters[3])
  gsb::DevBuf ent_key;    // uint64 (FP64 depth high word << 32 | gid) per entry, tile grouped
  gsb::DevBuf ent_gid;    // uint32 gid per entry -> depth-sorted tile lists
  bool ranks_valid = false;  // rank-order arrays (rec, aux, rank_of_g) hold this frame
  // RenderOutput export for config.tile_size != 16 (k_export.cu): tile lists /
  // ranges / contrib_count of the requested tile size, built on first export
  bool exp_valid = false;
  int32_t exp_tiles_x = 0, exp_tiles_y = 0;
  int64_t exp_k = 0;
  gsb::DevBuf exp_lists, exp_ranges, exp_contrib;
  // what the raster kernels read: tile lists of record ids, records, aux
  const uint32_t* list() const {
    return binning == gsb::kBinTileLocal ? ent_gid.as<uint32_t>() : eval_[sorted_sel].as<uint32_t>();
  }
  const gsb::SplatRec* list_rec() const {
    return binning == gsb::kBinTileLocal ? rec_g.as<gsb::SplatRec>() : rec.as<gsb::SplatRec>();
  }
  const gsb::SplatAux* list_aux() const {
    return binning == gsb::kBinTileLocal ? aux_g.as<gsb::SplatAux>() : aux.as<gsb::SplatAux>();
  }
};
