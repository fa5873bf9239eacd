// api.cu — the C ABI (include/gsb200.h): context / cloud / frame objects and
// the host orchestration of the hot path (render -> loss -> backward -> pose
// step) on one CUDA stream. All arithmetic runs in the kernels of
// k_*.cu; the host only sizes buffers, converts the reference's FP64
// host layouts at the boundary and sequences launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <dlfcn.h>
#include <nccl.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gsb_internal.cuh"

namespace gsb {

// kernels (k_*.cu)
int launch_preprocess(cudaStream_t st, const gsb_cloud* cloud, const CamDev* cam, const RasterDev& rc, gsb_frame* f);
int launch_preprocess_multi(cudaStream_t st, const gsb_cloud* cloud, const RasterDev& rc, const CamDev* const* cams,
                            gsb_frame* const* frames, int nviews);
int scan_exclusive(cudaStream_t st, const uint32_t* in, int64_t cap, const uint32_t* n_dev, bool flag, uint32_t* out,
                   uint32_t* scratch, uint32_t* total, int64_t* launches);
size_t scan_words(int64_t n);
int radix_sort_pairs(cudaStream_t st, uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                     int total_bits, uint32_t* hist, int* result_sel, int64_t* launches);
size_t radix_hist_words(int64_t n, int total_bits);
int scan_onepass(cudaStream_t st, const uint32_t* in, int64_t cap, const uint32_t* n_dev, bool flag, uint32_t* out,
                 uint32_t* status, uint32_t* total, int64_t* launches);
size_t scan_onepass_words(int64_t cap);
int onesweep_sort_pairs(cudaStream_t st, uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                        int total_bits, uint32_t* ws, int* result_sel, int64_t* launches);
size_t onesweep_words(int64_t cap, int total_bits);
int launch_compact(cudaStream_t st, const uint32_t* cnt_g, const uint32_t* vis_pos, const double* depth_g, int64_t n,
                   uint32_t* vis_idx, uint32_t* dkey, uint32_t* dval);
int launch_depth_tie_fix(cudaStream_t st, const uint32_t* key, uint32_t* val, const uint32_t* vis_idx,
                         const double* depth_g, int64_t cap, const uint32_t* nv_dev);
int launch_gather_ranks(cudaStream_t st, const uint32_t* sorted_v, const uint32_t* vis_idx, const SplatRec* rec_g,
                        const uint2* rect_g, const uint32_t* cnt_g, int64_t cap, const uint32_t* nv_dev, SplatRec* rec,
                        SplatAux* aux, uint32_t* cnt_r, int32_t* rank_of_g);
int launch_duplicate(cudaStream_t st, const uint32_t* offs, SplatAux* aux, int64_t cap, const uint32_t* nv_dev,
                     int tiles_x, int64_t k_cap, uint32_t* ekey, uint32_t* eval, uint32_t* off_g);
int launch_tile_ranges(cudaStream_t st, const uint32_t* ekey, int64_t k_cap, const uint32_t* k_dev, int n_tiles,
                       uint2* ranges);
int launch_tile_bin(cudaStream_t st, gsb_frame* f, int64_t n, int64_t* launches);
size_t bin_hist_words(int64_t n, int n_tiles);
int init_bin_attributes();
int launch_composite(cudaStream_t st, gsb_frame* f, const RasterDev& rc);
bool hit_masks_enabled();
int hit_words();
int build_export_tiles(cudaStream_t st, gsb_frame* f, int S);
int launch_expected_depth(cudaStream_t st, gsb_frame* f, const RasterDev& rc, float* depth_out, float* weight_out);
int launch_backward_raster(cudaStream_t st, gsb_frame* f, const RasterDev& rc, bool pose_only);
int64_t bwd_geom_blocks(int64_t n);
int launch_backward_geom(cudaStream_t st, const gsb_cloud* cloud, gsb_frame* f, const RasterDev& rc, bool full,
                         float* grads, int64_t* launches, bool reduce = true);
int launch_rgb_loss(cudaStream_t st, const float* ren, const float* tgt, int W, int H, double beta, float* gmaps,
                    double* block_sums, double* out3, float* d_image, int64_t* launches, const float* mask_t = nullptr,
                    double mask_thr = 0.0, void* mask_ws = nullptr);
size_t loss_block_count(int W, int H);
int init_loss_constants();
int init_loss_attributes();
int init_preprocess_attributes();
int launch_pose_iter(cudaStream_t st, void* state, const double* pose_blocks, int64_t nb, double* dpose_out,
                     const double* loss3, double lr_start, double lr_end, double eps, int budget, CamDev* cam,
                     double* trace_pose, double* trace_loss, const uint32_t* k_dev, int64_t k_cap);
int32_t pose_state_take_aborted(void* host_state, uint32_t* k_max, uint32_t* tile_ovf);
int32_t pose_state_aborted(const void* host_state);
size_t pose_state_bytes();
int pose_state_init(void* host_state, const double pose[12]);
void pose_state_read(const void* host_state, double best_pose[12], double cur_pose[12], double* final_loss,
                     int32_t* steps_used, int32_t* converged, int32_t* stop, double applied[6], double m[6],
                     double v[6], int64_t* step);
void pose_state_set_adam(void* host_state, const double m[6], const double v[6], int64_t step);
int launch_pose_step(cudaStream_t st, void* states, const double* dpose, double lr, int nb);
int launch_adam_f64(cudaStream_t st, double* p, const double* g, double* m, double* v, int64_t n, double lr,
                    const double* lrs, int64_t step);
int launch_joint_slot_begin(cudaStream_t st, const void* js, const int32_t* seq, const JointCtl& ctl, int b,
                            const CamDev* cams, CamDev* frame_cam, const float* const* targets, float* tbuf,
                            int64_t n3p);
int launch_joint_slot_end(cudaStream_t st, const JointCtl& ctl, int b, const double* d_pose, const double* loss3,
                          const uint32_t* counters, int64_t k_cap, double* xchg);
int launch_joint_sum(cudaStream_t st, float* g0, const float* rest, int64_t len, int nrest, int64_t stride);
int64_t joint_adam_blocks(int64_t n);
int64_t joint_red_doubles(int64_t n);
int launch_joint_adam(cudaStream_t st, float* params, const float* grads, float* m, float* v, int64_t n,
                      int64_t n_pad, const void* js, const JointCtl& ctl, const double* xchg, double* red_blocks);
int launch_joint_finalize(cudaStream_t st, void* js, const int32_t* seq, const JointCtl& ctl, const double* xchg,
                          const double* red_blocks, int64_t nblocks, void* poses, CamDev* cams, double* trace_total,
                          double* trace_l1);
size_t joint_state_bytes();
size_t joint_xchg_doubles();
void joint_state_read(const void* host, int64_t* t, int32_t* diverged, int32_t* aborted, double* k_max,
                      int32_t* tile);
void joint_state_clear_abort(void* host);
int launch_grad_norm(cudaStream_t st, const float* grads, int nplanes, int64_t n_pad, int64_t n,
                     const uint32_t* cnt_g, double scale, double* stage);
int launch_grad_accum_commit(cudaStream_t st, const double* stage, int local, int64_t stride, int64_t n,
                             const void* js, const JointCtl& ctl, const double* xchg, double* gsum, int32_t* gcnt);
int densify_bbox_blocks();
int launch_densify_bbox(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, float* out);
int launch_densify_action(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, const double* gsum,
                          const int32_t* gcnt, double grad_threshold, double size_threshold, uint32_t* keep,
                          uint32_t* extra, uint32_t* split);
int launch_densify_build(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, int nplanes,
                         const uint32_t* keep, const uint32_t* keep_pos, const uint32_t* extra,
                         const uint32_t* extra_pos, const uint32_t* split_rank, const double* normals,
                         uint32_t n_keep, float* out, int64_t n_pad_o, int32_t* src_o);
int launch_densify_logit_keys(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, uint32_t* keys,
                              uint32_t* vals);
int launch_densify_prune_flag(cudaStream_t st, const float* params, int64_t n, int64_t n_pad, double threshold,
                              uint32_t* flag);
int launch_densify_gather(cudaStream_t st, const float* in, int64_t n, int64_t n_pad_i, int nplanes,
                          const uint32_t* flag, const uint32_t* pos, const int32_t* src_i, float* out,
                          int64_t n_pad_o, int32_t* src_o);
int launch_densify_adam_remap(cudaStream_t st, const float* m, const float* v, int64_t n_pad_i, int nplanes,
                              const int32_t* src, int64_t n_o, int64_t n_pad_o, float* m_o, float* v_o);
int launch_cloud_adam(cudaStream_t st, float* params, const float* grads, float* m, float* v, int64_t n,
                      int64_t n_pad, int sh_degree, const double lrs[6], const int64_t steps[5]);

// ---------------------------------------------------------------- errors
static thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }
int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? GSB_ERR_OUT_OF_MEMORY : GSB_ERR_CUDA;
}

// ---------------------------------------------------------- stage timer
struct StageTimer {
  struct Pair {
    cudaEvent_t a, b;
    int stage;
  };
  std::vector<Pair> pool;
  size_t used = 0;
  int open_stage = -1;
  double ms[kNumStages] = {0};
  int64_t count[kNumStages] = {0};
  cudaError_t begin(cudaStream_t st, int stage) {
    if (used == pool.size()) {
      Pair p;
      cudaEventCreate(&p.a);
      cudaEventCreate(&p.b);
      pool.push_back(p);
    }
    pool[used].stage = stage;
    open_stage = stage;
    return cudaEventRecord(pool[used].a, st);
  }
  cudaError_t end(cudaStream_t st) {
    cudaError_t e = cudaEventRecord(pool[used].b, st);
    ++used;
    open_stage = -1;
    return e;
  }
  cudaError_t collect() {
    for (size_t i = 0; i < used; ++i) {
      cudaError_t e = cudaEventSynchronize(pool[i].b);
      if (e != cudaSuccess) return e;
      float t = 0.f;
      cudaEventElapsedTime(&t, pool[i].a, pool[i].b);
      ms[pool[i].stage] += t;
      count[pool[i].stage] += 1;
    }
    used = 0;
    return cudaSuccess;
  }
  void reset() {
    used = 0;
    for (int k = 0; k < kNumStages; ++k) {
      ms[k] = 0;
      count[k] = 0;
    }
  }
  ~StageTimer() {
    for (auto& p : pool) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
  }
};

// Brackets a stage's launches with CUDA events on the context stream: into
// the context's event pool (eager launches) or, while a session graph is
// being captured with profiling on, into that session's per-stage events.
struct StageScope {
  gsb_ctx* ctx;
  int stage;
  StageScope(gsb_ctx* c, int s) : ctx(c), stage(s) {
    if (ctx->stage_events) {
      cudaEventRecordWithFlags(ctx->stage_events[stage][0], ctx->stream, cudaEventRecordExternal);
    } else if (ctx->profiling && ctx->timer) {
      if (ctx->timer->used > 4096) ctx->timer->collect();
      ctx->timer->begin(ctx->stream, stage);
    }
  }
  ~StageScope() {
    if (ctx->stage_events) cudaEventRecordWithFlags(ctx->stage_events[stage][1], ctx->stream, cudaEventRecordExternal);
    else if (ctx->profiling && ctx->timer) ctx->timer->end(ctx->stream);
  }
};

// --------------------------------------------------------------- helpers
static int cuda_fail_or_ok(cudaError_t e) { return e == cudaSuccess ? GSB_OK : cuda_fail(e, "cudaMemcpy"); }

// GSB_DEBUG=1: host-side events (graph captures, buffer growth, discarded
// iterations, binning fallbacks) on stderr, for diagnosing e2e overheads.
static bool debug_on() {
  static const bool on = [] {
    const char* e = std::getenv("GSB_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}
static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static int ensure_device(gsb_ctx* ctx) {
  if (!ctx) return fail(GSB_ERR_INVALID_ARGUMENT, "null context");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  return GSB_OK;
}

static void* pinned(gsb_ctx* ctx, size_t bytes) {
  if (bytes > ctx->host_pinned_bytes) {
    if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
    ctx->host_pinned = nullptr;
    ctx->host_pinned_bytes = 0;
    size_t cap = bytes + bytes / 4 + 4096;
    if (cudaMallocHost(&ctx->host_pinned, cap) != cudaSuccess) return nullptr;
    ctx->host_pinned_bytes = cap;
  }
  return ctx->host_pinned;
}

#define GSB_RESERVE(buf, bytes) GSB_CUDA((buf).reserve(bytes))

static uint64_t fnv1a(uint64_t h, const void* data, size_t n) {  // rasterizer.cpp:41-48
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// rasterizer.cpp:52-73: FNV-1a over the sizes, degrees and the full camera,
// then 64 strided samples of every parameter array. `exact` (exported forward
// states, gsb_render): when the cloud holds exactly what was last uploaded
// from the host, the samples are that upload's FP64 values and the result is
// the reference's fingerprint bit for bit. A cloud changed on the device
// (Adam, densify, synth, PLY) has no FP64 host copy: its (identity, version)
// pair stands in for the samples — every mutation goes through this API and
// bumps the version, so a stale forward state is still rejected. Internal
// forward states (sessions, joint; never exported) always use the cheap form.
static uint64_t fingerprint(const gsb_cloud* cloud, const gsb_camera* cam, bool exact) {
  uint64_t h = 0xcbf29ce484222325ull;
  const int64_t n = cloud->n;
  h = fnv1a(h, &n, sizeof n);
  h = fnv1a(h, &cloud->sh_degree, sizeof(int32_t));
  h = fnv1a(h, &cloud->active_sh_degree, sizeof(int32_t));
  const double f4[4] = {cam->fx, cam->fy, cam->cx, cam->cy};
  h = fnv1a(h, f4, sizeof f4);
  const int32_t wh[2] = {cam->width, cam->height};
  h = fnv1a(h, wh, sizeof wh);
  // Se3Pose::rotation.data(): Eigen matrices are column-major
  const double Rcm[9] = {cam->R[0], cam->R[3], cam->R[6], cam->R[1], cam->R[4], cam->R[7], cam->R[2], cam->R[5], cam->R[8]};
  h = fnv1a(h, Rcm, sizeof Rcm);
  h = fnv1a(h, cam->t, sizeof(double) * 3);
  if (exact && cloud->fp_version == cloud->version) return fnv1a(h, cloud->fp_samples.data(), cloud->fp_samples.size());
  const uintptr_t id = reinterpret_cast<uintptr_t>(cloud);
  h = fnv1a(h, &id, sizeof id);
  h = fnv1a(h, &cloud->host_fingerprint, sizeof(uint64_t));
  h = fnv1a(h, &cloud->version, sizeof(uint64_t));
  return h;
}

static CamDev make_camdev(const gsb_camera* c, int tile) {
  CamDev d;
  d.fx = c->fx;
  d.fy = c->fy;
  d.cx = c->cx;
  d.cy = c->cy;
  for (int k = 0; k < 9; ++k) d.R[k] = c->R[k];
  for (int k = 0; k < 3; ++k) d.t[k] = c->t[k];
  for (int i = 0; i < 3; ++i) {  // Camera::center = -(R^T t) (rasterizer.hpp:24)
    const double r = c->R[0 * 3 + i] * c->t[0] + c->R[1 * 3 + i] * c->t[1] + c->R[2 * 3 + i] * c->t[2];
    d.center[i] = -r;
  }
  d.width = c->width;
  d.height = c->height;
  d.tiles_x = (c->width + tile - 1) / tile;
  d.tiles_y = (c->height + tile - 1) / tile;
  return d;
}

static RasterDev make_rasterdev(const gsb_raster_config* c) {
  RasterDev r;
  r.cutoff_sigma = c->cutoff_sigma;
  r.alpha_clamp = c->alpha_clamp;
  r.dilation = c->dilation;
  r.early_termination = c->early_termination;
  r.z_near = c->z_near;
  r.cutoff2_f = (float)(c->cutoff_sigma * c->cutoff_sigma);
  r.alpha_clamp_f = (float)c->alpha_clamp;
  r.early_term_f = (float)c->early_termination;
  r.pad = 0.f;
  return r;
}

static int validate_config(const gsb_raster_config* cfg) {
  if (!cfg) return fail(GSB_ERR_INVALID_ARGUMENT, "null raster config");
  // any tile size is accepted: the kernels bin 16x16 tiles, and RenderOutput's
  // tile lists / ranges / contrib_count are exported for the requested size
  // (k_export.cu explains why nothing else depends on it)
  if (cfg->tile_size < 1 || cfg->tile_size > 4096) return fail(GSB_ERR_INVALID_CONFIG, "tile_size out of range");
  if (!(cfg->cutoff_sigma > 0.0) || !(cfg->alpha_clamp > 0.0) || cfg->alpha_clamp >= 1.0 || cfg->dilation < 0.0 ||
      cfg->early_termination < 0.0)
    return fail(GSB_ERR_INVALID_CONFIG, "raster config out of range");
  return GSB_OK;
}

// Copies `count` u32 device counters to host through pinned memory (one sync).
static int read_counters(gsb_ctx* ctx, const uint32_t* dev, uint32_t* host, int count) {
  uint32_t* h = static_cast<uint32_t*>(pinned(ctx, sizeof(uint32_t) * count));
  if (!h) return fail(GSB_ERR_OUT_OF_MEMORY, "pinned staging");
  GSB_CUDA(cudaMemcpyAsync(h, dev, sizeof(uint32_t) * count, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < count; ++i) host[i] = h[i];
  return GSB_OK;
}

// K2 primitives: reduce-then-scan scans and hist/scan/scatter LSD passes
// (default), or single-pass decoupled-lookback scan / Onesweep sort
// (GSB_SORT=onesweep). Both produce bit-identical results; on B200 at these
// sizes the whole-wave look-back chains make Onesweep slower (measured
// 0.48 vs 0.31 ms per sort stage), so it stays opt-in for A/B measurement.
static bool legacy_sort() {
  static const bool legacy = [] {
    const char* e = std::getenv("GSB_SORT");
    return !(e && std::strcmp(e, "onesweep") == 0);
  }();
  return legacy;
}
static int scan_any(cudaStream_t st, const uint32_t* in, int64_t cap, const uint32_t* n_dev, bool flag, uint32_t* out,
                    uint32_t* scratch, uint32_t* total, int64_t* launches) {
  return legacy_sort() ? scan_exclusive(st, in, cap, n_dev, flag, out, scratch, total, launches)
                       : scan_onepass(st, in, cap, n_dev, flag, out, scratch, total, launches);
}
static int sort_any(cudaStream_t st, uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                    int bits, uint32_t* ws, int* sel, int64_t* launches) {
  return legacy_sort() ? radix_sort_pairs(st, keys, vals, cap, n_dev, bits, ws, sel, launches)
                       : onesweep_sort_pairs(st, keys, vals, cap, n_dev, bits, ws, sel, launches);
}

static int tile_bits(int n_tiles) {
  int bits = 0;
  while ((1 << bits) < n_tiles) ++bits;
  return bits;
}

// Sizes every forward/backward buffer of the frame for (cloud, image size,
// entry capacity). Any reallocation bumps f->gen (captured graphs hold raw
// pointers and must be rebuilt).
// First entry capacity of a forward state: 4 entries per Gaussian (the C3
// scene has K ≈ 3.0 N at its views; 3 N left a few hundred entries of
// headroom). An overflow is still detected on the device and the iteration
// re-run with a larger capacity.
static int64_t initial_k_cap(int64_t n) { return std::max<int64_t>(4 * n, 1 << 16); }

static int frame_reserve(gsb_frame* f, const gsb_cloud* cloud, int64_t k_cap) {
  const int64_t n = std::max<int64_t>(cloud->n, 1);
  const int64_t np = std::max<int64_t>(cloud->n_pad, 1);
  const int n_tiles = std::max(f->tiles_x * f->tiles_y, 1);
  const int64_t npix = std::max<int64_t>((int64_t)f->width * f->height, 1);
  k_cap = std::max<int64_t>(k_cap, 1024);
  bool grew = false;
  GSB_CUDA(f->cam.reserve(sizeof(CamDev), &grew));
  GSB_CUDA(f->counters.reserve(64, &grew));
  GSB_CUDA(f->aux_g.reserve(sizeof(SplatAux) * n, &grew));
  GSB_CUDA(f->tile_hist.reserve(sizeof(uint32_t) * bin_hist_words(n, n_tiles), &grew));
  GSB_CUDA(f->tile_scan.reserve(sizeof(uint32_t) * scan_onepass_words(bin_hist_words(n, n_tiles)), &grew));
  GSB_CUDA(f->tile_big.reserve(sizeof(uint32_t) * n_tiles, &grew));
  GSB_CUDA(f->rec_g.reserve(sizeof(SplatRec) * n, &grew));
  GSB_CUDA(f->rect_g.reserve(sizeof(uint2) * n, &grew));
  GSB_CUDA(f->cnt_g.reserve(sizeof(uint32_t) * np, &grew));  // n_pad: TMA-staged by 16 B
  GSB_CUDA(f->depth_g.reserve(sizeof(double) * n, &grew));
  GSB_CUDA(f->radius_g.reserve(sizeof(double) * n, &grew));
  GSB_CUDA(f->rank_of_g.reserve(sizeof(int32_t) * n, &grew));
  GSB_CUDA(f->colj.reserve(sizeof(float) * 9 * np, &grew));
  GSB_CUDA(f->off_g.reserve(sizeof(uint32_t) * np, &grew));
  GSB_CUDA(f->vis_idx.reserve(sizeof(uint32_t) * n, &grew));
  GSB_CUDA(f->cnt_r.reserve(sizeof(uint32_t) * n, &grew));
  for (int b = 0; b < 2; ++b) {
    GSB_CUDA(f->dkey[b].reserve(sizeof(uint32_t) * n, &grew));
    GSB_CUDA(f->dval[b].reserve(sizeof(uint32_t) * n, &grew));
    GSB_CUDA(f->ekey[b].reserve(sizeof(uint32_t) * k_cap, &grew));
    GSB_CUDA(f->eval_[b].reserve(sizeof(uint32_t) * k_cap, &grew));
  }
  GSB_CUDA(f->ent_key.reserve(sizeof(uint64_t) * k_cap, &grew));
  GSB_CUDA(f->ent_gid.reserve(sizeof(uint32_t) * k_cap, &grew));
  GSB_CUDA(f->rec.reserve(sizeof(SplatRec) * n, &grew));
  GSB_CUDA(f->aux.reserve(sizeof(SplatAux) * n, &grew));
  GSB_CUDA(f->scan_tmp.reserve(sizeof(uint32_t) * (std::max(scan_onepass_words(n), scan_words(n)) + 64), &grew));
  const size_t hist = std::max(std::max(onesweep_words(n, 32), onesweep_words(k_cap, tile_bits(n_tiles))),
                               std::max(radix_hist_words(n, 32), radix_hist_words(k_cap, tile_bits(n_tiles))));
  GSB_CUDA(f->sort_hist.reserve(sizeof(uint32_t) * hist, &grew));
  GSB_CUDA(f->ranges.reserve(sizeof(uint2) * n_tiles, &grew));
  GSB_CUDA(f->tile_cut.reserve(sizeof(double2) * n_tiles, &grew));
  GSB_CUDA(f->image.reserve(sizeof(float) * 3 * npix, &grew));
  GSB_CUDA(f->final_t.reserve(sizeof(float) * npix, &grew));
  GSB_CUDA(f->pixstate.reserve(sizeof(uint32_t) * npix, &grew));
  GSB_CUDA(f->d_image.reserve(sizeof(float) * 3 * npix, &grew));
  GSB_CUDA(f->gmaps.reserve(sizeof(float) * 9 * npix, &grew));
  GSB_CUDA(f->loss_blocks.reserve(sizeof(double) * 2 * loss_block_count(f->width, f->height), &grew));
  GSB_CUDA(f->loss_val.reserve(sizeof(double) * 4, &grew));
  GSB_CUDA(f->partials.reserve(sizeof(float) * kPartial * k_cap, &grew));
  if (f->want_hits) GSB_CUDA(f->hits.reserve(sizeof(uint16_t) * hit_words() * k_cap, &grew));
  GSB_CUDA(f->pose_blocks.reserve(sizeof(double) * 6 * ((n + 63) / 64 + 1), &grew));  // K4b blocks of >= 64
  GSB_CUDA(f->d_pose.reserve(sizeof(double) * 6, &grew));
  if (grew) {
    ++f->gen;
    if (debug_on()) std::fprintf(stderr, "[gsb] frame_reserve grew (k_cap request %lld)\n", (long long)k_cap);
  }
  f->k_cap = (int64_t)(f->ekey[0].bytes / sizeof(uint32_t));
  f->k_cap = std::min<int64_t>(f->k_cap, (int64_t)(f->partials.bytes / (sizeof(float) * kPartial)));
  f->k_cap = std::min<int64_t>(f->k_cap, (int64_t)(f->ent_key.bytes / sizeof(uint64_t)));
  f->k_cap = std::min<int64_t>(f->k_cap, (int64_t)(f->ent_gid.bytes / sizeof(uint32_t)));
  if (f->want_hits) f->k_cap = std::min<int64_t>(f->k_cap, (int64_t)(f->hits.bytes / (sizeof(uint16_t) * hit_words())));
  f->k_cap = std::min<int64_t>(f->k_cap, 0xffffffffll);
  return GSB_OK;
}

// Global depth order (reference rank order): compaction in index order, stable
// depth sort (FP32 bits, 4 passes) + FP64 tie fix, rank-order records. Leaves
// the rank-major entry offsets in *offs_out (a depth-key ping-pong buffer).
static int rank_order_async(gsb_ctx* ctx, const gsb_cloud* cloud, gsb_frame* f, uint32_t** offs_out) {
  cudaStream_t st = ctx->stream;
  const int64_t n = cloud->n;
  uint32_t* counters = f->counters.as<uint32_t>();
  if (int r = scan_any(st, f->cnt_g.as<uint32_t>(), n, nullptr, true, f->cnt_r.as<uint32_t>(),
                       f->scan_tmp.as<uint32_t>(), counters + 0, &ctx->launches))
    return r;
  if (int r = launch_compact(st, f->cnt_g.as<uint32_t>(), f->cnt_r.as<uint32_t>(), f->depth_g.as<double>(), n,
                             f->vis_idx.as<uint32_t>(), f->dkey[0].as<uint32_t>(), f->dval[0].as<uint32_t>()))
    return r;
  ctx->launches += n > 0 ? 1 : 0;
  uint32_t* dk[2] = {f->dkey[0].as<uint32_t>(), f->dkey[1].as<uint32_t>()};
  uint32_t* dv[2] = {f->dval[0].as<uint32_t>(), f->dval[1].as<uint32_t>()};
  int sel = 0;
  if (int r = sort_any(st, dk, dv, n, counters + 0, 32, f->sort_hist.as<uint32_t>(), &sel, &ctx->launches)) return r;
  if (int r = launch_depth_tie_fix(st, dk[sel], dv[sel], f->vis_idx.as<uint32_t>(), f->depth_g.as<double>(), n,
                                   counters + 0))
    return r;
  ctx->launches += n > 1 ? 1 : 0;
  if (int r = launch_gather_ranks(st, dv[sel], f->vis_idx.as<uint32_t>(), f->rec_g.as<SplatRec>(),
                                  f->rect_g.as<uint2>(), f->cnt_g.as<uint32_t>(), n, counters + 0,
                                  f->rec.as<SplatRec>(), f->aux.as<SplatAux>(), f->cnt_r.as<uint32_t>(),
                                  f->rank_of_g.as<int32_t>()))
    return r;
  ctx->launches += n > 0 ? 1 : 0;
  *offs_out = dk[sel ^ 1];
  return GSB_OK;
}

// The forward pass as a fixed launch sequence (no host synchronisation; live
// counts V -> counters[0], K -> counters[1] stay on the device, counters[2]
// flags a tile too large for tile-local binning). Camera in f->cam.
static int render_post(gsb_ctx* ctx, const gsb_cloud* cloud, gsb_frame* f, const RasterDev& rc);

static int render_async(gsb_ctx* ctx, const gsb_cloud* cloud, gsb_frame* f, const RasterDev& rc) {
  cudaStream_t st = ctx->stream;
  const int64_t n = cloud->n;
  {
    StageScope sc(ctx, kStPreprocess);
    GSB_CUDA(cudaMemsetAsync(f->counters.p, 0, 4 * sizeof(uint32_t), st));
    if (int r = launch_preprocess(st, cloud, f->cam.as<CamDev>(), rc, f)) return r;
    ctx->launches += n > 0 ? 1 : 0;
  }
  return render_post(ctx, cloud, f, rc);
}

// Everything of the forward pass after K1 (binning + compositing).
static int render_post(gsb_ctx* ctx, const gsb_cloud* cloud, gsb_frame* f, const RasterDev& rc) {
  cudaStream_t st = ctx->stream;
  const int64_t n = cloud->n;
  const int n_tiles = f->tiles_x * f->tiles_y;
  uint32_t* counters = f->counters.as<uint32_t>();
  const bool tile_local = f->binning == kBinTileLocal;
  {
    StageScope sc(ctx, kStSort);
    if (tile_local) {
      // tile ranges from the preprocess counts, scatter, per-tile (depth, gid) sort
      if (int r = launch_tile_bin(st, f, n, &ctx->launches)) return r;
    } else {
      uint32_t* offs = nullptr;
      if (int r = rank_order_async(ctx, cloud, f, &offs)) return r;
      if (int r = scan_any(st, f->cnt_r.as<uint32_t>(), n, counters + 0, false, offs, f->scan_tmp.as<uint32_t>(),
                           counters + 1, &ctx->launches))
        return r;
      // duplicate (tile, rank) entries, stable sort by tile, ranges
      if (int r = launch_duplicate(st, offs, f->aux.as<SplatAux>(), n, counters + 0, f->tiles_x, f->k_cap,
                                   f->ekey[0].as<uint32_t>(), f->eval_[0].as<uint32_t>(), f->off_g.as<uint32_t>()))
        return r;
      ctx->launches += n > 0 ? 1 : 0;
      uint32_t* ek[2] = {f->ekey[0].as<uint32_t>(), f->ekey[1].as<uint32_t>()};
      uint32_t* ev[2] = {f->eval_[0].as<uint32_t>(), f->eval_[1].as<uint32_t>()};
      int esel = 0;
      if (int r = sort_any(st, ek, ev, f->k_cap, counters + 1, tile_bits(n_tiles), f->sort_hist.as<uint32_t>(),
                           &esel, &ctx->launches))
        return r;
      f->sorted_sel = esel;
      if (int r = launch_tile_ranges(st, ek[esel], f->k_cap, counters + 1, n_tiles, f->ranges.as<uint2>())) return r;
      ctx->launches += n_tiles > 0 ? 1 : 0;
    }
    f->ranks_valid = !tile_local;
  }
  {
    StageScope sc(ctx, kStComposite);
    if (int r = launch_composite(st, f, rc)) return r;
    ctx->launches += n_tiles > 0 ? 1 : 0;
  }
  return GSB_OK;
}

// A tile held more entries than the per-tile sort takes: this frame uses the
// global binning path from now on (buffers unchanged; graphs are rebuilt).
static void fall_back_to_global(gsb_frame* f) {
  f->fallback_global = true;
  f->binning = kBinGlobal;
  ++f->gen;
}

// Synchronous forward for the host API: runs the async pass, reads (V, K)
// and re-runs with a larger entry capacity if K overflowed it.
static int render_sync(gsb_ctx* ctx, const gsb_cloud* cloud, gsb_frame* f, const RasterDev& rc) {
  int64_t want = f->k_cap > 0 ? f->k_cap : initial_k_cap(cloud->n);
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (int r = frame_reserve(f, cloud, want)) return r;
    if (int r = render_async(ctx, cloud, f, rc)) return r;
    uint32_t cnt[3];
    if (int r = read_counters(ctx, f->counters.as<uint32_t>(), cnt, 3)) return r;
    f->n_splats = cnt[0];
    f->n_entries = cnt[1];
    if (cnt[2] != 0u) {
      fall_back_to_global(f);
      continue;
    }
    if ((int64_t)cnt[1] <= f->k_cap) return GSB_OK;
    want = (int64_t)cnt[1] + (int64_t)cnt[1] / 4 + 4096;
  }
  return fail(GSB_ERR_OUT_OF_MEMORY, "entry capacity did not converge");
}

static int frame_setup(gsb_ctx* ctx, gsb_frame* f, const gsb_cloud* cloud, const gsb_camera* cam,
                       const double bg[3], const gsb_raster_config* cfg, bool upload_camera) {
  if (cam->width <= 0 || cam->height <= 0) return fail(GSB_ERR_INVALID_ARGUMENT, "camera size must be positive");
  f->width = cam->width;
  f->height = cam->height;
  f->tiles_x = (cam->width + kTile - 1) / kTile;
  f->tiles_y = (cam->height + kTile - 1) / kTile;
  if (f->tiles_x > 65535 || f->tiles_y > 65535) return fail(GSB_ERR_INVALID_ARGUMENT, "image too large");
  f->camera = *cam;
  f->config = *cfg;
  f->exp_valid = false;
  const bool local_ok = (int64_t)f->tiles_x * f->tiles_y <= kBinMaxTiles;  // per-tile counters fit shared memory
  const int binning =
      (ctx->binning == kBinGlobal || f->fallback_global || !local_ok) ? kBinGlobal : kBinTileLocal;
  if (binning != f->binning) {
    f->binning = binning;
    ++f->gen;
  }
  for (int c = 0; c < 3; ++c) f->background[c] = bg ? bg[c] : 0.0;
  f->n_gaussians = cloud->n;
  f->cloud = cloud;
  f->fingerprint = fingerprint(cloud, cam, !f->lean);
  f->cloud_version = cloud->version;
  f->valid = false;
  f->has_dimage = false;
  GSB_RESERVE(f->cam, sizeof(CamDev));
  if (upload_camera) {
    CamDev cd = make_camdev(cam, kTile);
    CamDev* h = static_cast<CamDev*>(pinned(ctx, sizeof(CamDev)));
    if (!h) return fail(GSB_ERR_OUT_OF_MEMORY, "pinned staging");
    GSB_CUDA(cudaStreamSynchronize(ctx->stream));  // staging buffer reuse
    *h = cd;
    GSB_CUDA(cudaMemcpyAsync(f->cam.p, h, sizeof(CamDev), cudaMemcpyHostToDevice, ctx->stream));
  }
  return GSB_OK;
}

// Host-side (de)interleave of an image between the caller's FP64 HWC buffer
// and the pinned FP32 planes, split over the host cores for frame-sized
// images (it is the e2e path's only O(pixels) host work).
template <typename F>
static void host_parallel(size_t n, F fn) {
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const size_t chunks = n < (size_t)1 << 16 ? 1 : std::min<size_t>(hw, (n + 65535) / 65536);
  if (chunks <= 1) {
    fn((size_t)0, n);
    return;
  }
  std::vector<std::thread> th;
  const size_t step = (n + chunks - 1) / chunks;
  for (size_t c = 1; c < chunks; ++c) {
    const size_t b = c * step, e = std::min(n, b + step);
    if (b < e) th.emplace_back([=, &fn] { fn(b, e); });
  }
  fn((size_t)0, std::min(n, step));
  for (auto& t : th) t.join();
}

// planar FP32 [3][P] -> interleaved FP64 host
static int download_image(gsb_ctx* ctx, const float* dev_planes, int W, int H, double* out) {
  const size_t P = (size_t)W * H;
  float* h = static_cast<float*>(pinned(ctx, sizeof(float) * 3 * P));
  if (!h) return fail(GSB_ERR_OUT_OF_MEMORY, "pinned staging");
  GSB_CUDA(cudaMemcpyAsync(h, dev_planes, sizeof(float) * 3 * P, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  host_parallel(P, [&](size_t b, size_t e) {
    for (size_t p = b; p < e; ++p) {
      out[3 * p] = h[p];
      out[3 * p + 1] = h[P + p];
      out[3 * p + 2] = h[2 * P + p];
    }
  });
  return GSB_OK;
}
// A rendered frame's image to host FP64 HWC. Pixels no splat touched
// (final T == 1 exactly and the stored value is the FP32 background) are the
// background in FP64 exactly, as the reference composes them (C = 0 + bg * 1,
// rasterizer.cpp:260-268; empty cloud = background, test_rasterizer.cpp:127-142).
static int download_frame_image(gsb_ctx* ctx, const gsb_frame* f, double* out) {
  if (int r = download_image(ctx, f->image.as<float>(), f->width, f->height, out)) return r;
  const size_t P = (size_t)f->width * f->height;
  std::vector<float> ft(P);
  GSB_CUDA(cudaMemcpyAsync(ft.data(), f->final_t.p, sizeof(float) * P, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  double bg[3];
  float bgf[3];
  for (int c = 0; c < 3; ++c) {
    bg[c] = std::min(f->background[c], 1.0);
    bgf[c] = std::min((float)f->background[c], 1.0f);
  }
  host_parallel(P, [&](size_t b, size_t e) {
    for (size_t p = b; p < e; ++p)
      if (ft[p] == 1.0f)
        for (int c = 0; c < 3; ++c)
          if (out[3 * p + c] == (double)bgf[c]) out[3 * p + c] = bg[c];
  });
  return GSB_OK;
}
static int rank_order_async(gsb_ctx* ctx, const gsb_cloud* cloud, gsb_frame* f, uint32_t** offs_out);
// Exported tile geometry of a frame rendered with tile_size != 16.
static int ensure_export(gsb_ctx* ctx, gsb_frame* f) {
  if (f->config.tile_size == kTile || f->exp_valid) return GSB_OK;
  if (!f->ranks_valid && f->cloud) {
    uint32_t* offs = nullptr;
    if (int r = rank_order_async(ctx, f->cloud, f, &offs)) return r;
    f->ranks_valid = true;
  }
  return build_export_tiles(ctx->stream, f, f->config.tile_size);
}
// interleaved FP64 host -> planar FP32 device
// Host FP64 HWC image -> device FP32 planes, stream ordered on ctx->stream.
// Two pinned staging slots alternate: the conversion of the next image
// overlaps the DMA of the previous one, and the call returns without waiting
// for its own copy (only for the copy that last used the slot it takes).
static int upload_image(gsb_ctx* ctx, const double* img, int W, int H, float* dev_planes) {
  const size_t P = (size_t)W * H;
  const size_t bytes = sizeof(float) * 3 * P;
  const int k = ctx->up_next;
  ctx->up_next ^= 1;
  if (ctx->up_ev[k]) {
    GSB_CUDA(cudaEventSynchronize(ctx->up_ev[k]));  // the slot's previous copy has landed
  } else {
    GSB_CUDA(cudaEventCreateWithFlags(&ctx->up_ev[k], cudaEventDisableTiming));
  }
  if (bytes > ctx->up_bytes[k]) {
    if (ctx->up_buf[k]) cudaFreeHost(ctx->up_buf[k]);
    ctx->up_buf[k] = nullptr;
    ctx->up_bytes[k] = 0;
    const size_t cap = bytes + bytes / 4 + 4096;
    if (cudaMallocHost(&ctx->up_buf[k], cap) != cudaSuccess) return fail(GSB_ERR_OUT_OF_MEMORY, "pinned staging");
    ctx->up_bytes[k] = cap;
  }
  float* h = static_cast<float*>(ctx->up_buf[k]);
  const double t0 = debug_on() ? now_ms() : 0.0;
  host_parallel(P, [&](size_t b, size_t e) {
    for (size_t p = b; p < e; ++p) {
      h[p] = (float)img[3 * p];
      h[P + p] = (float)img[3 * p + 1];
      h[2 * P + p] = (float)img[3 * p + 2];
    }
  });
  if (debug_on())
    std::fprintf(stderr, "[gsb] upload_image: convert %.2f ms (%u threads)\n", now_ms() - t0,
                 std::thread::hardware_concurrency());
  GSB_CUDA(cudaMemcpyAsync(dev_planes, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaEventRecord(ctx->up_ev[k], ctx->stream));
  return GSB_OK;
}

// Loss on the frame's image (buffers sized by frame_reserve or here).
// mask_t (nullable): masked_rgb_loss on accum = 1 - mask_t > mask_thr.
static int loss_device(gsb_ctx* ctx, gsb_frame* f, const float* target, double beta, bool want_grad,
                       const float* mask_t = nullptr, double mask_thr = 0.0) {
  const int W = f->width, H = f->height;
  const int64_t P = std::max<int64_t>((int64_t)W * H, 1);
  GSB_RESERVE(f->gmaps, sizeof(float) * 9 * P);
  GSB_RESERVE(f->loss_blocks, sizeof(double) * 2 * loss_block_count(W, H));
  GSB_RESERVE(f->loss_val, sizeof(double) * 4);
  if (mask_t) GSB_RESERVE(f->mask_ws, 64);
  if (want_grad) GSB_RESERVE(f->d_image, sizeof(float) * 3 * P);
  StageScope sc(ctx, kStLoss);
  int r = launch_rgb_loss(ctx->stream, f->image.as<float>(), target, W, H, beta, f->gmaps.as<float>(),
                          f->loss_blocks.as<double>(), f->loss_val.as<double>(), want_grad ? f->d_image.as<float>() : nullptr,
                          &ctx->launches, mask_t, mask_thr, mask_t ? f->mask_ws.p : nullptr);
  if (r) return r;
  if (want_grad) f->has_dimage = true;
  return GSB_OK;
}

// Backward pass (buffers sized by frame_reserve).
static int backward_device(gsb_ctx* ctx, const gsb_cloud* cloud, gsb_frame* f, bool full, float* grads,
                           bool reduce_pose = true) {
  const RasterDev rc = make_rasterdev(&f->config);
  {
    StageScope sc(ctx, kStBwdRaster);
    if (int r = launch_backward_raster(ctx->stream, f, rc, !full)) return r;
    ctx->launches += f->tiles_x * f->tiles_y > 0 ? 1 : 0;
  }
  {
    StageScope sc(ctx, kStBwdGeom);
    if (int r = launch_backward_geom(ctx->stream, cloud, f, rc, full, grads, &ctx->launches, reduce_pose)) return r;
  }
  return GSB_OK;
}

}  // namespace gsb

using namespace gsb;

// ===================================================================== ABI
namespace gsb {
static int ctx_free(gsb_ctx* ctx) {
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->scratch_small.release();
  if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
  for (auto& pb : ctx->pinned_pool) cudaFreeHost(pb.first);
  for (int k = 0; k < 2; ++k) {
    if (ctx->up_buf[k]) cudaFreeHost(ctx->up_buf[k]);
    if (ctx->up_ev[k]) cudaEventDestroy(ctx->up_ev[k]);
  }
  ctx->pinned_pool.clear();
  delete ctx->timer;
  if (ctx->work) gsb_frame_destroy(ctx->work);
  for (gsb_frame* f : ctx->frame_pool) gsb_frame_destroy(f);
  for (DevBuf& b : ctx->image_pool) b.release();
  ctx->image_pool.clear();
  if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
  if (ctx->ev_stop) cudaEventDestroy(ctx->ev_stop);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return GSB_OK;
}
void ctx_retain(gsb_ctx* ctx) { ++ctx->refs; }
void ctx_release(gsb_ctx* ctx) {
  if (--ctx->refs == 0 && ctx->closing) ctx_free(ctx);
}
}  // namespace gsb

extern "C" {

const char* gsb_last_error(void) { return gsb::g_error.c_str(); }
const char* gsb_version(void) { return "gsb200 0.1 (sm_100a)"; }

void gsb_default_raster_config(gsb_raster_config* c) {  // rasterizer.hpp:30-38
  c->tile_size = 16;
  c->cutoff_sigma = 3.0;
  c->alpha_clamp = 0.99;
  c->dilation = 0.3;
  c->early_termination = 1e-4;
  c->z_near = 0.01;
  c->deterministic = 1;
}
void gsb_default_pose_config(gsb_pose_config* c) {  // trainer.hpp:21-60
  c->cam_lr_start = 1e-2;
  c->cam_lr_end = 1e-4;
  c->beta = 0.2;
  c->pose_converged_eps = 1e-7;
  c->background[0] = c->background[1] = c->background[2] = 0.0;
  gsb_default_raster_config(&c->raster);
  c->budget = 1000;
}

int gsb_ctx_create(int32_t device, gsb_ctx** out) {
  if (!out) return fail(GSB_ERR_INVALID_ARGUMENT, "null out");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return fail(GSB_ERR_NO_DEVICE, "no CUDA device visible (no CPU fallback exists)");
  if (device < 0 || device >= ndev) return fail(GSB_ERR_INVALID_ARGUMENT, "device index out of range");
  GSB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  GSB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) return fail(GSB_ERR_NO_DEVICE, "device is not sm_100 class (this build targets sm_100a only)");
  gsb_ctx* c = new gsb_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaStreamCreate");
  }
  c->timer = new StageTimer();
  if (int r = init_loss_constants()) {
    gsb_ctx_destroy(c);
    return r;
  }
  if (int r = init_loss_attributes()) {
    gsb_ctx_destroy(c);
    return r;
  }
  if (int r = init_preprocess_attributes()) {
    gsb_ctx_destroy(c);
    return r;
  }
  if (int r = init_bin_attributes()) {
    gsb_ctx_destroy(c);
    return r;
  }
  *out = c;
  return GSB_OK;
}

int gsb_ctx_destroy(gsb_ctx* ctx) {
  if (!ctx) return GSB_OK;
  if (ctx->refs > 0) {  // objects still live: free with the last of them
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->closing = true;
    return GSB_OK;
  }
  return ctx_free(ctx);
}

int gsb_ctx_synchronize(gsb_ctx* ctx) {
  if (int r = ensure_device(ctx)) return r;
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return GSB_OK;
}

int gsb_ctx_set_binning(gsb_ctx* ctx, int32_t mode) {
  if (int r = ensure_device(ctx)) return r;
  if (mode != GSB_BINNING_TILE_LOCAL && mode != GSB_BINNING_GLOBAL)
    return fail(GSB_ERR_INVALID_ARGUMENT, "unknown binning mode");
  ctx->binning = mode == GSB_BINNING_GLOBAL ? kBinGlobal : kBinTileLocal;
  return GSB_OK;
}

int gsb_ctx_set_profiling(gsb_ctx* ctx, int32_t enable) {
  if (int r = ensure_device(ctx)) return r;
  ctx->profiling = enable != 0;
  return GSB_OK;
}

int gsb_ctx_stage_times(gsb_ctx* ctx, double* ms_out, int64_t* launches_out, int32_t reset) {
  if (int r = ensure_device(ctx)) return r;
  GSB_CUDA(ctx->timer->collect());
  for (int k = 0; k < kNumStages; ++k) {
    if (ms_out) ms_out[k] = ctx->timer->ms[k];
    if (launches_out) launches_out[k] = ctx->timer->count[k];
  }
  if (reset) ctx->timer->reset();
  return GSB_OK;
}

int64_t gsb_ctx_launch_count(gsb_ctx* ctx) { return ctx ? ctx->launches : -1; }

// ------------------------------------------------------------------ cloud
int gsb_cloud_create(gsb_ctx* ctx, int64_t n, int32_t sh_degree, gsb_cloud** out) {
  if (int r = ensure_device(ctx)) return r;
  if (!out || n < 0 || sh_degree < 0 || sh_degree > 3) return fail(GSB_ERR_INVALID_ARGUMENT, "bad cloud shape");
  if (n > (int64_t)0x7fffffff) return fail(GSB_ERR_INVALID_ARGUMENT, "cloud too large for int32 ids");
  gsb_cloud* c = new gsb_cloud();
  c->ctx = ctx;
  c->n = n;
  c->n_pad = std::max<int64_t>(32, (n + 31) / 32 * 32);
  c->sh_degree = sh_degree;
  c->active_sh_degree = sh_degree;
  cudaError_t e = c->params.reserve(sizeof(float) * num_planes(sh_degree) * c->n_pad);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cloud alloc");
  }
  cudaMemsetAsync(c->params.p, 0, sizeof(float) * num_planes(sh_degree) * c->n_pad, ctx->stream);
  ctx_retain(ctx);
  c->ctx_ref = true;
  *out = c;
  return GSB_OK;
}

int gsb_cloud_destroy(gsb_cloud* c) {
  if (!c) return GSB_OK;
  cudaSetDevice(c->ctx->device);
  cudaStreamSynchronize(c->ctx->stream);
  c->params.release();
  gsb_ctx* owner = c->ctx_ref ? c->ctx : nullptr;
  delete c;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_cloud_upload(gsb_cloud* c, const double* means, const double* rotations, const double* log_scales,
                     const double* opacity_logits, const double* sh, int32_t active) {
  GSB_NVTX("gsb_cloud_upload");
  if (!c) return fail(GSB_ERR_INVALID_ARGUMENT, "null cloud");
  gsb_ctx* ctx = c->ctx;
  if (int r = ensure_device(ctx)) return r;
  const int64_t n = c->n, np = c->n_pad;
  const int B = (c->sh_degree + 1) * (c->sh_degree + 1);
  const int NP = num_planes(c->sh_degree);
  if (n > 0 && (!means || !rotations || !log_scales || !opacity_logits || !sh))
    return fail(GSB_ERR_INVALID_ARGUMENT, "null parameter array");
  for (int64_t i = 0; i < n; ++i) {  // GaussianCloud::validate (scene.cpp:135-148)
    bool ok = std::isfinite(means[3 * i]) && std::isfinite(means[3 * i + 1]) && std::isfinite(means[3 * i + 2]) &&
              std::isfinite(log_scales[3 * i]) && std::isfinite(log_scales[3 * i + 1]) &&
              std::isfinite(log_scales[3 * i + 2]) && std::isfinite(opacity_logits[i]);
    for (int k = 0; k < 4; ++k) ok = ok && std::isfinite(rotations[4 * i + k]);
    if (!ok) return fail(GSB_ERR_DIVERGED, "GaussianCloud: non-finite parameter at index " + std::to_string(i));
  }
  float* h = static_cast<float*>(pinned(ctx, sizeof(float) * NP * np));
  if (!h) return fail(GSB_ERR_OUT_OF_MEMORY, "pinned staging");
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memset(h, 0, sizeof(float) * NP * np);
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) h[(kMeanX + k) * np + i] = (float)means[3 * i + k];
    for (int k = 0; k < 4; ++k) h[(kQuatW + k) * np + i] = (float)rotations[4 * i + k];
    for (int k = 0; k < 3; ++k) h[(kScaleX + k) * np + i] = (float)log_scales[3 * i + k];
    h[kOpacity * np + i] = (float)opacity_logits[i];
    const double* s = sh + (size_t)i * 3 * B;
    for (int k = 0; k < 3 * B; ++k) h[(kShBase + k) * np + i] = (float)s[k];
  }
  GSB_CUDA(cudaMemcpyAsync(c->params.p, h, sizeof(float) * NP * np, cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  c->active_sh_degree = std::min(std::max(active, 0), c->sh_degree);
  // content hash of the uploaded FP64 arrays at 64 strided samples (rasterizer.cpp:62-71)
  uint64_t hsh = 0xcbf29ce484222325ull;
  const int64_t stride = std::max<int64_t>(1, n / 64);
  c->fp_samples.clear();
  auto put = [&](const double* p, size_t k) {
    const unsigned char* b = reinterpret_cast<const unsigned char*>(p);
    c->fp_samples.insert(c->fp_samples.end(), b, b + sizeof(double) * k);
    hsh = fnv1a(hsh, p, sizeof(double) * k);
  };
  for (int64_t i = 0; i < n; i += stride) {
    put(means + 3 * i, 3);
    put(rotations + 4 * i, 4);
    put(log_scales + 3 * i, 3);
    put(opacity_logits + i, 1);
    put(sh + (size_t)i * 3 * B, (size_t)3 * B);
  }
  c->host_fingerprint = hsh;
  c->version += 1;
  c->fp_version = c->version;
  return GSB_OK;
}

int gsb_cloud_download(gsb_cloud* c, double* means, double* rotations, double* log_scales, double* opacity_logits,
                       double* sh) {
  GSB_NVTX("gsb_cloud_download");
  if (!c) return fail(GSB_ERR_INVALID_ARGUMENT, "null cloud");
  gsb_ctx* ctx = c->ctx;
  if (int r = ensure_device(ctx)) return r;
  const int64_t n = c->n, np = c->n_pad;
  const int B = (c->sh_degree + 1) * (c->sh_degree + 1);
  const int NP = num_planes(c->sh_degree);
  float* h = static_cast<float*>(pinned(ctx, sizeof(float) * NP * np));
  if (!h) return fail(GSB_ERR_OUT_OF_MEMORY, "pinned staging");
  GSB_CUDA(cudaMemcpyAsync(h, c->params.p, sizeof(float) * NP * np, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int64_t i = 0; i < n; ++i) {
    if (means) for (int k = 0; k < 3; ++k) means[3 * i + k] = h[(kMeanX + k) * np + i];
    if (rotations) for (int k = 0; k < 4; ++k) rotations[4 * i + k] = h[(kQuatW + k) * np + i];
    if (log_scales) for (int k = 0; k < 3; ++k) log_scales[3 * i + k] = h[(kScaleX + k) * np + i];
    if (opacity_logits) opacity_logits[i] = h[kOpacity * np + i];
    if (sh) for (int k = 0; k < 3 * B; ++k) sh[(size_t)i * 3 * B + k] = h[(kShBase + k) * np + i];
  }
  return GSB_OK;
}

int gsb_cloud_info(gsb_cloud* c, int64_t* n, int32_t* deg, int32_t* active) {
  if (!c) return fail(GSB_ERR_INVALID_ARGUMENT, "null cloud");
  if (n) *n = c->n;
  if (deg) *deg = c->sh_degree;
  if (active) *active = c->active_sh_degree;
  return GSB_OK;
}

int gsb_cloud_set_active_sh_degree(gsb_cloud* c, int32_t active) {
  if (!c) return fail(GSB_ERR_INVALID_ARGUMENT, "null cloud");
  c->active_sh_degree = std::min(std::max(active, 0), c->sh_degree);
  c->version += 1;
  return GSB_OK;
}

// ------------------------------------------------------------------ frame
int gsb_frame_create(gsb_ctx* ctx, gsb_frame** out) {
  if (int r = ensure_device(ctx)) return r;
  if (!out) return fail(GSB_ERR_INVALID_ARGUMENT, "null out");
  gsb_frame* f = new gsb_frame();
  f->ctx = ctx;
  ctx_retain(ctx);
  f->ctx_ref = true;
  *out = f;
  return GSB_OK;
}

int gsb_frame_destroy(gsb_frame* f) {
  if (!f) return GSB_OK;
  cudaSetDevice(f->ctx->device);
  cudaStreamSynchronize(f->ctx->stream);
  DevBuf* bufs[] = {&f->cam, &f->rec_g, &f->rect_g, &f->cnt_g, &f->depth_g, &f->radius_g, &f->rank_of_g,
                    &f->colj, &f->off_g, &f->vis_idx, &f->dkey[0], &f->dkey[1], &f->dval[0], &f->dval[1], &f->rec, &f->aux,
                    &f->cnt_r, &f->ekey[0], &f->ekey[1], &f->eval_[0], &f->eval_[1], &f->ranges, &f->tile_cut, &f->image,
                    &f->final_t, &f->pixstate, &f->d_image, &f->partials, &f->pose_blocks, &f->d_pose,
                    &f->loss_blocks, &f->loss_val, &f->mask_ws, &f->gmaps, &f->scan_tmp, &f->sort_hist, &f->counters,
                    &f->aux_g, &f->tile_hist, &f->tile_scan, &f->tile_big, &f->ent_key, &f->ent_gid, &f->hits, &f->exp_lists,
                    &f->exp_ranges, &f->exp_contrib};
  for (DevBuf* b : bufs) b->release();
  gsb_ctx* owner = f->ctx_ref ? f->ctx : nullptr;
  delete f;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_render(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, const double bg[3],
               const gsb_raster_config* cfg, gsb_frame* f, double* image_out) {
  GSB_NVTX("gsb_render");
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !cam || !f) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  gsb_raster_config dflt;
  gsb_default_raster_config(&dflt);
  if (!cfg) cfg = &dflt;
  if (int r = validate_config(cfg)) return r;
  f->want_hits = hit_masks_enabled();  // a pose-only gsb_render_backward may follow
  if (int r = frame_setup(ctx, f, cloud, cam, bg, cfg, true)) return r;
  const RasterDev rc = make_rasterdev(cfg);
  if (int r = render_sync(ctx, cloud, f, rc)) return r;
  f->valid = true;
  if (image_out) return download_frame_image(ctx, f, image_out);
  return GSB_OK;
}

int gsb_state_fingerprint(gsb_cloud* cloud, const gsb_camera* cam, uint64_t* out) {
  if (!cloud || !cam || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  *out = fingerprint(cloud, cam, true);  // what gsb_render stamps on a (non-lean) frame
  return GSB_OK;
}

int gsb_render_expected_depth(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, const gsb_raster_config* cfg,
                              float* depth_out, float* weight_out) {
  GSB_NVTX("gsb_render_expected_depth");
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !cam || !depth_out || !weight_out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  gsb_raster_config dflt;
  gsb_default_raster_config(&dflt);
  if (!cfg) cfg = &dflt;
  if (int r = validate_config(cfg)) return r;
  gsb_frame* f = nullptr;
  if (int r = gsb_frame_create(ctx, &f)) return r;
  f->lean = true;
  const RasterDev rc = make_rasterdev(cfg);
  const int64_t P = (int64_t)cam->width * cam->height;
  DevBuf out;
  int r = frame_setup(ctx, f, cloud, cam, nullptr, cfg, true);
  if (!r) r = render_sync(ctx, cloud, f, rc);
  if (!r && out.reserve(sizeof(float) * 2 * std::max<int64_t>(P, 1)) != cudaSuccess)
    r = fail(GSB_ERR_OUT_OF_MEMORY, "expected depth buffers");
  if (!r) r = launch_expected_depth(ctx->stream, f, rc, out.as<float>(), out.as<float>() + P);
  if (!r && P > 0) {
    cudaError_t e = cudaMemcpyAsync(depth_out, out.p, sizeof(float) * P, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(weight_out, out.as<float>() + P, sizeof(float) * P, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) r = cuda_fail(e, "expected depth download");
  }
  out.release();
  gsb_frame_destroy(f);
  return r;
}

int gsb_frame_get_info(gsb_frame* f, gsb_frame_info* info) {
  if (!f || !info) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  info->n_gaussians = f->n_gaussians;
  info->n_splats = f->n_splats;
  info->n_entries = f->n_entries;
  info->width = f->width;
  info->height = f->height;
  info->tiles_x = f->tiles_x;
  info->tiles_y = f->tiles_y;
  if (f->valid && f->config.tile_size != kTile) {  // RenderOutput geometry of the requested tile size
    if (int r = ensure_export(f->ctx, f)) return r;
    info->tiles_x = f->exp_tiles_x;
    info->tiles_y = f->exp_tiles_y;
    info->n_entries = f->exp_k;
  }
  info->state_fingerprint = f->fingerprint;
  info->binning = f->binning == kBinGlobal ? GSB_BINNING_GLOBAL : GSB_BINNING_TILE_LOCAL;
  info->reserved = 0;
  return GSB_OK;
}

int gsb_frame_download(gsb_frame* f, double* image, double* accum_t, double* final_t, int32_t* contrib,
                       uint8_t* overflow, int32_t* s_gauss, double* s_mu2d, double* s_depth, double* s_conic,
                       double* s_color, double* s_opacity, double* s_radius, uint8_t* s_clamped, int32_t* tile_lists,
                       int32_t* tile_ranges) {
  GSB_NVTX("gsb_frame_download");
  if (!f || !f->valid) return fail(GSB_ERR_INVALID_ARGUMENT, "frame holds no forward state");
  gsb_ctx* ctx = f->ctx;
  if (int r = ensure_device(ctx)) return r;
  if (int r = ensure_export(ctx, f)) return r;
  const bool exp = f->config.tile_size != kTile;
  const int64_t P = (int64_t)f->width * f->height, V = f->n_splats, K = exp ? f->exp_k : f->n_entries;
  const int T = exp ? f->exp_tiles_x * f->exp_tiles_y : f->tiles_x * f->tiles_y;
  if (image)
    if (int r = download_frame_image(ctx, f, image)) return r;
  std::vector<float> ft(P);
  std::vector<uint32_t> ps(P);
  GSB_CUDA(cudaMemcpyAsync(ft.data(), f->final_t.p, sizeof(float) * P, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(ps.data(), f->pixstate.p, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost, ctx->stream));
  if (!f->ranks_valid && f->cloud) {
    // tile-local frames never build the global rank order; materialise it
    // (the reference's ProjectedSplat order) for the export
    uint32_t* offs = nullptr;
    if (int r = rank_order_async(ctx, f->cloud, f, &offs)) return r;
    f->ranks_valid = true;
  }
  std::vector<SplatRec> rec(V);
  std::vector<SplatAux> aux(V);
  if (V > 0) {
    GSB_CUDA(cudaMemcpyAsync(rec.data(), f->rec.p, sizeof(SplatRec) * V, cudaMemcpyDeviceToHost, ctx->stream));
    GSB_CUDA(cudaMemcpyAsync(aux.data(), f->aux.p, sizeof(SplatAux) * V, cudaMemcpyDeviceToHost, ctx->stream));
  }
  std::vector<double> depth_g(f->n_gaussians), radius_g(f->n_gaussians);
  if (f->n_gaussians > 0 && (s_depth || s_radius)) {
    GSB_CUDA(cudaMemcpyAsync(depth_g.data(), f->depth_g.p, sizeof(double) * f->n_gaussians, cudaMemcpyDeviceToHost,
                             ctx->stream));
    GSB_CUDA(cudaMemcpyAsync(radius_g.data(), f->radius_g.p, sizeof(double) * f->n_gaussians,
                             cudaMemcpyDeviceToHost, ctx->stream));
  }
  std::vector<int32_t> rank_of(!exp && f->binning == kBinTileLocal && tile_lists ? f->n_gaussians : 0);
  if (tile_lists && K > 0) {
    GSB_CUDA(cudaMemcpyAsync(tile_lists, exp ? f->exp_lists.p : f->list(), sizeof(uint32_t) * K,
                             cudaMemcpyDeviceToHost, ctx->stream));
    if (!rank_of.empty())
      GSB_CUDA(cudaMemcpyAsync(rank_of.data(), f->rank_of_g.p, sizeof(int32_t) * rank_of.size(),
                               cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (tile_ranges && T > 0)
    GSB_CUDA(cudaMemcpyAsync(tile_ranges, exp ? f->exp_ranges.p : f->ranges.p, sizeof(uint2) * T,
                             cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<int32_t> contrib_s(exp && contrib ? P : 0);
  if (!contrib_s.empty())
    GSB_CUDA(cudaMemcpyAsync(contrib_s.data(), f->exp_contrib.p, sizeof(int32_t) * P, cudaMemcpyDeviceToHost,
                             ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (!rank_of.empty())  // tile-local lists hold gids: export them as ranks
    for (int64_t e = 0; e < K; ++e) tile_lists[e] = rank_of[(uint32_t)tile_lists[e]];
  for (int64_t p = 0; p < P; ++p) {
    if (final_t) final_t[p] = ft[p];
    if (accum_t) accum_t[p] = 1.0 - (double)ft[p];  // rasterizer.cpp:271-273
    if (contrib) contrib[p] = exp ? contrib_s[p] : (int32_t)(ps[p] & 0x1fffffffu);
    if (overflow) overflow[p] = (uint8_t)(ps[p] >> 29);
  }
  for (int64_t r = 0; r < V; ++r) {
    const int gid = aux[r].gid;
    if (s_gauss) s_gauss[r] = gid;
    if (s_mu2d) {
      s_mu2d[2 * r] = rec[r].mu_x;
      s_mu2d[2 * r + 1] = rec[r].mu_y;
    }
    if (s_depth) s_depth[r] = depth_g[gid];
    if (s_radius) s_radius[r] = radius_g[gid];
    if (s_conic) {
      s_conic[4 * r] = rec[r].conic_a;
      s_conic[4 * r + 1] = rec[r].conic_b;
      s_conic[4 * r + 2] = rec[r].conic_b;
      s_conic[4 * r + 3] = rec[r].conic_c;
    }
    if (s_color) {
      s_color[3 * r] = rec[r].col_r;
      s_color[3 * r + 1] = rec[r].col_g;
      s_color[3 * r + 2] = rec[r].col_b;
    }
    if (s_opacity) s_opacity[r] = rec[r].opacity;
    if (s_clamped) s_clamped[r] = (uint8_t)rec[r].clamp_bits;
  }
  return GSB_OK;
}

// ------------------------------------------------------------------- loss
int gsb_image_create(gsb_ctx* ctx, const double* img, int32_t W, int32_t H, gsb_image** out) {
  GSB_NVTX("gsb_image_create");
  if (int r = ensure_device(ctx)) return r;
  if (!img || !out || W <= 0 || H <= 0) return fail(GSB_ERR_INVALID_ARGUMENT, "bad image");
  gsb_image* im = new gsb_image();
  im->ctx = ctx;
  im->width = W;
  im->height = H;
  const double t0 = debug_on() ? now_ms() : 0.0;
  const size_t need = sizeof(float) * 3 * (size_t)W * H;
  for (size_t i = 0; i < ctx->image_pool.size(); ++i)  // a destroyed image's planes of a fitting size
    if (ctx->image_pool[i].bytes >= need && ctx->image_pool[i].bytes <= 2 * need + 4096) {
      im->planes = ctx->image_pool[i];
      ctx->image_pool.erase(ctx->image_pool.begin() + (ptrdiff_t)i);
      break;
    }
  cudaError_t e = im->planes.reserve(need);
  if (e != cudaSuccess) {
    delete im;
    return cuda_fail(e, "image alloc");
  }
  const double t1 = debug_on() ? now_ms() : 0.0;
  const int ru = upload_image(ctx, img, W, H, im->planes.as<float>());
  if (debug_on()) std::fprintf(stderr, "[gsb] image_create: alloc %.2f upload %.2f ms\n", t1 - t0, now_ms() - t1);
  if (int r = ru) {
    im->planes.release();
    delete im;
    return r;
  }
  ctx_retain(ctx);
  im->ctx_ref = true;
  *out = im;
  return GSB_OK;
}

int gsb_image_destroy(gsb_image* im) {
  if (!im) return GSB_OK;
  cudaSetDevice(im->ctx->device);
  cudaStreamSynchronize(im->ctx->stream);
  if (im->planes.p && im->ctx->image_pool.size() < 64) {  // keep the planes for the next image of this size
    im->ctx->image_pool.push_back(im->planes);
    im->planes = DevBuf();
  }
  im->planes.release();
  gsb_ctx* owner = im->ctx_ref ? im->ctx : nullptr;
  delete im;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_rgb_loss(gsb_ctx* ctx, const double* rendered, const double* target, int32_t W, int32_t H, double beta,
                 double* loss_out, double* d_rendered) {
  GSB_NVTX("gsb_rgb_loss");
  if (int r = ensure_device(ctx)) return r;
  if (!rendered || !target || W <= 0 || H <= 0) return fail(GSB_ERR_INVALID_ARGUMENT, "bad images");
  static thread_local gsb_frame* work = nullptr;
  static thread_local DevBuf tgt;
  if (!work || work->ctx != ctx) {
    work = new gsb_frame();
    work->ctx = ctx;
  }
  work->width = W;
  work->height = H;
  const int64_t P = (int64_t)W * H;
  GSB_RESERVE(work->image, sizeof(float) * 3 * P);
  GSB_RESERVE(tgt, sizeof(float) * 3 * P);
  if (int r = upload_image(ctx, rendered, W, H, work->image.as<float>())) return r;
  if (int r = upload_image(ctx, target, W, H, tgt.as<float>())) return r;
  if (int r = loss_device(ctx, work, tgt.as<float>(), beta, d_rendered != nullptr)) return r;
  double out3[4];
  GSB_CUDA(cudaMemcpyAsync(out3, work->loss_val.p, sizeof(double) * 3, cudaMemcpyDeviceToHost, ctx->stream));
  if (d_rendered)
    if (int r = download_image(ctx, work->d_image.as<float>(), W, H, d_rendered)) return r;
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (loss_out) *loss_out = out3[2];
  return GSB_OK;
}

int gsb_frame_rgb_loss(gsb_ctx* ctx, gsb_frame* f, gsb_image* target, double beta, double* loss_out) {
  GSB_NVTX("gsb_frame_rgb_loss");
  if (int r = ensure_device(ctx)) return r;
  if (!f || !f->valid || !target) return fail(GSB_ERR_INVALID_ARGUMENT, "frame / target missing");
  if (target->width != f->width || target->height != f->height)
    return fail(GSB_ERR_DIMENSION_MISMATCH, "rgb_loss: image shapes differ");
  if (int r = loss_device(ctx, f, target->planes.as<float>(), beta, true)) return r;
  if (loss_out) {
    double out3[4];
    GSB_CUDA(cudaMemcpyAsync(out3, f->loss_val.p, sizeof(double) * 3, cudaMemcpyDeviceToHost, ctx->stream));
    GSB_CUDA(cudaStreamSynchronize(ctx->stream));
    *loss_out = out3[2];
  }
  return GSB_OK;
}

// masked_rgb_loss (losses.cpp:273-289) on host FP64 images and a host mask.
// The mask enters the device loss as a transmittance plane (0 where set, 1
// elsewhere) with threshold 0.5, i.e. through the same kernels as the
// frame-resident variant below.
int gsb_masked_rgb_loss(gsb_ctx* ctx, const double* rendered, const double* target, int32_t W, int32_t H,
                        const uint8_t* mask, double beta, double* loss_out, double* d_rendered) {
  if (int r = ensure_device(ctx)) return r;
  if (!rendered || !target || !mask || W <= 0 || H <= 0) return fail(GSB_ERR_INVALID_ARGUMENT, "bad images / mask");
  const int64_t P = (int64_t)W * H;
  int64_t count = 0;
  for (int64_t p = 0; p < P; ++p) count += mask[p] != 0;
  if (count == 0) return fail(GSB_ERR_EMPTY_MASK, "masked_l1: no pixel passes the mask");
  static thread_local gsb_frame* work = nullptr;
  static thread_local DevBuf tgt, mplane;
  if (!work || work->ctx != ctx) {
    work = new gsb_frame();
    work->ctx = ctx;
  }
  work->width = W;
  work->height = H;
  GSB_RESERVE(work->image, sizeof(float) * 3 * P);
  GSB_RESERVE(tgt, sizeof(float) * 3 * P);
  GSB_RESERVE(mplane, sizeof(float) * P);
  if (int r = upload_image(ctx, rendered, W, H, work->image.as<float>())) return r;
  if (int r = upload_image(ctx, target, W, H, tgt.as<float>())) return r;
  std::vector<float> mt(P);
  for (int64_t p = 0; p < P; ++p) mt[p] = mask[p] ? 0.f : 1.f;
  GSB_CUDA(cudaMemcpyAsync(mplane.p, mt.data(), sizeof(float) * P, cudaMemcpyHostToDevice, ctx->stream));
  if (int r = loss_device(ctx, work, tgt.as<float>(), beta, d_rendered != nullptr, mplane.as<float>(), 0.5)) return r;
  double out3[4];
  GSB_CUDA(cudaMemcpyAsync(out3, work->loss_val.p, sizeof(double) * 3, cudaMemcpyDeviceToHost, ctx->stream));
  if (d_rendered)
    if (int r = download_image(ctx, work->d_image.as<float>(), W, H, d_rendered)) return r;
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (loss_out) *loss_out = out3[2];
  return GSB_OK;
}

// masked_rgb_loss of the frame's image with the frame's own transmittance
// mask (transmittance_mask(accum, threshold), losses.cpp:259-263); the
// gradient stays in the frame. GSB_ERR_EMPTY_MASK (masked_out = 0) when no
// pixel passes, like masked_l1's empty_mask.
int gsb_frame_masked_rgb_loss(gsb_ctx* ctx, gsb_frame* f, gsb_image* target, double beta, double threshold,
                              double* loss_out, int64_t* masked_out) {
  if (int r = ensure_device(ctx)) return r;
  if (!f || !f->valid || !target) return fail(GSB_ERR_INVALID_ARGUMENT, "frame / target missing");
  if (target->width != f->width || target->height != f->height)
    return fail(GSB_ERR_DIMENSION_MISMATCH, "masked_rgb_loss: image shapes differ");
  if (int r = loss_device(ctx, f, target->planes.as<float>(), beta, true, f->final_t.as<float>(), threshold)) return r;
  double out3[4];
  uint64_t counts[2];
  GSB_CUDA(cudaMemcpyAsync(out3, f->loss_val.p, sizeof(double) * 3, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(counts, f->mask_ws.p, sizeof(counts), cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (masked_out) *masked_out = (int64_t)counts[0];
  if (counts[0] == 0) {
    f->has_dimage = false;
    return fail(GSB_ERR_EMPTY_MASK, "masked_l1: no pixel passes the mask");
  }
  if (loss_out) *loss_out = out3[2];
  return GSB_OK;
}

// ---------------------------------------------------------------- backward
int gsb_grads_create(gsb_ctx* ctx, gsb_cloud* cloud, gsb_grads** out) {
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  gsb_grads* g = new gsb_grads();
  g->ctx = ctx;
  g->n = cloud->n;
  g->n_pad = cloud->n_pad;
  g->sh_degree = cloud->sh_degree;
  cudaError_t e = g->planes.reserve(sizeof(float) * (num_planes(cloud->sh_degree) + 2) * cloud->n_pad);
  if (e == cudaSuccess) e = g->pose.reserve(sizeof(double) * 6);
  if (e != cudaSuccess) {
    g->planes.release();
    delete g;
    return cuda_fail(e, "grads alloc");
  }
  ctx_retain(ctx);
  g->ctx_ref = true;
  *out = g;
  return GSB_OK;
}

int gsb_grads_destroy(gsb_grads* g) {
  if (!g) return GSB_OK;
  cudaSetDevice(g->ctx->device);
  cudaStreamSynchronize(g->ctx->stream);
  g->planes.release();
  g->pose.release();
  gsb_ctx* owner = g->ctx_ref ? g->ctx : nullptr;
  delete g;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_grads_download(gsb_grads* g, double* d_means, double* d_rot, double* d_ls, double* d_op, double* d_sh,
                       double* d_mu2d, double d_pose[6]) {
  if (!g || !g->valid) return fail(GSB_ERR_INVALID_ARGUMENT, "grads hold no result");
  gsb_ctx* ctx = g->ctx;
  if (int r = ensure_device(ctx)) return r;
  const int64_t n = g->n, np = g->n_pad;
  const int NP = num_planes(g->sh_degree);
  const int B = (g->sh_degree + 1) * (g->sh_degree + 1);
  std::vector<float> h((size_t)(NP + 2) * np);
  GSB_CUDA(cudaMemcpyAsync(h.data(), g->planes.p, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
  double pose[6];
  GSB_CUDA(cudaMemcpyAsync(pose, g->pose.p, sizeof(double) * 6, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int64_t i = 0; i < n; ++i) {
    if (d_means) for (int k = 0; k < 3; ++k) d_means[3 * i + k] = h[(kMeanX + k) * np + i];
    if (d_rot) for (int k = 0; k < 4; ++k) d_rot[4 * i + k] = h[(kQuatW + k) * np + i];
    if (d_ls) for (int k = 0; k < 3; ++k) d_ls[3 * i + k] = h[(kScaleX + k) * np + i];
    if (d_op) d_op[i] = h[kOpacity * np + i];
    if (d_sh) for (int k = 0; k < 3 * B; ++k) d_sh[(size_t)i * 3 * B + k] = h[(kShBase + k) * np + i];
    if (d_mu2d) {
      d_mu2d[2 * i] = h[(size_t)NP * np + i];
      d_mu2d[2 * i + 1] = h[(size_t)(NP + 1) * np + i];
    }
  }
  if (d_pose) for (int k = 0; k < 6; ++k) d_pose[k] = pose[k];
  return GSB_OK;
}

static int backward_common(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, gsb_frame* f, uint32_t flags,
                           gsb_grads* grads, double d_pose_out[6]) {
  const bool full = !(flags & GSB_BWD_POSE_ONLY);
  if (full && !grads) return fail(GSB_ERR_INVALID_ARGUMENT, "full backward needs a grads object");
  if (grads && grads->n != cloud->n) return fail(GSB_ERR_DIMENSION_MISMATCH, "grads / cloud size mismatch");
  if (int r = backward_device(ctx, cloud, f, full, full ? grads->planes.as<float>() : nullptr)) return r;
  if (grads) {
    GSB_CUDA(cudaMemcpyAsync(grads->pose.p, f->d_pose.p, sizeof(double) * 6, cudaMemcpyDeviceToDevice, ctx->stream));
    grads->valid = true;
  }
  if (d_pose_out) {
    double h[6];
    GSB_CUDA(cudaMemcpyAsync(h, f->d_pose.p, sizeof(double) * 6, cudaMemcpyDeviceToHost, ctx->stream));
    GSB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < 6; ++k) d_pose_out[k] = h[k];
  }
  return GSB_OK;
}

static int check_state(gsb_cloud* cloud, const gsb_camera* cam, gsb_frame* f) {
  if (!f->valid || f->fingerprint != fingerprint(cloud, cam, !f->lean) || f->n_gaussians != cloud->n ||
      f->cloud != cloud)
    return fail(GSB_ERR_STATE_MISMATCH, "render_backward: output does not match (cloud, camera)");
  return GSB_OK;
}

int gsb_render_backward(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, gsb_frame* f, const double* d_image,
                        int32_t W, int32_t H, uint32_t flags, gsb_grads* grads, double d_pose_out[6]) {
  GSB_NVTX("gsb_render_backward");
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !cam || !f || !d_image) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = check_state(cloud, cam, f)) return r;  // rasterizer.cpp:338-340
  if (W != cam->width || H != cam->height)
    return fail(GSB_ERR_DIMENSION_MISMATCH, "render_backward: d_image size mismatch");  // 341-343
  GSB_RESERVE(f->d_image, sizeof(float) * 3 * (size_t)W * H);
  if (int r = upload_image(ctx, d_image, W, H, f->d_image.as<float>())) return r;
  f->has_dimage = true;
  return backward_common(ctx, cloud, cam, f, flags, grads, d_pose_out);
}

int gsb_render_backward_device(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, gsb_frame* f, uint32_t flags,
                               gsb_grads* grads, double d_pose_out[6]) {
  GSB_NVTX("gsb_render_backward_device");
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !cam || !f) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = check_state(cloud, cam, f)) return r;
  if (!f->has_dimage) return fail(GSB_ERR_INVALID_ARGUMENT, "no upstream gradient in frame (run gsb_frame_rgb_loss)");
  return backward_common(ctx, cloud, cam, f, flags, grads, d_pose_out);
}

int gsb_render_backward_image(gsb_ctx* ctx, gsb_cloud* cloud, const gsb_camera* cam, gsb_frame* f,
                              const gsb_image* d_image, uint32_t flags, gsb_grads* grads, double d_pose_out[6]) {
  GSB_NVTX("gsb_render_backward_image");
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !cam || !f || !d_image) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = check_state(cloud, cam, f)) return r;  // rasterizer.cpp:338-340
  if (d_image->width != cam->width || d_image->height != cam->height)
    return fail(GSB_ERR_DIMENSION_MISMATCH, "render_backward: d_image size mismatch");  // 341-343
  const size_t bytes = sizeof(float) * 3 * (size_t)cam->width * cam->height;
  GSB_RESERVE(f->d_image, bytes);
  GSB_CUDA(cudaMemcpyAsync(f->d_image.p, d_image->planes.p, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  f->has_dimage = true;
  return backward_common(ctx, cloud, cam, f, flags, grads, d_pose_out);
}

// --------------------------------------------------------------- optimiser
double gsb_schedule(int32_t kind, double start, double end, int64_t step, int64_t total) {  // trainer.cpp:30-38
  if (total <= 0) return end;
  double s = std::clamp((double)step / (double)total, 0.0, 1.0);
  if (kind == 0) return end + (start - end) * 0.5 * (1.0 + std::cos(M_PI * s));
  return start * std::pow(end / start, s);
}

int gsb_pose_step(gsb_ctx* ctx, const double pose[12], const double d_pose[6], double lr, gsb_pose_adam* state,
                  double pose_out[12], double applied[6]) {
  GSB_NVTX("gsb_pose_step");
  if (int r = ensure_device(ctx)) return r;
  if (!pose || !d_pose || !state || !pose_out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  const size_t sb = pose_state_bytes();
  char* h = static_cast<char*>(pinned(ctx, sb + 64));
  if (!h) return fail(GSB_ERR_OUT_OF_MEMORY, "pinned staging");
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  pose_state_init(h, pose);
  pose_state_set_adam(h, state->m, state->v, state->step);
  double* hd = reinterpret_cast<double*>(h + ((sb + 15) / 16) * 16);
  for (int k = 0; k < 6; ++k) hd[k] = d_pose[k];
  GSB_RESERVE(ctx->scratch_small, 4096);
  char* dev = ctx->scratch_small.as<char>();
  const size_t off = ((sb + 15) / 16) * 16;
  GSB_CUDA(cudaMemcpyAsync(dev, h, off + sizeof(double) * 6, cudaMemcpyHostToDevice, ctx->stream));
  if (int r = launch_pose_step(ctx->stream, dev, reinterpret_cast<double*>(dev + off), lr, 1)) return r;
  ctx->launches += 1;
  GSB_CUDA(cudaMemcpyAsync(h, dev, sb, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  double cur[12], app[6];
  pose_state_read(h, nullptr, cur, nullptr, nullptr, nullptr, nullptr, app, state->m, state->v, &state->step);
  bool zero = true;
  for (int k = 0; k < 6; ++k) zero = zero && app[k] == 0.0;
  for (int k = 0; k < 12; ++k) pose_out[k] = zero ? pose[k] : cur[k];  // trainer.cpp:86 (bitwise identity)
  if (applied) for (int k = 0; k < 6; ++k) applied[k] = app[k];
  return GSB_OK;
}

namespace gsb {
// Both adam_step overloads (trainer.cpp:40-69): lrs == nullptr -> scalar lr.
static int adam_step_host(gsb_ctx* ctx, double* params, const double* grads, double* m, double* v, int64_t* step,
                          int64_t n, double lr, const double* lrs) {
  if (int r = ensure_device(ctx)) return r;
  if (n < 0 || (n > 0 && (!params || !grads || !m || !v)) || !step) return fail(GSB_ERR_INVALID_ARGUMENT, "bad adam args");
  *step += 1;
  if (n == 0) return GSB_OK;
  DevBuf buf;
  GSB_CUDA(buf.reserve(sizeof(double) * (lrs ? 5 : 4) * n));
  double* d = buf.as<double>();
  GSB_CUDA(cudaMemcpyAsync(d, params, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(d + n, grads, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(d + 2 * n, m, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(d + 3 * n, v, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  if (lrs) GSB_CUDA(cudaMemcpyAsync(d + 4 * n, lrs, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  int r = launch_adam_f64(ctx->stream, d, d + n, d + 2 * n, d + 3 * n, n, lr, lrs ? d + 4 * n : nullptr, *step);
  if (r) {
    buf.release();
    return r;
  }
  ctx->launches += 1;
  GSB_CUDA(cudaMemcpyAsync(params, d, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(m, d + 2 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(v, d + 3 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  buf.release();
  return GSB_OK;
}
}  // namespace gsb

int gsb_adam_step(gsb_ctx* ctx, double* params, const double* grads, double* m, double* v, int64_t* step, int64_t n,
                  double lr) {
  return adam_step_host(ctx, params, grads, m, v, step, n, lr, nullptr);
}

int gsb_adam_step_lrs(gsb_ctx* ctx, double* params, const double* grads, double* m, double* v, int64_t* step,
                      int64_t n, const double* lr_of) {
  if (n > 0 && !lr_of) return fail(GSB_ERR_INVALID_ARGUMENT, "null lr_of");
  return adam_step_host(ctx, params, grads, m, v, step, n, 0.0, lr_of);
}

int gsb_adam_create(gsb_ctx* ctx, gsb_cloud* cloud, gsb_adam** out) {
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  gsb_adam* a = new gsb_adam();
  a->ctx = ctx;
  a->n = cloud->n;
  a->n_pad = cloud->n_pad;
  a->sh_degree = cloud->sh_degree;
  const size_t bytes = sizeof(float) * num_planes(cloud->sh_degree) * cloud->n_pad;
  cudaError_t e = a->m.reserve(bytes);
  if (e == cudaSuccess) e = a->v.reserve(bytes);
  if (e != cudaSuccess) {
    a->m.release();
    a->v.release();
    delete a;
    return cuda_fail(e, "adam alloc");
  }
  cudaMemsetAsync(a->m.p, 0, bytes, ctx->stream);
  cudaMemsetAsync(a->v.p, 0, bytes, ctx->stream);
  ctx_retain(ctx);
  a->ctx_ref = true;
  *out = a;
  return GSB_OK;
}

int gsb_adam_destroy(gsb_adam* a) {
  if (!a) return GSB_OK;
  cudaSetDevice(a->ctx->device);
  cudaStreamSynchronize(a->ctx->stream);
  a->m.release();
  a->v.release();
  gsb_ctx* owner = a->ctx_ref ? a->ctx : nullptr;
  delete a;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_cloud_adam_step(gsb_ctx* ctx, gsb_cloud* cloud, gsb_grads* grads, gsb_adam* adam, const double lrs[6]) {
  GSB_NVTX("gsb_cloud_adam_step");
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !grads || !adam || !lrs) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (grads->n != cloud->n || adam->n != cloud->n) return fail(GSB_ERR_DIMENSION_MISMATCH, "adam/grads/cloud sizes");
  if (cloud->n == 0) return GSB_OK;
  for (int k = 0; k < 5; ++k) adam->step[k] += 1;
  StageScope sc(ctx, kStOptim);
  int r = launch_cloud_adam(ctx->stream, cloud->params.as<float>(), grads->planes.as<float>(), adam->m.as<float>(),
                            adam->v.as<float>(), cloud->n, cloud->n_pad, cloud->sh_degree, lrs, adam->step);
  if (r) return r;
  ctx->launches += 1;
  cloud->version += 1;
  return GSB_OK;
}

// ------------------------------------------------------------ timer API
int gsb_ctx_timer_start(gsb_ctx* ctx) {
  if (int r = ensure_device(ctx)) return r;
  if (!ctx->ev_start) GSB_CUDA(cudaEventCreate(&ctx->ev_start));
  if (!ctx->ev_stop) GSB_CUDA(cudaEventCreate(&ctx->ev_stop));
  GSB_CUDA(cudaEventRecord(ctx->ev_start, ctx->stream));
  return GSB_OK;
}

int gsb_ctx_timer_stop(gsb_ctx* ctx, double* ms) {
  if (int r = ensure_device(ctx)) return r;
  if (!ctx->ev_start || !ctx->ev_stop) return fail(GSB_ERR_INVALID_ARGUMENT, "timer not started");
  GSB_CUDA(cudaEventRecord(ctx->ev_stop, ctx->stream));
  GSB_CUDA(cudaEventSynchronize(ctx->ev_stop));
  float t = 0.f;
  GSB_CUDA(cudaEventElapsedTime(&t, ctx->ev_start, ctx->ev_stop));
  if (ms) *ms = t;
  return GSB_OK;
}

}  // extern "C"

// ------------------------------------------------------------ sessions
// A session's pose_descent iteration is one fixed launch sequence, captured
// once into a CUDA graph and replayed (one cudaGraphLaunch per iteration).
// The graph is rebuilt when the shared scratch frame's buffers move
// (frame gen), the entry capacity changes, or profiling is toggled.
struct gsb_session {
  gsb_ctx* ctx = nullptr;
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  gsb_cloud* cloud = nullptr;
  gsb_image* target = nullptr;
  gsb_camera cam{};
  gsb_pose_config cfg{};
  DevBuf state;   // PoseState
  DevBuf camdev;  // CamDev of the current pose
  DevBuf trace;   // pose (12) + loss (1) per iteration
  void* host_state = nullptr;  // pinned, from / back to ctx->pinned_pool
  size_t host_state_bytes = 0;
  uint32_t* host_counters = nullptr;
  int64_t n_splats = 0, n_entries = 0;
  int32_t stopped = 0;
  int32_t pending = 0;  // iterations launched since the last status check
  int64_t discarded = 0;  // iterations the device discarded (capacity growth) and the host re-ran
  cudaGraphExec_t exec = nullptr;
  int64_t graph_launches = 0;  // kernels per replay
  const gsb_frame* graph_frame = nullptr;
  uint64_t graph_gen = 0;
  int64_t graph_kcap = 0;
  bool graph_profiled = false;
  cudaEvent_t ev[kNumStages][2] = {};
  bool have_events = false;
  bool batch_events = false;  // the events were last recorded by a profiled pose-batch graph
  gsb_frame* own = nullptr;      // private forward state while the session is in a pose batch
  gsb_pose_batch* batch = nullptr;
};

// A pose batch advances several sessions by one pose_descent iteration per
// graph replay: each session's launch sequence is a parallel branch of one
// CUDA graph (fork/join over side streams), on its own forward state, so the
// branches fill each other's wave tails and serial single-block kernels.
struct gsb_pose_batch {
  gsb_ctx* ctx = nullptr;
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  std::vector<gsb_session*> sessions;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> joins;
  cudaEvent_t fork = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<uint64_t> graph_gen;
  std::vector<int64_t> graph_kcap;
  std::vector<int> graph_binning;
  bool graph_profiled = false;  // branches carry per-stage event nodes (ctx profiling on at capture)
  int64_t graph_launches = 0;
};

namespace gsb {

// One pose_descent iteration of the session on forward state f. pre_done:
// K1 already ran for this iteration (a pose batch's shared multi-view launch,
// which also copied the camera into f).
static int session_launch_iteration(gsb_ctx* ctx, gsb_session* s, gsb_frame* f, bool pre_done = false) {
  const gsb_pose_config& cfg = s->cfg;
  const RasterDev rc = make_rasterdev(&cfg.raster);
  double* tp = s->trace.as<double>();
  double* tl = tp + 12 * (size_t)cfg.budget;
  if (pre_done) {
    if (int r = render_post(ctx, s->cloud, f, rc)) return r;
  } else {
    {
      StageScope sc(ctx, kStOther);
      GSB_CUDA(cudaMemcpyAsync(f->cam.p, s->camdev.p, sizeof(CamDev), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (int r = render_async(ctx, s->cloud, f, rc)) return r;
  }
  if (int r = loss_device(ctx, f, s->target->planes.as<float>(), cfg.beta, true)) return r;
  if (int r = backward_device(ctx, s->cloud, f, false, nullptr, /*reduce_pose=*/false)) return r;
  StageScope sc(ctx, kStOptim);
  if (int r = launch_pose_iter(ctx->stream, s->state.p, f->pose_blocks.as<double>(), bwd_geom_blocks(s->cloud->n),
                               f->d_pose.as<double>(), f->loss_val.as<double>(),
                               cfg.cam_lr_start, cfg.cam_lr_end, cfg.pose_converged_eps, cfg.budget,
                               s->camdev.as<CamDev>(), tp, tl, f->counters.as<uint32_t>() + 1, f->k_cap))
    return r;
  ctx->launches += 1;
  return GSB_OK;
}

static int session_capture(gsb_ctx* ctx, gsb_session* s, gsb_frame* f) {
  const double t_dbg = debug_on() ? now_ms() : 0.0;
  if (s->exec) {
    cudaGraphExecDestroy(s->exec);
    s->exec = nullptr;
  }
  if (ctx->profiling && !s->have_events) {
    for (int k = 0; k < kNumStages; ++k)
      for (int j = 0; j < 2; ++j) GSB_CUDA(cudaEventCreate(&s->ev[k][j]));
    s->have_events = true;
  }
  const int64_t launches0 = ctx->launches;
  GSB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  ctx->stage_events = ctx->profiling ? s->ev : nullptr;
  int r = session_launch_iteration(ctx, s, f);
  ctx->stage_events = nullptr;
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (r) {
    if (graph) cudaGraphDestroy(graph);
    return r;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
  e = cudaGraphInstantiate(&s->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  s->graph_launches = ctx->launches - launches0;
  ctx->launches = launches0;  // counted per replay instead
  s->graph_frame = f;
  s->graph_gen = f->gen;
  s->graph_kcap = f->k_cap;
  s->graph_profiled = ctx->profiling;
  s->batch_events = false;
  if (debug_on())
    std::fprintf(stderr, "[gsb] session graph captured: %lld kernels, %.2f ms (binning %d, k_cap %lld)\n",
                 (long long)s->graph_launches, now_ms() - t_dbg, f->binning, (long long)f->k_cap);
  return GSB_OK;
}

static gsb_frame* work_frame(gsb_ctx* ctx) {
  if (!ctx->work) {
    ctx->work = new gsb_frame();
    ctx->work->ctx = ctx;
  }
  return ctx->work;
}

static gsb_frame* session_frame(gsb_ctx* ctx, gsb_session* s) { return s->own ? s->own : work_frame(ctx); }

// Frame set-up + buffer sizing for one session iteration (no capture).
static int session_frame_ready(gsb_ctx* ctx, gsb_session* s, gsb_frame** out) {
  gsb_frame* f = session_frame(ctx, s);
  f->lean = true;  // never exported (not reachable through gsb_frame_download)
  f->want_hits = hit_masks_enabled();  // pose-only backward: K4a may walk the composite's hit masks
  if (int r = frame_setup(ctx, f, s->cloud, &s->cam, s->cfg.background, &s->cfg.raster, false)) return r;
  const int64_t want = f->k_cap > 0 ? f->k_cap : initial_k_cap(s->cloud->n);
  if (int r = frame_reserve(f, s->cloud, want)) return r;
  *out = f;
  return GSB_OK;
}

static int session_prepare(gsb_ctx* ctx, gsb_session* s, gsb_frame** out) {
  gsb_frame* f = nullptr;
  if (int r = session_frame_ready(ctx, s, &f)) return r;
  if (!s->exec || s->graph_frame != f || s->graph_gen != f->gen || s->graph_kcap != f->k_cap ||
      s->graph_profiled != ctx->profiling)
    if (int r = session_capture(ctx, s, f)) return r;
  *out = f;
  return GSB_OK;
}

static int session_launch(gsb_ctx* ctx, gsb_session* s, int32_t iterations) {
  gsb_frame* f = nullptr;
  if (int r = session_prepare(ctx, s, &f)) return r;
  for (int32_t i = 0; i < iterations; ++i) GSB_CUDA(cudaGraphLaunch(s->exec, ctx->stream));
  ctx->launches += s->graph_launches * iterations;
  s->pending += iterations;
  return GSB_OK;
}

// Waits for the session's launched iterations; re-runs any the device
// discarded for an entry-capacity overflow (after growing the capacity).
static int session_sync(gsb_ctx* ctx, gsb_session* s) {
  const size_t sb = pose_state_bytes();
  for (int round = 0; round < 8; ++round) {
    gsb_frame* f = session_frame(ctx, s);
    GSB_CUDA(cudaMemcpyAsync(s->host_state, s->state.p, sb, cudaMemcpyDeviceToHost, ctx->stream));
    if (f->counters.p)
      GSB_CUDA(cudaMemcpyAsync(s->host_counters, f->counters.p, 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               ctx->stream));
    GSB_CUDA(cudaStreamSynchronize(ctx->stream));
    pose_state_read(s->host_state, nullptr, nullptr, nullptr, nullptr, nullptr, &s->stopped, nullptr, nullptr, nullptr,
                    nullptr);
    uint32_t abort_k = 0, abort_tile = 0;
    const int32_t aborted = pose_state_take_aborted(s->host_state, &abort_k, &abort_tile);
    s->n_splats = s->host_counters[0];
    s->n_entries = s->host_counters[1];
    if (aborted == 0) {
      s->pending = 0;
      return GSB_OK;
    }
    s->discarded += aborted;
    if (debug_on())
      std::fprintf(stderr, "[gsb] %d iteration(s) discarded: K %u (cap %lld), tile overflow %u\n", aborted, abort_k,
                   (long long)f->k_cap, abort_tile);
    // clear the device-side abort counter, grow the entry capacity (or leave
    // tile-local binning), replay
    GSB_CUDA(cudaMemcpyAsync(s->state.p, s->host_state, sb, cudaMemcpyHostToDevice, ctx->stream));
    if (abort_tile != 0u) fall_back_to_global(f);
    const int64_t k = std::max<int64_t>(abort_k, s->host_counters[1]);
    if (int r = frame_reserve(f, s->cloud, std::max<int64_t>(f->k_cap, k + k / 4 + 4096))) return r;
    s->pending = 0;
    if (int r = session_launch(ctx, s, aborted)) return r;
  }
  return fail(GSB_ERR_OUT_OF_MEMORY, "entry capacity did not converge");
}

}  // namespace gsb

extern "C" {

int gsb_session_create(gsb_ctx* ctx, gsb_cloud* cloud, gsb_image* target, const double intr[4],
                       const double init_pose[12], const gsb_pose_config* cfg, gsb_session** out) {
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !target || !intr || !init_pose || !cfg || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = validate_config(&cfg->raster)) return r;
  if (cfg->budget <= 0) return fail(GSB_ERR_INVALID_CONFIG, "budget must be > 0");
  gsb_session* s = new gsb_session();
  s->ctx = ctx;
  s->cloud = cloud;
  s->target = target;
  s->cfg = *cfg;
  s->cam.fx = intr[0];
  s->cam.fy = intr[1];
  s->cam.cx = intr[2];
  s->cam.cy = intr[3];
  s->cam.width = target->width;
  s->cam.height = target->height;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) s->cam.R[r * 3 + c] = init_pose[r * 4 + c];
    s->cam.t[r] = init_pose[r * 4 + 3];
  }
  const size_t sb = pose_state_bytes();
  const size_t host_bytes = ((sb + 63) / 64) * 64 + 64 + sizeof(CamDev);
  cudaError_t e = s->state.reserve(sb);
  if (e == cudaSuccess) e = s->camdev.reserve(sizeof(CamDev));
  if (e == cudaSuccess) e = s->trace.reserve(sizeof(double) * 13 * (size_t)cfg->budget);
  // pinned status block from the context's pool (cudaMallocHost / cudaFreeHost
  // cost up to hundreds of ms per call under load)
  if (e == cudaSuccess) {
    for (size_t i = 0; i < ctx->pinned_pool.size(); ++i)
      if (ctx->pinned_pool[i].second >= host_bytes) {
        s->host_state = ctx->pinned_pool[i].first;
        s->host_state_bytes = ctx->pinned_pool[i].second;
        ctx->pinned_pool.erase(ctx->pinned_pool.begin() + i);
        break;
      }
    if (!s->host_state) {
      e = cudaMallocHost(&s->host_state, host_bytes);
      if (e == cudaSuccess) s->host_state_bytes = host_bytes;
    }
  }
  if (e != cudaSuccess) {
    gsb_session_destroy(s);
    return cuda_fail(e, "session alloc");
  }
  char* hb = static_cast<char*>(s->host_state);
  s->host_counters = reinterpret_cast<uint32_t*>(hb + ((sb + 63) / 64) * 64);
  CamDev* hcam = reinterpret_cast<CamDev*>(hb + ((sb + 63) / 64) * 64 + 64);
  pose_state_init(s->host_state, init_pose);
  *hcam = make_camdev(&s->cam, kTile);
  GSB_CUDA(cudaMemcpyAsync(s->camdev.p, hcam, sizeof(CamDev), cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(s->state.p, s->host_state, sb, cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx_retain(ctx);
  s->ctx_ref = true;
  *out = s;
  return GSB_OK;
}

int gsb_session_destroy(gsb_session* s) {
  if (!s) return GSB_OK;
  cudaSetDevice(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  if (gsb_pose_batch* b = s->batch) {  // leave the batch: its graph is rebuilt without this branch
    for (size_t i = 0; i < b->sessions.size(); ++i)
      if (b->sessions[i] == s) {
        cudaStreamDestroy(b->streams[i]);
        cudaEventDestroy(b->joins[i]);
        b->sessions.erase(b->sessions.begin() + i);
        b->streams.erase(b->streams.begin() + i);
        b->joins.erase(b->joins.begin() + i);
        b->graph_gen.erase(b->graph_gen.begin() + i);
        b->graph_kcap.erase(b->graph_kcap.begin() + i);
        b->graph_binning.erase(b->graph_binning.begin() + i);
        break;
      }
    if (b->exec) cudaGraphExecDestroy(b->exec);
    b->exec = nullptr;
  }
  if (s->exec) cudaGraphExecDestroy(s->exec);
  if (s->own) s->ctx->frame_pool.push_back(s->own);
  if (s->have_events)
    for (int k = 0; k < kNumStages; ++k)
      for (int j = 0; j < 2; ++j) cudaEventDestroy(s->ev[k][j]);
  s->state.release();
  s->camdev.release();
  s->trace.release();
  if (s->host_state) s->ctx->pinned_pool.emplace_back(s->host_state, s->host_state_bytes);
  gsb_ctx* owner = s->ctx_ref ? s->ctx : nullptr;
  delete s;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_session_step(gsb_ctx* ctx, gsb_session* s, int32_t iterations) {
  GSB_NVTX("gsb_session_step");
  if (int r = ensure_device(ctx)) return r;
  if (!s || s->ctx != ctx) return fail(GSB_ERR_INVALID_ARGUMENT, "session / context mismatch");
  const int32_t chunk = 16;
  while (iterations > 0 && !s->stopped) {
    const int32_t now = std::min(iterations, chunk);
    if (int r = session_launch(ctx, s, now)) return r;
    if (int r = session_sync(ctx, s)) return r;
    iterations -= now;
  }
  return GSB_OK;
}

int gsb_session_step_async(gsb_ctx* ctx, gsb_session* s, int32_t iterations) {
  GSB_NVTX("gsb_session_step_async");
  if (int r = ensure_device(ctx)) return r;
  if (!s || s->ctx != ctx) return fail(GSB_ERR_INVALID_ARGUMENT, "session / context mismatch");
  if (iterations <= 0) return GSB_OK;
  return session_launch(ctx, s, iterations);
}

int gsb_session_stage_times(gsb_session* s, double* ms_out) {
  if (!s || !ms_out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = ensure_device(s->ctx)) return r;
  for (int k = 0; k < kNumStages; ++k) ms_out[k] = 0.0;
  if (!s->have_events || !(s->graph_profiled || s->batch_events)) return GSB_OK;
  GSB_CUDA(cudaStreamSynchronize(s->ctx->stream));
  for (int k = 0; k < kNumStages; ++k) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, s->ev[k][0], s->ev[k][1]) == cudaSuccess) ms_out[k] = t;
  }
  cudaGetLastError();  // stages never recorded report cudaErrorInvalidResourceHandle
  return GSB_OK;
}

int gsb_session_read(gsb_session* s, double pose[12], double best_pose[12], double* final_loss, int32_t* steps_used,
                     int32_t* converged, int32_t* stopped) {
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "null session");
  gsb_ctx* ctx = s->ctx;
  if (int r = ensure_device(ctx)) return r;
  if (int r = session_sync(ctx, s)) return r;  // also re-runs discarded iterations
  pose_state_read(s->host_state, best_pose, pose, final_loss, steps_used, converged, stopped, nullptr, nullptr,
                  nullptr, nullptr);
  return GSB_OK;
}

int gsb_session_frame_info(gsb_session* s, gsb_frame_info* info) {
  if (!s || !info) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  std::memset(info, 0, sizeof *info);
  info->n_gaussians = s->cloud->n;
  info->n_splats = s->n_splats;
  info->n_entries = s->n_entries;
  info->width = s->cam.width;
  info->height = s->cam.height;
  info->tiles_x = (s->cam.width + kTile - 1) / kTile;
  info->tiles_y = (s->cam.height + kTile - 1) / kTile;
  if (gsb_frame* f = session_frame(s->ctx, s)) info->binning = f->binning == kBinGlobal ? GSB_BINNING_GLOBAL : GSB_BINNING_TILE_LOCAL;
  return GSB_OK;
}

// pipelines.cpp:218-222 -> pose_descent (58-92), device resident.
int gsb_estimate_pose(gsb_ctx* ctx, gsb_cloud* cloud, gsb_image* target, const double intr[4],
                      const double init_pose[12], const gsb_pose_config* cfg, double pose_out[12], double* final_loss,
                      int32_t* steps_used, int32_t* converged, double* trace_pose, double* trace_loss) {
  GSB_NVTX("gsb_estimate_pose");
  if (!pose_out) return fail(GSB_ERR_INVALID_ARGUMENT, "null pose_out");
  gsb_session* s = nullptr;
  if (int r = gsb_session_create(ctx, cloud, target, intr, init_pose, cfg, &s)) return r;
  int r = gsb_session_step(ctx, s, cfg->budget);
  int32_t su = 0;
  if (!r) r = gsb_session_read(s, nullptr, pose_out, final_loss, &su, converged, nullptr);
  if (!r && steps_used) *steps_used = su;
  if (!r && su > 0 && (trace_pose || trace_loss)) {
    const double* tp = s->trace.as<double>();
    if (trace_pose)
      r = cuda_fail_or_ok(cudaMemcpy(trace_pose, tp, sizeof(double) * 12 * su, cudaMemcpyDeviceToHost));
    if (!r && trace_loss)
      r = cuda_fail_or_ok(cudaMemcpy(trace_loss, tp + 12 * (size_t)cfg->budget, sizeof(double) * su,
                                     cudaMemcpyDeviceToHost));
  }
  gsb_session_destroy(s);
  return r;
}

}  // extern "C"

namespace gsb {

static void batch_drop_graph(gsb_pose_batch* b) {
  if (b->exec) cudaGraphExecDestroy(b->exec);
  b->exec = nullptr;
}

// One graph: fork -> one branch per session (its own stream while capturing)
// -> join. ctx->stream is pointed at the branch stream while a session's
// launch sequence is recorded, so the launch code is the single-session code.
static int batch_capture(gsb_ctx* ctx, gsb_pose_batch* b) {
  batch_drop_graph(b);
  const size_t n = b->sessions.size();
  std::vector<gsb_frame*> frames(n);
  for (size_t i = 0; i < n; ++i)
    if (int r = session_frame_ready(ctx, b->sessions[i], &frames[i])) return r;
  const double t_dbg = debug_on() ? now_ms() : 0.0;
  const int64_t launches0 = ctx->launches;
  cudaStream_t main = ctx->stream;
  // With profiling on, each branch brackets its stages with its session's
  // events, so stage times are those of the concurrent batch (the eager event
  // pool stays off while capturing).
  const bool profiling = ctx->profiling;
  ctx->profiling = false;
  if (profiling)
    for (gsb_session* s : b->sessions)
      if (!s->have_events) {
        for (int k = 0; k < kNumStages; ++k)
          for (int j = 0; j < 2; ++j) GSB_CUDA(cudaEventCreate(&s->ev[k][j]));
        s->have_events = true;
      }
  GSB_CUDA(cudaStreamBeginCapture(main, cudaStreamCaptureModeThreadLocal));
  int r = GSB_OK;
  cudaError_t e = cudaSuccess;
  // K1 for every session of one cloud in one launch (the cloud is read once);
  // sessions on other clouds run their own K1 inside their branch.
  std::vector<char> shared(n, 0);
  {
    std::vector<const CamDev*> cams;
    std::vector<gsb_frame*> fr;
    const gsb_cloud* c0 = b->sessions[0]->cloud;
    bool same_cfg = true;
    for (size_t i = 0; i < n; ++i)
      same_cfg = same_cfg && std::memcmp(&b->sessions[i]->cfg.raster, &b->sessions[0]->cfg.raster,
                                         sizeof(gsb_raster_config)) == 0;
    for (size_t i = 0; i < n && same_cfg; ++i)
      if (b->sessions[i]->cloud == c0) {
        shared[i] = 1;
        cams.push_back(b->sessions[i]->camdev.as<CamDev>());
        fr.push_back(frames[i]);
        e = cudaMemsetAsync(frames[i]->counters.p, 0, 4 * sizeof(uint32_t), main);
        if (e != cudaSuccess) break;
      }
    if (e == cudaSuccess && !fr.empty()) {
      // profiling: the shared multi-view preprocess is charged to session 0's preprocess stage
      if (profiling) e = cudaEventRecordWithFlags(b->sessions[0]->ev[kStPreprocess][0], main, cudaEventRecordExternal);
      if (e == cudaSuccess)
        r = launch_preprocess_multi(main, c0, make_rasterdev(&b->sessions[0]->cfg.raster), cams.data(), fr.data(),
                                    (int)fr.size());
      if (profiling && !r && e == cudaSuccess)
        e = cudaEventRecordWithFlags(b->sessions[0]->ev[kStPreprocess][1], main, cudaEventRecordExternal);
      ctx->launches += (int64_t)((fr.size() + 15) / 16);
    }
  }
  if (!r && e == cudaSuccess) e = cudaEventRecord(b->fork, main);
  for (size_t i = 0; i < n && !r && e == cudaSuccess; ++i) {
    e = cudaStreamWaitEvent(b->streams[i], b->fork, 0);
    if (e != cudaSuccess) break;
    ctx->stream = b->streams[i];
    ctx->stage_events = profiling ? b->sessions[i]->ev : nullptr;
    r = session_launch_iteration(ctx, b->sessions[i], frames[i], shared[i] != 0);
    ctx->stage_events = nullptr;
    ctx->stream = main;
    if (!r) e = cudaEventRecord(b->joins[i], b->streams[i]);
    if (!r && e == cudaSuccess) e = cudaStreamWaitEvent(main, b->joins[i], 0);
  }
  ctx->stream = main;
  ctx->profiling = profiling;
  cudaGraph_t graph = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(main, &graph);
  if (r || e != cudaSuccess || e2 != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    ctx->launches = launches0;
    if (r) return r;
    return cuda_fail(e != cudaSuccess ? e : e2, "pose batch capture");
  }
  e = cudaGraphInstantiate(&b->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate (pose batch)");
  b->graph_launches = ctx->launches - launches0;
  ctx->launches = launches0;
  for (size_t i = 0; i < n; ++i) {
    b->graph_gen[i] = frames[i]->gen;
    b->graph_kcap[i] = frames[i]->k_cap;
    b->graph_binning[i] = frames[i]->binning;
    b->sessions[i]->batch_events = profiling;
  }
  b->graph_profiled = profiling;
  if (debug_on())
    std::fprintf(stderr, "[gsb] pose batch graph captured: %zu sessions, %lld kernels, %.2f ms\n", n,
                 (long long)b->graph_launches, now_ms() - t_dbg);
  return GSB_OK;
}

static int batch_prepare(gsb_ctx* ctx, gsb_pose_batch* b) {
  bool stale = b->exec == nullptr || b->graph_profiled != ctx->profiling;
  for (size_t i = 0; i < b->sessions.size() && !stale; ++i) {
    const gsb_frame* f = b->sessions[i]->own;
    stale = f->gen != b->graph_gen[i] || f->k_cap != b->graph_kcap[i] || f->binning != b->graph_binning[i];
  }
  return stale ? batch_capture(ctx, b) : GSB_OK;
}

}  // namespace gsb

extern "C" {

int gsb_pose_batch_create(gsb_ctx* ctx, gsb_session* const* sessions, int32_t count, gsb_pose_batch** out) {
  if (int r = ensure_device(ctx)) return r;
  if (!sessions || count <= 0 || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "empty pose batch");
  for (int32_t i = 0; i < count; ++i) {
    if (!sessions[i] || sessions[i]->ctx != ctx) return fail(GSB_ERR_INVALID_ARGUMENT, "session / context mismatch");
    if (sessions[i]->batch) return fail(GSB_ERR_INVALID_ARGUMENT, "session already belongs to a pose batch");
    for (int32_t j = 0; j < i; ++j)
      if (sessions[j] == sessions[i]) return fail(GSB_ERR_INVALID_ARGUMENT, "session listed twice");
  }
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  gsb_pose_batch* b = new gsb_pose_batch();
  b->ctx = ctx;
  cudaError_t e = cudaEventCreateWithFlags(&b->fork, cudaEventDisableTiming);
  for (int32_t i = 0; i < count && e == cudaSuccess; ++i) {
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) b->streams.push_back(st);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) b->joins.push_back(ev);
  }
  if (e != cudaSuccess) {
    gsb_pose_batch_destroy(b);
    return cuda_fail(e, "pose batch streams");
  }
  for (int32_t i = 0; i < count; ++i) {
    gsb_session* s = sessions[i];
    if (!ctx->frame_pool.empty()) {
      s->own = ctx->frame_pool.back();
      ctx->frame_pool.pop_back();
    } else {
      s->own = new gsb_frame();
      s->own->ctx = ctx;
    }
    s->batch = b;
    b->sessions.push_back(s);
  }
  b->graph_gen.assign(count, 0);
  b->graph_kcap.assign(count, 0);
  b->graph_binning.assign(count, -1);
  ctx_retain(ctx);
  b->ctx_ref = true;
  *out = b;
  return GSB_OK;
}

int gsb_pose_batch_destroy(gsb_pose_batch* b) {
  if (!b) return GSB_OK;
  gsb_ctx* ctx = b->ctx;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  batch_drop_graph(b);
  for (gsb_session* s : b->sessions) {
    if (s->exec && s->graph_frame == s->own) {  // its single-session graph points at the private frame
      cudaGraphExecDestroy(s->exec);
      s->exec = nullptr;
    }
    if (s->own) ctx->frame_pool.push_back(s->own);  // keeps its sized buffers for the next batch
    s->own = nullptr;
    s->batch = nullptr;
  }
  for (cudaStream_t st : b->streams) cudaStreamDestroy(st);
  for (cudaEvent_t ev : b->joins) cudaEventDestroy(ev);
  if (b->fork) cudaEventDestroy(b->fork);
  gsb_ctx* owner = b->ctx_ref ? b->ctx : nullptr;
  delete b;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_pose_batch_step_async(gsb_ctx* ctx, gsb_pose_batch* b, int32_t iterations) {
  GSB_NVTX("gsb_pose_batch_step_async");
  if (int r = ensure_device(ctx)) return r;
  if (!b || b->ctx != ctx) return fail(GSB_ERR_INVALID_ARGUMENT, "pose batch / context mismatch");
  if (iterations <= 0) return GSB_OK;
  if (int r = batch_prepare(ctx, b)) return r;
  for (int32_t i = 0; i < iterations; ++i) GSB_CUDA(cudaGraphLaunch(b->exec, ctx->stream));
  ctx->launches += b->graph_launches * iterations;
  for (gsb_session* s : b->sessions) s->pending += iterations;
  return GSB_OK;
}

int gsb_pose_batch_sync(gsb_ctx* ctx, gsb_pose_batch* b) {
  GSB_NVTX("gsb_pose_batch_sync");
  if (int r = ensure_device(ctx)) return r;
  if (!b || b->ctx != ctx) return fail(GSB_ERR_INVALID_ARGUMENT, "pose batch / context mismatch");
  // Every session's status block in one round trip; only sessions that had
  // iterations discarded go through session_sync, which re-runs them on the
  // session's own graph.
  const size_t sb = pose_state_bytes();
  for (gsb_session* s : b->sessions) {
    GSB_CUDA(cudaMemcpyAsync(s->host_state, s->state.p, sb, cudaMemcpyDeviceToHost, ctx->stream));
    gsb_frame* f = session_frame(ctx, s);
    if (f->counters.p)
      GSB_CUDA(cudaMemcpyAsync(s->host_counters, f->counters.p, 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               ctx->stream));
  }
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (gsb_session* s : b->sessions) {
    if (pose_state_aborted(s->host_state) != 0) {
      if (int r = session_sync(ctx, s)) return r;
      continue;
    }
    pose_state_read(s->host_state, nullptr, nullptr, nullptr, nullptr, nullptr, &s->stopped, nullptr, nullptr, nullptr,
                    nullptr);
    s->n_splats = s->host_counters[0];
    s->n_entries = s->host_counters[1];
    s->pending = 0;
  }
  return GSB_OK;
}

int gsb_pose_batch_discarded(const gsb_pose_batch* b, int64_t* out) {
  if (!b || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  int64_t t = 0;
  for (const gsb_session* s : b->sessions) t += s->discarded;
  *out = t;
  return GSB_OK;
}

int gsb_pose_batch_step(gsb_ctx* ctx, gsb_pose_batch* b, int32_t iterations) {
  GSB_NVTX("gsb_pose_batch_step");
  const int32_t chunk = 16;
  while (iterations > 0) {
    bool all_stopped = true;
    for (gsb_session* s : b->sessions) all_stopped = all_stopped && s->stopped;
    if (all_stopped) break;
    const int32_t now = std::min(iterations, chunk);
    if (int r = gsb_pose_batch_step_async(ctx, b, now)) return r;
    if (int r = gsb_pose_batch_sync(ctx, b)) return r;
    iterations -= now;
  }
  return GSB_OK;
}

// C3's call: pose_descent for `count` independent views of one cloud
// (pipelines.cpp:218-222 per view), advanced together as one pose batch.
int gsb_estimate_poses(gsb_ctx* ctx, gsb_cloud* cloud, gsb_image* const* targets, const double intr[4],
                       const double* init_poses, int32_t count, const gsb_pose_config* cfg, double* poses_out,
                       double* final_losses, int32_t* steps_used) {
  GSB_NVTX("gsb_estimate_poses");
  if (!targets || !init_poses || !poses_out || count <= 0) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  // Views run in pose batches of kBatchViews (8: one batch's branches fill
  // the GPU; more branches only add memory traffic — 64 views in one batch
  // measured 1474 iters/s against 1923 at 8). Per-view results do not depend
  // on the grouping (batches are bit-identical to sessions stepped alone).
  static const int32_t kBatchViews = [] {
    const char* e = std::getenv("GSB_POSE_BATCH_VIEWS");
    const int v = e ? std::atoi(e) : 8;
    return v > 0 ? v : 8;
  }();
  int r = GSB_OK;
  for (int32_t g0 = 0; g0 < count && !r; g0 += kBatchViews) {
    const int32_t gn = std::min(kBatchViews, count - g0);
    std::vector<gsb_session*> ss(gn, nullptr);
    double t[6] = {debug_on() ? now_ms() : 0.0};
    for (int32_t i = 0; i < gn && !r; ++i)
      r = gsb_session_create(ctx, cloud, targets[g0 + i], intr, init_poses + 12 * (size_t)(g0 + i), cfg, &ss[i]);
    if (debug_on()) t[1] = now_ms();
    gsb_pose_batch* b = nullptr;
    if (!r) r = gsb_pose_batch_create(ctx, ss.data(), gn, &b);
    if (debug_on()) t[2] = now_ms();
    if (!r) r = gsb_pose_batch_step(ctx, b, cfg->budget);
    if (debug_on()) t[3] = now_ms();
    for (int32_t i = 0; i < gn && !r; ++i) {
      int32_t su = 0;
      const size_t v = (size_t)(g0 + i);
      r = gsb_session_read(ss[i], nullptr, poses_out + 12 * v, final_losses ? final_losses + v : nullptr, &su,
                           nullptr, nullptr);
      if (!r && steps_used) steps_used[v] = su;
    }
    if (debug_on()) t[4] = now_ms();
    if (b) gsb_pose_batch_destroy(b);
    for (gsb_session* s : ss)
      if (s) gsb_session_destroy(s);
    if (debug_on()) {
      t[5] = now_ms();
      std::fprintf(stderr, "[gsb] estimate_poses views %d..%d: create %.2f batch %.2f step %.2f read %.2f destroy %.2f ms\n",
                   g0, g0 + gn - 1, t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[5] - t[4]);
    }
  }
  return r;
}

}  // extern "C"


// ------------------------------------------------------ densify_and_prune
namespace gsb {

static int64_t pad_n(int64_t n) { return std::max<int64_t>(32, (n + 31) / 32 * 32); }

struct DensifyParams {
  double grad_threshold, size_ratio, prune_opacity;
  int32_t n_target;
};

// trainer.cpp:144-239 on the device (k_densify.cu); d_gsum / d_gcnt are the
// GradAccum arrays (device, cloud->n). Rebuilds cloud->params (new n, n_pad)
// and remaps the Adam moment planes (m, v: [planes][n_pad], may be null).
static int densify_device(gsb_ctx* ctx, gsb_cloud* cloud, const double* d_gsum, const int32_t* d_gcnt,
                          const DensifyParams& p, uint64_t* rng_state, DevBuf* adam_m, DevBuf* adam_v,
                          int32_t report[3]) {
  cudaStream_t st = ctx->stream;
  const int64_t n = cloud->n, np = cloud->n_pad;
  const int nplanes = num_planes(cloud->sh_degree);
  report[0] = report[1] = report[2] = 0;
  if (n == 0) return GSB_OK;
  // bounding box -> extent -> size threshold (trainer.cpp:148-155), exact
  DevBuf bb;
  GSB_CUDA(bb.reserve(sizeof(float) * 6 * densify_bbox_blocks()));
  if (int r = launch_densify_bbox(st, cloud->params.as<float>(), n, np, bb.as<float>())) return r;
  std::vector<float> hb(6 * densify_bbox_blocks());
  GSB_CUDA(cudaMemcpyAsync(hb.data(), bb.p, sizeof(float) * hb.size(), cudaMemcpyDeviceToHost, st));
  GSB_CUDA(cudaStreamSynchronize(st));
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = hb[k];
    hi[k] = hb[3 + k];
    for (int b = 1; b < densify_bbox_blocks(); ++b) {
      lo[k] = std::min(lo[k], (double)hb[6 * b + k]);
      hi[k] = std::max(hi[k], (double)hb[6 * b + 3 + k]);
    }
  }
  const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  const double extent = std::sqrt(dx * dx + dy * dy + dz * dz);
  const double size_threshold = p.size_ratio * std::max(extent, 1e-6);
  // actions + positions
  DevBuf keep, extra, split, keep_pos, extra_pos, split_rank, tmp, tot;
  GSB_CUDA(keep.reserve(sizeof(uint32_t) * n));
  GSB_CUDA(extra.reserve(sizeof(uint32_t) * n));
  GSB_CUDA(split.reserve(sizeof(uint32_t) * n));
  GSB_CUDA(keep_pos.reserve(sizeof(uint32_t) * n));
  GSB_CUDA(extra_pos.reserve(sizeof(uint32_t) * n));
  GSB_CUDA(split_rank.reserve(sizeof(uint32_t) * n));
  GSB_CUDA(tmp.reserve(sizeof(uint32_t) * (scan_onepass_words(n) + 64)));
  GSB_CUDA(tot.reserve(sizeof(uint32_t) * 4));
  if (int r = launch_densify_action(st, cloud->params.as<float>(), n, np, d_gsum, d_gcnt, p.grad_threshold,
                                    size_threshold, keep.as<uint32_t>(), extra.as<uint32_t>(), split.as<uint32_t>()))
    return r;
  int64_t launches = 0;
  uint32_t* t = tot.as<uint32_t>();
  if (int r = scan_onepass(st, keep.as<uint32_t>(), n, nullptr, false, keep_pos.as<uint32_t>(), tmp.as<uint32_t>(),
                           t + 0, &launches))
    return r;
  if (int r = scan_onepass(st, extra.as<uint32_t>(), n, nullptr, false, extra_pos.as<uint32_t>(), tmp.as<uint32_t>(),
                           t + 1, &launches))
    return r;
  if (int r = scan_onepass(st, split.as<uint32_t>(), n, nullptr, false, split_rank.as<uint32_t>(),
                           tmp.as<uint32_t>(), t + 2, &launches))
    return r;
  uint32_t ht[3];
  GSB_CUDA(cudaMemcpyAsync(ht, t, sizeof ht, cudaMemcpyDeviceToHost, st));
  GSB_CUDA(cudaStreamSynchronize(st));
  const uint32_t n_keep = ht[0], n_extra = ht[1], n_split = ht[2];
  report[1] = (int32_t)n_split;
  report[0] = (int32_t)(n_extra - 2 * n_split);
  // split children's normals from the run's Rng, in the reference's draw order
  std::vector<double> nh(6 * (size_t)n_split + 1);
  if (int r = gsb_rng_child_normals(rng_state, 2 * (int64_t)n_split, nh.data())) return r;
  DevBuf normals;
  GSB_CUDA(normals.reserve(sizeof(double) * nh.size()));
  GSB_CUDA(cudaMemcpyAsync(normals.p, nh.data(), sizeof(double) * nh.size(), cudaMemcpyHostToDevice, st));
  // post-densify population
  const int64_t total = (int64_t)n_keep + n_extra, np_t = pad_n(total);
  DevBuf next, src_next;
  GSB_CUDA(next.reserve(sizeof(float) * nplanes * np_t));
  GSB_CUDA(src_next.reserve(sizeof(int32_t) * std::max<int64_t>(total, 1)));
  GSB_CUDA(cudaMemsetAsync(next.p, 0, sizeof(float) * nplanes * np_t, st));
  if (int r = launch_densify_build(st, cloud->params.as<float>(), n, np, nplanes, keep.as<uint32_t>(),
                                   keep_pos.as<uint32_t>(), extra.as<uint32_t>(), extra_pos.as<uint32_t>(),
                                   split_rank.as<uint32_t>(), normals.as<double>(), n_keep, next.as<float>(), np_t,
                                   src_next.as<int32_t>()))
    return r;
  // prune threshold: max(prune_opacity, (n_target+1)-th largest opacity)
  double threshold = p.prune_opacity;
  if (total > p.n_target && p.n_target >= 0) {
    DevBuf kv[2][2], hist;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) GSB_CUDA(kv[a][b].reserve(sizeof(uint32_t) * total));
    GSB_CUDA(hist.reserve(sizeof(uint32_t) * (radix_hist_words(total, 32) + 64)));
    if (int r = launch_densify_logit_keys(st, next.as<float>(), total, np_t, kv[0][0].as<uint32_t>(),
                                          kv[1][0].as<uint32_t>()))
      return r;
    uint32_t* keys[2] = {kv[0][0].as<uint32_t>(), kv[0][1].as<uint32_t>()};
    uint32_t* vals[2] = {kv[1][0].as<uint32_t>(), kv[1][1].as<uint32_t>()};
    int sel = 0;
    if (int r = radix_sort_pairs(st, keys, vals, total, nullptr, 32, hist.as<uint32_t>(), &sel, &launches)) return r;
    uint32_t kbits = 0;  // ascending: the (n_target+1)-th largest sits at total - 1 - n_target
    GSB_CUDA(cudaMemcpyAsync(&kbits, keys[sel] + (total - 1 - p.n_target), sizeof(uint32_t), cudaMemcpyDeviceToHost,
                             st));
    GSB_CUDA(cudaStreamSynchronize(st));
    const uint32_t b = (kbits & 0x80000000u) ? (kbits & 0x7fffffffu) : ~kbits;
    float logit;
    std::memcpy(&logit, &b, sizeof logit);
    threshold = std::max(threshold, 1.0 / (1.0 + std::exp(-(double)logit)));
  }
  DevBuf flag, pos;
  GSB_CUDA(flag.reserve(sizeof(uint32_t) * total));
  GSB_CUDA(pos.reserve(sizeof(uint32_t) * total));
  if (int r = launch_densify_prune_flag(st, next.as<float>(), total, np_t, threshold, flag.as<uint32_t>())) return r;
  GSB_CUDA(tmp.reserve(sizeof(uint32_t) * (scan_onepass_words(total) + 64)));
  if (int r = scan_onepass(st, flag.as<uint32_t>(), total, nullptr, false, pos.as<uint32_t>(), tmp.as<uint32_t>(),
                           t + 3, &launches))
    return r;
  uint32_t m = 0;
  GSB_CUDA(cudaMemcpyAsync(&m, t + 3, sizeof m, cudaMemcpyDeviceToHost, st));
  GSB_CUDA(cudaStreamSynchronize(st));
  report[2] = (int32_t)(total - m);
  const int64_t np_m = pad_n(m);
  DevBuf fin, src_fin;
  GSB_CUDA(fin.reserve(sizeof(float) * nplanes * np_m));
  GSB_CUDA(src_fin.reserve(sizeof(int32_t) * std::max<int64_t>(m, 1)));
  GSB_CUDA(cudaMemsetAsync(fin.p, 0, sizeof(float) * nplanes * np_m, st));
  if (int r = launch_densify_gather(st, next.as<float>(), total, np_t, nplanes, flag.as<uint32_t>(),
                                    pos.as<uint32_t>(), src_next.as<int32_t>(), fin.as<float>(), np_m,
                                    src_fin.as<int32_t>()))
    return r;
  if (adam_m && adam_v && adam_m->p && adam_v->p) {
    DevBuf mo, vo;
    GSB_CUDA(mo.reserve(sizeof(float) * nplanes * np_m));
    GSB_CUDA(vo.reserve(sizeof(float) * nplanes * np_m));
    GSB_CUDA(cudaMemsetAsync(mo.p, 0, sizeof(float) * nplanes * np_m, st));
    GSB_CUDA(cudaMemsetAsync(vo.p, 0, sizeof(float) * nplanes * np_m, st));
    if (int r = launch_densify_adam_remap(st, adam_m->as<float>(), adam_v->as<float>(), np, nplanes,
                                          src_fin.as<int32_t>(), m, np_m, mo.as<float>(), vo.as<float>()))
      return r;
    GSB_CUDA(cudaStreamSynchronize(st));
    std::swap(*adam_m, mo);
    std::swap(*adam_v, vo);
    mo.release();
    vo.release();
  }
  GSB_CUDA(cudaStreamSynchronize(st));
  std::swap(cloud->params, fin);
  fin.release();
  cloud->n = m;
  cloud->n_pad = np_m;
  ++cloud->version;
  ctx->launches += launches + 7;
  DevBuf* tmps[] = {&bb, &keep, &extra, &split, &keep_pos, &extra_pos, &split_rank, &tmp, &tot, &normals, &next,
                    &src_next, &flag, &pos, &src_fin};
  for (DevBuf* b : tmps) b->release();
  return GSB_OK;
}

}  // namespace gsb

extern "C" {

int gsb_densify_and_prune(gsb_ctx* ctx, gsb_cloud* cloud, const double* grad_sum, const int32_t* count,
                          double grad_threshold, double densify_size_ratio, int32_t n_target, double prune_opacity,
                          uint64_t* rng_state, gsb_adam* adam, int32_t report[3]) {
  GSB_NVTX("gsb_densify_and_prune");
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !grad_sum || !count || !rng_state || !report) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (adam && (adam->n != cloud->n || adam->n_pad != cloud->n_pad))
    return fail(GSB_ERR_DIMENSION_MISMATCH, "adam state does not match the cloud");
  const int64_t n = cloud->n;
  DevBuf gs, gc;
  GSB_CUDA(gs.reserve(sizeof(double) * std::max<int64_t>(n, 1)));
  GSB_CUDA(gc.reserve(sizeof(int32_t) * std::max<int64_t>(n, 1)));
  GSB_CUDA(cudaMemcpyAsync(gs.p, grad_sum, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaMemcpyAsync(gc.p, count, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  DensifyParams p{grad_threshold, densify_size_ratio, prune_opacity, n_target};
  int r = densify_device(ctx, cloud, gs.as<double>(), gc.as<int32_t>(), p, rng_state, adam ? &adam->m : nullptr,
                         adam ? &adam->v : nullptr, report);
  if (!r && adam) {
    adam->n = cloud->n;
    adam->n_pad = cloud->n_pad;
  }
  gs.release();
  gc.release();
  return r;
}

}  // extern "C"

// ------------------------------------------------------------ NCCL (dlopen)
namespace gsb {

struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

// libnccl.so.2 is resolved at run time: the library (and every non-DP path)
// loads without it; a process that already loaded NCCL (e.g. torch's) shares it.
static NcclApi& nccl() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
  api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
  api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.group_start && api.group_end &&
           api.comm_destroy && api.error_string;
  return api;
}

static int nccl_fail(ncclResult_t r, const char* what) {
  return fail(GSB_ERR_CUDA + 4, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "nccl"));
}

}  // namespace gsb

struct gsb_comm {
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  gsb_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int32_t rank = 0, world = 1;
};

extern "C" {

int gsb_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) return fail(GSB_ERR_INVALID_ARGUMENT, "null id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!nccl().ok) return fail(GSB_ERR_NO_DEVICE, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  if (ncclResult_t r = nccl().get_unique_id(&id)) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof id);
  return GSB_OK;
}

int gsb_comm_create(gsb_ctx* ctx, const uint8_t id[128], int32_t rank, int32_t world, gsb_comm** out) {
  if (int r = ensure_device(ctx)) return r;
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return fail(GSB_ERR_INVALID_ARGUMENT, "bad comm args");
  if (!nccl().ok) return fail(GSB_ERR_NO_DEVICE, "libnccl.so.2 not loadable");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  gsb_comm* c = new gsb_comm();
  c->ctx = ctx;
  c->rank = rank;
  c->world = world;
  if (ncclResult_t r = nccl().comm_init_rank(&c->comm, world, uid, rank)) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  ctx_retain(ctx);
  c->ctx_ref = true;
  *out = c;
  return GSB_OK;
}

int gsb_comm_destroy(gsb_comm* c) {
  if (!c) return GSB_OK;
  cudaSetDevice(c->ctx->device);
  cudaStreamSynchronize(c->ctx->stream);
  if (c->comm) nccl().comm_destroy(c->comm);
  gsb_ctx* owner = c->ctx_ref ? c->ctx : nullptr;
  delete c;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_comm_allreduce_f32(gsb_comm* c, float* dev_buf, int64_t n) {
  if (!c) return fail(GSB_ERR_INVALID_ARGUMENT, "null comm");
  if (int r = ensure_device(c->ctx)) return r;
  if (n <= 0) return GSB_OK;
  if (ncclResult_t r = nccl().all_reduce(dev_buf, dev_buf, (size_t)n, ncclFloat32, ncclSum, c->comm, c->ctx->stream))
    return nccl_fail(r, "ncclAllReduce");
  GSB_CUDA(cudaStreamSynchronize(c->ctx->stream));
  return GSB_OK;
}

void gsb_default_joint_config(gsb_joint_config* c) {  // trainer.hpp:21-60, losses.hpp:15-19
  c->iterations = 30000;
  c->cam_lr_start = 1e-2;
  c->cam_lr_end = 1e-4;
  c->pos_lr_start = 1.6e-2;
  c->pos_lr_end = 1.6e-4;
  c->rot_lr = 1e-3;
  c->scale_lr = 5e-3;
  c->opacity_lr = 5e-2;
  c->sh_dc_lr = 2.5e-3;
  c->sh_rest_lr = 2.5e-3 / 20.0;
  c->opacity_l1_steps = 10000;
  c->sh_degree = 3;
  c->sh_degree_interval = 1000;
  c->optimize_poses = 1;
  c->beta = 0.2;
  c->aniso_ratio = 10.0;
  c->opacity_l1_weight = 0.01;
  c->background[0] = c->background[1] = c->background[2] = 0.0;
  gsb_default_raster_config(&c->raster);
  c->densify_interval = 100;
  c->densify_start = 500;
  c->densify_stop = 15000;
  c->n_target = 256000;
  c->grad_threshold = 2e-4;
  c->densify_size_ratio = 0.01;
  c->prune_opacity = 0.005;
}

}  // extern "C"

// ------------------------------------------------------------- joint loop
// joint_optimize (pipelines.cpp:96-216, densification off) on the device:
// one CUDA graph per step covers the rank's `local` slots (camera + target
// selection, render, loss, full backward), the slot sum, the NCCL
// all-reduce of the gradient planes and of the FP64 exchange slots (d_pose,
// losses, overflow flags), the Adam step with the regularisers and the pose
// steps. Every rank sees identical reduced bytes, so replicas stay bitwise
// in sync without broadcasting parameters.
struct gsb_joint {
  gsb_ctx* ctx = nullptr;
  bool ctx_ref = false;  // holds a reference on ctx (public create)
  gsb_cloud* cloud = nullptr;
  gsb_comm* comm = nullptr;
  gsb_joint_config cfg{};
  JointCtl ctl{};
  int32_t n_views = 0, local = 1, world = 1, rank = 0;
  gsb_camera cam{};  // intrinsics + size (pose per view lives on the device)
  std::vector<gsb_frame*> frames;
  DevBuf grads, adam_m, adam_v, state, seq, poses, cams, tptrs, tbuf, xchg, red, trace_total, trace_l1;
  int64_t glen = 0;  // floats per gradient copy ((planes + 2) * n_pad)
  void* host_state = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t graph_launches = 0;
  std::vector<uint64_t> graph_gen;
  std::vector<int64_t> graph_kcap;
  int graph_active = -1;
  int64_t t = 0;  // steps completed as of the last sync
  int64_t sh_grown_t = -1;  // step at which the active SH degree last grew
  // training-view sequence, produced lazily so its shuffles interleave with
  // densify_and_prune's draws from the same Rng (pipelines.cpp:123-129, 182-186)
  uint64_t rng_state = 0;
  std::vector<int32_t> order;
  int64_t seq_next = 0;
  // GradAccum (trainer.cpp:134-142) on the device + densification bookkeeping
  DevBuf acc_sum, acc_cnt, acc_stage;  // acc_stage: per local slot, [local][n_pad] staged increments
  const void* graph_params = nullptr;
  int64_t graph_n = -1;
  int32_t densify_report[3] = {0, 0, 0};
  int32_t densify_events = 0;
};

namespace gsb {

static bool joint_densify_due(const gsb_joint* j, int64_t t) {  // after step t (pipelines.cpp:182-183)
  const gsb_joint_config& c = j->cfg;
  return c.densify_interval > 0 && t >= c.densify_start && t <= c.densify_stop && t > 0 &&
         (t - c.densify_start) % c.densify_interval == 0;
}

// Extends the device view sequence to `upto` slots (epoch shuffles drawn now,
// i.e. before any later densify draws, as in the reference loop).
static int joint_sched_extend(gsb_ctx* ctx, gsb_joint* j, int64_t upto) {
  const int64_t cap = (int64_t)std::max(j->cfg.iterations, 1) * j->ctl.slots;
  upto = std::min(upto, cap);
  if (upto <= j->seq_next) return GSB_OK;
  std::vector<int32_t> add;
  add.reserve((size_t)(upto - j->seq_next));
  for (int64_t k = j->seq_next; k < upto; ++k) {
    if (k % j->n_views == 0)
      if (int r = gsb_rng_shuffle(&j->rng_state, j->n_views, j->order.data())) return r;
    add.push_back(j->order[k % j->n_views]);
  }
  GSB_CUDA(cudaMemcpyAsync(j->seq.as<int32_t>() + j->seq_next, add.data(), sizeof(int32_t) * add.size(),
                           cudaMemcpyHostToDevice, ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));  // host staging vector
  j->seq_next = upto;
  return GSB_OK;
}

static bool joint_accumulates(const gsb_joint* j) { return j->cfg.densify_interval > 0; }

// Per-Gaussian buffers sized by the cloud (after creation and after every
// densify_and_prune): gradient copies, reduction blocks, GradAccum.
static int joint_size_buffers(gsb_ctx* ctx, gsb_joint* j) {
  const int64_t n = std::max<int64_t>(j->cloud->n, 1);
  const int np = num_planes(j->cloud->sh_degree);
  j->glen = (int64_t)(np + 2) * j->cloud->n_pad;
  GSB_CUDA(j->grads.reserve(sizeof(float) * j->glen * j->local));
  GSB_CUDA(j->red.reserve(sizeof(double) * joint_red_doubles(n)));
  GSB_CUDA(cudaMemsetAsync(j->grads.p, 0, sizeof(float) * j->glen * j->local, ctx->stream));
  if (joint_accumulates(j)) {
    GSB_CUDA(j->acc_sum.reserve(sizeof(double) * n));
    GSB_CUDA(j->acc_cnt.reserve(sizeof(int32_t) * n));
    GSB_CUDA(j->acc_stage.reserve(sizeof(double) * j->cloud->n_pad * j->local));
    GSB_CUDA(cudaMemsetAsync(j->acc_sum.p, 0, sizeof(double) * n, ctx->stream));
    GSB_CUDA(cudaMemsetAsync(j->acc_cnt.p, 0, sizeof(int32_t) * n, ctx->stream));
  }
  return GSB_OK;
}

static int joint_launch_step(gsb_ctx* ctx, gsb_joint* j) {
  cudaStream_t st = ctx->stream;
  const RasterDev rc = make_rasterdev(&j->cfg.raster);
  const int64_t P = (int64_t)j->cam.width * j->cam.height;
  const size_t xbytes = sizeof(double) * joint_xchg_doubles() * (size_t)j->ctl.slots;
  GSB_CUDA(cudaMemsetAsync(j->xchg.p, 0, xbytes, st));
  for (int b = 0; b < j->local; ++b) {
    gsb_frame* f = j->frames[b];
    float* tb = j->tbuf.as<float>() + (size_t)b * 3 * P;
    float* gb = j->grads.as<float>() + (size_t)b * j->glen;
    if (int r = launch_joint_slot_begin(st, j->state.p, j->seq.as<int32_t>(), j->ctl, b, j->cams.as<CamDev>(),
                                        f->cam.as<CamDev>(), j->tptrs.as<const float*>(), tb, 3 * P))
      return r;
    if (int r = render_async(ctx, j->cloud, f, rc)) return r;
    if (int r = loss_device(ctx, f, tb, j->cfg.beta, true)) return r;
    if (int r = backward_device(ctx, j->cloud, f, true, gb)) return r;
    if (joint_accumulates(j)) {  // GradAccum::add for this view (trainer.cpp:134-142), staged
      if (int r = launch_grad_norm(st, gb, num_planes(j->cloud->sh_degree), j->cloud->n_pad, j->cloud->n,
                                   f->cnt_g.as<uint32_t>(), 0.5 * std::max(j->cam.width, j->cam.height),
                                   j->acc_stage.as<double>() + (size_t)b * j->cloud->n_pad))
        return r;
      ctx->launches += 1;
    }
    if (int r = launch_joint_slot_end(st, j->ctl, b, f->d_pose.as<double>(), f->loss_val.as<double>(),
                                      f->counters.as<uint32_t>(), f->k_cap, j->xchg.as<double>()))
      return r;
    ctx->launches += 2;
  }
  if (j->local > 1) {
    if (int r = launch_joint_sum(st, j->grads.as<float>(), j->grads.as<float>() + j->glen, j->glen, j->local - 1,
                                 j->glen))
      return r;
    ctx->launches += 1;
  }
  if (j->comm && j->world > 1) {  // gradient planes (FP32) and exchange slots (FP64), one NCCL group
    NcclApi& nc = nccl();
    if (ncclResult_t r = nc.group_start()) return nccl_fail(r, "ncclGroupStart");
    ncclResult_t r1 = nc.all_reduce(j->grads.p, j->grads.p, (size_t)j->glen, ncclFloat32, ncclSum, j->comm->comm, st);
    ncclResult_t r2 = nc.all_reduce(j->xchg.p, j->xchg.p, joint_xchg_doubles() * (size_t)j->ctl.slots, ncclFloat64,
                                    ncclSum, j->comm->comm, st);
    ncclResult_t r3 = nc.group_end();
    if (r1 || r2 || r3) return nccl_fail(r1 ? r1 : (r2 ? r2 : r3), "ncclAllReduce (joint)");
  }
  if (joint_accumulates(j)) {  // commit the staged GradAccum rows unless the step is discarded
    if (int r = launch_grad_accum_commit(st, j->acc_stage.as<double>(), j->local, j->cloud->n_pad, j->cloud->n,
                                         j->state.p, j->ctl, j->xchg.as<double>(), j->acc_sum.as<double>(),
                                         j->acc_cnt.as<int32_t>()))
      return r;
    ctx->launches += 1;
  }
  const int64_t nb = joint_adam_blocks(j->cloud->n);
  if (int r = launch_joint_adam(st, j->cloud->params.as<float>(), j->grads.as<float>(), j->adam_m.as<float>(),
                                j->adam_v.as<float>(), j->cloud->n, j->cloud->n_pad, j->state.p, j->ctl,
                                j->xchg.as<double>(), j->red.as<double>()))
    return r;
  if (int r = launch_joint_finalize(st, j->state.p, j->seq.as<int32_t>(), j->ctl, j->xchg.as<double>(),
                                    j->red.as<double>(), nb, j->poses.p, j->cams.as<CamDev>(),
                                    j->trace_total.as<double>(), j->trace_l1.as<double>()))
    return r;
  ctx->launches += 3;  // joint_adam, joint_adam_sh, joint_finalize
  return GSB_OK;
}

static int joint_frames_ready(gsb_ctx* ctx, gsb_joint* j) {
  for (gsb_frame* f : j->frames) {
    f->lean = true;
    if (int r = frame_setup(ctx, f, j->cloud, &j->cam, j->cfg.background, &j->cfg.raster, false)) return r;
    // after densify_and_prune grows the cloud the capacity follows it
    const int64_t want = std::max(f->k_cap, initial_k_cap(j->cloud->n));
    if (int r = frame_reserve(f, j->cloud, want)) return r;
  }
  return GSB_OK;
}

static int joint_prepare(gsb_ctx* ctx, gsb_joint* j) {
  if (int r = joint_frames_ready(ctx, j)) return r;
  bool stale = !j->exec || j->graph_active != j->cloud->active_sh_degree || j->graph_params != j->cloud->params.p ||
               j->graph_n != j->cloud->n;
  for (size_t b = 0; b < j->frames.size() && !stale; ++b)
    stale = j->frames[b]->gen != j->graph_gen[b] || j->frames[b]->k_cap != j->graph_kcap[b];
  if (!stale) return GSB_OK;
  if (j->exec) cudaGraphExecDestroy(j->exec);
  j->exec = nullptr;
  const bool profiling = ctx->profiling;
  ctx->profiling = false;
  const int64_t launches0 = ctx->launches;
  GSB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int r = joint_launch_step(ctx, j);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  ctx->profiling = profiling;
  if (r || e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    ctx->launches = launches0;
    return r ? r : cuda_fail(e, "joint capture");
  }
  e = cudaGraphInstantiate(&j->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate (joint)");
  j->graph_launches = ctx->launches - launches0;
  ctx->launches = launches0;
  for (size_t b = 0; b < j->frames.size(); ++b) {
    j->graph_gen[b] = j->frames[b]->gen;
    j->graph_kcap[b] = j->frames[b]->k_cap;
  }
  j->graph_active = j->cloud->active_sh_degree;
  j->graph_params = j->cloud->params.p;
  j->graph_n = j->cloud->n;
  if (debug_on()) std::fprintf(stderr, "[gsb] joint graph captured: %lld kernels\n", (long long)j->graph_launches);
  return GSB_OK;
}

// Launches `k` replays, waits, re-runs steps discarded for entry-capacity
// growth (every rank sees the same discard count through the exchange slots).
static int joint_run(gsb_ctx* ctx, gsb_joint* j, int64_t k) {
  const size_t sb = joint_state_bytes();
  for (int round = 0; round < 8 && k > 0; ++round) {
    if (int r = joint_prepare(ctx, j)) return r;
    for (int64_t i = 0; i < k; ++i) GSB_CUDA(cudaGraphLaunch(j->exec, ctx->stream));
    ctx->launches += j->graph_launches * k;
    ++j->cloud->version;
    GSB_CUDA(cudaMemcpyAsync(j->host_state, j->state.p, sb, cudaMemcpyDeviceToHost, ctx->stream));
    GSB_CUDA(cudaStreamSynchronize(ctx->stream));
    int64_t t = 0;
    int32_t div = 0, aborted = 0, tile = 0;
    double kmax = 0.0;
    joint_state_read(j->host_state, &t, &div, &aborted, &kmax, &tile);
    j->t = t;
    if (div) return fail(GSB_ERR_DIVERGED, "joint_optimize: non-finite loss at step " + std::to_string(div - 1));
    if (aborted == 0) return GSB_OK;
    if (debug_on()) std::fprintf(stderr, "[gsb] joint: %d step(s) discarded (K %.0f, tile overflow %d)\n", aborted, kmax, tile);
    joint_state_clear_abort(j->host_state);
    GSB_CUDA(cudaMemcpyAsync(j->state.p, j->host_state, sb, cudaMemcpyHostToDevice, ctx->stream));
    for (gsb_frame* f : j->frames) {
      if (tile) fall_back_to_global(f);
      if (int r = frame_reserve(f, j->cloud, std::max<int64_t>(f->k_cap, (int64_t)kmax + (int64_t)kmax / 4 + 4096)))
        return r;
    }
    k = aborted;
  }
  return k > 0 ? fail(GSB_ERR_OUT_OF_MEMORY, "joint: entry capacity did not converge") : GSB_OK;
}

}  // namespace gsb

extern "C" {

int gsb_joint_create(gsb_ctx* ctx, gsb_cloud* cloud, gsb_image* const* targets, int32_t n_views,
                     const double intr[4], const double* init_poses, const gsb_joint_config* cfg, uint64_t seed,
                     int32_t local_views, gsb_comm* comm, gsb_joint** out) {
  if (int r = ensure_device(ctx)) return r;
  if (!cloud || !targets || !intr || !init_poses || !cfg || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  if (n_views < 2) return fail(GSB_ERR_INVALID_CONFIG, "joint_optimize: need >= 2 images");  // pipelines.cpp:101
  if (local_views < 1 || cfg->iterations < 0) return fail(GSB_ERR_INVALID_CONFIG, "bad joint config");
  if (int r = validate_config(&cfg->raster)) return r;
  if (comm && comm->ctx != ctx) return fail(GSB_ERR_INVALID_ARGUMENT, "comm / context mismatch");
  const int W = targets[0]->width, H = targets[0]->height;
  for (int32_t v = 0; v < n_views; ++v)
    if (!targets[v] || targets[v]->width != W || targets[v]->height != H)
      return fail(GSB_ERR_DIMENSION_MISMATCH, "joint_optimize: target sizes differ");
  gsb_joint* j = new gsb_joint();
  j->ctx = ctx;
  j->cloud = cloud;
  j->comm = comm;
  j->cfg = *cfg;
  j->n_views = n_views;
  j->local = local_views;
  j->world = comm ? comm->world : 1;
  j->rank = comm ? comm->rank : 0;
  j->cam.fx = intr[0];
  j->cam.fy = intr[1];
  j->cam.cx = intr[2];
  j->cam.cy = intr[3];
  j->cam.width = W;
  j->cam.height = H;
  for (int k = 0; k < 9; ++k) j->cam.R[k] = (k % 4 == 0) ? 1.0 : 0.0;
  const int slots = j->local * j->world;
  const int np = num_planes(cloud->sh_degree);
  JointCtl& c = j->ctl;
  c.iterations = cfg->iterations;
  c.slots = slots;
  c.slot0 = j->rank * j->local;
  c.local = j->local;
  c.n_views = n_views;
  c.opacity_l1_steps = cfg->opacity_l1_steps;
  c.optimize_poses = cfg->optimize_poses;
  c.nplanes = np;
  c.basis = (cloud->sh_degree + 1) * (cloud->sh_degree + 1);
  c.pos_lr_start = cfg->pos_lr_start;
  c.pos_lr_end = cfg->pos_lr_end;
  c.rot_lr = cfg->rot_lr;
  c.scale_lr = cfg->scale_lr;
  c.opacity_lr = cfg->opacity_lr;
  c.sh_dc_lr = cfg->sh_dc_lr;
  c.sh_rest_lr = cfg->sh_rest_lr;
  c.cam_lr_start = cfg->cam_lr_start;
  c.cam_lr_end = cfg->cam_lr_end;
  c.aniso_ratio = cfg->aniso_ratio;
  c.opacity_l1_weight = cfg->opacity_l1_weight;
  c.inv_slots = 1.0 / (double)slots;
  j->glen = (int64_t)(np + 2) * cloud->n_pad;
  const int64_t P = (int64_t)W * H;
  const int64_t iters = std::max(cfg->iterations, 1);
  const int64_t nb = joint_adam_blocks(std::max<int64_t>(cloud->n, 1));
  const size_t sb = joint_state_bytes();
  cudaError_t e = j->adam_m.reserve(sizeof(float) * np * cloud->n_pad);
  if (e == cudaSuccess) e = j->adam_v.reserve(sizeof(float) * np * cloud->n_pad);
  if (e == cudaSuccess) e = j->state.reserve(sb);
  if (e == cudaSuccess) e = j->seq.reserve(sizeof(int32_t) * iters * slots);
  if (e == cudaSuccess) e = j->poses.reserve(pose_state_bytes() * n_views);
  if (e == cudaSuccess) e = j->cams.reserve(sizeof(CamDev) * n_views);
  if (e == cudaSuccess) e = j->tptrs.reserve(sizeof(float*) * n_views);
  if (e == cudaSuccess) e = j->tbuf.reserve(sizeof(float) * 3 * P * j->local);
  if (e == cudaSuccess) e = j->xchg.reserve(sizeof(double) * joint_xchg_doubles() * slots);
  if (e == cudaSuccess) e = j->trace_total.reserve(sizeof(double) * iters);
  if (e == cudaSuccess) e = j->trace_l1.reserve(sizeof(double) * iters);
  if (e == cudaSuccess) e = cudaMallocHost(&j->host_state, std::max<size_t>(sb, 64));
  if (e != cudaSuccess) {
    gsb_joint_destroy(j);
    return cuda_fail(e, "joint alloc");
  }
  (void)nb;
  if (int r = joint_size_buffers(ctx, j)) {
    gsb_joint_destroy(j);
    return r;
  }
  // host-side initial state: the Rng of the view sequence (extended lazily),
  // per-view PoseState + CamDev, target pointers
  j->rng_state = seed ? seed : 0x9e3779b97f4a7c15ull;
  j->order.resize(n_views);
  for (int32_t v = 0; v < n_views; ++v) j->order[v] = v;
  std::vector<char> ps(pose_state_bytes() * n_views);
  std::vector<CamDev> cams(n_views);
  std::vector<const float*> tp(n_views);
  for (int32_t v = 0; v < n_views; ++v) {
    pose_state_init(ps.data() + pose_state_bytes() * v, init_poses + 12 * (size_t)v);
    gsb_camera cv = j->cam;
    for (int r = 0; r < 3; ++r) {
      for (int k = 0; k < 3; ++k) cv.R[r * 3 + k] = init_poses[12 * (size_t)v + r * 4 + k];
      cv.t[r] = init_poses[12 * (size_t)v + r * 4 + 3];
    }
    cams[v] = make_camdev(&cv, kTile);
    tp[v] = targets[v]->planes.as<float>();
  }
  std::memset(j->host_state, 0, sb);
  cudaStream_t st = ctx->stream;
  GSB_CUDA(cudaMemcpyAsync(j->poses.p, ps.data(), ps.size(), cudaMemcpyHostToDevice, st));
  GSB_CUDA(cudaMemcpyAsync(j->cams.p, cams.data(), sizeof(CamDev) * n_views, cudaMemcpyHostToDevice, st));
  GSB_CUDA(cudaMemcpyAsync(j->tptrs.p, tp.data(), sizeof(float*) * n_views, cudaMemcpyHostToDevice, st));
  GSB_CUDA(cudaMemcpyAsync(j->state.p, j->host_state, sb, cudaMemcpyHostToDevice, st));
  GSB_CUDA(cudaMemsetAsync(j->adam_m.p, 0, sizeof(float) * np * cloud->n_pad, st));
  GSB_CUDA(cudaMemsetAsync(j->adam_v.p, 0, sizeof(float) * np * cloud->n_pad, st));
  GSB_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < j->local; ++b) {
    gsb_frame* f = new gsb_frame();
    f->ctx = ctx;
    j->frames.push_back(f);
  }
  j->graph_gen.assign(j->local, 0);
  j->graph_kcap.assign(j->local, 0);
  ctx_retain(ctx);
  j->ctx_ref = true;
  *out = j;
  return GSB_OK;
}

int gsb_joint_destroy(gsb_joint* j) {
  if (!j) return GSB_OK;
  cudaSetDevice(j->ctx->device);
  cudaStreamSynchronize(j->ctx->stream);
  if (j->exec) cudaGraphExecDestroy(j->exec);
  for (gsb_frame* f : j->frames) gsb_frame_destroy(f);
  DevBuf* bufs[] = {&j->grads, &j->adam_m, &j->adam_v, &j->state, &j->seq, &j->poses, &j->cams, &j->tptrs,
                    &j->tbuf, &j->xchg, &j->red, &j->trace_total, &j->trace_l1, &j->acc_sum, &j->acc_cnt,
                    &j->acc_stage};
  for (DevBuf* b : bufs) b->release();
  if (j->host_state) cudaFreeHost(j->host_state);
  gsb_ctx* owner = j->ctx_ref ? j->ctx : nullptr;
  delete j;
  if (owner) ctx_release(owner);
  return GSB_OK;
}

int gsb_joint_step(gsb_ctx* ctx, gsb_joint* j, int32_t steps) {
  GSB_NVTX("gsb_joint_step");
  if (int r = ensure_device(ctx)) return r;
  if (!j || j->ctx != ctx) return fail(GSB_ERR_INVALID_ARGUMENT, "joint / context mismatch");
  int64_t left = std::min<int64_t>(steps, (int64_t)j->cfg.iterations - j->t);
  const int interval = j->cfg.sh_degree_interval;
  while (left > 0) {
    // SH degree growth at the start of step t (pipelines.cpp:130-133): chunks end on growth steps
    if (interval > 0 && j->t > 0 && j->t % interval == 0 && j->sh_grown_t != j->t) {
      j->cloud->active_sh_degree = std::min(j->cloud->active_sh_degree + 1, j->cfg.sh_degree);
      j->sh_grown_t = j->t;
    }
    int64_t chunk = std::min<int64_t>(left, 16);
    if (interval > 0) chunk = std::min<int64_t>(chunk, interval - (j->t % interval));
    for (int64_t k = 0; k < chunk; ++k)  // densification after step t ends the chunk
      if (joint_densify_due(j, j->t + k)) {
        chunk = k + 1;
        break;
      }
    if (int r = joint_sched_extend(ctx, j, (j->t + chunk) * j->ctl.slots)) return r;
    const int64_t t0 = j->t;
    if (int r = joint_run(ctx, j, chunk)) return r;
    left -= j->t - t0;
    if (j->t == t0) return fail(GSB_ERR_CUDA, "joint: no progress");
    if (j->t - t0 == chunk && joint_densify_due(j, j->t - 1)) {
      // densify_and_prune (pipelines.cpp:182-186): GradAccum summed over ranks,
      // then the identical rebuild on every replica (same Rng)
      if (j->comm && j->world > 1) {
        NcclApi& nc = nccl();
        if (ncclResult_t r = nc.group_start()) return nccl_fail(r, "ncclGroupStart");
        ncclResult_t r1 = nc.all_reduce(j->acc_sum.p, j->acc_sum.p, (size_t)j->cloud->n, ncclFloat64, ncclSum,
                                        j->comm->comm, ctx->stream);
        ncclResult_t r2 = nc.all_reduce(j->acc_cnt.p, j->acc_cnt.p, (size_t)j->cloud->n, ncclInt32, ncclSum,
                                        j->comm->comm, ctx->stream);
        ncclResult_t r3 = nc.group_end();
        if (r1 || r2 || r3) return nccl_fail(r1 ? r1 : (r2 ? r2 : r3), "ncclAllReduce (GradAccum)");
      }
      DensifyParams dp{j->cfg.grad_threshold, j->cfg.densify_size_ratio, j->cfg.prune_opacity, j->cfg.n_target};
      if (int r = densify_device(ctx, j->cloud, j->acc_sum.as<double>(), j->acc_cnt.as<int32_t>(), dp, &j->rng_state,
                                 &j->adam_m, &j->adam_v, j->densify_report))
        return r;
      ++j->densify_events;
      if (int r = joint_size_buffers(ctx, j)) return r;
      if (debug_on())
        std::fprintf(stderr, "[gsb] joint densify after step %lld: cloned %d split %d pruned %d -> n %lld\n",
                     (long long)(j->t - 1), j->densify_report[0], j->densify_report[1], j->densify_report[2],
                     (long long)j->cloud->n);
    }
  }
  return GSB_OK;
}

int gsb_joint_rng_state(const gsb_joint* j, uint64_t* rng_state) {
  if (!j || !rng_state) return fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  *rng_state = j->rng_state;
  return GSB_OK;
}

int gsb_joint_info(gsb_joint* j, int64_t* n_gaussians, int32_t* densify_events, int32_t last_report[3]) {
  if (!j) return fail(GSB_ERR_INVALID_ARGUMENT, "null joint");
  if (n_gaussians) *n_gaussians = j->cloud->n;
  if (densify_events) *densify_events = j->densify_events;
  if (last_report)
    for (int k = 0; k < 3; ++k) last_report[k] = j->densify_report[k];
  return GSB_OK;
}

int gsb_joint_read(gsb_joint* j, double* poses_out, int64_t* steps_done, double* trace_total, double* trace_l1) {
  if (!j) return fail(GSB_ERR_INVALID_ARGUMENT, "null joint");
  gsb_ctx* ctx = j->ctx;
  if (int r = ensure_device(ctx)) return r;
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (steps_done) *steps_done = j->t;
  if (poses_out) {
    std::vector<char> ps(pose_state_bytes() * j->n_views);
    GSB_CUDA(cudaMemcpy(ps.data(), j->poses.p, ps.size(), cudaMemcpyDeviceToHost));
    for (int32_t v = 0; v < j->n_views; ++v)
      pose_state_read(ps.data() + pose_state_bytes() * v, nullptr, poses_out + 12 * (size_t)v, nullptr, nullptr,
                      nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  }
  const size_t nt = (size_t)std::max<int64_t>(j->t, 0);
  if (trace_total && nt) GSB_CUDA(cudaMemcpy(trace_total, j->trace_total.p, sizeof(double) * nt, cudaMemcpyDeviceToHost));
  if (trace_l1 && nt) GSB_CUDA(cudaMemcpy(trace_l1, j->trace_l1.p, sizeof(double) * nt, cudaMemcpyDeviceToHost));
  return GSB_OK;
}

}  // extern "C"
