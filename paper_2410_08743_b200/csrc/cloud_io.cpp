// cloud_io.cpp — the 3DGS PLY cloud format (reference: proj/src/ply.cpp,
// save_cloud_ply 29-60 / load_cloud_ply 62-148) straight to and from the
// device's plane-major FP32 layout: rows are transposed into parameter
// planes on the host and moved with one copy, no FP64 intermediate.
//
// Format: binary_little_endian 1.0, one `vertex` element of float properties
// x y z rot_0..3 scale_0..2 opacity f_dc_0..2 f_rest_0..44 (saved zero-padded
// to SH degree 3, so a saved cloud always reloads as degree 3 — the
// reference's behaviour, tests/test_io.cpp:54). f_rest is channel-major
// (channel c, band b >= 1 at c * (B - 1) + b - 1). Errors map to
// GSB_ERR_CORRUPT_FILE like the reference's ErrorCode::corrupt_file.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "gsb_internal.cuh"

namespace {

int sh_basis_of(int degree) { return (degree + 1) * (degree + 1); }

std::vector<std::string> ply_columns() {
  std::vector<std::string> c = {"x",       "y",       "z",       "rot_0",   "rot_1",  "rot_2",  "rot_3",
                                "scale_0", "scale_1", "scale_2", "opacity", "f_dc_0", "f_dc_1", "f_dc_2"};
  for (int k = 0; k < 45; ++k) c.push_back("f_rest_" + std::to_string(k));
  return c;
}

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

}  // namespace

extern "C" {

int gsb_cloud_load_ply(gsb_ctx* ctx, const char* path, gsb_cloud** out) {
  if (!ctx || !path || !out) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  std::ifstream in(path, std::ios::binary);
  if (!in) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("load_ply: cannot open ") + path);
  std::string line;
  if (!std::getline(in, line) || line != "ply") return gsb::fail(GSB_ERR_CORRUPT_FILE, "load_ply: not a PLY file");
  if (!std::getline(in, line) || line != "format binary_little_endian 1.0")
    return gsb::fail(GSB_ERR_CORRUPT_FILE, "load_ply: unsupported format");
  int64_t n = -1;
  std::vector<std::string> cols;
  bool ended = false;
  while (std::getline(in, line)) {
    std::istringstream ls(line);
    std::string w;
    ls >> w;
    if (w == "end_header") {
      ended = true;
      break;
    }
    if (w == "comment") continue;
    if (w == "element") {
      std::string kind;
      ls >> kind >> n;
      if (kind != "vertex") return gsb::fail(GSB_ERR_CORRUPT_FILE, "load_ply: unsupported element " + kind);
    } else if (w == "property") {
      std::string type, name;
      ls >> type >> name;
      if (type != "float") return gsb::fail(GSB_ERR_CORRUPT_FILE, "load_ply: non-float property " + name);
      cols.push_back(name);
    }
  }
  if (!ended || n < 0) return gsb::fail(GSB_ERR_CORRUPT_FILE, "load_ply: missing header / vertex count");
  std::map<std::string, int> at;
  for (size_t i = 0; i < cols.size(); ++i) at[cols[i]] = (int)i;
  int n_rest = 0;
  while (at.count("f_rest_" + std::to_string(n_rest))) ++n_rest;
  int degree = -1;
  for (int d = 0; d <= 3; ++d)
    if (n_rest % 3 == 0 && sh_basis_of(d) == n_rest / 3 + 1) degree = d;
  if (degree < 0) return gsb::fail(GSB_ERR_CORRUPT_FILE, "load_ply: f_rest count is not a full SH band");
  const int B = sh_basis_of(degree);
  // source column of every device plane (kMeanX.. kOpacity, then SH c * B + b)
  const int NP = gsb::num_planes(degree);
  std::vector<int> src(NP, -1);
  const char* fixed[gsb::kShBase] = {"x",       "y",       "z",       "rot_0",   "rot_1",  "rot_2",
                                     "rot_3",   "scale_0", "scale_1", "scale_2", "opacity"};
  for (int p = 0; p < gsb::kShBase; ++p) {
    auto it = at.find(fixed[p]);
    if (it == at.end()) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("load_ply: missing property ") + fixed[p]);
    src[p] = it->second;
  }
  for (int c = 0; c < 3; ++c) {
    auto it = at.find("f_dc_" + std::to_string(c));
    if (it == at.end()) return gsb::fail(GSB_ERR_CORRUPT_FILE, "load_ply: missing f_dc");
    src[gsb::kShBase + c * B] = it->second;
    for (int b = 1; b < B; ++b) src[gsb::kShBase + c * B + b] = at["f_rest_" + std::to_string(c * (B - 1) + b - 1)];
  }
  gsb_cloud* cloud = nullptr;
  if (int r = gsb_cloud_create(ctx, n, degree, &cloud)) return r;
  const int64_t np = cloud->n_pad;
  std::vector<float> planes((size_t)NP * np, 0.f);
  const size_t ncol = cols.size();
  std::vector<float> rows;
  const int64_t chunk = 1 << 16;
  for (int64_t i0 = 0; i0 < n; i0 += chunk) {
    const int64_t m = std::min(chunk, n - i0);
    rows.resize((size_t)m * ncol);
    in.read(reinterpret_cast<char*>(rows.data()), (std::streamsize)(rows.size() * sizeof(float)));
    if (!in) {
      gsb_cloud_destroy(cloud);
      return gsb::fail(GSB_ERR_CORRUPT_FILE, "load_ply: truncated vertex data");
    }
    for (int p = 0; p < NP; ++p) {
      float* dst = planes.data() + (size_t)p * np + i0;
      const int s = src[p];
      for (int64_t i = 0; i < m; ++i) dst[i] = rows[(size_t)i * ncol + s];
    }
  }
  cudaSetDevice(ctx->device);
  GSB_CUDA(cudaMemcpyAsync(cloud->params.p, planes.data(), sizeof(float) * planes.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  cloud->active_sh_degree = degree;
  uint64_t h = 0xcbf29ce484222325ull;  // identity of the loaded content (64 strided rows)
  const int64_t stride = std::max<int64_t>(1, n / 64);
  for (int64_t i = 0; i < n; i += stride)
    for (int p = 0; p < NP; ++p) h = fnv(h, &planes[(size_t)p * np + i], sizeof(float));
  cloud->host_fingerprint = h;
  cloud->version += 1;
  *out = cloud;
  return GSB_OK;
}

int gsb_cloud_save_ply(gsb_cloud* cloud, const char* path) {
  if (!cloud || !path) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  gsb_ctx* ctx = cloud->ctx;
  const int64_t n = cloud->n, np = cloud->n_pad;
  const int B = sh_basis_of(cloud->sh_degree);
  const int NP = gsb::num_planes(cloud->sh_degree);
  std::vector<float> planes((size_t)NP * np);
  cudaSetDevice(ctx->device);
  GSB_CUDA(cudaStreamSynchronize(ctx->stream));
  GSB_CUDA(cudaMemcpy(planes.data(), cloud->params.p, sizeof(float) * planes.size(), cudaMemcpyDeviceToHost));
  std::ofstream out(path, std::ios::binary);
  if (!out) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("save_ply: cannot open ") + path);
  const auto names = ply_columns();
  out << "ply\nformat binary_little_endian 1.0\nelement vertex " << n << "\n";
  for (const auto& c : names) out << "property float " << c << "\n";
  out << "end_header\n";
  // row layout: the 11 fixed columns, f_dc (band 0 per channel), then f_rest
  // channel-major with bands 1..15 (zero beyond the cloud's degree)
  std::vector<float> rows;
  const int64_t chunk = 1 << 16;
  const size_t W = names.size();
  for (int64_t i0 = 0; i0 < n; i0 += chunk) {
    const int64_t m = std::min(chunk, n - i0);
    rows.assign((size_t)m * W, 0.f);
    for (int64_t i = 0; i < m; ++i) {
      float* r = rows.data() + (size_t)i * W;
      for (int p = 0; p < gsb::kShBase; ++p) r[p] = planes[(size_t)p * np + i0 + i];
      for (int c = 0; c < 3; ++c) {
        r[gsb::kShBase + c] = planes[(size_t)(gsb::kShBase + c * B) * np + i0 + i];
        for (int b = 1; b < 16; ++b)
          r[gsb::kShBase + 3 + c * 15 + b - 1] = b < B ? planes[(size_t)(gsb::kShBase + c * B + b) * np + i0 + i] : 0.f;
      }
    }
    out.write(reinterpret_cast<const char*>(rows.data()), (std::streamsize)(rows.size() * sizeof(float)));
  }
  if (!out) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("save_ply: write failed for ") + path);
  return GSB_OK;
}

}  // extern "C"
