// scene_io.cpp — the reference's small on-disk formats around the hot path
// (SURVEY.md §8f row 3), host C++:
//   f32map depth / transmittance maps   image.cpp:105-141
//   pose lists  {"poses": [[12], ...]}  scene_io.cpp:64-79 (pose_to_json 38-50)
//   cameras.json intrinsics + frames    scene_io.cpp:254-279 (load_cameras_json)
// Poses are row-major 3x4 [R | t] world_to_cam (lie.hpp:59-61). JSON is read by
// a small recursive-descent parser (objects, arrays, numbers, strings,
// literals) and written with 17 significant digits, so pose lists round-trip
// losslessly (tests/test_io.cpp:71-84). PNG frames (load_scene's images/) need
// libpng, which is absent from this image: scene bundles are out of scope.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "gsb_internal.cuh"

namespace {

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const char* p;
  const char* end;
  std::string err;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool lit(const char* s) {
    const size_t n = std::strlen(s);
    if ((size_t)(end - p) < n || std::strncmp(p, s, n) != 0) return false;
    p += n;
    return true;
  }
  bool string(std::string* out) {
    if (p >= end || *p != '"') return false;
    ++p;
    while (p < end && *p != '"') {
      if (*p == '\\') {
        if (++p >= end) return false;
        switch (*p) {
          case 'n': out->push_back('\n'); break;
          case 't': out->push_back('\t'); break;
          case 'r': out->push_back('\r'); break;
          case 'b': out->push_back('\b'); break;
          case 'f': out->push_back('\f'); break;
          case 'u': {  // BMP code point as UTF-8
            if (end - p < 5) return false;
            const unsigned cp = (unsigned)std::strtoul(std::string(p + 1, p + 5).c_str(), nullptr, 16);
            if (cp < 0x80) {
              out->push_back((char)cp);
            } else if (cp < 0x800) {
              out->push_back((char)(0xC0 | (cp >> 6)));
              out->push_back((char)(0x80 | (cp & 0x3F)));
            } else {
              out->push_back((char)(0xE0 | (cp >> 12)));
              out->push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
              out->push_back((char)(0x80 | (cp & 0x3F)));
            }
            p += 4;
            break;
          }
          default: out->push_back(*p);
        }
        ++p;
      } else {
        out->push_back(*p++);
      }
    }
    if (p >= end) return false;
    ++p;
    return true;
  }
  bool value(Json* v, int depth) {
    if (depth > 64) return false;
    ws();
    if (p >= end) return false;
    if (*p == '{') {
      v->kind = Json::Obj;
      ++p;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return true;
      }
      for (;;) {
        ws();
        std::string k;
        if (!string(&k)) return false;
        ws();
        if (p >= end || *p != ':') return false;
        ++p;
        Json child;
        if (!value(&child, depth + 1)) return false;
        v->obj.emplace_back(std::move(k), std::move(child));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (*p == '[') {
      v->kind = Json::Arr;
      ++p;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return true;
      }
      for (;;) {
        Json child;
        if (!value(&child, depth + 1)) return false;
        v->arr.push_back(std::move(child));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (*p == '"') {
      v->kind = Json::Str;
      return string(&v->str);
    }
    if (lit("true")) {
      v->kind = Json::Bool;
      v->b = true;
      return true;
    }
    if (lit("false")) {
      v->kind = Json::Bool;
      return true;
    }
    if (lit("null")) return true;
    char* e = nullptr;
    const std::string tok(p, (size_t)std::min<ptrdiff_t>(end - p, 64));
    const double d = std::strtod(tok.c_str(), &e);
    if (e == tok.c_str()) return false;
    v->kind = Json::Num;
    v->num = d;
    p += e - tok.c_str();
    return true;
  }
};

int load_json(const char* path, Json* out) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("cannot open ") + path);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string s = ss.str();
  Parser ps{s.data(), s.data() + s.size(), {}};
  if (!ps.value(out, 0)) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("invalid JSON in ") + path);
  ps.ws();
  if (ps.p != ps.end) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("invalid JSON in ") + path);
  return GSB_OK;
}

// pose_from_json (scene_io.cpp:42-50): exactly 12 numbers
int pose_from_json(const Json& j, const char* path, double* out12) {
  if (j.kind != Json::Arr || j.arr.size() != 12)
    return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("pose must be 12 numbers in ") + path);
  for (int i = 0; i < 12; ++i) {
    if (j.arr[i].kind != Json::Num)
      return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("pose must be 12 numbers in ") + path);
    out12[i] = j.arr[i].num;
  }
  return GSB_OK;
}

void identity12(double* p) {
  static const double I[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
  std::memcpy(p, I, sizeof I);
}

std::string num17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

}  // namespace

extern "C" {

int gsb_load_float_map(const char* path, float* values, int64_t capacity, int32_t* width, int32_t* height) {
  if (!path || !width || !height) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  std::ifstream in(path, std::ios::binary);
  if (!in) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("load_float_map: cannot open ") + path);
  std::string header;
  std::getline(in, header);
  std::istringstream hs(header);
  std::string magic;
  long long w = 0, h = 0;
  double scale = 1.0;
  hs >> magic >> w >> h >> scale;
  if (magic != "f32map" || w <= 0 || h <= 0 || !hs)
    return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("load_float_map: bad header in ") + path);
  *width = (int32_t)w;
  *height = (int32_t)h;
  if (!values) return GSB_OK;  // size query
  if (capacity < w * h) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "load_float_map: buffer too small");
  in.read(reinterpret_cast<char*>(values), (std::streamsize)(w * h * (long long)sizeof(float)));
  if (!in) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("load_float_map: truncated data in ") + path);
  if (scale != 1.0)
    for (long long i = 0; i < w * h; ++i) values[i] = (float)(values[i] * scale);
  return GSB_OK;
}

int gsb_save_float_map(const float* values, int32_t width, int32_t height, const char* path, double scale) {
  if (!values || !path || width <= 0 || height <= 0) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "bad float map");
  std::ofstream out(path, std::ios::binary);
  if (!out) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("save_float_map: cannot open ") + path);
  out << "f32map " << width << " " << height << " " << scale << "\n";
  out.write(reinterpret_cast<const char*>(values), (std::streamsize)((size_t)width * height * sizeof(float)));
  if (!out) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("save_float_map: write failed for ") + path);
  return GSB_OK;
}

// f32map as a depth map the way load_scene reads depth/<stem>.f32
// (scene_io.cpp:203-215): FP64 values, valid = finite and > 0.
int gsb_load_depth_map(const char* path, double* depth, uint8_t* valid, int64_t capacity, int32_t* width,
                       int32_t* height) {
  if (int r = gsb_load_float_map(path, nullptr, 0, width, height)) return r;
  if (!depth && !valid) return GSB_OK;
  const int64_t n = (int64_t)*width * *height;
  if (capacity < n) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "load_depth_map: buffer too small");
  std::vector<float> v((size_t)n);
  if (int r = gsb_load_float_map(path, v.data(), n, width, height)) return r;
  for (int64_t k = 0; k < n; ++k) {
    if (depth) depth[k] = v[k];
    if (valid) valid[k] = (std::isfinite(v[k]) && v[k] > 0.0f) ? 1 : 0;
  }
  return GSB_OK;
}

int gsb_save_poses_json(const double* poses, int32_t n, const char* path) {
  if ((!poses && n > 0) || !path || n < 0) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "bad poses");
  std::ofstream out(path);
  if (!out) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("cannot open ") + path);
  out << "{\n  \"poses\": [";
  for (int32_t i = 0; i < n; ++i) {
    out << (i ? ",\n    [" : "\n    [");
    for (int k = 0; k < 12; ++k) out << (k ? ", " : "") << num17(poses[12 * i + k]);
    out << "]";
  }
  out << (n ? "\n  ]\n}\n" : "]\n}\n");
  if (!out) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("write failed for ") + path);
  return GSB_OK;
}

int gsb_load_poses_json(const char* path, double* poses, int32_t capacity, int32_t* n_out) {
  if (!path || !n_out) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  Json j;
  if (int r = load_json(path, &j)) return r;
  const Json* ps = j.kind == Json::Obj ? j.get("poses") : nullptr;
  if (!ps || ps->kind != Json::Arr) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("missing poses array in ") + path);
  *n_out = (int32_t)ps->arr.size();
  if (!poses) return GSB_OK;
  if (capacity < (int32_t)ps->arr.size()) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "load_poses_json: buffer too small");
  for (size_t i = 0; i < ps->arr.size(); ++i)
    if (int r = pose_from_json(ps->arr[i], path, poses + 12 * i)) return r;
  return GSB_OK;
}

// load_cameras_json (scene_io.cpp:254-279). intr = {fx, fy, cx, cy}, size =
// {width, height}; poses (n x 12, identity where a frame has none) and names
// ('\n'-separated, NUL-terminated) are optional; has_poses = every frame has one.
int gsb_load_cameras_json(const char* path, double intr[4], int32_t size[2], double* poses, int32_t capacity,
                          int32_t* n_frames, int32_t* has_poses, char* names, int64_t names_capacity) {
  if (!path || !intr || !size || !n_frames) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "null argument");
  Json j;
  if (int r = load_json(path, &j)) return r;
  const char* keys[7] = {"fx", "fy", "cx", "cy", "width", "height", "frames"};
  for (const char* k : keys)
    if (j.kind != Json::Obj || !j.get(k))
      return gsb::fail(GSB_ERR_MISSING_INTRINSICS,
                       std::string("cameras.json missing key '") + k + "' in " + path);
  for (int i = 0; i < 6; ++i)
    if (j.get(keys[i])->kind != Json::Num)
      return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("cameras.json: '") + keys[i] + "' is not a number");
  intr[0] = j.get("fx")->num;
  intr[1] = j.get("fy")->num;
  intr[2] = j.get("cx")->num;
  intr[3] = j.get("cy")->num;
  size[0] = (int32_t)j.get("width")->num;
  size[1] = (int32_t)j.get("height")->num;
  const Json* fr = j.get("frames");
  if (fr->kind != Json::Arr) return gsb::fail(GSB_ERR_CORRUPT_FILE, std::string("frames is not an array in ") + path);
  *n_frames = (int32_t)fr->arr.size();
  if (poses && capacity < *n_frames) return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "load_cameras_json: buffer too small");
  bool any = false, all = true;
  std::string joined;
  for (size_t i = 0; i < fr->arr.size(); ++i) {
    const Json& f = fr->arr[i];
    const Json* file = f.kind == Json::Obj ? f.get("file") : nullptr;
    if (i) joined.push_back('\n');
    if (file && file->kind == Json::Str) joined += file->str;
    const Json* pose = f.kind == Json::Obj ? f.get("pose") : nullptr;
    if (pose) {
      any = true;
      double tmp[12];
      if (int r = pose_from_json(*pose, path, tmp)) return r;
      if (poses) std::memcpy(poses + 12 * i, tmp, sizeof tmp);
    } else {
      all = false;
      if (poses) identity12(poses + 12 * i);
    }
  }
  if (has_poses) *has_poses = (any && all) ? 1 : 0;
  if (names) {
    if (names_capacity < (int64_t)joined.size() + 1)
      return gsb::fail(GSB_ERR_INVALID_ARGUMENT, "load_cameras_json: names buffer too small");
    std::memcpy(names, joined.c_str(), joined.size() + 1);
  }
  return GSB_OK;
}

}  // extern "C"
