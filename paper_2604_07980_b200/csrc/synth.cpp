// synth.cpp -- synthetic rectified stereo frames (host side of the library).
//
// Input generator for tests and bench: reproduces the reference renderer
// render_stereo_pair (synth.hpp:142-230) and ground_truth_detections
// (synth.hpp:253-274) bit for bit, with the canonical calibration
// make_calibration(f, b, cx, cy, h_cam) (geometry.hpp:108-133).  Rows are
// independent until the radiometric/shift/noise epilogue, so the image body
// is rendered by a pool of std::threads.  Compiled with -ffp-contract=off so
// every double rounds exactly as the reference's build.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "../../include/ranger_cuda.h"
#include "synth_scene.h"

namespace {

inline uint64_t mix64(uint64_t x) {  // splitmix64 finaliser, synth.hpp:56-61
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Bilinear value-noise texture field (synth.hpp:65-89).
struct NoiseField {
  uint64_t seed;
  double cell, contrast;
  int quant;

  double node(long gx, long gy) const {
    const uint64_t k = uint64_t(gx) * 0x100000001B3ull ^ uint64_t(gy);
    return double(mix64(seed ^ mix64(k)) >> 11) * 0x1.0p-53;
  }
  double at(double x, double y) const {
    const double u = x / cell, v = y / cell;
    const long iu = long(std::floor(u)), iv = long(std::floor(v));
    const double tu = u - iu, tv = v - iv;
    const double top = node(iu, iv) * (1 - tu) + node(iu + 1, iv) * tu;
    const double bot = node(iu, iv + 1) * (1 - tu) + node(iu + 1, iv + 1) * tu;
    const double mixv = top * (1 - tv) + bot * tv;
    double val = 128.0 + contrast * (2.0 * mixv - 1.0);
    if (quant > 1) val = std::round(val / quant) * quant;
    return val < 0.0 ? 0.0 : (val > 255.0 ? 255.0 : val);
  }
};

struct Cam {  // canonical camera: cam = R^T (p - t), R = [0 0 1; -1 0 0; 0 -1 0]
  double x, y, z;
};
inline Cam to_camera(const rg_scene_object& o, const rg_scene_config& c) {
  const double vx = o.px - 0.0, vy = o.py - 0.0, vz = o.pz - c.h_cam;
  // R^T rows: (0,-1,0), (0,0,-1), (1,0,0); same summation order as Mat3*Vec3
  return {0.0 * vx + -1.0 * vy + 0.0 * vz, 0.0 * vx + 0.0 * vy + -1.0 * vz,
          1.0 * vx + 0.0 * vy + 0.0 * vz};
}

struct Proj {  // synth.hpp:91-112
  double u0, u1, v0, v1, uc, z, disp;
};
inline Proj project(const rg_scene_object& o, const rg_scene_config& c, const Cam& p) {
  Proj r;
  r.z = p.z;
  r.u0 = c.cx + c.f * (p.x - o.width_m / 2) / p.z;
  r.u1 = c.cx + c.f * (p.x + o.width_m / 2) / p.z;
  r.v0 = c.cy + c.f * (p.y - o.height_m / 2) / p.z;
  r.v1 = c.cy + c.f * (p.y + o.height_m / 2) / p.z;
  r.uc = c.cx + c.f * p.x / p.z;
  r.disp = c.f * c.b / p.z;
  return r;
}

inline uint8_t to_byte(double v) { return uint8_t(std::lround(v)); }

template <typename Fn>
void rows_parallel(int n, Fn&& fn) {
  unsigned hc = std::thread::hardware_concurrency();
  int k = int(std::min<unsigned>(hc ? hc : 1, 32u));
  if (n < 64) k = 1;
  if (k <= 1) {
    for (int y = 0; y < n; ++y) fn(y);
    return;
  }
  std::vector<std::thread> pool;
  const int chunk = (n + k - 1) / k;
  for (int t = 0; t < k; ++t) {
    const int lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([lo, hi, &fn] {
      for (int y = lo; y < hi; ++y) fn(y);
    });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

namespace rg_synth {

rg_status prepare_scene(const rg_scene_config& c, const rg_scene_object* objs, int n_obj,
                        std::vector<RenderObj>& out) {
  out.clear();
  if (n_obj < 0 || (n_obj > 0 && !objs)) return RG_EINVAL;
  if (c.width < 8 || c.height < 8 || c.gamma <= 0) return RG_EINVAL;
  const int w = c.width, h = c.height;
  std::vector<Proj> pr(static_cast<size_t>(n_obj));
  for (int i = 0; i < n_obj; ++i) {
    const Cam p = to_camera(objs[i], c);
    if (p.z <= 0) return RG_EINVAL;  // object behind the camera
    pr[i] = project(objs[i], c, p);
  }
  std::vector<int> order(static_cast<size_t>(n_obj));
  for (int i = 0; i < n_obj; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {  // far to near, synth.hpp:168
    if (pr[a].z != pr[b].z) return pr[a].z > pr[b].z;
    return objs[a].id < objs[b].id;
  });
  for (int i : order)
    if (std::abs(objs[i].disparity_ramp) >= 1) return RG_EINVAL;
  for (int i : order) {
    const rg_scene_object& o = objs[i];
    const Proj& p = pr[i];
    RenderObj s{};
    s.ly0 = std::max(0, int(std::ceil(p.v0)));
    s.ly1 = std::min(h - 1, int(std::floor(p.v1)));
    s.lx0 = std::max(0, int(std::ceil(p.u0)));
    s.lx1 = std::min(w - 1, int(std::floor(p.u1)));
    s.k = 1.0 - o.disparity_ramp;
    s.c0 = p.disp + c.disparity_bias_px - o.disparity_ramp * p.uc;
    const double ru0 = p.u0 * s.k - s.c0, ru1 = p.u1 * s.k - s.c0;
    s.rx0 = std::max(0, int(std::ceil(std::min(ru0, ru1))));
    s.rx1 = std::min(w - 1, int(std::floor(std::max(ru0, ru1))));
    s.id = o.id;
    s.u0 = p.u0;
    s.u1 = p.u1;
    s.v0 = p.v0;
    s.uc = p.uc;
    s.disp = p.disp;
    s.ramp = o.disparity_ramp;
    s.tex_seed = o.texture_seed;
    s.contrast = o.contrast;
    out.push_back(s);
  }
  return RG_OK;
}

void radiometric_lut(const rg_scene_config& c, uint8_t lut[256]) {  // synth.hpp:212-217
  const bool apply = c.gain != 1 || c.rad_bias != 0 || c.gamma != 1;
  for (int v = 0; v < 256; ++v) {
    if (!apply) {
      lut[v] = uint8_t(v);
      continue;
    }
    const double m = c.gain * std::pow(v / 255.0, c.gamma) * 255.0 + c.rad_bias;
    const long r = std::lround(m);
    lut[v] = uint8_t(r < 0 ? 0 : (r > 255 ? 255 : r));
  }
}

}  // namespace rg_synth

extern "C" rg_status rg_render_stereo_pair(const rg_scene_config* cfg, const rg_scene_object* objs,
                                           int n_obj, uint8_t* left, uint8_t* right,
                                           double* true_disp, int32_t* object_id) {
  if (!cfg || !left || !right) return RG_EINVAL;
  const rg_scene_config& c = *cfg;
  std::vector<rg_synth::RenderObj> sp;
  if (rg_synth::prepare_scene(c, objs, n_obj, sp) != RG_OK) return RG_EINVAL;
  const int w = c.width, h = c.height;
  const NoiseField bg{c.background_seed, c.texture_cell_px, c.background_contrast, c.texture_quant};
  std::vector<NoiseField> tex;
  for (const auto& s : sp) tex.push_back({s.tex_seed, c.texture_cell_px, s.contrast, c.texture_quant});
  const bool shift = c.vertical_offset_px != 0;
  std::vector<uint8_t> rtmp;
  uint8_t* rbody = right;
  if (shift) {
    rtmp.resize(size_t(w) * h);
    rbody = rtmp.data();
  }

  rows_parallel(h, [&](int y) {
    uint8_t* lrow = left + size_t(y) * w;
    uint8_t* rrow = rbody + size_t(y) * w;
    for (int x = 0; x < w; ++x) {
      lrow[x] = to_byte(bg.at(x, y));
      rrow[x] = to_byte(bg.at(x + c.disparity_bias_px, y));
    }
    if (true_disp) std::fill(true_disp + size_t(y) * w, true_disp + size_t(y + 1) * w, 0.0);
    if (object_id) std::fill(object_id + size_t(y) * w, object_id + size_t(y + 1) * w, -1);
    for (size_t t = 0; t < sp.size(); ++t) {
      const rg_synth::RenderObj& s = sp[t];
      if (y < s.ly0 || y > s.ly1) continue;
      for (int x = s.lx0; x <= s.lx1; ++x) {
        lrow[x] = to_byte(tex[t].at(x - s.u0, y - s.v0));
        if (true_disp) true_disp[size_t(y) * w + x] = s.disp + s.ramp * (x - s.uc);
        if (object_id) object_id[size_t(y) * w + x] = s.id;
      }
      for (int xr = s.rx0; xr <= s.rx1; ++xr) {
        const double u = (xr + s.c0) / s.k;
        if (u < s.u0 || u > s.u1) continue;
        rrow[xr] = to_byte(tex[t].at(u - s.u0, y - s.v0));
      }
    }
  });

  if (c.gain != 1 || c.rad_bias != 0 || c.gamma != 1) {
    uint8_t lut[256];
    rg_synth::radiometric_lut(c, lut);
    for (size_t i = 0; i < size_t(w) * h; ++i) rbody[i] = lut[rbody[i]];
  }
  if (shift) {  // image.hpp:145-154: out(y) = in(clamp(y - dy))
    for (int y = 0; y < h; ++y) {
      int sy = y - c.vertical_offset_px;
      sy = sy < 0 ? 0 : (sy >= h ? h - 1 : sy);
      std::memcpy(right + size_t(y) * w, rbody + size_t(sy) * w, size_t(w));
    }
  }
  if (c.noise_sigma > 0) {
    std::mt19937_64 rng(c.seed);
    std::normal_distribution<double> nd(0.0, c.noise_sigma);
    for (uint8_t* img : {left, right})
      for (size_t i = 0; i < size_t(w) * h; ++i) {
        const long v = std::lround(img[i] + nd(rng));
        img[i] = uint8_t(v < 0 ? 0 : (v > 255 ? 255 : v));
      }
  }
  return RG_OK;
}

extern "C" rg_status rg_ground_truth_detections(const rg_scene_config* cfg,
                                                const rg_scene_object* objs, int n_obj,
                                                rg_detection* out, int* n_out) {
  if (!cfg || !out || !n_out || n_obj < 0) return RG_EINVAL;
  int n = 0;
  for (int i = 0; i < n_obj; ++i) {
    const Cam p = to_camera(objs[i], *cfg);
    if (p.z <= 0) continue;
    const Proj r = project(objs[i], *cfg, p);
    const double x0 = std::max(0.0, r.u0 / cfg->width), x1 = std::min(1.0, r.u1 / cfg->width);
    const double y0 = std::max(0.0, r.v0 / cfg->height), y1 = std::min(1.0, r.v1 / cfg->height);
    if (x1 - x0 <= 0 || y1 - y0 <= 0) continue;
    rg_detection d;
    d.cx = (x0 + x1) / 2;
    d.cy = (y0 + y1) / 2;
    d.w = x1 - x0;
    d.h = y1 - y0;
    d.id = objs[i].id;
    d.class_id = objs[i].class_id;
    out[n++] = d;
  }
  *n_out = n;
  return RG_OK;
}
