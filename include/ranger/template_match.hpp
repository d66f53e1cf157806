#pragma once
// Drop-in replacement for ranger/template_match.hpp (proj/include/ranger/
// template_match.hpp:1-365).  estimate_object_disparities runs the whole
// frame on the B200 (census K1, planner K3, fused sampler+matcher K2,
// aggregation K4); the helper functions run the same device code one call
// at a time so the reference's unit tests exercise it.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <vector>

#include "ranger/census.hpp"
#include "ranger/detection.hpp"
#include "ranger/image.hpp"

namespace ranger {

struct ObjectDisparity {
  int det_id = -1;
  double disparity = 0;
  ObjectKind kind = ObjectKind::kFar;
  int n_blocks_used = 0;
  bool valid = false;
};

struct FrontalCrop {
  double x0 = 0.25, y0 = 0.25, x1 = 0.75, y1 = 0.75;
  bool contains(double cx, double cy) const { return cx >= x0 && cx < x1 && cy >= y0 && cy < y1; }
};

struct RangerConfig {
  double tau_s = 48;
  int close_scale = 2;
  int grid_side_points = 8;
  int max_total_points = 64;
  int close_block_side_points = 5;
  double tau_d = 1.0;
  int n_min = 3;
  double tau_v = 1.0;
  int max_objects = 16;
  FrontalCrop frontal_crop;
  int dx_max_far = 64;
  int dx_max_close = 192;
};

namespace cuda {
inline rg_ranger_config to_c(const RangerConfig& c) {
  rg_ranger_config r;
  r.tau_s = c.tau_s;
  r.close_scale = c.close_scale;
  r.grid_side_points = c.grid_side_points;
  r.max_total_points = c.max_total_points;
  r.close_block_side_points = c.close_block_side_points;
  r.tau_d = c.tau_d;
  r.n_min = c.n_min;
  r.max_objects = c.max_objects;
  r.tau_v = c.tau_v;
  r.crop_x0 = c.frontal_crop.x0;
  r.crop_y0 = c.frontal_crop.y0;
  r.crop_x1 = c.frontal_crop.x1;
  r.crop_y1 = c.frontal_crop.y1;
  r.dx_max_far = c.dx_max_far;
  r.dx_max_close = c.dx_max_close;
  r.census_9x7 = 0;  // the reference has only the 5x5 transform
  r.reserved = 0;
  return r;
}
inline const rg_detection* to_c(const std::vector<Detection>& d) {
  static_assert(sizeof(Detection) == sizeof(rg_detection), "Detection layout must match rg_detection");
  return reinterpret_cast<const rg_detection*>(d.data());
}
}  // namespace cuda

/// template_match.hpp:48-61
inline void validate(const RangerConfig& c) {
  const rg_ranger_config r = cuda::to_c(c);
  cuda::check(rg_validate_ranger_config(cuda::ctx(), &r));
}

/// template_match.hpp:63-67
inline ObjectKind classify_far_close(const Detection& d, int img_w, int img_h, double tau_s) {
  return std::max(d.w * img_w, d.h * img_h) < tau_s ? ObjectKind::kFar : ObjectKind::kClose;
}

/// template_match.hpp:71-89 -> rg_find_occluders (device)
inline std::vector<std::vector<int>> find_occluders(const std::vector<Detection>& dets) {
  const int n = int(dets.size());
  std::vector<std::int32_t> off(static_cast<std::size_t>(n) + 1), idx(static_cast<std::size_t>(n) * n + 1);
  cuda::check(rg_find_occluders(cuda::ctx(), cuda::to_c(dets), n, off.data(), idx.data()));
  std::vector<std::vector<int>> occ(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) occ[i].assign(idx.begin() + off[i], idx.begin() + off[i + 1]);
  return occ;
}

/// template_match.hpp:94-114 -> rg_select_objects (device rank kernel)
inline std::vector<int> select_objects(const std::vector<Detection>& dets, const RangerConfig& cfg) {
  const rg_ranger_config c = cuda::to_c(cfg);
  std::vector<std::int32_t> idx(dets.size() + 1);
  int n = 0;
  cuda::check(rg_select_objects(cuda::ctx(), cuda::to_c(dets), int(dets.size()), &c, idx.data(), &n));
  return std::vector<int>(idx.begin(), idx.begin() + n);
}

struct AggregationResult {
  bool valid = false;
  double disparity = 0;
  int run_length = 0;
};

/// template_match.hpp:126-148 -> rg_aggregate_close_disparities (device)
inline AggregationResult aggregate_close_disparities(std::vector<double> disps, double tau_d, int n_min) {
  std::int32_t valid = 0, len = 0;
  double d = 0;
  cuda::check(rg_aggregate_close_disparities(cuda::ctx(), disps.data(), int(disps.size()), tau_d, n_min, &valid,
                                             &d, &len));
  return AggregationResult{valid != 0, d, len};
}

/// template_match.hpp:155-223 -> rg_sample_query_points (device sampler)
inline std::vector<QueryBlock> sample_query_points(const Detection& det, ObjectKind kind,
                                                   const std::vector<PixelBox>& occluder_boxes,
                                                   const RangerConfig& cfg, int img_w, int img_h) {
  const rg_ranger_config c = cuda::to_c(cfg);
  std::vector<double> occ;
  for (const auto& b : occluder_boxes) occ.insert(occ.end(), {b.x0, b.y0, b.x1, b.y1});
  const PixelBox box = to_pixel_box(det, img_w, img_h);
  const double half_tau = cfg.tau_s / 2;
  const int cap_blocks = kind == ObjectKind::kFar
                             ? 1
                             : std::max(2, int(box.width() / half_tau)) * std::max(2, int(box.height() / half_tau));
  const std::int64_t cap_points = std::int64_t(cap_blocks) * std::max(cfg.max_total_points, 1);
  std::vector<std::int64_t> offs(static_cast<std::size_t>(cap_blocks) + 1);
  std::vector<std::int32_t> pts(2 * static_cast<std::size_t>(cap_points) + 2);
  std::vector<rg_search_range> rg(static_cast<std::size_t>(cap_blocks));
  int nb = 0;
  cuda::check(rg_sample_query_points(cuda::ctx(), reinterpret_cast<const rg_detection*>(&det),
                                     kind == ObjectKind::kFar ? RG_KIND_FAR : RG_KIND_CLOSE, occ.data(),
                                     int(occluder_boxes.size()), &c, img_w, img_h, offs.data(), pts.data(),
                                     rg.data(), cap_blocks, cap_points, &nb));
  std::vector<QueryBlock> blocks(static_cast<std::size_t>(nb));
  for (int b = 0; b < nb; ++b) {
    for (std::int64_t k = offs[b]; k < offs[b + 1]; ++k) blocks[b].points.emplace_back(pts[2 * k], pts[2 * k + 1]);
    blocks[b].dx_min = rg[b].dx_min;
    blocks[b].dx_max = rg[b].dx_max;
    blocks[b].dy_min = rg[b].dy_min;
    blocks[b].dy_max = rg[b].dy_max;
    blocks[b].kind = kind;
  }
  return blocks;
}

/// template_match.hpp:229-234
struct CensusCache {
  CensusImage full_left, full_right;
  CensusImage scaled_left, scaled_right;
  bool has_full = false;
  bool has_scaled = false;
};

/// template_match.hpp:236-241
struct RangerStats {
  std::size_t query_points = 0;
  std::size_t image_pixels = 0;
  int n_far = 0;
  int n_close = 0;
};

namespace detail {

/// template_match.hpp:243-255: the census ROI of a box in a raster scaled by
/// (sx, sy) -- floor/ceil of the scaled edges, dilated, clipped to w x h (the
/// right/bottom edges half-open, hence the + 1).  The device path computes
/// the same rows (census_rows_kernel); this helper keeps the API surface.
inline void add_roi(std::vector<CensusRoi>& rois, const PixelBox& b, double sx, double sy, int dilate_x,
                    int dilate_y, int w, int h) {
  CensusRoi r;
  r.x0 = std::max(0, int(std::floor(b.x0 * sx)) - dilate_x);
  r.y0 = std::max(0, int(std::floor(b.y0 * sy)) - dilate_y);
  r.x1 = std::min(w, int(std::ceil(b.x1 * sx)) + dilate_x + 1);
  r.y1 = std::min(h, int(std::ceil(b.y1 * sy)) + dilate_y + 1);
  rois.push_back(r);
}

}  // namespace detail

/// template_match.hpp:260-363 -> rg_estimate_object_disparities (whole frame on device)
inline std::vector<ObjectDisparity> estimate_object_disparities(const GrayImage& left, const GrayImage& right,
                                                                const std::vector<Detection>& dets,
                                                                const RangerConfig& cfg,
                                                                CensusCache* cache = nullptr, int workers = 1,
                                                                RangerStats* stats = nullptr) {
  (void)workers;
  validate(cfg);
  if (left.width != right.width || left.height != right.height)
    throw std::invalid_argument("estimate_object_disparities: image dims differ");
  const int w = left.width, h = left.height;
  const rg_ranger_config c = cuda::to_c(cfg);
  std::vector<rg_object_disparity> out(std::max<std::size_t>(dets.size(), 1));
  int n_out = 0;
  rg_ranger_stats st{};
  rg_census_cache cc{};
  const int cw = w / cfg.close_scale, ch = h / cfg.close_scale;
  std::vector<std::uint32_t> fl, fr, sl, sr;
  // A pre-filled cache whose images are not w x h (or the CLOSE scale) is
  // laid out on the frame's raster with zeros outside its extent: the
  // reference drops samples that are not inside() the cached image exactly
  // like undefined (0) codes (census.hpp:195-216), and the device path reads
  // w*h (cw*ch) codes.
  std::vector<std::uint32_t> rl[4];
  // (rg_census_cache points are writable for the fill case; pre-filled codes are only read)
  auto fit = [](const CensusImage& img, int ww, int hh, std::vector<std::uint32_t>& buf) -> std::uint32_t* {
    if (img.width == ww && img.height == hh && img.codes.size() == std::size_t(ww) * hh)
      return const_cast<std::uint32_t*>(img.codes.data());
    buf.assign(std::size_t(std::max(ww, 0)) * std::max(hh, 0), 0u);
    for (int y = 0; y < std::min(hh, img.height); ++y)
      for (int x = 0; x < std::min(ww, img.width); ++x)
        if (std::size_t(y) * img.width + x < img.codes.size()) buf[std::size_t(y) * ww + x] = img.code(x, y);
    return buf.data();
  };
  if (cache) {
    cc.has_full = cache->has_full;
    cc.has_scaled = cache->has_scaled;
    if (cache->has_full) {
      cc.full_left = fit(cache->full_left, w, h, rl[0]);
      cc.full_right = fit(cache->full_right, w, h, rl[1]);
    } else {
      fl.assign(std::size_t(w) * h, 0);
      fr.assign(std::size_t(w) * h, 0);
      cc.full_left = fl.data();
      cc.full_right = fr.data();
    }
    if (cache->has_scaled) {
      cc.scaled_left = fit(cache->scaled_left, cw, ch, rl[2]);
      cc.scaled_right = fit(cache->scaled_right, cw, ch, rl[3]);
    } else {
      sl.assign(std::size_t(std::max(cw, 0)) * std::max(ch, 0), 0);
      sr.assign(sl.size(), 0);
      cc.scaled_left = sl.data();
      cc.scaled_right = sr.data();
    }
  }
  cuda::check(rg_estimate_object_disparities(cuda::ctx(), left.data.data(), right.data.data(), w, h,
                                             cuda::to_c(dets), int(dets.size()), &c, cache ? &cc : nullptr, 0.0,
                                             0.0, out.data(), &n_out, &st));
  if (cache) {
    auto adopt = [](CensusImage& img, std::vector<std::uint32_t>& codes, int ww, int hh, double sx, double sy) {
      img.width = ww;
      img.height = hh;
      img.codes = std::move(codes);
      img.scale_x = sx;
      img.scale_y = sy;
    };
    if (!cache->has_full && cc.has_full) {
      adopt(cache->full_left, fl, w, h, 1.0, 1.0);
      adopt(cache->full_right, fr, w, h, 1.0, 1.0);
      cache->has_full = true;
    }
    if (!cache->has_scaled && cc.has_scaled) {
      adopt(cache->scaled_left, sl, cw, ch, double(cw) / w, double(ch) / h);
      adopt(cache->scaled_right, sr, cw, ch, double(cw) / w, double(ch) / h);
      cache->has_scaled = true;
    }
  }
  if (stats) {
    stats->query_points = std::size_t(st.query_points);
    stats->image_pixels = std::size_t(st.image_pixels);
    stats->n_far = st.n_far;
    stats->n_close = st.n_close;
  }
  std::vector<ObjectDisparity> res(static_cast<std::size_t>(n_out));
  for (int i = 0; i < n_out; ++i)
    res[i] = ObjectDisparity{out[i].det_id, out[i].disparity,
                             out[i].kind == RG_KIND_FAR ? ObjectKind::kFar : ObjectKind::kClose,
                             out[i].n_blocks_used, out[i].valid != 0};
  return res;
}

}  // namespace ranger
