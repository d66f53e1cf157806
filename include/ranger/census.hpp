#pragma once
// Drop-in replacement for ranger/census.hpp (proj/include/ranger/census.hpp:
// 1-327).  Same declarations; the transforms and the matcher run on the
// B200 (K1 census, K2 matcher) via include/ranger_cuda.h.
#include <bit>
#include <cstdint>
#include <fstream>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ranger/cuda_context.hpp"
#include "ranger/image.hpp"

namespace ranger {

/// 26-bit census descriptors (sentinel bit 25), 0 = undefined (census.hpp:21-39).
struct CensusImage {
  static constexpr int kSpan = 2;
  static constexpr std::uint32_t kSentinel = 1u << 25;

  int width = 0;
  int height = 0;
  std::vector<std::uint32_t> codes;
  double scale_x = 1.0;
  double scale_y = 1.0;

  CensusImage() = default;
  CensusImage(int w, int h) : width(w), height(h), codes(static_cast<std::size_t>(w) * h, 0) {}
  std::uint32_t code(int x, int y) const { return codes[static_cast<std::size_t>(y) * width + x]; }
  bool inside(int x, int y) const { return 0 <= x && x < width && 0 <= y && y < height; }
};

/// census.hpp:43-56 -> rg_census_code_at
inline std::uint32_t census_code_at(const GrayImage& img, int sx, int sy) {
  std::uint32_t code = 0;
  cuda::check(rg_census_code_at(cuda::ctx(), img.data.data(), img.width, img.height, sx, sy, &code));
  return code;
}

/// census.hpp:69-86 -> rg_census_transform (workers: the CUDA grid is the parallelism)
inline CensusImage census_transform(const GrayImage& img, int out_w, int out_h, int workers = 1) {
  (void)workers;
  if (out_w > img.width || out_h > img.height)
    throw std::invalid_argument("census_transform: output dims exceed source");
  if (out_w < 1 || out_h < 1) throw std::invalid_argument("census_transform: empty output");
  CensusImage out(out_w, out_h);
  out.scale_x = double(out_w) / img.width;
  out.scale_y = double(out_h) / img.height;
  cuda::check(rg_census_transform(cuda::ctx(), img.data.data(), img.width, img.height, out_w, out_h,
                                  out.codes.data()));
  return out;
}

inline CensusImage census_transform(const GrayImage& img, int workers = 1) {
  return census_transform(img, img.width, img.height, workers);
}

struct CensusRoi {
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
};

/// census.hpp:100-138 -> rg_census_transform_rois
inline CensusImage census_transform_rois(const GrayImage& img, int out_w, int out_h,
                                         const std::vector<CensusRoi>& rois, int workers = 1) {
  (void)workers;
  if (out_w > img.width || out_h > img.height)
    throw std::invalid_argument("census_transform_rois: output dims exceed source");
  CensusImage out(out_w, out_h);
  out.scale_x = double(out_w) / img.width;
  out.scale_y = double(out_h) / img.height;
  if (out_w < 1 || out_h < 1) return out;
  std::vector<rg_rect> r;
  r.reserve(rois.size());
  for (const auto& q : rois) r.push_back({q.x0, q.y0, q.x1, q.y1});
  cuda::check(rg_census_transform_rois(cuda::ctx(), img.data.data(), img.width, img.height, out_w, out_h,
                                       r.data(), int(r.size()), out.codes.data()));
  return out;
}

/// census.hpp:141
inline int hamming_cost(std::uint32_t a, std::uint32_t b) { return std::popcount(a ^ b); }

enum class ObjectKind { kFar, kClose };

/// census.hpp:146-152
struct QueryBlock {
  std::vector<std::pair<int, int>> points;
  int dx_min = 0, dx_max = 0;
  int dy_min = 0, dy_max = 0;
  int owner = -1;
  ObjectKind kind = ObjectKind::kFar;
};

/// census.hpp:154-163
struct MatchResult {
  int dx_int = 0;
  int dy_int = 0;
  double dx_subpix = 0.0;
  double cost = 0.0;
  double cost_minus = -1.0;
  double cost_plus = -1.0;
  int valid_points = 0;
  bool verified = false;
};

/// census.hpp:167-171 (pure arithmetic, also used by the reference's BM/SGM)
inline double subpixel_refine(double cost_minus, double cost_at, double cost_plus) {
  const double denom = cost_minus + cost_plus - 2.0 * cost_at;
  return denom <= 0.0 ? 0.0 : -(cost_plus - cost_minus) / (2.0 * denom);
}

namespace cuda {
inline std::vector<std::optional<MatchResult>> match(const std::vector<QueryBlock>& blocks,
                                                     const CensusImage& left, const CensusImage& right,
                                                     int mode, double tau_v) {
  std::vector<std::optional<MatchResult>> out(blocks.size());
  if (blocks.empty()) return out;
  std::vector<std::int64_t> offs(blocks.size() + 1, 0);
  std::vector<std::int32_t> pts;
  std::vector<rg_search_range> rg(blocks.size());
  for (std::size_t b = 0; b < blocks.size(); ++b) {
    for (const auto& [x, y] : blocks[b].points) {
      pts.push_back(x);
      pts.push_back(y);
    }
    offs[b + 1] = std::int64_t(pts.size() / 2);
    rg[b] = {blocks[b].dx_min, blocks[b].dx_max, blocks[b].dy_min, blocks[b].dy_max};
  }
  std::vector<rg_match_result> res(blocks.size());
  check(rg_match_blocks(ctx(), left.codes.data(), left.width, left.height, right.codes.data(), right.width,
                        right.height, pts.data(), offs.data(), rg.data(), int(blocks.size()), mode, tau_v,
                        res.data()));
  for (std::size_t b = 0; b < blocks.size(); ++b) {
    if (!res[b].has_value) continue;
    const rg_match_result& r = res[b];
    out[b] = MatchResult{r.dx_int,     r.dy_int,        r.dx_subpix,  r.cost, r.cost_minus,
                         r.cost_plus,  r.valid_points,  r.verified != 0};
  }
  return out;
}
}  // namespace cuda

/// census.hpp:178-272 -> rg_match_blocks(RG_MATCH_FORWARD)
inline std::optional<MatchResult> block_match(const QueryBlock& block, const CensusImage& left,
                                              const CensusImage& right) {
  return cuda::match({block}, left, right, RG_MATCH_FORWARD, 0.0)[0];
}

/// census.hpp:281-303 -> rg_match_blocks(RG_MATCH_FWD_BWD)
inline std::optional<MatchResult> forward_backward_match(const QueryBlock& block, const CensusImage& left,
                                                         const CensusImage& right, double tau_v) {
  return cuda::match({block}, left, right, RG_MATCH_FWD_BWD, tau_v)[0];
}

/// census.hpp:307-315: one CTA per block, results by block index
inline std::vector<std::optional<MatchResult>> batch_match(const std::vector<QueryBlock>& blocks,
                                                           const CensusImage& left, const CensusImage& right,
                                                           double tau_v, int workers = 1) {
  (void)workers;
  return cuda::match(blocks, left, right, RG_MATCH_FWD_BWD, tau_v);
}

/// census.hpp:318-325: 8-byte width/height header then raw codes
inline void dump_census(const CensusImage& img, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("dump_census: cannot open " + path);
  const std::uint32_t dims[2] = {std::uint32_t(img.width), std::uint32_t(img.height)};
  f.write(reinterpret_cast<const char*>(dims), sizeof(dims));
  f.write(reinterpret_cast<const char*>(img.codes.data()), std::streamsize(img.codes.size() * 4));
}

}  // namespace ranger
