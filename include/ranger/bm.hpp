#pragma once
// Drop-in replacement for ranger/bm.hpp (proj/include/ranger/bm.hpp:1-137):
// the SAD block matcher runs on the B200 (K5) via include/ranger_cuda.h.
#include <cstdint>
#include <stdexcept>

#include "ranger/census.hpp"
#include "ranger/image.hpp"

namespace ranger {

struct BmParams {
  int num_disparities = 64;
  int block_size = 9;
  int min_disparity = 0;
  double texture_threshold = 10;
  double uniqueness_ratio = 10;
  int downscale = 1;
};

namespace cuda {
inline rg_bm_params to_c(const BmParams& p) {
  rg_bm_params r;
  r.num_disparities = p.num_disparities;
  r.block_size = p.block_size;
  r.min_disparity = p.min_disparity;
  r.downscale = p.downscale;
  r.texture_threshold = p.texture_threshold;
  r.uniqueness_ratio = p.uniqueness_ratio;
  return r;
}
}  // namespace cuda

/// bm.hpp:24-32
inline void validate(const BmParams& p) {
  const rg_bm_params c = cuda::to_c(p);
  cuda::check(rg_validate_bm_params(cuda::ctx(), &c));
}

/// bm.hpp:113-135 -> rg_bm_disparity
inline DisparityMap bm_disparity(const GrayImage& left, const GrayImage& right, const BmParams& p,
                                 int workers = 1) {
  (void)workers;
  validate(p);
  if (left.width != right.width || left.height != right.height)
    throw std::invalid_argument("bm_disparity: image dims differ");
  DisparityMap out(left.width, left.height);
  const rg_bm_params c = cuda::to_c(p);
  cuda::check(rg_bm_disparity(cuda::ctx(), left.data.data(), right.data.data(), left.width, left.height, &c,
                              out.raw.data()));
  return out;
}

}  // namespace ranger
