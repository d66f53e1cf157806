#pragma once
// Drop-in replacement for ranger/sgm.hpp (proj/include/ranger/sgm.hpp:1-157):
// census cost volume, the four directional aggregation passes and the
// winner-take-all run on the B200 (sgm.cu) via include/ranger_cuda.h.  The
// detail:: entry points the reference's tests use as building blocks
// (sgm_cost_volume, sgm_direction_pass) are the same device kernels.
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "ranger/census.hpp"
#include "ranger/image.hpp"

namespace ranger {

/// sgm.hpp:14-19
struct SgmParams {
  int num_disparities = 64;  // N_d
  int min_disparity = 0;     // d_min
  int p1 = 8;
  int p2 = 32;
};

namespace cuda {
inline rg_sgm_params to_c(const SgmParams& p) {
  rg_sgm_params r;
  r.num_disparities = p.num_disparities;
  r.min_disparity = p.min_disparity;
  r.p1 = p.p1;
  r.p2 = p.p2;
  return r;
}
}  // namespace cuda

/// sgm.hpp:21-28
inline void validate(const SgmParams& p) {
  const rg_sgm_params c = cuda::to_c(p);
  cuda::check(rg_validate_sgm_params(cuda::ctx(), &c));
}

namespace detail {

/// sgm.hpp:35: cost of a disparity whose right column leaves the frame
constexpr int kSgmNoData = 27;

/// sgm.hpp:37-56 -> rg_sgm_cost_volume ([y][x][i] bytes)
inline std::vector<std::uint8_t> sgm_cost_volume(const CensusImage& cl, const CensusImage& cr,
                                                 const SgmParams& p) {
  const rg_sgm_params c = cuda::to_c(p);
  std::vector<std::uint8_t> cost(static_cast<std::size_t>(cl.width) * cl.height * p.num_disparities);
  cuda::check(rg_sgm_cost_volume(cuda::ctx(), cl.codes.data(), cr.codes.data(), cl.width, cl.height, &c,
                                 cost.data()));
  return cost;
}

/// sgm.hpp:60-110 -> rg_sgm_direction_pass (adds L_r into acc)
inline void sgm_direction_pass(const std::vector<std::uint8_t>& cost, int w, int h, int nd, int p1, int p2,
                               int sx, int sy, std::vector<std::int32_t>& acc) {
  cuda::check(rg_sgm_direction_pass(cuda::ctx(), cost.data(), w, h, nd, p1, p2, sx, sy, acc.data()));
}

}  // namespace detail

/// sgm.hpp:118-155 -> rg_sgm_disparity
inline DisparityMap sgm_disparity(const GrayImage& left, const GrayImage& right, const SgmParams& p,
                                  int workers = 1) {
  (void)workers;
  validate(p);
  if (left.width != right.width || left.height != right.height)
    throw std::invalid_argument("sgm_disparity: image dims differ");
  DisparityMap out(left.width, left.height);
  const rg_sgm_params c = cuda::to_c(p);
  cuda::check(rg_sgm_disparity(cuda::ctx(), left.data.data(), right.data.data(), left.width, left.height, &c,
                               out.raw.data()));
  return out;
}

}  // namespace ranger
