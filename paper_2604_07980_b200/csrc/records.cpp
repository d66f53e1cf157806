// records.cpp -- the sequential per-frame tail of Pipeline::process_frame
// (pipeline.hpp:180-265, the tracker excluded): object refiner, monocular and
// stereo depth cues, priority fusion into DepthRecord, refiner log.
//
// This is host code by design: it runs once per frame over <= max_objects
// entries after the device batch (census -> matcher -> aggregation) is back,
// and the object refiner carries state from frame to frame.  Every FP64
// expression keeps the reference's operation order (built with
// -ffp-contract=off), so the records are bit-identical.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/ranger_cuda.h"

namespace {

struct V3 {
  double x, y, z;
};
V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double norm3(V3 v) { return std::sqrt(v.x * v.x + v.y * v.y + v.z * v.z); }  // geometry.hpp:23-24
// Mat3 * Vec3 (geometry.hpp:42-46); trans = use R^T
V3 mul(const double* r, V3 v, bool trans) {
  auto a = [&](int i, int j) { return trans ? r[j * 3 + i] : r[i * 3 + j]; };
  return {a(0, 0) * v.x + a(0, 1) * v.y + a(0, 2) * v.z, a(1, 0) * v.x + a(1, 1) * v.y + a(1, 2) * v.z,
          a(2, 0) * v.x + a(2, 1) * v.y + a(2, 2) * v.z};
}

// reproject (geometry.hpp:142-146) through the Q of make_calibration
// (geometry.hpp:122-126), evaluated as Mat4 * array (geometry.hpp:89-94)
V3 reproject(double u, double v, double d, const rg_calibration& c) {
  const double q[16] = {1, 0, 0, -c.cx, 0, 1, 0, -c.cy, 0, 0, 0, c.f, 0, 0, 1 / c.b, 0};
  const double in[4] = {u, v, d, 1.0};
  double h[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) h[i] += q[i * 4 + k] * in[k];
  if (h[3] == 0.0) throw std::invalid_argument("reproject: degenerate point (W = 0)");
  return {h[0] / h[3], h[1] / h[3], h[2] / h[3]};
}
V3 cam_to_imu(V3 p, const rg_calibration& c) { return add(mul(c.R, p, false), V3{c.t[0], c.t[1], c.t[2]}); }
V3 imu_to_cam(V3 p, const rg_calibration& c) { return mul(c.R, sub(p, V3{c.t[0], c.t[1], c.t[2]}), true); }

// project_radar_to_disparity(...).d (radar_refiner.hpp:21-27)
double radar_disparity(V3 p_imu, const rg_calibration& c) {
  const V3 p = imu_to_cam(p_imu, c);
  if (p.z <= 0) throw std::invalid_argument("project_radar_to_disparity: point behind camera");
  return c.f * c.b / p.z;
}

struct Obs {
  double u, v, d;
};

// default_offset_candidates (object_refiner.hpp:37-43)
std::vector<double> offset_candidates(double half_range, double step) {
  std::vector<double> c;
  const int n = int(std::lround(half_range / step));
  for (int i = -n; i <= n; ++i) c.push_back(i * step);
  return c;
}

// object_refiner_coarse (object_refiner.hpp:50-106): per candidate offset,
// greedy 1-to-1 pairing by ascending 3-D distance, score, consistency bonus
double refiner_coarse(const std::vector<Obs>& stereo, const std::vector<V3>& radar,
                      const std::vector<double>& cands, const rg_obj_refiner_state& st, const rg_calibration& c,
                      std::vector<std::pair<double, double>>& best_pairs) {
  if (cands.empty()) throw std::invalid_argument("object_refiner_coarse: no candidates");
  double best_off = 0, best_score = 0;
  bool first = true;
  std::vector<V3> pts(stereo.size());
  std::vector<char> usable(stereo.size());
  std::vector<std::tuple<double, int, int>> edges;
  for (const double cand : cands) {
    for (std::size_t i = 0; i < stereo.size(); ++i) {
      const double d = stereo[i].d + cand;
      usable[i] = d > 0;
      if (usable[i]) pts[i] = cam_to_imu(reproject(stereo[i].u, stereo[i].v, d, c), c);
    }
    edges.clear();
    for (std::size_t i = 0; i < stereo.size(); ++i) {
      if (!usable[i]) continue;
      for (std::size_t j = 0; j < radar.size(); ++j) {
        const double dist = norm3(sub(pts[i], radar[j]));
        if (dist < st.r_max) edges.emplace_back(dist, int(i), int(j));
      }
    }
    std::sort(edges.begin(), edges.end());  // (dist, i, j): a total order
    std::vector<char> s_used(stereo.size(), 0), r_used(radar.size(), 0);
    double score = 0;
    std::vector<std::pair<double, double>> pairs;
    for (const auto& [dist, i, j] : edges) {
      if (s_used[i] || r_used[j]) continue;
      s_used[i] = r_used[j] = 1;
      score += std::max(1.0 - dist / st.r_max, 0.0);
      pairs.emplace_back(stereo[i].d, radar_disparity(radar[j], c));
    }
    if (cand == st.prev_offset) score += st.beta;
    bool better = first || score > best_score;
    if (!first && score == best_score) {
      if (std::abs(cand) < std::abs(best_off))
        better = true;
      else if (std::abs(cand) == std::abs(best_off) && cand < best_off)
        better = true;
    }
    if (better) {
      best_off = cand;
      best_score = score;
      best_pairs = std::move(pairs);
      first = false;
    }
  }
  return best_off;
}

// object_refiner_iterate (object_refiner.hpp:113-134)
double refiner_iterate(const std::vector<std::pair<double, double>>& pairs, double coarse,
                       rg_obj_refiner_state& st) {
  double sum = 0;
  int n = 0;
  for (const auto& [ds, dr] : pairs) {
    const double diff = dr - ds;
    if (std::abs(diff - coarse) < st.tau) {
      sum += diff;
      ++n;
    }
  }
  const double refined = (n == 0 && st.w_p == 0) ? st.prev_offset : (sum + st.w_p * st.prev_offset) / (n + st.w_p);
  const double step = std::clamp(refined - st.prev_offset, -st.rate_limit, st.rate_limit);
  st.prev_offset += step;
  return st.prev_offset;
}

struct Cue {
  bool has = false;
  double z = 0, d = 0;
};

}  // namespace

extern "C" {

rg_status rg_obj_refiner_state_init(rg_obj_refiner_state* st) {
  if (!st) return RG_EINVAL;
  *st = rg_obj_refiner_state{0.0, 0.1, 5.0, 1.0, 0.5, 0.5};
  return RG_OK;
}

rg_status rg_make_calibration(double f, double b, double cx, double cy, double h_cam, rg_calibration* out) {
  if (!out || !(f > 0) || !(b > 0)) return RG_EINVAL;  // geometry.hpp:108-109
  *out = rg_calibration{f, b, cx, cy, h_cam, {0, 0, 1, -1, 0, 0, 0, -1, 0}, {0, 0, h_cam}};
  return RG_OK;
}

rg_status rg_frame_records(const rg_record_params* p, int frame_id, int img_w, int img_h, int dense,
                           const rg_detection* dets, int n_dets, const int32_t* sel,
                           rg_object_disparity* objects, int n_obj, const rg_vec3* radar, int n_radar,
                           rg_obj_refiner_state* st, double rect_applied, rg_depth_record* records,
                           rg_refiner_log* log) {
  if (!p || !st || n_obj < 0 || n_dets < 0 || n_radar < 0 || img_w < 1 || img_h < 1) return RG_EINVAL;
  if (n_obj > 0 && (!dets || !sel || !objects || !records)) return RG_EINVAL;
  if (n_radar > 0 && !radar) return RG_EINVAL;
  if (p->n_class_widths > 0 && !p->class_widths) return RG_EINVAL;
  for (int k = 0; k < n_obj; ++k)
    if (sel[k] < 0 || sel[k] >= n_dets) return RG_EINVAL;
  const rg_calibration& c = p->calib;
  try {
    // object refiner (pipeline.hpp:185-205)
    double obj_applied = st->prev_offset;
    if (!dense && p->object_refiner) {
      std::vector<Obs> obs;
      for (int k = 0; k < n_obj; ++k)
        if (objects[k].valid && objects[k].disparity > 0) {
          const rg_detection& d = dets[sel[k]];
          obs.push_back({d.cx * img_w, d.cy * img_h, objects[k].disparity});
        }
      std::vector<V3> rp;
      for (int j = 0; j < n_radar; ++j) rp.push_back({radar[j].x, radar[j].y, radar[j].z});
      if (!obs.empty() && !rp.empty()) {
        std::vector<std::pair<double, double>> pairs;
        const double coarse = refiner_coarse(obs, rp, offset_candidates(p->obj_cand_half_px, p->obj_cand_step_px),
                                             *st, c, pairs);
        obj_applied = refiner_iterate(pairs, coarse, *st);
      }
      for (int k = 0; k < n_obj; ++k)
        if (objects[k].valid) objects[k].disparity += obj_applied;
    }
    // cues, fusion, records (pipeline.hpp:151-160, 208-249)
    const double nan = std::numeric_limits<double>::quiet_NaN();
    for (int k = 0; k < n_obj; ++k) {
      const rg_detection& det = dets[sel[k]];
      Cue stereo, gpt, size;
      if ((det.cy + det.h / 2) * img_h > c.cy) {  // ground_point_depth, geometry.hpp:214-229
        const double v_bottom = (det.cy + det.h / 2) * img_h;
        gpt.has = true;
        gpt.z = c.h_cam * c.f / (v_bottom - c.cy);
      }
      for (int q = 0; q < p->n_class_widths; ++q)
        if (p->class_widths[q].class_id == det.class_id) {
          if (det.w * img_w > 0) {  // size_based_depth, geometry.hpp:231-246
            size.has = true;
            size.z = c.f * p->class_widths[q].width_m / (det.w * img_w);
          }
          break;
        }
      const rg_object_disparity& o = objects[k];
      if (o.valid && o.disparity > 0) {  // make_stereo_estimate, geometry.hpp:198-211
        stereo.has = true;
        stereo.d = o.disparity;
        stereo.z = reproject(det.cx * img_w, det.cy * img_h, o.disparity, c).z;
      }
      rg_depth_record r;
      r.frame_id = frame_id;
      r.det_id = det.id;
      r.disparity = stereo.has ? stereo.d : nan;
      r.valid = stereo.has;
      r.clp_by_stereo = stereo.has ? stereo.z : nan;
      r.clp_by_gpt = gpt.has ? gpt.z : nan;
      r.clp_by_size = size.has ? size.z : nan;
      r.z_fused = nan;
      r.source = RG_SRC_STEREO;
      if (stereo.has || gpt.has || size.has) {  // fuse_depth, tracking.hpp:383-394
        const Cue& mono = gpt.has ? gpt : size;
        int src = -1;
        if (stereo.has) {
          if (!mono.has) {
            src = RG_SRC_STEREO;
          } else {
            const double zm = mono.z;
            if (zm > 0 && std::abs(stereo.z - zm) / zm <= p->fuse_sanity_ratio) src = RG_SRC_STEREO;
          }
        }
        if (src < 0) src = gpt.has ? RG_SRC_GPT : RG_SRC_SIZE;
        r.source = src;
        r.z_fused = src == RG_SRC_STEREO ? stereo.z : src == RG_SRC_GPT ? gpt.z : size.z;
      }
      records[k] = r;
    }
    if (log) *log = rg_refiner_log{frame_id, 0, rect_applied, 0.0, obj_applied};
  } catch (const std::exception&) {
    return RG_EINVAL;
  }
  return RG_OK;
}

// ---------------------------------------------------------------- radar refiner
// Host halves of radar_refine_step (radar_refiner.hpp:49-167); the pixel
// search and the map update run on the device (dense.cu).

rg_status rg_vote_state_init(rg_vote_state* st, int k_px, double lambda, double smooth_sigma_px) {
  if (!st) return RG_EINVAL;
  if (k_px < 1 || lambda <= 0 || lambda > 1) return RG_EINVAL;  // VoteState ctor throws
  if (2 * k_px * 16 + 1 > RG_VOTE_MAX_BINS) return RG_EINVAL;
  std::memset(st, 0, sizeof(*st));
  st->k_px = k_px;
  st->n_bins = 2 * k_px * 16 + 1;
  st->lambda = lambda;
  st->smooth_sigma_px = smooth_sigma_px;
  return RG_OK;
}

rg_status rg_radar_boxes(const rg_radar_detection* radar, int n, const rg_calibration* calib, int w, int h,
                         int32_t* boxes, double* d_radar, int* n_boxes) {
  if (!calib || !n_boxes || n < 0 || (n > 0 && (!radar || !boxes || !d_radar))) return RG_EINVAL;
  const rg_calibration& c = *calib;
  int m = 0;
  for (int i = 0; i < n; ++i) {
    const rg_radar_detection& det = radar[i];
    const V3 pc = imu_to_cam(V3{det.position.x, det.position.y, det.position.z}, c);
    if (pc.z <= 0) continue;
    const double dr = c.f * c.b / pc.z;
    // detail::radar_extent_box (radar_refiner.hpp:71-100)
    double u_min = std::numeric_limits<double>::infinity(), u_max = -u_min, v_min = u_min, v_max = -u_min;
    int np = 0;
    for (int k = 0; k < 8; ++k) {
      const V3 corner{det.position.x + (k & 1 ? 0.5 : -0.5) * det.extent.x,
                      det.position.y + (k & 2 ? 0.5 : -0.5) * det.extent.y,
                      det.position.z + (k & 4 ? 0.5 : -0.5) * det.extent.z};
      const V3 p = imu_to_cam(corner, c);
      if (p.z <= 0) continue;
      const double u = c.cx + c.f * p.x / p.z, v = c.cy + c.f * p.y / p.z;
      u_min = std::min(u_min, u);
      u_max = std::max(u_max, u);
      v_min = std::min(v_min, v);
      v_max = std::max(v_max, v);
      ++np;
    }
    if (np == 0) continue;
    const int x0 = std::max(0, int(std::floor(u_min))), x1 = std::min(w - 1, int(std::ceil(u_max)));
    const int y0 = std::max(0, int(std::floor(v_min))), y1 = std::min(h - 1, int(std::ceil(v_max)));
    if (!(x0 <= x1 && y0 <= y1)) continue;
    boxes[4 * m] = x0, boxes[4 * m + 1] = y0, boxes[4 * m + 2] = x1, boxes[4 * m + 3] = y1;
    d_radar[m] = dr;
    ++m;
  }
  *n_boxes = m;
  return RG_OK;
}

rg_status rg_radar_vote_update(rg_vote_state* st, const double* best_off, const int32_t* found, int n_boxes,
                               double* applied, int* raw_off) {
  if (!st || st->n_bins != 2 * st->k_px * 16 + 1 || n_boxes < 0 || (n_boxes > 0 && (!best_off || !found)))
    return RG_EINVAL;
  const int bins = st->n_bins;
  std::vector<double> votes(bins, 0.0);
  int n_votes = 0;
  for (int i = 0; i < n_boxes; ++i) {
    const double best = best_off[i];
    if (!found[i] || std::abs(best) > st->k_px) continue;
    const int bin = std::clamp(int(std::lround((best + st->k_px) * 16)), 0, bins - 1);
    votes[bin] += 1.0;  // one vote per detection
    ++n_votes;
  }
  if (n_votes > 0) {
    // detail::gaussian_smooth_bins (radar_refiner.hpp:51-69)
    std::vector<double> sm;
    const double sigma_bins = st->smooth_sigma_px * 16;
    if (sigma_bins <= 0) {
      sm = votes;
    } else {
      const int radius = std::max(1, int(std::ceil(3 * sigma_bins)));
      std::vector<double> kernel(2 * radius + 1);
      double sum = 0;
      for (int i = -radius; i <= radius; ++i) {
        kernel[i + radius] = std::exp(-0.5 * (i / sigma_bins) * (i / sigma_bins));
        sum += kernel[i + radius];
      }
      for (auto& k : kernel) k /= sum;
      sm.assign(bins, 0.0);
      for (int i = 0; i < bins; ++i) {
        if (votes[i] == 0) continue;
        for (int j = -radius; j <= radius; ++j) {
          const int t = i + j;
          if (t >= 0 && t < bins) sm[t] += votes[i] * kernel[j + radius];
        }
      }
    }
    double l1 = 0;
    for (double v : sm) l1 += v;
    if (l1 > 0)
      for (auto& v : sm) v /= l1;
    for (int i = 0; i < bins; ++i) st->memory[i] = (1 - st->lambda) * st->memory[i] + st->lambda * sm[i];
    int best_bin = 0;
    for (int i = 1; i < bins; ++i)
      if (st->memory[i] > st->memory[best_bin]) best_bin = i;
    const double d_star = best_bin / 16.0 - st->k_px;  // VoteState::bin_center
    st->smoothed_offset = (1 - st->lambda) * st->smoothed_offset + st->lambda * d_star;
  }
  const double a = std::clamp(st->smoothed_offset, -3.0, 3.0);
  if (applied) *applied = a;
  if (raw_off) *raw_off = int(std::lround(a * 16));  // DisparityMap::kSubLevels
  return RG_OK;
}

}  // extern "C"
