// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Compiles the reference's own header-only implementation IN PLACE
// (-I /root/reference/proj/include, nothing copied) and exposes it through the
// oracle's C interface as ref_*, so the C restatement (orc_*) and the CUDA
// path can be checked against the reference itself, and so bench.py can time
// the reference on the host cores (cpu_baseline kind "reference").
// Built by oracle/Makefile into oracle/_ref/libranger_ref.so.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ranger/autorect.hpp"
#include "ranger/bm.hpp"
#include "ranger/census.hpp"
#include "ranger/pipeline.hpp"
#include "ranger/synth.hpp"
#include "ranger/template_match.hpp"

#include "oracle.h"

using namespace ranger;

namespace {

GrayImage to_gray(const uint8_t* p, int w, int h) {
  GrayImage g(w, h);
  std::memcpy(g.data.data(), p, std::size_t(w) * h);
  return g;
}

CensusImage to_census(const uint32_t* c, int w, int h) {
  CensusImage img(w, h);
  std::memcpy(img.codes.data(), c, sizeof(uint32_t) * std::size_t(w) * h);
  return img;
}

RangerConfig to_cfg(const rg_ranger_config* c) {
  RangerConfig r;
  r.tau_s = c->tau_s;
  r.close_scale = c->close_scale;
  r.grid_side_points = c->grid_side_points;
  r.max_total_points = c->max_total_points;
  r.close_block_side_points = c->close_block_side_points;
  r.tau_d = c->tau_d;
  r.n_min = c->n_min;
  r.tau_v = c->tau_v;
  r.max_objects = c->max_objects;
  r.frontal_crop.x0 = c->crop_x0;
  r.frontal_crop.y0 = c->crop_y0;
  r.frontal_crop.x1 = c->crop_x1;
  r.frontal_crop.y1 = c->crop_y1;
  r.dx_max_far = c->dx_max_far;
  r.dx_max_close = c->dx_max_close;
  return r;
}

std::vector<Detection> to_dets(const rg_detection* d, int n) {
  std::vector<Detection> v(std::size_t(n > 0 ? n : 0));
  for (int i = 0; i < n; ++i) {
    v[i].cx = d[i].cx;
    v[i].cy = d[i].cy;
    v[i].w = d[i].w;
    v[i].h = d[i].h;
    v[i].class_id = d[i].class_id;
    v[i].id = d[i].id;
  }
  return v;
}

BmParams to_bm(const rg_bm_params* p) {
  BmParams b;
  b.num_disparities = p->num_disparities;
  b.block_size = p->block_size;
  b.min_disparity = p->min_disparity;
  b.texture_threshold = p->texture_threshold;
  b.uniqueness_ratio = p->uniqueness_ratio;
  b.downscale = p->downscale;
  return b;
}

void fill_match(const std::optional<MatchResult>& m, rg_match_result* o) {
  std::memset(o, 0, sizeof(*o));
  o->cost_minus = -1.0;
  o->cost_plus = -1.0;
  if (!m) return;
  o->has_value = 1;
  o->dx_int = m->dx_int;
  o->dy_int = m->dy_int;
  o->dx_subpix = m->dx_subpix;
  o->cost = m->cost;
  o->cost_minus = m->cost_minus;
  o->cost_plus = m->cost_plus;
  o->valid_points = m->valid_points;
  o->verified = m->verified ? 1 : 0;
}

SceneConfig to_scene(const rg_scene_config* c, const rg_scene_object* o, int n) {
  SceneConfig s;
  s.calib = make_calibration(c->f, c->b, c->cx, c->cy, c->h_cam);
  s.width = c->width;
  s.height = c->height;
  s.background_seed = c->background_seed;
  s.background_contrast = c->background_contrast;
  s.vertical_offset_px = c->vertical_offset_px;
  s.disparity_bias_px = c->disparity_bias_px;
  s.gain = c->gain;
  s.rad_bias = c->rad_bias;
  s.gamma = c->gamma;
  s.noise_sigma = c->noise_sigma;
  s.seed = c->seed;
  s.texture_quant = c->texture_quant;
  s.texture_cell_px = c->texture_cell_px;
  for (int i = 0; i < n; ++i) {
    SceneObject so;
    so.id = o[i].id;
    so.class_id = o[i].class_id;
    so.position = {o[i].px, o[i].py, o[i].pz};
    so.width_m = o[i].width_m;
    so.height_m = o[i].height_m;
    so.depth_m = o[i].depth_m;
    so.contrast = o[i].contrast;
    so.disparity_ramp = o[i].disparity_ramp;
    so.texture_seed = o[i].texture_seed;
    s.objects.push_back(so);
  }
  return s;
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument&) {
    return RG_EINVAL;
  } catch (...) {
    return RG_ECUDA;
  }
}

}  // namespace

extern "C" {

int ref_census_transform(const uint8_t* img, int w, int h, int ow, int oh, uint32_t* out) {
  return guarded([&] {
    const CensusImage c = census_transform(to_gray(img, w, h), ow, oh, 1);
    std::memcpy(out, c.codes.data(), sizeof(uint32_t) * c.codes.size());
    return RG_OK;
  });
}

int ref_census_transform_rois(const uint8_t* img, int w, int h, int ow, int oh,
                              const rg_rect* rois, int n_rois, uint32_t* out) {
  return guarded([&] {
    std::vector<CensusRoi> r(std::size_t(n_rois > 0 ? n_rois : 0));
    for (int i = 0; i < n_rois; ++i) r[i] = {rois[i].x0, rois[i].y0, rois[i].x1, rois[i].y1};
    const CensusImage c = census_transform_rois(to_gray(img, w, h), ow, oh, r, 1);
    std::memcpy(out, c.codes.data(), sizeof(uint32_t) * c.codes.size());
    return RG_OK;
  });
}

int ref_match_blocks(const uint32_t* left, int lw, int lh, const uint32_t* right, int rw, int rh,
                     const int32_t* points_xy, const int64_t* offsets,
                     const rg_search_range* ranges, int n_blocks, int mode, double tau_v,
                     rg_match_result* out) {
  return guarded([&] {
    const CensusImage L = to_census(left, lw, lh), R = to_census(right, rw, rh);
    for (int b = 0; b < n_blocks; ++b) {
      QueryBlock q;
      for (int64_t k = offsets[b]; k < offsets[b + 1]; ++k)
        q.points.emplace_back(points_xy[2 * k], points_xy[2 * k + 1]);
      q.dx_min = ranges[b].dx_min;
      q.dx_max = ranges[b].dx_max;
      q.dy_min = ranges[b].dy_min;
      q.dy_max = ranges[b].dy_max;
      fill_match(mode == RG_MATCH_FWD_BWD ? forward_backward_match(q, L, R, tau_v)
                                          : block_match(q, L, R),
                 &out[b]);
    }
    return RG_OK;
  });
}

int ref_select_objects(const rg_detection* dets, int n, const rg_ranger_config* cfg,
                       int32_t* out_idx, int* n_out) {
  return guarded([&] {
    const auto sel = select_objects(to_dets(dets, n), to_cfg(cfg));
    for (std::size_t i = 0; i < sel.size(); ++i) out_idx[i] = sel[i];
    *n_out = int(sel.size());
    return RG_OK;
  });
}

int ref_find_occluders(const rg_detection* dets, int n, int32_t* occ_offsets, int32_t* occ_idx) {
  return guarded([&] {
    const auto occ = find_occluders(to_dets(dets, n));
    int k = 0;
    for (int i = 0; i < n; ++i) {
      occ_offsets[i] = k;
      for (int j : occ[i]) occ_idx[k++] = j;
    }
    occ_offsets[n] = k;
    return RG_OK;
  });
}

int ref_sample_query_points(const rg_detection* det, int kind, const double* occ_boxes, int n_occ,
                            const rg_ranger_config* cfg, int w, int h, int64_t* block_offsets,
                            int32_t* points_xy, rg_search_range* ranges, int cap_blocks,
                            int64_t cap_points, int* n_blocks) {
  return guarded([&] {
    std::vector<PixelBox> ob(std::size_t(n_occ > 0 ? n_occ : 0));
    for (int i = 0; i < n_occ; ++i)
      ob[i] = {occ_boxes[4 * i], occ_boxes[4 * i + 1], occ_boxes[4 * i + 2], occ_boxes[4 * i + 3]};
    const auto blocks =
        sample_query_points(to_dets(det, 1)[0], kind == RG_KIND_FAR ? ObjectKind::kFar : ObjectKind::kClose,
                            ob, to_cfg(cfg), w, h);
    if (int(blocks.size()) > cap_blocks) return RG_EOVERFLOW;
    int64_t np = 0;
    block_offsets[0] = 0;
    for (std::size_t b = 0; b < blocks.size(); ++b) {
      for (const auto& [x, y] : blocks[b].points) {
        if (np >= cap_points) return RG_EOVERFLOW;
        points_xy[2 * np] = x;
        points_xy[2 * np + 1] = y;
        ++np;
      }
      block_offsets[b + 1] = np;
      ranges[b] = {blocks[b].dx_min, blocks[b].dx_max, blocks[b].dy_min, blocks[b].dy_max};
    }
    *n_blocks = int(blocks.size());
    return RG_OK;
  });
}

int ref_aggregate_close_disparities(const double* disps, int n, double tau_d, int n_min,
                                    int32_t* valid, double* disparity, int32_t* run_length) {
  return guarded([&] {
    const auto a = aggregate_close_disparities(std::vector<double>(disps, disps + n), tau_d, n_min);
    *valid = a.valid;
    *disparity = a.disparity;
    *run_length = a.run_length;
    return RG_OK;
  });
}

int ref_estimate_object_disparities(const uint8_t* left, const uint8_t* right, int w, int h,
                                    const rg_detection* dets, int n_dets, const rg_ranger_config* cfg,
                                    rg_census_cache* cache, double focal_px, double baseline_m,
                                    rg_object_disparity* out, int* n_out, rg_ranger_stats* stats) {
  if (cfg->census_9x7) return RG_EINVAL;  // the reference has only the 5x5 census
  return guarded([&] {
    const GrayImage L = to_gray(left, w, h), R = to_gray(right, w, h);
    const RangerConfig rc = to_cfg(cfg);
    CensusCache cc;
    const int s = rc.close_scale > 0 ? rc.close_scale : 1;
    const int cw = w / s, ch = h / s;
    if (cache) {
      if (cache->has_full) {
        cc.full_left = to_census(cache->full_left, w, h);
        cc.full_right = to_census(cache->full_right, w, h);
        cc.has_full = true;
      }
      if (cache->has_scaled) {
        cc.scaled_left = to_census(cache->scaled_left, cw, ch);
        cc.scaled_right = to_census(cache->scaled_right, cw, ch);
        cc.has_scaled = true;
      }
    }
    RangerStats st;
    const auto res = estimate_object_disparities(L, R, to_dets(dets, n_dets), rc, cache ? &cc : nullptr,
                                                 1, &st);
    if (cache) {
      if (!cache->has_full && cc.has_full) {
        std::memcpy(cache->full_left, cc.full_left.codes.data(), sizeof(uint32_t) * std::size_t(w) * h);
        std::memcpy(cache->full_right, cc.full_right.codes.data(), sizeof(uint32_t) * std::size_t(w) * h);
        cache->has_full = 1;
      }
      if (!cache->has_scaled && cc.has_scaled) {
        std::memcpy(cache->scaled_left, cc.scaled_left.codes.data(), sizeof(uint32_t) * std::size_t(cw) * ch);
        std::memcpy(cache->scaled_right, cc.scaled_right.codes.data(), sizeof(uint32_t) * std::size_t(cw) * ch);
        cache->has_scaled = 1;
      }
    }
    const StereoCalibration cal =
        (focal_px > 0 && baseline_m > 0) ? make_calibration(focal_px, baseline_m, w / 2.0, h / 2.0, 1.5)
                                         : StereoCalibration{};
    for (std::size_t i = 0; i < res.size(); ++i) {
      rg_object_disparity& o = out[i];
      std::memset(&o, 0, sizeof(o));
      o.det_id = res[i].det_id;
      o.kind = res[i].kind == ObjectKind::kFar ? RG_KIND_FAR : RG_KIND_CLOSE;
      o.n_blocks_used = res[i].n_blocks_used;
      o.valid = res[i].valid;
      o.disparity = res[i].disparity;
      if (res[i].valid && res[i].disparity > 0 && focal_px > 0 && baseline_m > 0) o.z_cam = reproject(0.0, 0.0, res[i].disparity, cal).z;
    }
    *n_out = int(res.size());
    if (stats) {
      stats->query_points = int64_t(st.query_points);
      stats->image_pixels = int64_t(st.image_pixels);
      stats->n_far = st.n_far;
      stats->n_close = st.n_close;
    }
    return RG_OK;
  });
}

int ref_bm_disparity(const uint8_t* left, const uint8_t* right, int w, int h, const rg_bm_params* p,
                     int16_t* out_raw) {
  return guarded([&] {
    const DisparityMap d = bm_disparity(to_gray(left, w, h), to_gray(right, w, h), to_bm(p), 1);
    std::memcpy(out_raw, d.raw.data(), sizeof(int16_t) * d.raw.size());
    return RG_OK;
  });
}

int ref_auto_rect_search(const uint8_t* left, const uint8_t* right, int w, int h, const rg_rect* roi,
                         int delta_min, int delta_max, const rg_bm_params* p, int32_t* best_delta,
                         int64_t* counts) {
  return guarded([&] {
    const GrayImage L = to_gray(left, w, h), R = to_gray(right, w, h);
    const BmParams bm = to_bm(p);
    const ImageRoi r{roi->x0, roi->y0, roi->x1, roi->y1};
    *best_delta = auto_rect_search(L, R, r, delta_min, delta_max, bm, 1);
    if (counts) {
      // per-delta counts as the search body computes them (autorect.hpp:37-44)
      const GrayImage rcrop = crop(R, r.x0, r.y0, r.width(), r.height());
      for (int d = delta_min; d <= delta_max; ++d) {
        const GrayImage lcrop = crop(shift_vertical(L, d), r.x0, r.y0, r.width(), r.height());
        const DisparityMap dm = bm_disparity(lcrop, rcrop, bm, 1);
        int64_t c = 0;
        const int lo = bm.min_disparity * DisparityMap::kSubLevels;
        for (std::int16_t v : dm.raw)
          if (v != DisparityMap::kInvalid && v > lo) ++c;
        counts[d - delta_min] = c;
      }
    }
    return RG_OK;
  });
}

/* auto_rect_search at `workers` (autorect.hpp:22-58: bm_disparity's rows in
 * `workers` threads per delta) plus the per-delta counts as the search body
 * computes them, the deltas spread over `workers` threads (each
 * bm_disparity at workers = 1; results are worker-count invariant,
 * test_bm.cpp / image.hpp:158-178). */
int ref_auto_rect_search_mt(const uint8_t* left, const uint8_t* right, int w, int h, const rg_rect* roi,
                            int delta_min, int delta_max, const rg_bm_params* p, int workers,
                            int32_t* best_delta, int64_t* counts) {
  return guarded([&] {
    const GrayImage L = to_gray(left, w, h), R = to_gray(right, w, h);
    const BmParams bm = to_bm(p);
    const ImageRoi r{roi->x0, roi->y0, roi->x1, roi->y1};
    if (workers < 1) workers = 1;
    *best_delta = auto_rect_search(L, R, r, delta_min, delta_max, bm, workers);
    if (counts) {
      const GrayImage rcrop = crop(R, r.x0, r.y0, r.width(), r.height());
      const int n = delta_max - delta_min + 1;
      std::vector<std::thread> pool;
      for (int t = 0; t < workers; ++t)
        pool.emplace_back([&, t] {
          for (int k = t; k < n; k += workers) {
            const int d = delta_min + k;
            const GrayImage lcrop = crop(shift_vertical(L, d), r.x0, r.y0, r.width(), r.height());
            const DisparityMap dm = bm_disparity(lcrop, rcrop, bm, 1);
            int64_t c = 0;
            const int lo = bm.min_disparity * DisparityMap::kSubLevels;
            for (std::int16_t v : dm.raw)
              if (v != DisparityMap::kInvalid && v > lo) ++c;
            counts[k] = c;
          }
        });
      for (auto& th : pool) th.join();
    }
    return RG_OK;
  });
}

int ref_render_stereo_pair(const rg_scene_config* cfg, const rg_scene_object* objs, int n_obj,
                           uint8_t* left, uint8_t* right) {
  return guarded([&] {
    const RenderResult r = render_stereo_pair(to_scene(cfg, objs, n_obj));
    std::memcpy(left, r.left.data.data(), r.left.data.size());
    std::memcpy(right, r.right.data.data(), r.right.data.size());
    return RG_OK;
  });
}

int ref_ground_truth_detections(const rg_scene_config* cfg, const rg_scene_object* objs, int n_obj,
                                rg_detection* out, int* n_out) {
  return guarded([&] {
    const auto d = ground_truth_detections(to_scene(cfg, objs, n_obj));
    for (std::size_t i = 0; i < d.size(); ++i) {
      out[i].cx = d[i].cx;
      out[i].cy = d[i].cy;
      out[i].w = d[i].w;
      out[i].h = d[i].h;
      out[i].class_id = d[i].class_id;
      out[i].id = d[i].id;
    }
    *n_out = int(d.size());
    return RG_OK;
  });
}

/* Frame-parallel ranging by the reference (SURVEY 8(d) mode iii): `threads`
 * host threads, each ranging whole frames with estimate_object_disparities
 * at workers = 1.  Records as rg_object_disparity (z_cam through the
 * reference's reproject when focal_px, baseline_m > 0, as
 * ref_estimate_object_disparities).  Returns the wall seconds of the ranging
 * (frame/detection marshalling excluded). */
double ref_range_frames(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                        const rg_detection* dets, const int32_t* det_offsets, const rg_ranger_config* cfg,
                        int threads, double focal_px, double baseline_m, rg_object_disparity* out,
                        int out_stride, int32_t* out_count) {
  const RangerConfig rc = to_cfg(cfg);
  std::vector<GrayImage> Ls, Rs;
  std::vector<std::vector<Detection>> D;
  for (int f = 0; f < n_frames; ++f) {
    Ls.push_back(to_gray(left + std::size_t(f) * w * h, w, h));
    Rs.push_back(to_gray(right + std::size_t(f) * w * h, w, h));
    D.push_back(to_dets(dets + det_offsets[f], det_offsets[f + 1] - det_offsets[f]));
  }
  const bool range_z = focal_px > 0 && baseline_m > 0;
  const StereoCalibration cal =
      range_z ? make_calibration(focal_px, baseline_m, w / 2.0, h / 2.0, 1.5) : StereoCalibration{};
  if (threads < 1) threads = 1;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (int f = t; f < n_frames; f += threads) {
        const auto res = estimate_object_disparities(Ls[f], Rs[f], D[f], rc, nullptr, 1, nullptr);
        if (out) {
          for (std::size_t i = 0; i < res.size() && int(i) < out_stride; ++i) {
            rg_object_disparity& o = out[std::size_t(f) * out_stride + i];
            std::memset(&o, 0, sizeof(o));
            o.det_id = res[i].det_id;
            o.kind = res[i].kind == ObjectKind::kFar ? RG_KIND_FAR : RG_KIND_CLOSE;
            o.n_blocks_used = res[i].n_blocks_used;
            o.valid = res[i].valid;
            o.disparity = res[i].disparity;
            if (range_z && res[i].valid && res[i].disparity > 0) o.z_cam = reproject(0.0, 0.0, res[i].disparity, cal).z;
          }
          out_count[f] = int32_t(res.size());
        }
      }
    });
  for (auto& th : pool) th.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double ref_bench_estimate(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                          const rg_detection* dets, const int32_t* det_offsets,
                          const rg_ranger_config* cfg, int threads, rg_object_disparity* out,
                          int out_stride, int32_t* out_count) {
  return ref_range_frames(left, right, w, h, n_frames, dets, det_offsets, cfg, threads, 0.0, 0.0, out, out_stride,
                          out_count);
}

/* The reference's render_stereo_pair + ground_truth_detections over a batch of
 * scenes on `threads` host threads (scene f = cfgs[f] with objects
 * objs[obj_offsets[f] .. obj_offsets[f+1])); frame f at byte f*W*H of left /
 * right, its detections at dets[obj_offsets[f] ..] (n_dets[f] of them). */
int ref_render_frames(const rg_scene_config* cfgs, const rg_scene_object* objs, const int32_t* obj_offsets,
                      int n_frames, int threads, uint8_t* left, uint8_t* right, rg_detection* dets,
                      int32_t* n_dets) {
  return guarded([&] {
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    std::vector<int> st(std::size_t(threads), RG_OK);
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        st[t] = guarded([&] {
          for (int f = t; f < n_frames; f += threads) {
            const std::size_t px = std::size_t(cfgs[f].width) * cfgs[f].height;
            const int o0 = obj_offsets[f], no = obj_offsets[f + 1] - obj_offsets[f];
            const SceneConfig sc = to_scene(&cfgs[f], objs + o0, no);
            const RenderResult r = render_stereo_pair(sc);
            std::memcpy(left + std::size_t(f) * px, r.left.data.data(), px);
            std::memcpy(right + std::size_t(f) * px, r.right.data.data(), px);
            if (dets) {
              const auto d = ground_truth_detections(sc);
              for (std::size_t i = 0; i < d.size(); ++i) {
                rg_detection& o = dets[o0 + i];
                o.cx = d[i].cx;
                o.cy = d[i].cy;
                o.w = d[i].w;
                o.h = d[i].h;
                o.class_id = d[i].class_id;
                o.id = d[i].id;
              }
              n_dets[f] = int32_t(d.size());
            }
          }
          return RG_OK;
        });
      });
    for (auto& th : pool) th.join();
    for (int v : st)
      if (v != RG_OK) return v;
    return RG_OK;
  });
}

/* SURVEY 8(d) CPU baseline detail: median seconds of `reps` runs of one
 * frame through the reference at `workers`: [0] estimate_object_disparities
 * (the production ROI-census path), [1] census_transform of both images,
 * [2] auto_rect_search over `roi` / [delta_min, delta_max] with `bm`
 * (skipped when reps_rect == 0). */
int ref_bench_stages(const uint8_t* left, const uint8_t* right, int w, int h, const rg_detection* dets, int n_dets,
                     const rg_ranger_config* cfg, int workers, int reps, const rg_rect* roi, int delta_min,
                     int delta_max, const rg_bm_params* bm, int reps_rect, double* out_s) {
  return guarded([&] {
    const GrayImage L = to_gray(left, w, h), R = to_gray(right, w, h);
    const std::vector<Detection> D = to_dets(dets, n_dets);
    const RangerConfig rc = to_cfg(cfg);
    auto median_of = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v.empty() ? 0.0 : v[v.size() / 2];
    };
    auto timed = [&](int n, auto&& fn) {
      std::vector<double> t;
      for (int r = 0; r < n; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        fn();
        t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      }
      return median_of(t);
    };
    out_s[0] = timed(reps, [&] { (void)estimate_object_disparities(L, R, D, rc, nullptr, workers, nullptr); });
    out_s[1] = timed(reps, [&] {
      (void)census_transform(L, workers);
      (void)census_transform(R, workers);
    });
    out_s[2] = 0.0;
    if (reps_rect > 0) {
      const ImageRoi r{roi->x0, roi->y0, roi->x1, roi->y1};
      const BmParams p = to_bm(bm);
      out_s[2] = timed(reps_rect, [&] { (void)auto_rect_search(L, R, r, delta_min, delta_max, p, workers); });
    }
    return RG_OK;
  });
}

/* Pipeline::process_frame (pipeline.hpp:124-266), TEMPLATE_MATCHER (method 0) or STEREO_BM (1),
 * over n_frames consecutive frames (packed w*h images, dets CSR); no radar.
 * out[f*out_stride + k], out_count[f]: PipelineResult::objects of frame f;
 * rect_applied[f]: RefinerLogRecord::rect_delta. */
int ref_pipeline_sequence(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                          const rg_detection* dets, const int32_t* det_offsets, const rg_ranger_config* cfg,
                          const rg_rect_search_config* rect, double f, double b, double cx, double cy,
                          double h_cam, int method, const rg_bm_params* bm, rg_object_disparity* out,
                          int out_stride, int32_t* out_count, double* rect_applied) {
  return guarded([&] {
    PipelineConfig pc;
    pc.method = method == 1 ? DepthMethod::kStereoBm : DepthMethod::kTemplateMatcher;
    if (bm) pc.bm = to_bm(bm);
    pc.calib = make_calibration(f, b, cx, cy, h_cam);
    pc.ranger = to_cfg(cfg);
    pc.rect.enabled = rect->enabled != 0;
    pc.rect.delta_min = rect->delta_min;
    pc.rect.delta_max = rect->delta_max;
    pc.rect.window = rect->window;
    pc.rect.rate_limit = rect->rate_limit;
    pc.rect.bm = to_bm(&rect->bm);
    pc.workers = 1;
    Pipeline pipe(pc);
    const std::size_t img = std::size_t(w) * h;
    for (int t = 0; t < n_frames; ++t) {
      FrameInput in;
      in.frame_id = t;
      in.left = to_gray(left + img * t, w, h);
      in.right = to_gray(right + img * t, w, h);
      in.detections = to_dets(dets + det_offsets[t], det_offsets[t + 1] - det_offsets[t]);
      PipelineResult res;
      pipe.process_frame(in, res);
      int k = 0;
      for (const auto& fo : res.objects) {
        if (k >= out_stride) break;
        rg_object_disparity& o = out[std::size_t(t) * out_stride + k++];
        std::memset(&o, 0, sizeof(o));
        o.det_id = fo.obj.det_id;
        o.kind = fo.obj.kind == ObjectKind::kFar ? RG_KIND_FAR : RG_KIND_CLOSE;
        o.n_blocks_used = fo.obj.n_blocks_used;
        o.valid = fo.obj.valid;
        o.disparity = fo.obj.disparity;
      }
      out_count[t] = k;
      rect_applied[t] = res.refiner_log.empty() ? 0.0 : res.refiner_log.back().rect_delta;
    }
    return RG_OK;
  });
}


/* Pipeline::process_frame with radar and the per-frame records: objects,
 * DepthRecord and RefinerLogRecord per frame (pipeline.hpp:124-265).
 * radar_xyz: CSR (radar_offsets, n_frames + 1) of vehicle-frame positions. */
int ref_pipeline_records(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                         const rg_detection* dets, const int32_t* det_offsets, const double* radar_xyz,
                         const int32_t* radar_offsets, const rg_ranger_config* cfg,
                         const rg_rect_search_config* rect, const rg_record_params* rp, int method,
                         const rg_bm_params* bm, rg_object_disparity* out, int out_stride, int32_t* out_count,
                         rg_depth_record* recs, rg_refiner_log* logs) {
  return guarded([&] {
    PipelineConfig pc;
    pc.method = method == 1 ? DepthMethod::kStereoBm : DepthMethod::kTemplateMatcher;
    if (bm) pc.bm = to_bm(bm);
    Mat3 R;
    for (int i = 0; i < 9; ++i) R.m[i] = rp->calib.R[i];
    pc.calib = make_calibration(rp->calib.f, rp->calib.b, rp->calib.cx, rp->calib.cy, rp->calib.h_cam, R,
                                Vec3{rp->calib.t[0], rp->calib.t[1], rp->calib.t[2]});
    pc.ranger = to_cfg(cfg);
    pc.rect.enabled = rect->enabled != 0;
    pc.rect.delta_min = rect->delta_min;
    pc.rect.delta_max = rect->delta_max;
    pc.rect.window = rect->window;
    pc.rect.rate_limit = rect->rate_limit;
    pc.rect.bm = to_bm(&rect->bm);
    pc.object_refiner = rp->object_refiner != 0;
    pc.radar_refiner = false;
    pc.obj_cand_half_px = rp->obj_cand_half_px;
    pc.obj_cand_step_px = rp->obj_cand_step_px;
    pc.tracker.fuse_sanity_ratio = rp->fuse_sanity_ratio;
    pc.class_width_m.clear();
    for (int i = 0; i < rp->n_class_widths; ++i) pc.class_width_m[rp->class_widths[i].class_id] = rp->class_widths[i].width_m;
    pc.workers = 1;
    Pipeline pipe(pc);
    const std::size_t img = std::size_t(w) * h;
    for (int t = 0; t < n_frames; ++t) {
      FrameInput in;
      in.frame_id = t;
      in.left = to_gray(left + img * t, w, h);
      in.right = to_gray(right + img * t, w, h);
      in.detections = to_dets(dets + det_offsets[t], det_offsets[t + 1] - det_offsets[t]);
      for (int j = radar_offsets[t]; j < radar_offsets[t + 1]; ++j) {
        RadarDetection r;
        r.position = Vec3{radar_xyz[3 * j], radar_xyz[3 * j + 1], radar_xyz[3 * j + 2]};
        in.radar.push_back(r);
      }
      PipelineResult res;
      pipe.process_frame(in, res);
      int k = 0;
      for (const auto& fo : res.objects) {
        if (k >= out_stride) break;
        rg_object_disparity& o = out[std::size_t(t) * out_stride + k];
        std::memset(&o, 0, sizeof(o));
        o.det_id = fo.obj.det_id;
        o.kind = fo.obj.kind == ObjectKind::kFar ? RG_KIND_FAR : RG_KIND_CLOSE;
        o.n_blocks_used = fo.obj.n_blocks_used;
        o.valid = fo.obj.valid;
        o.disparity = fo.obj.disparity;
        const DepthRecord& d = res.depth[std::size_t(k)];
        rg_depth_record& r = recs[std::size_t(t) * out_stride + k];
        r.frame_id = d.frame_id;
        r.det_id = d.det_id;
        r.disparity = d.disparity;
        r.valid = d.valid;
        r.source = d.source == DepthSource::kStereo ? RG_SRC_STEREO : d.source == DepthSource::kGpt ? RG_SRC_GPT : RG_SRC_SIZE;
        r.clp_by_stereo = d.clp_by_stereo;
        r.clp_by_gpt = d.clp_by_gpt;
        r.clp_by_size = d.clp_by_size;
        r.z_fused = d.z_fused;
        ++k;
      }
      out_count[t] = k;
      const RefinerLogRecord& lg = res.refiner_log.back();
      logs[t] = rg_refiner_log{lg.frame_id, 0, lg.rect_delta, lg.radar_offset, lg.obj_offset};
    }
    return RG_OK;
  });
}

/* Pipeline::process_frame with DepthMethod::kStereoBm and the radar
 * (dense-map) refiner on (pipeline.hpp:69, 182-183, 207-224), rect search
 * off: per frame the objects (box medians of the refined map) and the
 * refiner log's radar offset.  radar: CSR (radar_offsets) of position +
 * extent records. */
int ref_pipeline_dense_radar(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                             const rg_detection* dets, const int32_t* det_offsets, const rg_radar_detection* radar,
                             const int32_t* radar_offsets, const rg_ranger_config* cfg, const rg_calibration* cal,
                             const rg_bm_params* bm, int k_px, double lambda, double sigma_px,
                             rg_object_disparity* out, int out_stride, int32_t* out_count, double* radar_applied) {
  return guarded([&] {
    PipelineConfig pc;
    pc.method = DepthMethod::kStereoBm;
    pc.bm = to_bm(bm);
    Mat3 R;
    for (int i = 0; i < 9; ++i) R.m[i] = cal->R[i];
    pc.calib = make_calibration(cal->f, cal->b, cal->cx, cal->cy, cal->h_cam, R, Vec3{cal->t[0], cal->t[1], cal->t[2]});
    pc.ranger = to_cfg(cfg);
    pc.rect.enabled = false;
    pc.radar_refiner = true;
    pc.vote_half_range_px = k_px;
    pc.vote_lambda = lambda;
    pc.vote_smooth_sigma_px = sigma_px;
    pc.workers = 1;
    Pipeline pipe(pc);
    const std::size_t img = std::size_t(w) * h;
    for (int t = 0; t < n_frames; ++t) {
      FrameInput in;
      in.frame_id = t;
      in.left = to_gray(left + img * t, w, h);
      in.right = to_gray(right + img * t, w, h);
      in.detections = to_dets(dets + det_offsets[t], det_offsets[t + 1] - det_offsets[t]);
      for (int j = radar_offsets[t]; j < radar_offsets[t + 1]; ++j) {
        RadarDetection r;
        r.position = Vec3{radar[j].position.x, radar[j].position.y, radar[j].position.z};
        r.extent = Vec3{radar[j].extent.x, radar[j].extent.y, radar[j].extent.z};
        r.id = radar[j].id;
        in.radar.push_back(r);
      }
      PipelineResult res;
      pipe.process_frame(in, res);
      int k = 0;
      for (const auto& fo : res.objects) {
        if (k >= out_stride) break;
        rg_object_disparity& o = out[std::size_t(t) * out_stride + k];
        std::memset(&o, 0, sizeof(o));
        o.det_id = fo.obj.det_id;
        o.kind = fo.obj.kind == ObjectKind::kFar ? RG_KIND_FAR : RG_KIND_CLOSE;
        o.n_blocks_used = fo.obj.n_blocks_used;
        o.valid = fo.obj.valid;
        o.disparity = fo.obj.disparity;
        ++k;
      }
      out_count[t] = k;
      radar_applied[t] = res.refiner_log.back().radar_offset;
    }
    return RG_OK;
  });
}

/* make_synthetic_frames + save_synthetic_run (pipeline.hpp:415-471): a
 * reference-written run directory. */
int ref_save_synthetic_run(const rg_scene_config* sc, const rg_scene_object* objs, int n_obj, int n_frames,
                           double dt, const char* dir) {
  return guarded([&] {
    const SceneConfig scene = to_scene(sc, objs, n_obj);
    save_synthetic_run(make_synthetic_frames(scene, n_frames, dt), scene, dir);
    return RG_OK;
  });
}

/* load_run_directory -> Pipeline (TEMPLATE_MATCHER, calib.txt of the run,
 * radar refiner off) -> save_pipeline_outputs (pipeline.hpp:354-406). */
int ref_run_directory(const char* dir, const char* out_dir, const rg_ranger_config* cfg,
                      const rg_rect_search_config* rect, int object_refiner, double fuse_ratio) {
  return guarded([&] {
    PipelineConfig pc;
    pc.method = DepthMethod::kTemplateMatcher;
    pc.calib = load_calibration(std::string(dir) + "/calib.txt");
    pc.ranger = to_cfg(cfg);
    pc.rect.enabled = rect->enabled != 0;
    pc.rect.delta_min = rect->delta_min;
    pc.rect.delta_max = rect->delta_max;
    pc.rect.window = rect->window;
    pc.rect.rate_limit = rect->rate_limit;
    pc.rect.bm = to_bm(&rect->bm);
    pc.object_refiner = object_refiner != 0;
    pc.radar_refiner = false;
    pc.tracker.fuse_sanity_ratio = fuse_ratio;
    pc.workers = 1;
    save_pipeline_outputs(run_pipeline(pc, load_run_directory(dir)), out_dir);
    return RG_OK;
  });
}

int ref_dynamic_disparity_variance(const double* near_s, int n_near, const double* all_s, int n_all,
                                   double sigma_obs2, double gamma, double sigma_sys2, double* out) {
  return guarded([&] {
    const std::vector<double> a(near_s, near_s + n_near), b(all_s, all_s + n_all);
    *out = dynamic_disparity_variance(a, b, sigma_obs2, gamma, sigma_sys2);
    return RG_OK;
  });
}

int ref_sgm_direction_pass(const uint8_t* cost, int w, int h, int nd, int p1, int p2, int sx, int sy,
                           int32_t* acc) {
  return guarded([&] {
    const std::vector<std::uint8_t> c(cost, cost + std::size_t(w) * h * nd);
    std::vector<std::int32_t> a(acc, acc + std::size_t(w) * h * nd);
    detail::sgm_direction_pass(c, w, h, nd, p1, p2, sx, sy, a);
    std::memcpy(acc, a.data(), sizeof(int32_t) * a.size());
    return RG_OK;
  });
}

int ref_sgm_disparity(const uint8_t* left, const uint8_t* right, int w, int h, int nd, int d_lo, int p1, int p2,
                      int16_t* out) {
  return guarded([&] {
    SgmParams p;
    p.num_disparities = nd;
    p.min_disparity = d_lo;
    p.p1 = p1;
    p.p2 = p2;
    const DisparityMap m = sgm_disparity(to_gray(left, w, h), to_gray(right, w, h), p, 1);
    std::memcpy(out, m.raw.data(), sizeof(int16_t) * m.raw.size());
    return RG_OK;
  });
}

}  // extern "C"
