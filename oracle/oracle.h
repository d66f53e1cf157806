/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU checker for the B200 census ranger.  Two implementations share this
 * interface:
 *   orc_*  ranger_oracle.c : a plain-C restatement of the reference algorithm
 *                            (each function cites the reference file:line).
 *   ref_*  ref_shim.cpp    : the reference's own headers
 *                            (/root/reference/proj/include) compiled in place
 *                            into oracle/_ref/libranger_ref.so.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load either library, and only as the checker / baseline -- never as the
 * product path.  Types come from the public C ABI header so both sides of a
 * parity test read the same structs.
 */
#ifndef RANGER_ORACLE_H_
#define RANGER_ORACLE_H_

#include "../include/ranger_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_DECL(prefix)                                                                  \
  int prefix##census_transform(const uint8_t* img, int w, int h, int ow, int oh,        \
                               uint32_t* out);                                           \
  int prefix##census_transform_rois(const uint8_t* img, int w, int h, int ow, int oh,   \
                                    const rg_rect* rois, int n_rois, uint32_t* out);     \
  int prefix##match_blocks(const uint32_t* left, int lw, int lh, const uint32_t* right,  \
                           int rw, int rh, const int32_t* points_xy,                     \
                           const int64_t* offsets, const rg_search_range* ranges,        \
                           int n_blocks, int mode, double tau_v, rg_match_result* out);  \
  int prefix##select_objects(const rg_detection* dets, int n, const rg_ranger_config* cfg, \
                             int32_t* out_idx, int* n_out);                              \
  int prefix##find_occluders(const rg_detection* dets, int n, int32_t* occ_offsets,      \
                             int32_t* occ_idx);                                          \
  int prefix##sample_query_points(const rg_detection* det, int kind,                     \
                                  const double* occ_boxes, int n_occ,                    \
                                  const rg_ranger_config* cfg, int w, int h,             \
                                  int64_t* block_offsets, int32_t* points_xy,            \
                                  rg_search_range* ranges, int cap_blocks,               \
                                  int64_t cap_points, int* n_blocks);                    \
  int prefix##aggregate_close_disparities(const double* disps, int n, double tau_d,      \
                                          int n_min, int32_t* valid, double* disparity,  \
                                          int32_t* run_length);                          \
  int prefix##estimate_object_disparities(                                               \
      const uint8_t* left, const uint8_t* right, int w, int h, const rg_detection* dets, \
      int n_dets, const rg_ranger_config* cfg, rg_census_cache* cache, double focal_px,  \
      double baseline_m, rg_object_disparity* out, int* n_out, rg_ranger_stats* stats);  \
  int prefix##bm_disparity(const uint8_t* left, const uint8_t* right, int w, int h,      \
                           const rg_bm_params* p, int16_t* out_raw);                     \
  int prefix##auto_rect_search(const uint8_t* left, const uint8_t* right, int w, int h,  \
                               const rg_rect* roi, int delta_min, int delta_max,         \
                               const rg_bm_params* p, int32_t* best_delta,               \
                               int64_t* counts);

ORC_DECL(orc_)
ORC_DECL(ref_)

/* 9x7 / uint64 extension (restatement only; no reference function) */
int orc_census_transform64(const uint8_t* img, int w, int h, int ow, int oh, uint64_t* out);
int orc_match_blocks64(const uint64_t* left, int lw, int lh, const uint64_t* right, int rw, int rh,
                       const int32_t* points_xy, const int64_t* offsets,
                       const rg_search_range* ranges, int n_blocks, int mode, double tau_v,
                       rg_match_result* out);

/* SGM (8f row 2): sgm.hpp:37-155 */
int orc_sgm_direction_pass(const uint8_t* cost, int w, int h, int nd, int p1, int p2, int sx, int sy,
                           int32_t* acc);
int orc_sgm_disparity(const uint8_t* left, const uint8_t* right, int w, int h, int nd, int d_lo, int p1, int p2,
                      int16_t* out);
int ref_sgm_direction_pass(const uint8_t* cost, int w, int h, int nd, int p1, int p2, int sx, int sy,
                           int32_t* acc);
int ref_sgm_disparity(const uint8_t* left, const uint8_t* right, int w, int h, int nd, int d_lo, int p1, int p2,
                      int16_t* out);

/* dense BM objects (8f row 3): pipeline.hpp:304-328 */
int orc_box_disparity(const int16_t* raw, int w, int h, const rg_detection* dets, int n, double sigma_obs2,
                      double gamma, double sigma_sys2, rg_box_stats* out);
/* geometry.hpp:162-178 on explicit samples (pins the restatement's variance) */
int ref_dynamic_disparity_variance(const double* near_s, int n_near, const double* all_s, int n_all,
                                   double sigma_obs2, double gamma, double sigma_sys2, double* out);

/* reference-only extras (ref_shim.cpp) */
int ref_render_stereo_pair(const rg_scene_config* cfg, const rg_scene_object* objs,
                           int n_obj, uint8_t* left, uint8_t* right);
int ref_ground_truth_detections(const rg_scene_config* cfg, const rg_scene_object* objs,
                                int n_obj, rg_detection* out, int* n_out);
int ref_pipeline_sequence(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                          const rg_detection* dets, const int32_t* det_offsets, const rg_ranger_config* cfg,
                          const rg_rect_search_config* rect, double f, double b, double cx, double cy,
                          double h_cam, int method, const rg_bm_params* bm, rg_object_disparity* out,
                          int out_stride, int32_t* out_count, double* rect_applied);
int ref_pipeline_records(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                         const rg_detection* dets, const int32_t* det_offsets, const double* radar_xyz,
                         const int32_t* radar_offsets, const rg_ranger_config* cfg,
                         const rg_rect_search_config* rect, const rg_record_params* rp, int method,
                         const rg_bm_params* bm, rg_object_disparity* out, int out_stride, int32_t* out_count,
                         rg_depth_record* recs, rg_refiner_log* logs);
int ref_pipeline_dense_radar(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                             const rg_detection* dets, const int32_t* det_offsets, const rg_radar_detection* radar,
                             const int32_t* radar_offsets, const rg_ranger_config* cfg, const rg_calibration* cal,
                             const rg_bm_params* bm, int k_px, double lambda, double sigma_px,
                             rg_object_disparity* out, int out_stride, int32_t* out_count, double* radar_applied);
int ref_save_synthetic_run(const rg_scene_config* sc, const rg_scene_object* objs, int n_obj, int n_frames,
                           double dt, const char* dir);
int ref_run_directory(const char* dir, const char* out_dir, const rg_ranger_config* cfg,
                      const rg_rect_search_config* rect, int object_refiner, double fuse_ratio);
/* CPU baseline: range n_frames frames (left/right packed w*h each, dets CSR)
 * with `threads` host threads, each thread ranging whole frames at workers=1
 * (SURVEY.md 8(d) mode iii); returns wall seconds, fills out like
 * rg_range_frames (out_stride per frame). */
double ref_bench_estimate(const uint8_t* left, const uint8_t* right, int w, int h,
                          int n_frames, const rg_detection* dets,
                          const int32_t* det_offsets, const rg_ranger_config* cfg,
                          int threads, rg_object_disparity* out, int out_stride,
                          int32_t* out_count);
/* ref_bench_estimate with z_cam (reference reproject) when focal_px,
 * baseline_m > 0 -- the checker for the bench's parity sweep. */
double ref_range_frames(const uint8_t* left, const uint8_t* right, int w, int h, int n_frames,
                        const rg_detection* dets, const int32_t* det_offsets, const rg_ranger_config* cfg,
                        int threads, double focal_px, double baseline_m, rg_object_disparity* out,
                        int out_stride, int32_t* out_count);
/* The reference's render_stereo_pair + ground_truth_detections for a batch of
 * scenes on `threads` host threads (frame f at byte f*W*H; dets at
 * dets[obj_offsets[f]..], n_dets[f] of them; dets may be NULL). */
int ref_render_frames(const rg_scene_config* cfgs, const rg_scene_object* objs, const int32_t* obj_offsets,
                      int n_frames, int threads, uint8_t* left, uint8_t* right, rg_detection* dets,
                      int32_t* n_dets);
/* auto_rect_search at `workers` + per-delta counts over `workers` threads */
int ref_auto_rect_search_mt(const uint8_t* left, const uint8_t* right, int w, int h, const rg_rect* roi,
                            int delta_min, int delta_max, const rg_bm_params* p, int workers,
                            int32_t* best_delta, int64_t* counts);
int ref_bench_stages(const uint8_t* left, const uint8_t* right, int w, int h, const rg_detection* dets, int n_dets,
                     const rg_ranger_config* cfg, int workers, int reps, const rg_rect* roi, int delta_min,
                     int delta_max, const rg_bm_params* bm, int reps_rect, double* out_s);

#ifdef __cplusplus
}
#endif
#endif
