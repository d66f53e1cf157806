/*
 * ranger_cuda.h -- C ABI of the B200-native census template-matching ranger.
 *
 * This is the drop-in boundary for the reference's hot path (the header-only
 * C++ API in proj/include/ranger/ of arxiv/paper_2604_07980).  Every entry
 * point below names the reference interface it replaces (file:line, relative
 * to the reference's proj/include/ranger/).  The C++ facade in
 * include/ranger/ (*.hpp) keeps the reference declarations verbatim and forwards
 * here; Python binds the same symbols with ctypes.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / CUDA types in signatures
 *     (streams are passed as void* = cudaStream_t).
 *   - every function returns an rg_status; on failure rg_last_error(ctx)
 *     holds a message.  RG_EINVAL maps to std::invalid_argument in the
 *     facade (reference: census.hpp:71-74, template_match.hpp:48-61,
 *     autorect.hpp:25-32, bm.hpp:24-32), everything else to
 *     std::runtime_error.
 *   - "host" arguments are ordinary host memory; "d_" arguments are device
 *     pointers on the context's device.
 *   - a context is single-writer (one host thread at a time), like the
 *     reference's CensusCache; create one per host thread for concurrency.
 */
#ifndef RANGER_CUDA_H_
#define RANGER_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int rg_status;
#define RG_OK 0
#define RG_EINVAL 1   /* invalid argument  -> std::invalid_argument */
#define RG_ECUDA 2    /* CUDA runtime error -> std::runtime_error   */
#define RG_ENOMEM 3   /* allocation failure -> std::runtime_error   */
#define RG_EOVERFLOW 4 /* device work list overflowed; call again    */

/* Object kinds, reference census.hpp:143 (enum class ObjectKind). */
#define RG_KIND_FAR 0
#define RG_KIND_CLOSE 1

/* Match modes for rg_match_blocks. */
#define RG_MATCH_FORWARD 0 /* block_match, census.hpp:178-272            */
#define RG_MATCH_FWD_BWD 1 /* forward_backward_match, census.hpp:281-303 */

typedef struct rg_ctx rg_ctx;

/* ---------------------------------------------------------------- context */
rg_status rg_ctx_create(int device, rg_ctx** out);
void rg_ctx_destroy(rg_ctx* ctx);
const char* rg_last_error(const rg_ctx* ctx);
/* message of the last failed rg_ctx_create on this thread */
const char* rg_create_error(void);
/* library build identification: "sm_100a <git-describe-ish>" */
const char* rg_build_info(void);
/* Self-test of the matcher's integer division (Markstein correction on a
 * table of RN(1/b)) against IEEE division on the device, for every
 * b in [1, b_max] and 0 <= a <= 64 b; *mismatches = 0 when exact. */
rg_status rg_selftest_division(rg_ctx* ctx, int b_max, int64_t* mismatches);

/* Per-stage CUDA-event timing of the batched API (off by default). */
rg_status rg_set_profiling(rg_ctx* ctx, int on);
/* rg_range_frames schedule: 0 (default) = one stream, census then matcher
 * for the whole batch; 1 = chunks whose census runs on a low-priority stream
 * while the previous chunk's matcher runs on a high-priority one.  Results
 * are identical; on B200 the overlap measured 5-10 % SLOWER (the streaming
 * census evicts the matcher's L2-resident rows), so it is opt-in. */
rg_status rg_set_overlap(rg_ctx* ctx, int on);
/* on (default): batches of >= 12 frames compute only the census codes the
 * matcher reads (ROI tiles); off: the full-frame census for every batch
 * (same records; a measurement / comparison switch). */
rg_status rg_set_census_rois(rg_ctx* ctx, int on);
/* Accumulated stage milliseconds and launch counts since the last reset:
 * times[0..4] = census, plan, match, aggregate, autorect;
 * launches[0..4] likewise; returns the total kernel launch count in *total. */
rg_status rg_get_counters(rg_ctx* ctx, double times_ms[5], int64_t launches[5],
                          int64_t* total_launches);
rg_status rg_reset_counters(rg_ctx* ctx);
/* Algorithmic work of the batched path since the last reset: Hamming
 * evaluations (sum over blocks and candidates of contributing points,
 * census.hpp:209-221, forward + backward) and planned blocks (slots). */
rg_status rg_get_work(rg_ctx* ctx, int64_t* hamming_evals, int64_t* blocks);
/* Host <-> device bytes moved by rg_range_frames_host since the last
 * rg_reset_counters (frames, detections, offsets, shifts in; records and
 * counts out).  With pinned caller frames and batches that take the ROI
 * census, only the image bytes the census reads are fetched (zero-copy, in
 * 16-B segments); otherwise whole frames are copied. */
rg_status rg_get_transfer(rg_ctx* ctx, int64_t* h2d_bytes, int64_t* d2h_bytes);

/* ---------------------------------------------------------------- types */

/* CensusRoi (census.hpp:93) and ImageRoi (autorect.hpp:13-17): half-open. */
typedef struct {
  int32_t x0, y0, x1, y1;
} rg_rect;

/* QueryBlock search ranges (census.hpp:146-152), inclusive. */
typedef struct {
  int32_t dx_min, dx_max, dy_min, dy_max;
} rg_search_range;

/* MatchResult (census.hpp:154-163) plus std::optional engagement. */
typedef struct {
  int32_t dx_int;
  int32_t dy_int;
  double dx_subpix;
  double cost;
  double cost_minus;
  double cost_plus;
  int32_t valid_points;
  int32_t verified;
  int32_t has_value; /* 0 = std::nullopt                                  */
  int32_t n_points;  /* sampled points of the block (planner path)        */
} rg_match_result;

/* Detection (detection.hpp:8-12); identical layout to ranger::Detection. */
typedef struct {
  double cx, cy, w, h;
  int32_t class_id;
  int32_t id;
} rg_detection;

/* RangerConfig (template_match.hpp:33-46) with FrontalCrop flattened. */
typedef struct {
  double tau_s;
  int32_t close_scale;
  int32_t grid_side_points;
  int32_t max_total_points;
  int32_t close_block_side_points;
  double tau_d;
  int32_t n_min;
  int32_t max_objects;
  double tau_v;
  double crop_x0, crop_y0, crop_x1, crop_y1;
  int32_t dx_max_far;
  int32_t dx_max_close;
  /* extension (BASELINE config 1): 1 = 9x7 census, 64-bit
   * descriptors (63 compares + sentinel bit 63); 0 = the reference's 5x5. */
  int32_t census_9x7;
  int32_t reserved;
} rg_ranger_config;

/* ObjectDisparity (template_match.hpp:18-24) plus the range z_cam
 * (geometry.hpp:142-146, 198-211) when a calibration is supplied. */
typedef struct {
  int32_t det_id;
  int32_t kind;
  int32_t n_blocks_used;
  int32_t valid;
  double disparity;
  double z_cam; /* 0 when invalid or no calibration */
} rg_object_disparity;

/* RangerStats (template_match.hpp:236-241). */
typedef struct {
  int64_t query_points;
  int64_t image_pixels;
  int32_t n_far;
  int32_t n_close;
} rg_ranger_stats;

/* CensusCache (template_match.hpp:229-234).  Buffers are caller-owned host
 * arrays: full_* hold w*h codes, scaled_* hold (w/s)*(h/s) codes.  has_* on
 * input: the buffer holds codes to be used as-is.  On output has_* is set to
 * 1 when this call filled the buffers (ROI-masked codes, as the reference). */
typedef struct {
  uint32_t* full_left;
  uint32_t* full_right;
  uint32_t* scaled_left;
  uint32_t* scaled_right;
  int32_t has_full;
  int32_t has_scaled;
} rg_census_cache;

/* BmParams (bm.hpp:15-22). */
typedef struct {
  int32_t num_disparities;
  int32_t block_size;
  int32_t min_disparity;
  int32_t downscale;
  double texture_threshold;
  double uniqueness_ratio;
} rg_bm_params;

/* ------------------------------------------------------ census (K1) */

/* census_code_at, census.hpp:43-56 */
rg_status rg_census_code_at(rg_ctx* ctx, const uint8_t* img, int w, int h, int sx,
                            int sy, uint32_t* code);
/* census_transform, census.hpp:69-90 (out = src dims gives census.hpp:88-90) */
rg_status rg_census_transform(rg_ctx* ctx, const uint8_t* img, int w, int h,
                              int out_w, int out_h, uint32_t* codes);
/* census_transform_rois, census.hpp:100-138 */
rg_status rg_census_transform_rois(rg_ctx* ctx, const uint8_t* img, int w, int h,
                                   int out_w, int out_h, const rg_rect* rois,
                                   int n_rois, uint32_t* codes);

/* 9x7 census extension: code = 1, then for window rows -3..3 and
 * columns -4..4 (row-major) code = code << 1 | (I(x+i, y+j) > I(x, y)); the
 * sentinel ends in bit 63; 0 when the window leaves the image (x < 4,
 * y < 3, x >= W-4, y >= H-3).  Same reduced-raster mapping as census.hpp:59-64.
 * No reference function exists (parity unpinned by the reference's tests). */
rg_status rg_census_transform64(rg_ctx* ctx, const uint8_t* img, int w, int h, int out_w,
                                int out_h, uint64_t* codes);

/* ------------------------------------------------------ matcher (K2) */

/* block_match (census.hpp:178-272), forward_backward_match (:281-303) and
 * batch_match (:307-315) over n_blocks blocks given in CSR form:
 * points_xy[2*k], points_xy[2*k+1] for k in [offsets[b], offsets[b+1]).
 * left/right are census rasters (lw x lh, rw x rh codes, row-major). */
rg_status rg_match_blocks(rg_ctx* ctx, const uint32_t* left, int lw, int lh,
                          const uint32_t* right, int rw, int rh,
                          const int32_t* points_xy, const int64_t* offsets,
                          const rg_search_range* ranges, int n_blocks, int mode,
                          double tau_v, rg_match_result* out);

/* rg_match_blocks over 64-bit (9x7) descriptors */
rg_status rg_match_blocks64(rg_ctx* ctx, const uint64_t* left, int lw, int lh,
                            const uint64_t* right, int rw, int rh, const int32_t* points_xy,
                            const int64_t* offsets, const rg_search_range* ranges, int n_blocks,
                            int mode, double tau_v, rg_match_result* out);

/* ------------------------------------------------------ object ranger */

/* validate(const RangerConfig&), template_match.hpp:48-61 */
rg_status rg_validate_ranger_config(rg_ctx* ctx, const rg_ranger_config* cfg);

/* select_objects, template_match.hpp:94-114 (priority order, truncated). */
rg_status rg_select_objects(rg_ctx* ctx, const rg_detection* dets, int n,
                            const rg_ranger_config* cfg, int32_t* out_idx,
                            int* n_out);
/* find_occluders, template_match.hpp:71-89; CSR out, occ_idx capacity n*n. */
rg_status rg_find_occluders(rg_ctx* ctx, const rg_detection* dets, int n,
                            int32_t* occ_offsets, int32_t* occ_idx);
/* sample_query_points, template_match.hpp:155-223.  occluder_boxes holds
 * n_occ PixelBoxes as (x0,y0,x1,y1) doubles.  Output CSR capacity:
 * cap_blocks blocks / cap_points points; *n_blocks receives the count. */
rg_status rg_sample_query_points(rg_ctx* ctx, const rg_detection* det, int kind,
                                 const double* occluder_boxes, int n_occ,
                                 const rg_ranger_config* cfg, int img_w, int img_h,
                                 int64_t* block_offsets, int32_t* points_xy,
                                 rg_search_range* ranges, int cap_blocks,
                                 int64_t cap_points, int* n_blocks);
/* aggregate_close_disparities, template_match.hpp:126-148 */
rg_status rg_aggregate_close_disparities(rg_ctx* ctx, const double* disps, int n,
                                         double tau_d, int n_min, int32_t* valid,
                                         double* disparity, int32_t* run_length);

/* estimate_object_disparities, template_match.hpp:260-363.  out has room for
 * n_dets entries; *n_out receives the number written (selected objects, in
 * input order).  cache and stats may be NULL.  focal_px/baseline_m > 0 also
 * fill z_cam (geometry.hpp:142-146). */
rg_status rg_estimate_object_disparities(rg_ctx* ctx, const uint8_t* left,
                                         const uint8_t* right, int w, int h,
                                         const rg_detection* dets, int n_dets,
                                         const rg_ranger_config* cfg,
                                         rg_census_cache* cache, double focal_px,
                                         double baseline_m, rg_object_disparity* out,
                                         int* n_out, rg_ranger_stats* stats);

/* Batched frame ranging -- the throughput path (one process per GPU).
 * Frames f in [0, n_frames): left/right images at base + f*frame_stride,
 * rows `pitch` bytes apart (pitch >= width, multiple of 16 for the fast
 * census path).  Detections of frame f: dets[det_offsets[f] .. det_offsets[f+1]).
 * Results: out[f*out_stride + k] for k < out_count[f] (selected objects in
 * input order); out_stride >= min(max_dets_per_frame, cfg.max_objects).
 * All pointers are device pointers.  The call is ASYNCHRONOUS on `stream`: it
 * returns once the batch is enqueued (no host synchronisation); the batch's
 * buffers must stay valid until the stream has run it.  Its planner counters
 * come back asynchronously and are inspected by later calls and by rg_sync:
 * a batch whose internal block list overflowed produced no results (its
 * out_count entries are not written), the list grows for later batches, and
 * the next rg_sync returns RG_EOVERFLOW -- resubmit that batch.  The list
 * starts at 512 blocks per frame (C2 plans 496), so a steady workload
 * overflows at most once.  Consecutive batches may use different streams
 * (the library orders them); every other entry point waits for the
 * context's pending batches first.  With rg_set_sync_mode(ctx, 1), or while
 * profiling / the overlap schedule is on, the call blocks and re-runs an
 * overflowed batch itself. */
typedef struct {
  int32_t n_frames;
  int32_t width;
  int32_t height;
  int32_t pitch;
  int64_t frame_stride;
  const uint8_t* d_left;
  const uint8_t* d_right;
  const rg_detection* d_dets;
  const int32_t* d_det_offsets; /* n_frames + 1 */
  int32_t max_dets_per_frame;
  int32_t out_stride;
  rg_object_disparity* d_out;
  int32_t* d_out_count;
  double focal_px;   /* <= 0: no range */
  double baseline_m;
  /* nullable, n_frames entries: vertical shift applied to frame f's LEFT image
   * before ranging, shift_vertical(left, s) (image.hpp:145-154; the rect
   * correction of pipeline.hpp:135-138), folded into the census row addressing */
  const int32_t* d_left_shift;
  /* nullable, n_frames*out_stride entries: receives the frame-local index of
   * the detection behind d_out[f*out_stride + k] (the sorted `sel` of
   * pipeline.hpp:140-141).  Device batches only: rg_range_frames_host rejects
   * a non-null value. */
  int32_t* d_out_index;
} rg_frame_batch;

rg_status rg_range_frames(rg_ctx* ctx, const rg_frame_batch* batch,
                          const rg_ranger_config* cfg, void* stream);

/* Wait for every asynchronous rg_range_frames batch of the context; returns
 * RG_EOVERFLOW if any of them overflowed since the last rg_sync (those
 * batches must be submitted again), else RG_OK. */
rg_status rg_sync(rg_ctx* ctx);
/* 1: rg_range_frames blocks until its batch is done and re-runs it itself on
 * overflow (the behaviour before asynchronous batches); 0 (default): async. */
rg_status rg_set_sync_mode(rg_ctx* ctx, int on);

/* Host-buffer variant of rg_range_frames: left/right/dets/offsets/out/count are
 * HOST pointers (pinned memory recommended).  The library streams frames
 * through device staging in chunks of `chunk` frames with copy/compute
 * overlap and returns after the results are on the host. */
rg_status rg_range_frames_host(rg_ctx* ctx, const rg_frame_batch* batch,
                               const rg_ranger_config* cfg, int chunk, void* stream);

/* ------------------------------------------------- multi-GPU */
/* Frames shard contiguously over devices: frame f of n runs on rank
 * floor(f * world / n), i.e. [lo, hi) = [ceil(rank n / world), ceil((rank+1) n / world)). */
rg_status rg_shard_bounds(int n_frames, int rank, int world, int* lo, int* hi);

/* One context, stream pair and host thread per device, NCCL communicators over
 * them (system libnccl.so.2, opened at create).  Devices must be distinct. */
typedef struct rg_multi rg_multi;
rg_status rg_multi_create(const int* devices, int n_devices, rg_multi** out);
void rg_multi_destroy(rg_multi* m);
const char* rg_multi_last_error(const rg_multi* m);

/* A HOST batch (pointers as rg_range_frames_host; no left shift or out index)
 * ranged with its frames sharded over the handle's devices: each device
 * stages its shard (pinned host -> device copies overlapping its asynchronous
 * batches of `chunk` frames) and ranges it; the per-box records are then
 * gathered IN FRAME ORDER to d_out0 / d_count0 (DEVICE pointers on the first
 * device, n_frames * out_stride records and n_frames counts; nullable) by
 * NCCL send/recv, and/or copied to h_out / h_count (HOST, nullable) by each
 * device over its own link.  Blocks until done.  Replaces the frame loop of
 * Pipeline::run (pipeline.hpp:338-344) for the ranging stage; the sequential
 * per-frame state stays with the caller. */
rg_status rg_multi_range_host(rg_multi* m, const rg_frame_batch* batch, const rg_ranger_config* cfg, int chunk,
                              rg_object_disparity* d_out0, int32_t* d_count0, rg_object_disparity* h_out,
                              int32_t* h_count);

/* ------------------------------------------------- sequence orchestration */

/* RectSearchConfig (pipeline.hpp:52-62): the per-frame vertical-offset search
 * and its filter, as Pipeline::process_frame runs them (pipeline.hpp:135-178). */
typedef struct {
  int32_t enabled;
  int32_t delta_min, delta_max;
  int32_t window;      /* median filter length, frames */
  double rate_limit;   /* max applied-offset change, px per frame */
  rg_bm_params bm;     /* reference default {32, 9, -4, 10, 10, 1} */
} rg_rect_search_config;

#define RG_RECT_MAX_WINDOW 64
/* RectOffsetState (autorect.hpp:62-75), carried across calls by the caller. */
typedef struct {
  int32_t window;
  int32_t n_hist;  /* history.size() */
  int32_t next;
  int32_t pad;
  double delta_max;
  double current;  /* applied offset */
  int32_t history[RG_RECT_MAX_WINDOW];
} rg_rect_state;

/* RectOffsetState(k, rate) (autorect.hpp:69-72); k in [1, RG_RECT_MAX_WINDOW]. */
rg_status rg_rect_state_init(rg_rect_state* st, int window, double rate);
/* filter_offset (autorect.hpp:77-90): push delta*, return the applied offset. */
rg_status rg_filter_offset(rg_rect_state* st, int delta_star, double* applied);

/* The TEMPLATE_MATCHER frame loop of Pipeline::process_frame over a batch of
 * consecutive frames (pipeline.hpp:124-178), as the two-pass schedule of
 * pass A runs the offset search on every UNCORRECTED pair
 * (rect_search_roi = central half, pipeline.hpp:268-275) on the device; the
 * host then walks the frames in order -- shift_f = lround(st.current) before
 * frame f's filter update (pipeline.hpp:135-138, 178); pass B ranges
 * shift_vertical(left_f, shift_f) with the shift folded into the census row
 * addressing.  `b` holds DEVICE pointers as for rg_range_frames (its
 * d_left_shift is ignored); `st` is updated in place; out_shift / out_delta
 * (HOST, n_frames entries, nullable) receive the applied shifts and the raw
 * search results; out_rect_applied (HOST, nullable) the filtered offset in
 * force for each frame (RefinerLogRecord::rect_delta).  Asynchronous on
 * `stream` after the host scan. */
rg_status rg_range_sequence(rg_ctx* ctx, const rg_frame_batch* b, const rg_ranger_config* cfg,
                            const rg_rect_search_config* rect, rg_rect_state* st,
                            int32_t* out_shift, int32_t* out_delta, double* out_rect_applied,
                            void* stream);

/* ------------------------------------------ per-frame records (host side) */

/* The sequential tail of Pipeline::process_frame (pipeline.hpp:180-265 minus
 * the tracker): object refiner, the stereo / ground-point / size cues,
 * fuse_depth -> DepthRecord, RefinerLogRecord.  Host code (a few hundred
 * flops per object), run after the device results of a batch are back. */

/* StereoCalibration (geometry.hpp:101-110); R row-major camera -> vehicle.
 * Q is derived as make_calibration does (geometry.hpp:118-127). */
typedef struct {
  double f, b, cx, cy, h_cam;
  double R[9];
  double t[3];
} rg_calibration;

typedef struct {
  double x, y, z;
} rg_vec3;

/* ObjRefinerState (object_refiner.hpp:14-21) */
typedef struct {
  double prev_offset, beta, r_max, w_p, tau, rate_limit;
} rg_obj_refiner_state;

/* one entry of PipelineConfig::class_width_m (pipeline.hpp:78) */
typedef struct {
  int32_t class_id;
  int32_t pad;
  double width_m;
} rg_class_width;

typedef struct {
  rg_calibration calib;
  const rg_class_width* class_widths; /* host, n_class_widths entries, distinct ids */
  int32_t n_class_widths;
  int32_t object_refiner;   /* PipelineConfig::object_refiner (pipeline.hpp:66) */
  double obj_cand_half_px;  /* pipeline.hpp:72 */
  double obj_cand_step_px;
  double fuse_sanity_ratio; /* TrackerConfig::fuse_sanity_ratio (tracker.hpp:18) */
} rg_record_params;

/* DepthSource (geometry.hpp:187) */
enum { RG_SRC_STEREO = 0, RG_SRC_GPT = 1, RG_SRC_SIZE = 2 };

/* DepthRecord (io.hpp:264-274); absent candidates are NaN */
typedef struct {
  int32_t frame_id;
  int32_t det_id;
  double disparity;
  int32_t valid;
  int32_t source;
  double clp_by_stereo, clp_by_gpt, clp_by_size, z_fused;
} rg_depth_record;

/* RefinerLogRecord (io.hpp:225-230) */
typedef struct {
  int32_t frame_id;
  int32_t pad;
  double rect_delta, radar_offset, obj_offset;
} rg_refiner_log;

/* ObjRefinerState defaults (object_refiner.hpp:15-20) */
rg_status rg_obj_refiner_state_init(rg_obj_refiner_state* st);
/* make_calibration(f, b, cx, cy, h_cam) with the canonical rotation and
 * t = (0, 0, h_cam) (geometry.hpp:130-133) */
rg_status rg_make_calibration(double f, double b, double cx, double cy, double h_cam, rg_calibration* out);

/* One frame of pipeline.hpp:180-249 for the TEMPLATE_MATCHER method
 * (dense = 0) or a dense method (dense = 1, objects[k] = box medians, the
 * radar refiner off).  dets: the frame's detections (HOST); sel[k]: the
 * frame-local index of objects[k] (rg_frame_batch.d_out_index); objects is
 * updated in place (object refiner offset); radar: the frame's radar
 * positions (vehicle frame).  Writes n_obj records and one log entry. */
rg_status rg_frame_records(const rg_record_params* p, int frame_id, int img_w, int img_h, int dense,
                           const rg_detection* dets, int n_dets, const int32_t* sel,
                           rg_object_disparity* objects, int n_obj, const rg_vec3* radar, int n_radar,
                           rg_obj_refiner_state* st, double rect_applied, rg_depth_record* records,
                           rg_refiner_log* log);

/* ------------------------------------------------------ BM / autorect (K5) */

/* validate(const BmParams&), bm.hpp:24-32 */
rg_status rg_validate_bm_params(rg_ctx* ctx, const rg_bm_params* p);
/* bm_disparity, bm.hpp:113-135 (downscale path: image.hpp:98-141) */
rg_status rg_bm_disparity(rg_ctx* ctx, const uint8_t* left, const uint8_t* right,
                          int w, int h, const rg_bm_params* p, int16_t* out_raw);
/* auto_rect_search, autorect.hpp:22-58.  counts (nullable) receives the
 * per-delta valid counts, delta_max - delta_min + 1 entries. */
rg_status rg_auto_rect_search(rg_ctx* ctx, const uint8_t* left, const uint8_t* right,
                              int w, int h, const rg_rect* roi, int delta_min,
                              int delta_max, const rg_bm_params* p, int32_t* best_delta,
                              int64_t* counts);
/* Batched device variant: frames as in rg_frame_batch (d_left/d_right, pitch,
 * frame_stride); d_best[n_frames], d_counts[n_frames * n_delta] (nullable). */
rg_status rg_auto_rect_frames(rg_ctx* ctx, const uint8_t* d_left,
                              const uint8_t* d_right, int n_frames, int64_t frame_stride,
                              int pitch, int w, int h, const rg_rect* roi, int delta_min,
                              int delta_max, const rg_bm_params* p, int32_t* d_best,
                              int64_t* d_counts, void* stream);

/* ------------------------------------------------------ dense BM objects (8f row 3) */

/* Pipeline::box_disparity (pipeline.hpp:304-328): median of the box's valid
 * dense disparities, their count, and dynamic_disparity_variance
 * (geometry.hpp:162-178) of the top-quartile "near" subset.  valid = 0: no
 * valid pixel (std::nullopt); -1: a raw value outside [raw_lo, raw_hi]. */
typedef struct {
  int32_t valid;
  int32_t count;
  double median;
  double variance;
} rg_box_stats;

/* box_disparity for n boxes of one raw map (HOST pointers; DisparityMap::raw,
 * 1/16 px, kInvalid = -32768); every valid raw value must lie in
 * [raw_lo, raw_hi] (the BM output range), raw_hi - raw_lo < 49152. */
rg_status rg_box_disparity(rg_ctx* ctx, const int16_t* raw, int w, int h, const rg_detection* dets,
                           int n, int raw_lo, int raw_hi, double sigma_obs2, double gamma,
                           double sigma_sys2, rg_box_stats* out);
/* The STEREO_BM branch of Pipeline::process_frame for one frame
 * (pipeline.hpp:140-141, 207-224): bm_disparity on the device, select_objects
 * (sorted, template_match.hpp:63-94), box_disparity per selected box;
 * out[k] = {det_id, kind = classify_far_close, n_blocks_used = count,
 * valid = has_value, disparity = median or 0, z_cam = 0}.  box_out and
 * raw_out (w*h) are optional. */
rg_status rg_dense_objects(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                           const rg_detection* dets, int n, const rg_ranger_config* cfg,
                           const rg_bm_params* bm, double sigma_obs2, double gamma,
                           double sigma_sys2, rg_object_disparity* out, rg_box_stats* box_out,
                           int* n_out, int16_t* raw_out);

/* ------------------------------------- radar (dense-map) refiner (8f row 3) */

/* RadarDetection, synth.hpp:19-23 */
typedef struct {
  rg_vec3 position; /* vehicle frame, m */
  rg_vec3 extent;   /* m */
  int32_t id;
  int32_t pad;
} rg_radar_detection;

/* VoteState, radar_refiner.hpp:30-47: bins cover [-K, K] px at 1/16 px
 * (2K*16 + 1 bins, K <= 32 here). */
#define RG_VOTE_MAX_BINS 1025
typedef struct {
  int32_t k_px;
  int32_t n_bins;
  double lambda;
  double smooth_sigma_px;
  double smoothed_offset;
  double memory[RG_VOTE_MAX_BINS];
} rg_vote_state;

/* VoteState(k, lambda, sigma_px) (defaults 4, 0.3, 1.0); RG_EINVAL as the
 * reference's constructor throws (K < 1, lambda outside (0, 1]) or K > 32. */
rg_status rg_vote_state_init(rg_vote_state* st, int k_px, double lambda, double smooth_sigma_px);

/* radar_refine_step (radar_refiner.hpp:111-167) on a DEVICE disparity map
 * d_raw (w*h int16, DisparityMap::raw): radar_extent_box per detection on the
 * host, the closest-offset search over each box on the device, the vote
 * smoothing / EMA of `st` on the host (sequential state), then the clamped
 * offset added to every valid raw value on the device.  *applied receives
 * the offset the reference returns.  Radar detections behind the camera or
 * without a projectable corner are skipped as in the reference. */
rg_status rg_radar_refine_step(rg_ctx* ctx, int16_t* d_raw, int w, int h, const rg_radar_detection* radar, int n,
                               rg_vote_state* st, const rg_calibration* calib, double* applied);

/* rg_radar_refine_step on a HOST map (uploaded, refined on the device,
 * copied back): the drop-in radar_refine_step of include/ranger/radar_refiner.hpp. */
rg_status rg_radar_refine_step_host(rg_ctx* ctx, int16_t* raw, int w, int h, const rg_radar_detection* radar, int n,
                                    rg_vote_state* st, const rg_calibration* calib, double* applied);

/* Host halves of rg_radar_refine_step (used by it; exposed for tests):
 * rg_radar_boxes -- per detection p_cam = imu_to_cam(position), skipped when
 * p_cam.z <= 0 or radar_extent_box fails, else box (x0, y0, x1, y1 inclusive)
 * and d_radar = f b / p_cam.z; *n_boxes of them.  rg_radar_vote_update --
 * the votes of the boxes' closest offsets (found[i] != 0) into `st`
 * (radar_refiner.hpp:129-155); *applied = clamp(smoothed offset, -3, 3),
 * *raw_off = lround(applied * 16). */
rg_status rg_radar_boxes(const rg_radar_detection* radar, int n, const rg_calibration* calib, int w, int h,
                         int32_t* boxes, double* d_radar, int* n_boxes);
rg_status rg_radar_vote_update(rg_vote_state* st, const double* best_off, const int32_t* found, int n_boxes,
                               double* applied, int* raw_off);

/* rg_dense_objects with the radar refiner between the dense map and the box
 * statistics (pipeline.hpp:182-183, 207-224; the PipelineConfig default
 * radar_refiner = true): radar (HOST, n_radar entries) of this frame, vote
 * state carried by the caller from frame to frame, *radar_applied receives
 * the refiner log's radar offset.  raw_out (optional) is the refined map. */
rg_status rg_dense_objects_refined(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                                   const rg_detection* dets, int n, const rg_ranger_config* cfg,
                                   const rg_bm_params* bm, double sigma_obs2, double gamma, double sigma_sys2,
                                   const rg_radar_detection* radar, int n_radar, rg_vote_state* st,
                                   const rg_calibration* calib, rg_object_disparity* out, rg_box_stats* box_out,
                                   int* n_out, int16_t* raw_out, double* radar_applied);

/* ------------------------------------------------------ SGM (8f row 2) */

/* SgmParams, sgm.hpp:14-19 */
typedef struct {
  int32_t num_disparities; /* <= 256 on the device path */
  int32_t min_disparity;
  int32_t p1;
  int32_t p2;
} rg_sgm_params;

/* validate(const SgmParams&), sgm.hpp:21-28 */
rg_status rg_validate_sgm_params(rg_ctx* ctx, const rg_sgm_params* p);
/* sgm_disparity, sgm.hpp:118-155: census cost, 4 directional passes
 * ({1,0},{0,1},{1,1},{-1,1}), winner-take-all + sub-pixel; raw int16 map
 * (DisparityMap::raw, kInvalid = -32768). */
rg_status rg_sgm_disparity(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                           const rg_sgm_params* p, int16_t* out_raw);
/* Batched device variant: frames as in rg_frame_batch; d_raw[n_frames * w * h]. */
rg_status rg_sgm_frames(rg_ctx* ctx, const uint8_t* d_left, const uint8_t* d_right, int n_frames,
                        int64_t frame_stride, int pitch, int w, int h, const rg_sgm_params* p,
                        int16_t* d_raw, void* stream);
/* detail::sgm_cost_volume, sgm.hpp:37-56 (codes: w*h reference-layout census;
 * cost: w*h*num_disparities bytes, [y][x][i]) */
rg_status rg_sgm_cost_volume(rg_ctx* ctx, const uint32_t* left_codes, const uint32_t* right_codes,
                             int w, int h, const rg_sgm_params* p, uint8_t* cost);
/* detail::sgm_direction_pass, sgm.hpp:60-110: adds L_r of direction (sx, sy)
 * into acc (w*h*nd int32, [y][x][d]) */
rg_status rg_sgm_direction_pass(rg_ctx* ctx, const uint8_t* cost, int w, int h, int nd, int p1,
                                int p2, int sx, int sy, int32_t* acc);

/* ------------------------------------------------------ synthetic frames */

/* SceneObject (synth.hpp:25-34) and SceneConfig (synth.hpp:36-52) with the
 * canonical calibration make_calibration(f, b, cx, cy, h_cam)
 * (geometry.hpp:130-133).  Used as the input generator for tests/bench. */
typedef struct {
  int32_t id;
  int32_t class_id;
  double px, py, pz; /* vehicle frame, m */
  double width_m, height_m, depth_m;
  double contrast;
  double disparity_ramp;
  uint64_t texture_seed;
} rg_scene_object;

typedef struct {
  double f, b, cx, cy, h_cam;
  int32_t width, height;
  uint64_t background_seed;
  double background_contrast;
  int32_t vertical_offset_px;
  int32_t texture_quant;
  double disparity_bias_px;
  double gain, rad_bias, gamma;
  double noise_sigma;
  uint64_t seed;
  double texture_cell_px;
} rg_scene_config;

/* render_stereo_pair, synth.hpp:142-230 (host, multi-threaded rows). */
rg_status rg_render_stereo_pair(const rg_scene_config* cfg, const rg_scene_object* objs,
                                int n_obj, uint8_t* left, uint8_t* right,
                                double* true_disparity, int32_t* object_id);
/* Device frame source: render_stereo_pair (synth.hpp:142-230) for n_frames
 * scenes rendered straight into device memory, byte-identical to
 * rg_render_stereo_pair (feeds device-resident streams without PCIe, SURVEY
 * 8(f) row 4).  cfgs[f] and objs[obj_offsets[f] .. obj_offsets[f+1]) are HOST
 * arrays; every frame must share width and height.  d_left / d_right receive
 * frame f at f * frame_stride as dense rows of `width` bytes.  Enqueued on
 * `stream`: returns with the upload of the scene tables (through a pinned
 * staging buffer) and the kernels enqueued -- order later work on that
 * stream or synchronise it before reading the frames.  stream NULL: the
 * context's stream, and the call blocks until the frames are rendered.
 * RG_EINVAL for any scene rg_render_stereo_pair rejects. */
rg_status rg_render_frames_device(rg_ctx* ctx, const rg_scene_config* cfgs, const rg_scene_object* objs,
                                  const int32_t* obj_offsets, int n_frames, uint8_t* d_left,
                                  uint8_t* d_right, int64_t frame_stride, void* stream);
/* ground_truth_detections, synth.hpp:253-274 (capacity n_obj). */
rg_status rg_ground_truth_detections(const rg_scene_config* cfg,
                                     const rg_scene_object* objs, int n_obj,
                                     rg_detection* out, int* n_out);

#ifdef __cplusplus
}
#endif

#endif /* RANGER_CUDA_H_ */
