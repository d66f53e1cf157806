// rg_common.cuh -- shared declarations of the B200 census ranger library.
//
// Device-side numerics follow SURVEY.md Appendix A: the whole library is
// compiled with -fmad=false and every double expression keeps the reference's
// operation order, so FP64 results (mean costs, sub-pixel offsets, sampling
// coordinates, ranges) are bit-identical to the reference's x86-64 build.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ranger_cuda.h"

namespace rg {

// NVTX ranges around the public entry points and the stages they enqueue
// (host-side ranges: visible to nsys / ncu --nvtx; header-only NVTX v3, a
// no-op unless a tool injects itself)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define RG_NVTX(name) ::rg::NvtxRange rg_nvtx_range_(name)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per DEVICE: one cache
// per kernel (a static of the call site) remembers the size raised on each
// device, so a process driving several GPUs raises it on every one.
constexpr size_t kSmemPerBlockOptIn = 227 * 1024;  // sm_100 opt-in limit per CTA (static + dynamic)

struct SmemAttr {
  static constexpr int kDevices = 64;
  std::atomic<int> raised[kDevices] = {};
  cudaError_t ensure(const void* fn, size_t bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDevices)
      return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (raised[dev].load(std::memory_order_relaxed) >= (int)bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) {
      int cur = raised[dev].load(std::memory_order_relaxed);
      while (cur < (int)bytes && !raised[dev].compare_exchange_weak(cur, (int)bytes)) {
      }
    }
    return e;
  }
};

// ------------------------------------------------------------ limits
constexpr int kMatchThreads = 256;     // CTA size of the matcher
constexpr int kWindowCodes = 12288;    // smem census window (48 KB)
constexpr int kMaxOccluders = 128;     // per-object occluder boxes kept in smem
constexpr int kAggCapacity = 4096;     // CLOSE blocks aggregated in smem
// per-launch device counters of the batched pipeline: [0] slots planned,
// [1] overflow flag, [2..3] Hamming evaluations (int64), [4] matcher work index
constexpr int kCounterInts = 8;

// Internal census layout of the batched pipeline: reference bits 0..24, bits
// 25..31 = 0x73 (sign set).  A constant high part cancels in l ^ r, so Hamming
// distances equal the reference's; the sign bit marks a defined code (0 =
// undefined).  0xE6 is the high byte of the fp16 accumulator -(1536 + B) that
// the fast census produces directly (census.cu).
constexpr uint32_t kInternalHigh = 0xE6000000u;

// ------------------------------------------------------------ device structs
template <typename CT>
struct RasterT {  // census raster in device memory
  const CT* p;
  int w, h;
  int pitch;  // elements
};
using Raster = RasterT<uint32_t>;              // 5x5 codes
using Raster64 = RasterT<unsigned long long>;  // 9x7 codes (extension)

// Layout of a census raster in device memory: `w x h` codes at `origin`
// inside a zero margin of padx columns / pady rows, rows `pitch` apart, frames
// `fstride` apart.  The batched path pads its rasters so the matcher can read
// any sample its search range reaches without bounds checks (margin codes are
// 0 = undefined, exactly the reference's inside() test); [sx0, sx1] x
// [sy0, sy1] is where a computed code is defined (non-zero).
struct PadGeom {
  int w, h, padx, pady, pitch;
  int64_t fstride, origin;
  int sx0, sx1, sy0, sy1;
};

__host__ __device__ inline PadGeom make_geom(int w, int h, int padx, int pady) {
  PadGeom g;
  g.w = w;
  g.h = h;
  g.padx = padx;
  g.pady = pady;
  g.pitch = w + 2 * padx;
  g.fstride = (int64_t)(h + 2 * pady) * g.pitch;
  g.origin = (int64_t)pady * g.pitch + padx;
  g.sx0 = g.sy0 = 0;
  g.sx1 = w - 1;
  g.sy1 = h - 1;
  return g;
}

// object table entry of the batched planner (one per selected detection)
struct ObjEntry {
  int32_t det;        // global detection index
  int32_t kind;       // RG_KIND_*
  int32_t slot_base;  // first slot in the global slot list
  int32_t n_slots;    // FAR 1, CLOSE rows*cols
  int32_t rows, cols; // CLOSE sub-block grid
  int32_t frame;
  int32_t occ_n;  // occluders in the planner's list (occ_list[g * kOccMax ..]); -1: more than kOccMax
};
constexpr int kOccMax = 32;  // occluders per object listed by the planner

// a slot = one potential QueryBlock (FAR block or CLOSE sub-block)
struct Slot {
  int32_t frame;
  int32_t obj;  // index into the object table
  int32_t sub;  // r*cols + c for CLOSE, 0 for FAR
  int32_t pad;  // r << 16 | c (planner); K2a overwrites it with the point count
};

}  // namespace rg

// ------------------------------------------------------------ context
struct rg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;  // stream of the synchronous compat API
  cudaStream_t copy_stream = nullptr;  // H2D staging of the host-fed batch API
  cudaStream_t census_stream = nullptr;  // K1 of chunk k+1 while K2 of chunk k runs (rg_range_frames)
  cudaStream_t match_stream = nullptr;   // K3/K2/K4 chunks (highest priority), joined back to the caller
  bool overlap = false;                  // chunked census/matcher overlap in rg_range_frames (opt-in)
  bool census_rois = true;               // ROI-tile census for batches of >= 12 frames (rg_set_census_rois)
  cudaEvent_t ev_sync[10] = {};          // cross-stream ordering events (no timing)
  cudaEvent_t ev_prof[40] = {};          // per-chunk stage timing when profiling
  int map_key[4] = {-1, -1, -1, -1};  // geometry of the cached inverse maps
  rg::PadGeom pad_key{}, pad_key_s{};  // layout of the zeroed census rasters
  int pad_wide = 0;                    // ... and their code width (1 = 64-bit)
  std::string err;
  bool profiling = false;
  double stage_ms[5] = {0, 0, 0, 0, 0};
  int64_t stage_launches[5] = {0, 0, 0, 0, 0};
  int64_t total_launches = 0;
  int64_t hamming_evals = 0;  // algorithmic matcher work of the batched path
  int64_t slots_total = 0;    // potential QueryBlocks planned
  int64_t h2d_bytes = 0, d2h_bytes = 0;  // host <-> device bytes of rg_range_frames_host
  cudaEvent_t ev[12] = {};
  int slot_capacity = 0;    // grows on RG_EOVERFLOW
  int64_t last_slots = 0;   // slots used by the last batch
  // grow-only device scratch, keyed by role
  void* buf[48] = {};
  size_t cap[48] = {};
  // pinned host scratch
  void* hbuf[8] = {};
  size_t hcap[8] = {};
  // asynchronous rg_range_frames: planner counters of batches still in
  // flight, retired (stats, overflow, capacity growth) by the next calls or
  // rg_sync; oldest first in a ring of kPending
  static constexpr int kPending = 8;
  struct Pending {
    cudaEvent_t ev = nullptr;
    int32_t* hc = nullptr;  // pinned copy of the batch's counters
  } pend[kPending];
  int pend_head = 0, pend_n = 0;
  int overflowed = 0;            // retired batches that overflowed since the last rg_sync
  int sync_mode = 0;             // 1: rg_range_frames blocks and re-runs on overflow (legacy)
  cudaStream_t last_stream = nullptr;  // stream of the last asynchronous batch
  cudaEvent_t ev_last = nullptr;       // orders a batch on another stream after it
  cudaEvent_t ev_stage = nullptr;      // pinned scene-table staging of rg_render_frames_device
};

namespace rg {

enum BufId {
  B_IMG_L, B_IMG_R, B_CEN_FL, B_CEN_FR, B_CEN_SL, B_CEN_SR, B_DETS, B_DET_OFF,
  B_OBJ, B_SLOTS, B_SLOT_RES, B_OUT, B_OUT_CNT, B_COUNTERS, B_MAPX, B_MAPY,
  B_PTS, B_OFFS, B_RANGES, B_MRES, B_TMP0, B_TMP1, B_TMP2, B_TMP3, B_STATS,
  B_BM_L, B_BM_R, B_BM_OUT, B_BM_CNT, B_ROIS, B_STAGE_L, B_STAGE_R, B_SHIFT,
  B_SEQ, B_SGM_COST, B_SGM_ACC, B_BOX_IDX, B_BOX_OUT, B_SYNTH, B_ROWMASK, B_SLOT_PTS, B_XFER, B_OCC, B_COUNT
};

// error helpers (defined in api.cu)
rg_status set_err(rg_ctx* ctx, rg_status st, const std::string& msg);
rg_status cuda_err(rg_ctx* ctx, cudaError_t e, const char* what);
void* dev_buf(rg_ctx* ctx, int id, size_t bytes);  // nullptr on failure
void* host_buf(rg_ctx* ctx, int id, size_t bytes);
void count_launch(rg_ctx* ctx, int stage, int n = 1);
rg_status wait_async(rg_ctx* ctx);  // blocks until the context's asynchronous batches are done

#define RG_CUDA(ctx, expr)                                  \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return rg::cuda_err(ctx, _e, #expr); \
  } while (0)

// ------------------------------------------------------------ launchers
// census (census.cu)
// internal: batched-pipeline layout (kInternalHigh; Hamming distances unchanged,
// distances unchanged; lets the matcher mask undefined codes by the sign bit)
cudaError_t launch_census_frames(const uint8_t* left, const uint8_t* right, int n_frames,
                                 int64_t frame_stride, int pitch, int w, int h,
                                 uint32_t* fl, uint32_t* fr, const PadGeom& gf, uint32_t* sl,
                                 uint32_t* sr, const PadGeom& gs, const int32_t* inv_x,
                                 const int32_t* inv_y, const int32_t* lshift, bool internal,
                                 cudaStream_t s);
size_t census_rois_scratch_words(int n_frames, int w, int h, int ch);
cudaError_t launch_census_rois(const uint8_t* left, const uint8_t* right, int n_frames, int64_t frame_stride,
                               int pitch, int w, int h, uint32_t* fl, uint32_t* fr, const PadGeom& gf, uint32_t* sl,
                               uint32_t* sr, const PadGeom& gs, const int32_t* lshift, bool internal,
                               const rg_detection* dets, const int32_t* det_off, double tau_s, int dx_far,
                               int dx_close_scaled, uint32_t* masks, cudaStream_t s,
                               cudaEvent_t full_done = nullptr, cudaStream_t side = nullptr,
                               cudaEvent_t ev_lists = nullptr, cudaEvent_t ev_red = nullptr);
cudaError_t launch_gather_rows(const uint8_t* hl, const uint8_t* hr, int64_t src_stride, int src_pitch, uint8_t* dl,
                               uint8_t* dr, int64_t dst_stride, int dst_pitch, int w, int h, int n_frames,
                               const rg_detection* dets, const int32_t* det_off, double tau_s, int close_scale,
                               int dx_far, int dx_close_scaled, bool wide, const int32_t* lshift,
                               unsigned long long* bytes, cudaStream_t s);
cudaError_t launch_census64_rois(const uint8_t* left, const uint8_t* right, int n_frames, int64_t frame_stride,
                                 int pitch, int w, int h, unsigned long long* fl, unsigned long long* fr,
                                 const PadGeom& gf, unsigned long long* sl, unsigned long long* sr,
                                 const PadGeom& gs, const int32_t* lshift, const rg_detection* dets,
                                 const int32_t* det_off, double tau_s, int dx_far, int dx_close_scaled,
                                 uint32_t* masks, cudaStream_t s, cudaStream_t side = nullptr,
                                 cudaEvent_t ev_lists = nullptr, cudaEvent_t ev_red = nullptr);
cudaError_t launch_census64_frames(const uint8_t* left, const uint8_t* right, int n_frames, int64_t frame_stride,
                                   int pitch, int w, int h, unsigned long long* fl, unsigned long long* fr,
                                   const PadGeom& gf, unsigned long long* sl, unsigned long long* sr,
                                   const PadGeom& gs, const int32_t* inv_x, const int32_t* inv_y,
                                   const int32_t* lshift, cudaStream_t s);
cudaError_t launch_roi_mask(uint32_t* codes, int w, int h, const rg_rect* rois, int n_rois,
                            cudaStream_t s);

// matcher (match.cu)
cudaError_t launch_match_blocks(Raster L, Raster R, const int32_t* pts, const int64_t* offs,
                                const rg_search_range* ranges, int n_blocks, int mode,
                                double tau_v, rg_match_result* out, int max_points,
                                cudaStream_t s);
cudaError_t launch_match_blocks64(Raster64 L, Raster64 R, const int32_t* pts, const int64_t* offs,
                                  const rg_search_range* ranges, int n_blocks, int mode,
                                  double tau_v, rg_match_result* out, int max_points,
                                  cudaStream_t s);
// c_recip table of the matcher's integer divisions (once per device) and its check
cudaError_t init_match_tables();
cudaError_t selftest_division(int b_max, unsigned long long* d_bad, cudaStream_t s);
// K2a slot sampler (match_warp.cu): the points of every planned slot into
// slot_pts (capacity x ((max_points + 1) & ~1)), counts in Slot::pad; whether
// the matcher for this batch reads them (else it samples in-warp)
bool match_presampled(int n_frames, int wide);
cudaError_t launch_sample_slots(Slot* slots, const int32_t* counters, int slot_capacity, const ObjEntry* objs,
                                const int16_t* occ_list, const rg_detection* dets, const int32_t* det_off, int img_w, int img_h,
                                rg_ranger_config cfg, int2* slot_pts, rg_ranger_stats* stats, int max_points,
                                cudaStream_t s);
// slot_pts: the K2a points (nullptr: the matcher samples in-warp)
cudaError_t launch_match_slots(const int2* slot_pts, const Slot* slots, int32_t* counters, int slot_capacity,
                               const ObjEntry* objs, const int16_t* occ_list, const rg_detection* dets,
                               const int32_t* det_off, const void* fl, const void* fr,
                               const PadGeom& gf, const void* sl, const void* sr,
                               const PadGeom& gs, int img_w, int img_h, int trusted, int wide,
                               rg_ranger_config cfg, rg_match_result* res,
                               rg_ranger_stats* stats, int max_points, cudaStream_t s,
                               int n_frames = 0, int region = 0);

// box statistics of dense maps (dense.cu)
cudaError_t launch_radar_votes(const int16_t* raw, int w, const int32_t* boxes, const double* d_radar, int n,
                               double* best_off, int32_t* found, cudaStream_t s);
cudaError_t launch_raw_offset(int16_t* raw, int64_t n, int raw_off, cudaStream_t s);
cudaError_t launch_box_disparity(const int16_t* raw, int w, int h, int64_t frame_stride, const rg_detection* dets,
                                 const int32_t* box_det, const int32_t* box_frame, int n_boxes, int raw_lo,
                                 int nbins, double sigma_obs2, double gamma, double sigma_sys2,
                                 rg_box_stats* out, cudaStream_t s);

// SGM (sgm.cu)
cudaError_t launch_sgm_cost(const uint32_t* cl, const uint32_t* cr, int w, int h, int nd, int d_lo, uint8_t* cost,
                            cudaStream_t s);
cudaError_t launch_sgm_pass(const uint8_t* cost, int w, int h, int nd, int p1, int p2, int sx, int sy,
                            int32_t* acc, cudaStream_t s);
cudaError_t launch_sgm_wta(const int32_t* acc, int w, int h, int nd, int d_lo, int16_t* out, cudaStream_t s);
int sgm_l_bytes(int p2);
cudaError_t launch_sgm_fast(const uint32_t* cl, const uint32_t* cr, int w, int h, int nd, int d_lo, int p1, int p2,
                            void* Lbuf, int16_t* out, cudaStream_t s);

// planner / aggregation / helpers (plan.cu)
cudaError_t launch_plan_frames(const rg_detection* dets, const int32_t* det_off, int n_frames,
                               int w, int h, rg_ranger_config cfg, int out_stride, ObjEntry* objs,
                               rg_object_disparity* out, int32_t* out_count, Slot* slots,
                               int slot_capacity, int32_t* counters, rg_ranger_stats* stats,
                               int32_t* out_index, int16_t* occ_list, bool list_occluders, cudaStream_t s);
cudaError_t launch_aggregate(const ObjEntry* objs, const int32_t* out_count, int n_frames,
                             int out_stride, const rg_match_result* res, int slot_capacity,
                             rg_ranger_config cfg, double focal, double baseline, double* scratch,
                             rg_object_disparity* out, const int32_t* counters, cudaStream_t s);
cudaError_t launch_select_objects(const rg_detection* dets, int n, rg_ranger_config cfg,
                                  int32_t* out_idx, int32_t* n_out, cudaStream_t s);
cudaError_t launch_find_occluders(const rg_detection* dets, int n, int32_t* counts,
                                  int32_t* lists, cudaStream_t s);
cudaError_t launch_sample_blocks(const rg_detection* det, int kind, const double* occ, int n_occ,
                                 rg_ranger_config cfg, int w, int h, int rows, int cols,
                                 int32_t* pts, int32_t* counts, int per_block, cudaStream_t s);
cudaError_t launch_aggregate_values(const double* v, int n, double tau_d, int n_min,
                                    double* scratch, int32_t* out_i, double* out_d,
                                    cudaStream_t s);

// BM / autorect (bm.cu)
cudaError_t launch_bm(const uint8_t* left, const uint8_t* right, int n_frames, int64_t stride,
                      int pitch, int img_h, int w, int h, int x0, int y0, int delta_min,
                      int n_delta, rg_bm_params p, int16_t* raw, int64_t* counts,
                      cudaStream_t s);
cudaError_t launch_downscale(const uint8_t* in, int w, int h, int s, uint8_t* out, cudaStream_t st);
cudaError_t launch_upscale(const int16_t* in, int w, int h, int s, int lo, int16_t* out, int ow,
                           int oh, cudaStream_t st);
cudaError_t launch_crop_shift(const uint8_t* src, int w, int h, int x0, int y0, int rw, int rh, int delta,
                              uint8_t* dst, cudaStream_t st);
cudaError_t launch_count_above(const int16_t* raw, int64_t n, int lo, int64_t* count, cudaStream_t st);
cudaError_t launch_autorect_pick(const int64_t* counts, int n_frames, int delta_min, int n_delta,
                                 int32_t* best, cudaStream_t s);

}  // namespace rg
