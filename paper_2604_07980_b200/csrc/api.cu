// api.cu -- the C ABI (include/ranger_cuda.h): context, buffers, the
// reference-compatible synchronous entry points and the batched pipeline.
//
// Every compute entry point runs on the GPU; there is no CPU fallback.  Host
// code here only validates arguments (mirroring the reference's
// std::invalid_argument checks), moves bytes, and assembles results.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "rg_common.cuh"

// Extra zero columns beyond the search reach on each side of a padded raster.
// 4 suffice for the matcher; 32 (with the pitch rounded to 32 words) keep every
// raster row 128-B aligned, so K1's 512-B warp stores fill whole lines instead
// of sharing a partial sector with the neighbouring tile: 1.467 -> 1.390 ms per
// 256 C2 frames on B200 (2, 3 and 5 x 32 measured the same as 32).
#ifndef RG_PAD_EXTRA
#define RG_PAD_EXTRA 32
#endif
#ifndef RG_BUILD_INFO
#define RG_BUILD_INFO "sm_100a"
#endif

namespace rg {

rg_status set_err(rg_ctx* ctx, rg_status st, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return st;
}

rg_status cuda_err(rg_ctx* ctx, cudaError_t e, const char* what) {
  if (ctx) ctx->err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? RG_ENOMEM : RG_ECUDA;
}

static_assert(B_COUNT <= 40, "rg_ctx::buf too small");

void* dev_buf(rg_ctx* ctx, int id, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (ctx->cap[id] >= bytes) return ctx->buf[id];
  const size_t old_cap = ctx->cap[id];
  if (ctx->buf[id]) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->buf[id]);
    ctx->buf[id] = nullptr;
    ctx->cap[id] = 0;
  }
  const size_t want = std::max(bytes, old_cap + old_cap / 4);  // grow geometrically
  void* p = nullptr;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    ctx->cap[id] = bytes;
  } else {
    ctx->cap[id] = want;
  }
  ctx->buf[id] = p;
  if (id == B_MAPX || id == B_MAPY) ctx->map_key[0] = -1;  // contents lost
  return p;
}

void* host_buf(rg_ctx* ctx, int id, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (ctx->hcap[id] >= bytes) return ctx->hbuf[id];
  if (ctx->hbuf[id]) {
    cudaStreamSynchronize(ctx->stream);
    cudaFreeHost(ctx->hbuf[id]);
    ctx->hbuf[id] = nullptr;
    ctx->hcap[id] = 0;
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  ctx->hbuf[id] = p;
  ctx->hcap[id] = bytes;
  return p;
}

void count_launch(rg_ctx* ctx, int stage, int n) {
  ctx->stage_launches[stage] += n;
  ctx->total_launches += n;
}

}  // namespace rg

using namespace rg;

namespace {

thread_local std::string g_create_err;

#define DBUF(T, ctx, id, n)                                                          \
  static_cast<T*>(rg::dev_buf(ctx, id, sizeof(T) * (size_t)(n)))
#define NEED(ptr)                                                                    \
  do {                                                                               \
    if (!(ptr)) return set_err(ctx, RG_ENOMEM, "device allocation failed");          \
  } while (0)
#define TRY(expr)                                                                    \
  do {                                                                               \
    rg_status _s = (expr);                                                           \
    if (_s != RG_OK) return _s;                                                      \
  } while (0)

enum Stage { ST_CENSUS = 0, ST_PLAN = 1, ST_MATCH = 2, ST_AGG = 3, ST_RECT = 4 };

rg_status retire_pending(rg_ctx* ctx, bool block);

// Every entry point binds the context's device; all but rg_range_frames also
// wait for its asynchronous batches (they share the internal buffers).
rg_status bind(rg_ctx* ctx, bool wait_async = true) {
  if (!ctx) return RG_EINVAL;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_err(ctx, e, "cudaSetDevice");
  if (wait_async && ctx->pend_n) {
    const rg_status st = retire_pending(ctx, true);
    if (st != RG_OK) return st;
    ctx->last_stream = nullptr;
  }
  return RG_OK;
}

// census.hpp:59-64 detail::scaled_coords
std::vector<int32_t> scaled_coords(int out, int src) {
  std::vector<int32_t> m(static_cast<size_t>(out));
  for (int i = 0; i < out; ++i)
    m[i] = (out == src) ? i : int(std::lround(i * double(src) / double(out)));
  return m;
}

// inverse of the reduced-raster gather maps: inv[src] = out index or -1.
// Cached per geometry; the maps only depend on (w, h, ow, oh).
rg_status upload_inverse_maps(rg_ctx* ctx, int w, int h, int ow, int oh, cudaStream_t s,
                              int32_t** inv_x, int32_t** inv_y) {
  const bool hit = ctx->map_key[0] == w && ctx->map_key[1] == h && ctx->map_key[2] == ow &&
                   ctx->map_key[3] == oh;
  int32_t* dx = DBUF(int32_t, ctx, B_MAPX, w);
  int32_t* dy = DBUF(int32_t, ctx, B_MAPY, h);
  NEED(dx);
  NEED(dy);
  if (!hit) {
    std::vector<int32_t> ix(static_cast<size_t>(w), -1), iy(static_cast<size_t>(h), -1);
    const auto mx = scaled_coords(ow, w), my = scaled_coords(oh, h);
    for (int i = 0; i < ow; ++i) ix[mx[i]] = i;
    for (int i = 0; i < oh; ++i) iy[my[i]] = i;
    RG_CUDA(ctx, cudaMemcpyAsync(dx, ix.data(), sizeof(int32_t) * w, cudaMemcpyHostToDevice, s));
    RG_CUDA(ctx, cudaMemcpyAsync(dy, iy.data(), sizeof(int32_t) * h, cudaMemcpyHostToDevice, s));
    RG_CUDA(ctx, cudaStreamSynchronize(s));  // host vectors die at scope exit
    ctx->map_key[0] = w;
    ctx->map_key[1] = h;
    ctx->map_key[2] = ow;
    ctx->map_key[3] = oh;
  }
  *inv_x = dx;
  *inv_y = dy;
  return RG_OK;
}

// upload a packed (w*h) host image into a device buffer with the same layout
rg_status upload_image(rg_ctx* ctx, int id, const uint8_t* img, int w, int h, uint8_t** out) {
  uint8_t* d = DBUF(uint8_t, ctx, id, (size_t)w * h);
  NEED(d);
  RG_CUDA(ctx, cudaMemcpyAsync(d, img, (size_t)w * h, cudaMemcpyHostToDevice, ctx->stream));
  *out = d;
  return RG_OK;
}

// one-image census into full (w*h) and optional reduced (ow*oh) device buffers
rg_status census_one(rg_ctx* ctx, const uint8_t* d_img, int w, int h, int ow, int oh,
                     uint32_t* d_full, uint32_t* d_red) {
  int32_t *ix = nullptr, *iy = nullptr;
  TRY(upload_inverse_maps(ctx, w, h, ow, oh, ctx->stream, &ix, &iy));
  RG_CUDA(ctx, launch_census_frames(d_img, nullptr, 1, 0, w, w, h, d_full, nullptr, make_geom(w, h, 0, 0),
                                    d_red, nullptr, make_geom(ow, oh, 0, 0), ix, iy, nullptr, false, ctx->stream));
  count_launch(ctx, ST_CENSUS);
  return RG_OK;
}

rg_status check_cfg(rg_ctx* ctx, const rg_ranger_config* c) {  // template_match.hpp:48-61
  if (!c) return set_err(ctx, RG_EINVAL, "RangerConfig: null");
  if (c->tau_s <= 0 || c->tau_d <= 0 || c->tau_v < 0)
    return set_err(ctx, RG_EINVAL, "RangerConfig: thresholds must be positive");
  if (c->n_min < 1) return set_err(ctx, RG_EINVAL, "RangerConfig: n_min must be >= 1");
  if (c->close_scale < 1) return set_err(ctx, RG_EINVAL, "RangerConfig: close_scale must be >= 1");
  if (c->grid_side_points < 1 || c->max_total_points < 1 || c->close_block_side_points < 1)
    return set_err(ctx, RG_EINVAL, "RangerConfig: point counts must be >= 1");
  if (c->max_objects < 0) return set_err(ctx, RG_EINVAL, "RangerConfig: max_objects must be >= 0");
  if (c->dx_max_far < 0 || c->dx_max_close < 0)
    return set_err(ctx, RG_EINVAL, "RangerConfig: search ceilings must be >= 0");
  return RG_OK;
}

rg_status check_bm(rg_ctx* ctx, const rg_bm_params* p) {  // bm.hpp:24-32
  if (!p) return set_err(ctx, RG_EINVAL, "BmParams: null");
  if (p->block_size < 3 || p->block_size % 2 == 0)
    return set_err(ctx, RG_EINVAL, "BmParams: block_size must be odd and >= 3");
  if (p->num_disparities < 1) return set_err(ctx, RG_EINVAL, "BmParams: num_disparities must be >= 1");
  if (p->uniqueness_ratio < 0) return set_err(ctx, RG_EINVAL, "BmParams: uniqueness_ratio must be >= 0");
  if (p->downscale < 1) return set_err(ctx, RG_EINVAL, "BmParams: downscale must be >= 1");
  return RG_OK;
}

// max points of any QueryBlock the planner can generate (template_match.hpp:165-194)
int planner_max_points(const rg_ranger_config& c) {
  const int cap = std::max(1, int(std::sqrt(double(c.max_total_points))));
  const int nf = std::min(c.grid_side_points, cap), nc = std::min(c.close_block_side_points, cap);
  return std::max(nf * nf, nc * nc);
}

size_t match_smem_bytes(int maxp, bool with_pts, size_t code_bytes = sizeof(uint32_t)) {
  const size_t mp = (size_t)((maxp + 3) & ~3);
  return code_bytes * (kWindowCodes + mp) + (with_pts ? 8 * mp : 0) + 12 * mp;
}
constexpr size_t kSmemLimit = 220 * 1024;

// ------------------------------------------------------------------------
// The batched pipeline over frames resident on the device.
struct FrameJob {
  const uint8_t* left;
  const uint8_t* right;
  int n_frames, w, h, pitch;
  int64_t frame_stride;
  const rg_detection* dets;
  const int32_t* det_off;
  int out_stride;
  rg_object_disparity* out;
  int32_t* out_count;
  rg_ranger_stats* stats;  // device, n_frames entries (nullable)
  double focal, baseline;
  // census override (compat path with a pre-filled cache): device codes
  const uint32_t* full_l = nullptr;
  const uint32_t* full_r = nullptr;
  const uint32_t* scaled_l = nullptr;
  const uint32_t* scaled_r = nullptr;
  const int32_t* left_shift = nullptr;  // device, n_frames entries (nullable)
  int32_t* out_index = nullptr;         // device, like out (nullable)
};

bool same_geom(const PadGeom& a, const PadGeom& b) {
  return a.w == b.w && a.h == b.h && a.padx == b.padx && a.pady == b.pady && a.pitch == b.pitch &&
         a.fstride == b.fstride && a.origin == b.origin;
}

struct PipelineBufs {
  uint32_t *fl, *fr, *sl, *sr;  // 5x5 rasters (9x7 runs keep 64-bit codes here)
  PadGeom gf, gs;
  ObjEntry* objs;
  Slot* slots;
  rg_match_result* res;
  int32_t* counters;
  double* scratch;
  int capacity;
};

// Geometry and device buffers of the padded census rasters for `frames`
// frames (the margins are zeroed on `s` whenever the layout changes).
struct Rasters {
  uint32_t *fl, *fr, *sl, *sr;
  PadGeom gf, gs;
  bool wide;
  int32_t *ix, *iy;
};

rg_status prepare_rasters(rg_ctx* ctx, const FrameJob& J, const rg_ranger_config& cfg, int frames, cudaStream_t s,
                          Rasters* R) {
  const int w = J.w, h = J.h, sc = cfg.close_scale;
  const int cw = w / sc, ch = h / sc;
  if (cw < 1 || ch < 1) return set_err(ctx, RG_EINVAL, "estimate_object_disparities: close raster empty");
  const int maxp = planner_max_points(cfg);
  // 9x7 extension: 64-bit codes, window rows +-3 / cols +-4
  const bool wide = cfg.census_9x7 != 0;
  const size_t csz = wide ? sizeof(unsigned long long) : sizeof(uint32_t);
  const int rx = wide ? 4 : 2, ry = wide ? 3 : 2;
  if ((sizeof(int2) + 2 * csz) * (size_t)(maxp + 1) * 8 > kSmemLimit)
    return set_err(ctx, RG_EINVAL, "RangerConfig: blocks too large for the device matcher");
  if (wide && (J.full_l || J.scaled_l))
    return set_err(ctx, RG_EINVAL, "RangerConfig: census_9x7 cannot use a CensusCache");
  // zero-padded census rasters: margins cover every sample the search reaches
  const int dxs = (cfg.dx_max_close + sc - 1) / sc;
  const int padf = 32 * ((cfg.dx_max_far + 1 + 31) / 32) + RG_PAD_EXTRA;
  const int pads = 32 * ((dxs + 1 + 31) / 32) + RG_PAD_EXTRA;
  PadGeom gf = make_geom(w, h, padf, 2), gs = make_geom(cw, ch, pads, 2);
  for (PadGeom* g : {&gf, &gs}) {  // 128-B aligned rows (right margin absorbs the rounding)
    g->pitch = (g->pitch + 31) & ~31;
    g->fstride = (int64_t)(g->h + 2 * g->pady) * g->pitch;
    g->origin = (int64_t)g->pady * g->pitch + g->padx;
  }
  // where a computed code is defined: full [rx, W-1-rx] (census.hpp:44); reduced
  // x' with lround(x' * W / cw) in that range (census.hpp:59-64)
  {
    const auto mx = scaled_coords(cw, w), my = scaled_coords(ch, h);
    gf.sx0 = rx, gf.sx1 = w - 1 - rx, gf.sy0 = ry, gf.sy1 = h - 1 - ry;
    gs.sx0 = cw, gs.sx1 = -1, gs.sy0 = ch, gs.sy1 = -1;
    for (int i = 0; i < cw; ++i)
      if (mx[i] >= rx && mx[i] <= w - 1 - rx) gs.sx0 = std::min(gs.sx0, i), gs.sx1 = std::max(gs.sx1, i);
    for (int i = 0; i < ch; ++i)
      if (my[i] >= ry && my[i] <= h - 1 - ry) gs.sy0 = std::min(gs.sy0, i), gs.sy1 = std::max(gs.sy1, i);
  }
  const size_t fbytes = csz * (size_t)gf.fstride * frames;
  const size_t sbytes = csz * (size_t)gs.fstride * frames;
  const bool regeom = ctx->cap[B_CEN_FL] < fbytes || ctx->cap[B_CEN_SL] < sbytes ||
                      !same_geom(ctx->pad_key, gf) || !same_geom(ctx->pad_key_s, gs) ||
                      ctx->pad_wide != (int)wide;
  uint32_t* fl = static_cast<uint32_t*>(dev_buf(ctx, B_CEN_FL, fbytes));
  uint32_t* fr = static_cast<uint32_t*>(dev_buf(ctx, B_CEN_FR, fbytes));
  uint32_t* sl = static_cast<uint32_t*>(dev_buf(ctx, B_CEN_SL, sbytes));
  uint32_t* sr = static_cast<uint32_t*>(dev_buf(ctx, B_CEN_SR, sbytes));
  NEED(fl);
  NEED(fr);
  NEED(sl);
  NEED(sr);
  if (regeom) {  // margins must read as 0; the census kernels never write them
    RG_CUDA(ctx, cudaMemsetAsync(fl, 0, ctx->cap[B_CEN_FL], s));
    RG_CUDA(ctx, cudaMemsetAsync(fr, 0, ctx->cap[B_CEN_FR], s));
    RG_CUDA(ctx, cudaMemsetAsync(sl, 0, ctx->cap[B_CEN_SL], s));
    RG_CUDA(ctx, cudaMemsetAsync(sr, 0, ctx->cap[B_CEN_SR], s));
    ctx->pad_key = gf;
    ctx->pad_key_s = gs;
    ctx->pad_wide = (int)wide;
  }
  int32_t *ix = nullptr, *iy = nullptr;
  TRY(upload_inverse_maps(ctx, w, h, cw, ch, s, &ix, &iy));
  *R = {fl, fr, sl, sr, gf, gs, wide, ix, iy};
  return RG_OK;
}

// K1 of job J into the rasters starting at raster frame `slot0`
rg_status enqueue_census(rg_ctx* ctx, const FrameJob& J, const rg_ranger_config& cfg, const Rasters& R, int slot0,
                         cudaStream_t s) {
  RG_NVTX("K1 census");
  const int w = J.w, h = J.h, F = J.n_frames;
  const size_t csz = R.wide ? sizeof(unsigned long long) : sizeof(uint32_t);
  auto at = [&](uint32_t* p, const PadGeom& g) {
    return reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(p) + csz * (size_t)g.fstride * slot0);
  };
  uint32_t *fl = at(R.fl, R.gf), *fr = at(R.fr, R.gf), *sl = at(R.sl, R.gs), *sr = at(R.sr, R.gs);
  if (R.wide) {
    using u64 = unsigned long long;
    RG_CUDA(ctx, launch_census64_frames(J.left, J.right, F, J.frame_stride, J.pitch, w, h, (u64*)fl, (u64*)fr,
                                        R.gf, (u64*)sl, (u64*)sr, R.gs, R.ix, R.iy, J.left_shift, s));
    count_launch(ctx, ST_CENSUS);
  } else if (!(J.full_l && J.scaled_l)) {
    // ROI rows only (census_transform_rois, template_match.hpp:300-321) when
    // no caller codes are mixed in and the fast layout applies
    static const bool rois_off = getenv("RG_CENSUS_FULL") != nullptr;  // A/B knob: full-frame K1
    cudaError_t e = cudaErrorNotSupported;
    if (!rois_off && !J.full_l && !J.scaled_l && J.dets) {
      const size_t words = (size_t)F * ((h + 31) / 32 + (R.gs.h + 31) / 32);
      uint32_t* masks = DBUF(uint32_t, ctx, B_ROWMASK, std::max<size_t>(words, 1));
      NEED(masks);
      e = launch_census_rois(J.left, J.right, F, J.frame_stride, J.pitch, w, h, fl, fr, R.gf, sl, sr, R.gs,
                             J.left_shift, true, J.dets, J.det_off, cfg.tau_s, masks, s);
      if (e != cudaSuccess && e != cudaErrorNotSupported) RG_CUDA(ctx, e);
    }
    if (e == cudaErrorNotSupported)
      RG_CUDA(ctx, launch_census_frames(J.left, J.right, F, J.frame_stride, J.pitch, w, h, fl, fr, R.gf, sl, sr,
                                        R.gs, R.ix, R.iy, J.left_shift, true, s));
    count_launch(ctx, ST_CENSUS);
  }
  // caller-supplied codes (a pre-filled CensusCache) into the padded layout
  auto put = [&](uint32_t* dst, const uint32_t* src, const PadGeom& g) -> rg_status {
    RG_CUDA(ctx, cudaMemcpy2DAsync(dst + g.origin, sizeof(uint32_t) * g.pitch, src, sizeof(uint32_t) * g.w,
                                   sizeof(uint32_t) * g.w, g.h, cudaMemcpyDefault, s));
    return RG_OK;
  };
  if (J.full_l) {
    TRY(put(fl, J.full_l, R.gf));
    TRY(put(fr, J.full_r, R.gf));
  }
  if (J.scaled_l) {
    TRY(put(sl, J.scaled_l, R.gs));
    TRY(put(sr, J.scaled_r, R.gs));
  }
  return RG_OK;
}

// K3 planner, K2 matcher, K4 aggregation of job J over the rasters at `slot0`.
// ev (nullable): 4 timing events recorded before K3, K2, K4 and after K4.
// plan_stream (nullable): run the counter reset and K3 there (the caller has
// made it wait for everything earlier on s), so K3 overlaps whatever s runs
// before this call (K1); s then waits for K3 before K2.
rg_status enqueue_match(rg_ctx* ctx, const FrameJob& J, const rg_ranger_config& cfg, const Rasters& R, int slot0,
                        cudaStream_t s, int32_t* counters, const cudaEvent_t* ev, PipelineBufs* pb,
                        cudaStream_t plan_stream = nullptr) {
  RG_NVTX("K3 plan + K2 match + K4 aggregate");
  const int w = J.w, h = J.h, F = J.n_frames;
  const size_t csz = R.wide ? sizeof(unsigned long long) : sizeof(uint32_t);
  auto at = [&](uint32_t* p, const PadGeom& g) {
    return reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(p) + csz * (size_t)g.fstride * slot0);
  };
  uint32_t *fl = at(R.fl, R.gf), *fr = at(R.fr, R.gf), *sl = at(R.sl, R.gs), *sr = at(R.sr, R.gs);
  const int maxp = planner_max_points(cfg);
  // initial list: 512 potential blocks per frame (C2 plans 496); grows on overflow
  if (ctx->slot_capacity < F * 512) ctx->slot_capacity = F * 512;
  const int capacity = ctx->slot_capacity;
  ObjEntry* objs = DBUF(ObjEntry, ctx, B_OBJ, (size_t)F * std::max(J.out_stride, 1));
  Slot* slots = DBUF(Slot, ctx, B_SLOTS, capacity);
  rg_match_result* res = DBUF(rg_match_result, ctx, B_SLOT_RES, capacity);
  double* scratch = DBUF(double, ctx, B_TMP3, 2 * (size_t)capacity);
  NEED(objs);
  NEED(slots);
  NEED(res);
  NEED(scratch);
  const cudaStream_t ps = plan_stream ? plan_stream : s;
  RG_CUDA(ctx, cudaMemsetAsync(counters, 0, kCounterInts * sizeof(int32_t), ps));
  if (ev) RG_CUDA(ctx, cudaEventRecord(ev[0], ps));
  // K3 planner
  RG_CUDA(ctx, launch_plan_frames(J.dets, J.det_off, F, w, h, cfg, J.out_stride, objs, J.out,
                                  J.out_count, slots, capacity, counters, J.stats, J.out_index, ps));
  count_launch(ctx, ST_PLAN);
  if (plan_stream) {
    RG_CUDA(ctx, cudaEventRecord(ctx->ev_sync[1], plan_stream));
    RG_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_sync[1], 0));
  }
  if (ev) RG_CUDA(ctx, cudaEventRecord(ev[1], s));
  // K2 fused sampler + forward/backward matcher, one warp per slot
  const int trusted = !(J.full_l || J.scaled_l);
  RG_CUDA(ctx, launch_match_slots(slots, counters, capacity, objs, J.dets, J.det_off, fl, fr, R.gf, sl, sr, R.gs,
                                  w, h, trusted, (int)R.wide, cfg, res, J.stats, maxp, s, F));
  count_launch(ctx, ST_MATCH);
  if (ev) RG_CUDA(ctx, cudaEventRecord(ev[2], s));
  // K4 aggregation + range
  RG_CUDA(ctx, launch_aggregate(objs, J.out_count, F, J.out_stride, res, capacity, cfg, J.focal,
                                J.baseline, scratch, J.out, counters, s));
  count_launch(ctx, ST_AGG);
  if (ev) RG_CUDA(ctx, cudaEventRecord(ev[3], s));
  if (pb) *pb = {fl, fr, sl, sr, R.gf, R.gs, objs, slots, res, counters, scratch, capacity};
  return RG_OK;
}

// census + match of J on one stream (timing events ev[0..4] when profiling)
rg_status enqueue_pipeline(rg_ctx* ctx, const FrameJob& J, const rg_ranger_config& cfg,
                           cudaStream_t s, int32_t* counters, PipelineBufs* pb) {
  Rasters R;
  TRY(prepare_rasters(ctx, J, cfg, J.n_frames, s, &R));
  const bool prof = ctx->profiling;
  // latency mode (a few frames, not profiling): K3 on the auxiliary stream
  // alongside K1 -- both are a few microseconds for one frame
  cudaStream_t aux = nullptr;
  if (!prof && J.n_frames <= 4 && ctx->match_stream) {
    aux = ctx->match_stream;  // high priority: the one planner CTA is dispatched ahead of K1's
    RG_CUDA(ctx, cudaEventRecord(ctx->ev_sync[0], s));
    RG_CUDA(ctx, cudaStreamWaitEvent(aux, ctx->ev_sync[0], 0));
  }
  if (prof) RG_CUDA(ctx, cudaEventRecord(ctx->ev[0], s));
  TRY(enqueue_census(ctx, J, cfg, R, 0, s));
  return enqueue_match(ctx, J, cfg, R, 0, s, counters, prof ? ctx->ev + 1 : nullptr, pb, aux);
}

void accumulate_profile(rg_ctx* ctx) {
  if (!ctx->profiling) return;
  for (int i = 0; i < 4; ++i) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ctx->ev[i], ctx->ev[i + 1]) == cudaSuccess) ctx->stage_ms[i] += ms;
  }
  cudaGetLastError();
}

// Overflow check after an enqueued pipeline: copies the counters back,
// waits, and on overflow grows the slot list and re-runs synchronously.
rg_status finish_pipeline(rg_ctx* ctx, const FrameJob& J, const rg_ranger_config& cfg,
                          cudaStream_t s, int32_t* counters, int32_t* hc, PipelineBufs* pb) {
  for (int attempt = 0;; ++attempt) {
    RG_CUDA(ctx, cudaMemcpyAsync(hc, counters, kCounterInts * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RG_CUDA(ctx, cudaStreamSynchronize(s));
    accumulate_profile(ctx);
    const int used = hc[0] + hc[4];  // FAR slots from the bottom, CLOSE slots from the top
    ctx->last_slots = used;
    if (!hc[1]) {
      int64_t ev;
      std::memcpy(&ev, hc + 2, sizeof(ev));
      ctx->hamming_evals += ev;
      ctx->slots_total += used;
      return RG_OK;
    }
    if (attempt >= 3) return set_err(ctx, RG_EOVERFLOW, "device block list overflow");
    ctx->slot_capacity = std::max(ctx->slot_capacity * 2, used + used / 4 + 64);
    TRY(enqueue_pipeline(ctx, J, cfg, s, counters, pb));
  }
}

// run + overflow check (synchronous)
rg_status run_pipeline(rg_ctx* ctx, const FrameJob& J, const rg_ranger_config& cfg, cudaStream_t s,
                       PipelineBufs* pb) {
  int32_t* counters = DBUF(int32_t, ctx, B_COUNTERS, kCounterInts);
  int32_t* hc = static_cast<int32_t*>(host_buf(ctx, 0, kCounterInts * sizeof(int32_t)));
  NEED(counters);
  NEED(hc);
  TRY(enqueue_pipeline(ctx, J, cfg, s, counters, pb));
  return finish_pipeline(ctx, J, cfg, s, counters, hc, pb);
}

// ---- asynchronous batches (rg_range_frames without host synchronisation)
// Planner counters of an enqueued batch: retire them (stats, overflow ->
// grown list for the following batches).  block = false stops at the first
// batch still running.
rg_status retire_pending(rg_ctx* ctx, bool block) {
  while (ctx->pend_n > 0) {
    rg_ctx::Pending& p = ctx->pend[ctx->pend_head];
    if (block) {
      RG_CUDA(ctx, cudaEventSynchronize(p.ev));
    } else {
      const cudaError_t q = cudaEventQuery(p.ev);
      if (q == cudaErrorNotReady) break;
      RG_CUDA(ctx, q);
    }
    const int32_t* hc = p.hc;
    const int used = hc[0] + hc[4];
    ctx->last_slots = used;
    if (hc[1]) {
      ++ctx->overflowed;
      ctx->slot_capacity = std::max(ctx->slot_capacity * 2, used + used / 4 + 64);
    } else {
      int64_t ev;
      std::memcpy(&ev, hc + 2, sizeof(ev));
      ctx->hamming_evals += ev;
      ctx->slots_total += used;
    }
    ctx->pend_head = (ctx->pend_head + 1) % rg_ctx::kPending;
    --ctx->pend_n;
  }
  return RG_OK;
}

// Enqueue J on s without waiting: the counters go to a pinned slot of the
// pending ring with an event; a batch on another stream than the previous
// one is ordered after it (the internal rasters and lists are shared).
rg_status run_pipeline_async(rg_ctx* ctx, const FrameJob& J, const rg_ranger_config& cfg, cudaStream_t s) {
  if (ctx->pend_n == rg_ctx::kPending) {  // ring full: wait for the oldest batch
    rg_ctx::Pending& p = ctx->pend[ctx->pend_head];
    RG_CUDA(ctx, cudaEventSynchronize(p.ev));
  }
  TRY(retire_pending(ctx, false));  // grows the list early when a finished batch overflowed
  if (!ctx->ev_last) RG_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_last, cudaEventDisableTiming));
  if (ctx->last_stream && ctx->last_stream != s) {
    RG_CUDA(ctx, cudaEventRecord(ctx->ev_last, ctx->last_stream));
    RG_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_last, 0));
  }
  const int slot = (ctx->pend_head + ctx->pend_n) % rg_ctx::kPending;
  rg_ctx::Pending& p = ctx->pend[slot];
  if (!p.ev) RG_CUDA(ctx, cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming));
  if (!p.hc) RG_CUDA(ctx, cudaMallocHost(&p.hc, kCounterInts * sizeof(int32_t)));
  int32_t* counters = DBUF(int32_t, ctx, B_COUNTERS, kCounterInts);
  NEED(counters);
  TRY(enqueue_pipeline(ctx, J, cfg, s, counters, nullptr));
  RG_CUDA(ctx, cudaMemcpyAsync(p.hc, counters, kCounterInts * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  RG_CUDA(ctx, cudaEventRecord(p.ev, s));
  ++ctx->pend_n;
  ctx->last_stream = s;
  return RG_OK;
}

int census_stream_priority() {  // lowest priority: census CTAs fill what the matcher leaves
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  const char* v = getenv("RG_CENSUS_PRIO");
  return v ? atoi(v) : lo;
}

int match_stream_priority() {  // greatest priority: the latency-bound matcher is scheduled first
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  const char* v = getenv("RG_MATCH_PRIO");
  return v ? atoi(v) : hi;
}

// rg_range_frames schedule: the batch is cut into chunks; K1 of chunk k+1 runs
// on the context's census stream while K3/K2/K4 of chunk k run on the caller's
// stream, so the HBM-bound census overlaps the latency-bound matcher.  The
// rasters are double-buffered by chunk parity (census k+2 waits for match k).
rg_status run_pipeline_overlapped(rg_ctx* ctx, const FrameJob& J, const rg_ranger_config& cfg, cudaStream_t s) {
  const int F = J.n_frames;
  constexpr int kMinChunk = 16;
  if (!ctx->overlap || F < 2 * kMinChunk || J.full_l || J.scaled_l) return run_pipeline(ctx, J, cfg, s, nullptr);
  static const int n_chunks = [] {
    const char* v = getenv("RG_CHUNKS");
    return v ? std::max(2, atoi(v)) : 4;
  }();
  const int chunk = std::max(kMinChunk, (F + n_chunks - 1) / n_chunks);
  const int nch = (F + chunk - 1) / chunk;
  if (nch > 6) return run_pipeline(ctx, J, cfg, s, nullptr);  // ev_prof holds 6 chunks
  Rasters R;
  TRY(prepare_rasters(ctx, J, cfg, 2 * chunk, s, &R));
  int32_t* counters = DBUF(int32_t, ctx, B_COUNTERS, kCounterInts * (size_t)nch);
  int32_t* hc = static_cast<int32_t*>(host_buf(ctx, 0, kCounterInts * sizeof(int32_t) * nch));
  NEED(counters);
  NEED(hc);
  cudaStream_t cs = ctx->census_stream, ms = ctx->match_stream;
  const bool prof = ctx->profiling;
  // both internal streams start after everything already queued on s
  RG_CUDA(ctx, cudaEventRecord(ctx->ev_sync[0], s));
  RG_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->ev_sync[0], 0));
  RG_CUDA(ctx, cudaStreamWaitEvent(ms, ctx->ev_sync[0], 0));
  auto sub = [&](int k) {
    FrameJob Jk = J;
    const int f0 = k * chunk;
    Jk.n_frames = std::min(F, f0 + chunk) - f0;
    Jk.left = J.left + (int64_t)f0 * J.frame_stride;
    Jk.right = J.right + (int64_t)f0 * J.frame_stride;
    Jk.det_off = J.det_off + f0;
    Jk.out = J.out + (int64_t)f0 * J.out_stride;
    Jk.out_count = J.out_count + f0;
    Jk.stats = J.stats ? J.stats + f0 : nullptr;
    Jk.left_shift = J.left_shift ? J.left_shift + f0 : nullptr;
    Jk.out_index = J.out_index ? J.out_index + (int64_t)f0 * J.out_stride : nullptr;
    return Jk;
  };
  for (int k = 0; k < nch; ++k) {
    const int slot = k & 1;
    const FrameJob Jk = sub(k);
    if (k >= 2) RG_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->ev_sync[2 + slot], 0));  // match k-2 released the slot
    if (prof) RG_CUDA(ctx, cudaEventRecord(ctx->ev_prof[6 * k], cs));
    TRY(enqueue_census(ctx, Jk, cfg, R, slot * chunk, cs));
    if (prof) RG_CUDA(ctx, cudaEventRecord(ctx->ev_prof[6 * k + 1], cs));
    RG_CUDA(ctx, cudaEventRecord(ctx->ev_sync[4 + slot], cs));
    RG_CUDA(ctx, cudaStreamWaitEvent(ms, ctx->ev_sync[4 + slot], 0));
    TRY(enqueue_match(ctx, Jk, cfg, R, slot * chunk, ms, counters + kCounterInts * k,
                      prof ? ctx->ev_prof + 6 * k + 2 : nullptr, nullptr));
    RG_CUDA(ctx, cudaEventRecord(ctx->ev_sync[2 + slot], ms));
  }
  // join: the caller's stream continues after the last matcher chunk (which
  // itself follows every census chunk)
  RG_CUDA(ctx, cudaEventRecord(ctx->ev_sync[1], ms));
  RG_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_sync[1], 0));
  RG_CUDA(ctx, cudaMemcpyAsync(hc, counters, kCounterInts * sizeof(int32_t) * nch, cudaMemcpyDeviceToHost, s));
  RG_CUDA(ctx, cudaStreamSynchronize(s));
  if (prof) {
    for (int k = 0; k < nch; ++k) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, ctx->ev_prof[6 * k], ctx->ev_prof[6 * k + 1]) == cudaSuccess)
        ctx->stage_ms[ST_CENSUS] += ms;
      for (int i = 0; i < 3; ++i)
        if (cudaEventElapsedTime(&ms, ctx->ev_prof[6 * k + 2 + i], ctx->ev_prof[6 * k + 3 + i]) == cudaSuccess)
          ctx->stage_ms[1 + i] += ms;
    }
    cudaGetLastError();
  }
  int64_t slots = 0;
  for (int k = 0; k < nch; ++k) {
    const int32_t* c = hc + kCounterInts * k;
    if (c[1]) {  // this chunk overflowed its slot list: grow and re-run it alone
      ctx->slot_capacity = std::max(ctx->slot_capacity * 2, c[0] + c[4] + (c[0] + c[4]) / 4 + 64);
      const FrameJob Jk = sub(k);
      TRY(run_pipeline(ctx, Jk, cfg, s, nullptr));
      continue;
    }
    int64_t ev;
    std::memcpy(&ev, c + 2, sizeof(ev));
    ctx->hamming_evals += ev;
    ctx->slots_total += c[0] + c[4];
    slots += c[0] + c[4];
  }
  ctx->last_slots = slots;
  return RG_OK;
}

}  // namespace

// =========================================================== C ABI: context
extern "C" {

rg_status rg_ctx_create(int device, rg_ctx** out) {
  if (!out) return RG_EINVAL;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    g_create_err = std::string("no CUDA device: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return RG_ECUDA;
  }
  if (device < 0 || device >= n) {
    g_create_err = "device index out of range";
    return RG_EINVAL;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) {
    g_create_err = "device is not sm_100 (Blackwell); this library is built for sm_100a only";
    return RG_ECUDA;
  }
  e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    g_create_err = cudaGetErrorString(e);
    return RG_ECUDA;
  }
  rg_ctx* c = new rg_ctx();
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->census_stream, cudaStreamNonBlocking, census_stream_priority()) !=
          cudaSuccess ||
      cudaStreamCreateWithPriority(&c->match_stream, cudaStreamNonBlocking, match_stream_priority()) != cudaSuccess) {
    g_create_err = "cudaStreamCreate failed";
    delete c;
    return RG_ECUDA;
  }
  for (auto& ev : c->ev) cudaEventCreate(&ev);
  for (auto& ev : c->ev_sync) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  for (auto& ev : c->ev_prof) cudaEventCreate(&ev);
  *out = c;
  return RG_OK;
}

void rg_ctx_destroy(rg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  retire_pending(ctx, true);
  for (cudaStream_t st : {ctx->stream, ctx->copy_stream, ctx->census_stream, ctx->match_stream})
    if (st) cudaStreamSynchronize(st);
  for (auto& p : ctx->pend) {
    if (p.ev) cudaEventDestroy(p.ev);
    if (p.hc) cudaFreeHost(p.hc);
  }
  if (ctx->ev_last) cudaEventDestroy(ctx->ev_last);
  for (void* p : ctx->buf)
    if (p) cudaFree(p);
  for (void* p : ctx->hbuf)
    if (p) cudaFreeHost(p);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : ctx->ev_sync)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : ctx->ev_prof)
    if (ev) cudaEventDestroy(ev);
  cudaStreamDestroy(ctx->stream);
  cudaStreamDestroy(ctx->copy_stream);
  cudaStreamDestroy(ctx->census_stream);
  cudaStreamDestroy(ctx->match_stream);
  delete ctx;
}

const char* rg_last_error(const rg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
const char* rg_create_error(void) { return g_create_err.c_str(); }
const char* rg_build_info(void) { return RG_BUILD_INFO; }

rg_status rg_set_profiling(rg_ctx* ctx, int on) {
  if (!ctx) return RG_EINVAL;
  ctx->profiling = on != 0;
  return RG_OK;
}

rg_status rg_set_overlap(rg_ctx* ctx, int on) {
  if (!ctx) return RG_EINVAL;
  ctx->overlap = on != 0;
  return RG_OK;
}

rg_status rg_get_counters(rg_ctx* ctx, double times_ms[5], int64_t launches[5], int64_t* total) {
  if (!ctx) return RG_EINVAL;
  for (int i = 0; i < 5; ++i) {
    if (times_ms) times_ms[i] = ctx->stage_ms[i];
    if (launches) launches[i] = ctx->stage_launches[i];
  }
  if (total) *total = ctx->total_launches;
  return RG_OK;
}

rg_status rg_get_work(rg_ctx* ctx, int64_t* hamming_evals, int64_t* blocks) {
  if (!ctx) return RG_EINVAL;
  if (hamming_evals) *hamming_evals = ctx->hamming_evals;
  if (blocks) *blocks = ctx->slots_total;
  return RG_OK;
}

rg_status rg_reset_counters(rg_ctx* ctx) {
  if (!ctx) return RG_EINVAL;
  ctx->hamming_evals = 0;
  ctx->slots_total = 0;
  for (int i = 0; i < 5; ++i) {
    ctx->stage_ms[i] = 0;
    ctx->stage_launches[i] = 0;
  }
  ctx->total_launches = 0;
  return RG_OK;
}

// =========================================================== census
rg_status rg_census_code_at(rg_ctx* ctx, const uint8_t* img, int w, int h, int sx, int sy,
                            uint32_t* code) {
  TRY(bind(ctx));
  if (!img || !code || w < 1 || h < 1) return set_err(ctx, RG_EINVAL, "census_code_at: bad image");
  *code = 0;
  if (sx < 2 || sy < 2 || sx >= w - 2 || sy >= h - 2) return RG_OK;  // census.hpp:44
  uint8_t patch[25];
  for (int j = 0; j < 5; ++j) std::memcpy(patch + 5 * j, img + (size_t)(sy - 2 + j) * w + sx - 2, 5);
  uint8_t* d = nullptr;
  TRY(upload_image(ctx, B_IMG_L, patch, 5, 5, &d));
  uint32_t* full = DBUF(uint32_t, ctx, B_TMP0, 25);
  NEED(full);
  TRY(census_one(ctx, d, 5, 5, 5, 5, full, nullptr));
  uint32_t out[25];
  RG_CUDA(ctx, cudaMemcpyAsync(out, full, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *code = out[12];
  return RG_OK;
}

static rg_status census_common(rg_ctx* ctx, const uint8_t* img, int w, int h, int ow, int oh,
                               const rg_rect* rois, int n_rois, bool masked, uint32_t* codes,
                               const char* name) {
  TRY(bind(ctx));
  if (!img || !codes || w < 1 || h < 1) return set_err(ctx, RG_EINVAL, std::string(name) + ": bad image");
  if (ow > w || oh > h) return set_err(ctx, RG_EINVAL, std::string(name) + ": output dims exceed source");
  if (ow < 1 || oh < 1) return set_err(ctx, RG_EINVAL, std::string(name) + ": empty output");
  uint8_t* d = nullptr;
  TRY(upload_image(ctx, B_IMG_L, img, w, h, &d));
  uint32_t* full = DBUF(uint32_t, ctx, B_TMP0, (size_t)w * h);
  NEED(full);
  uint32_t* red = nullptr;
  if (ow != w || oh != h) {
    red = DBUF(uint32_t, ctx, B_TMP1, (size_t)ow * oh);
    NEED(red);
  }
  TRY(census_one(ctx, d, w, h, ow, oh, full, red));
  uint32_t* res = red ? red : full;
  if (masked) {
    rg_rect* dr = DBUF(rg_rect, ctx, B_ROIS, std::max(n_rois, 1));
    NEED(dr);
    if (n_rois > 0)
      RG_CUDA(ctx, cudaMemcpyAsync(dr, rois, sizeof(rg_rect) * n_rois, cudaMemcpyHostToDevice, ctx->stream));
    RG_CUDA(ctx, launch_roi_mask(res, ow, oh, dr, n_rois, ctx->stream));
    count_launch(ctx, ST_CENSUS);
  }
  RG_CUDA(ctx, cudaMemcpyAsync(codes, res, sizeof(uint32_t) * (size_t)ow * oh, cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return RG_OK;
}

rg_status rg_census_transform(rg_ctx* ctx, const uint8_t* img, int w, int h, int ow, int oh,
                              uint32_t* codes) {
  RG_NVTX("rg_census_transform");
  return census_common(ctx, img, w, h, ow, oh, nullptr, 0, false, codes, "census_transform");
}

rg_status rg_census_transform_rois(rg_ctx* ctx, const uint8_t* img, int w, int h, int ow, int oh,
                                   const rg_rect* rois, int n_rois, uint32_t* codes) {
  if (n_rois < 0 || (n_rois > 0 && !rois)) return set_err(ctx, RG_EINVAL, "census_transform_rois: bad rois");
  if (ow < 1 || oh < 1) {  // reference builds an empty CensusImage (no empty-output check)
    if (ow > w || oh > h) return set_err(ctx, RG_EINVAL, "census_transform_rois: output dims exceed source");
    return RG_OK;
  }
  return census_common(ctx, img, w, h, ow, oh, rois, n_rois, true, codes, "census_transform_rois");
}

// =========================================================== matcher
}  // extern "C"

template <typename CT>
static rg_status match_blocks_common(rg_ctx* ctx, const CT* left, int lw, int lh, const CT* right,
                          int rw, int rh, const int32_t* points_xy, const int64_t* offsets,
                          const rg_search_range* ranges, int n_blocks, int mode, double tau_v,
                          rg_match_result* out) {
  TRY(bind(ctx));
  if (n_blocks < 0 || (n_blocks > 0 && (!offsets || !ranges || !out)))
    return set_err(ctx, RG_EINVAL, "match_blocks: bad arguments");
  if (n_blocks == 0) return RG_OK;
  if (lw < 0 || lh < 0 || rw < 0 || rh < 0) return set_err(ctx, RG_EINVAL, "match_blocks: bad raster");
  int64_t maxp = 0;
  for (int b = 0; b < n_blocks; ++b) {
    const int64_t np = offsets[b + 1] - offsets[b];
    if (np < 0) return set_err(ctx, RG_EINVAL, "match_blocks: bad offsets");
    maxp = std::max(maxp, np);
    if (np > 0 && (ranges[b].dx_min > ranges[b].dx_max || ranges[b].dy_min > ranges[b].dy_max))
      return set_err(ctx, RG_EINVAL, "block_match: empty search range");  // census.hpp:182-183
  }
  if (match_smem_bytes((int)std::min<int64_t>(maxp, 1 << 20), false, sizeof(CT)) > kSmemLimit)
    return set_err(ctx, RG_EINVAL, "block_match: block has too many points for the device matcher");
  const int64_t total = offsets[n_blocks] - offsets[0];
  const size_t lsz = std::max<size_t>((size_t)lw * lh, 1), rsz = std::max<size_t>((size_t)rw * rh, 1);
  CT* dl = DBUF(CT, ctx, B_CEN_FL, lsz);
  CT* dr = DBUF(CT, ctx, B_CEN_FR, rsz);
  ctx->pad_key = PadGeom{};  // the padded pipeline rasters are clobbered
  int32_t* dp = DBUF(int32_t, ctx, B_PTS, 2 * std::max<int64_t>(total, 1));
  int64_t* doff = DBUF(int64_t, ctx, B_OFFS, n_blocks + 1);
  rg_search_range* drg = DBUF(rg_search_range, ctx, B_RANGES, n_blocks);
  rg_match_result* dres = DBUF(rg_match_result, ctx, B_MRES, n_blocks);
  NEED(dl);
  NEED(dr);
  NEED(dp);
  NEED(doff);
  NEED(drg);
  NEED(dres);
  cudaStream_t s = ctx->stream;
  if ((size_t)lw * lh) RG_CUDA(ctx, cudaMemcpyAsync(dl, left, sizeof(CT) * lw * lh, cudaMemcpyHostToDevice, s));
  if ((size_t)rw * rh) RG_CUDA(ctx, cudaMemcpyAsync(dr, right, sizeof(CT) * rw * rh, cudaMemcpyHostToDevice, s));
  if (total > 0)
    RG_CUDA(ctx, cudaMemcpyAsync(dp, points_xy + 2 * offsets[0], sizeof(int32_t) * 2 * total,
                                 cudaMemcpyHostToDevice, s));
  std::vector<int64_t> off0(static_cast<size_t>(n_blocks + 1));
  for (int b = 0; b <= n_blocks; ++b) off0[b] = offsets[b] - offsets[0];
  RG_CUDA(ctx, cudaMemcpyAsync(doff, off0.data(), sizeof(int64_t) * (n_blocks + 1), cudaMemcpyHostToDevice, s));
  RG_CUDA(ctx, cudaMemcpyAsync(drg, ranges, sizeof(rg_search_range) * n_blocks, cudaMemcpyHostToDevice, s));
  const RasterT<CT> L = {dl, lw, lh, lw}, R = {dr, rw, rh, rw};
  if constexpr (sizeof(CT) == 4)
    RG_CUDA(ctx, launch_match_blocks(L, R, dp, doff, drg, n_blocks, mode, tau_v, dres,
                                     (int)std::max<int64_t>(maxp, 4), s));
  else
    RG_CUDA(ctx, launch_match_blocks64(L, R, dp, doff, drg, n_blocks, mode, tau_v, dres,
                                       (int)std::max<int64_t>(maxp, 4), s));
  count_launch(ctx, ST_MATCH);
  RG_CUDA(ctx, cudaMemcpyAsync(out, dres, sizeof(rg_match_result) * n_blocks, cudaMemcpyDeviceToHost, s));
  RG_CUDA(ctx, cudaStreamSynchronize(s));
  return RG_OK;
}

extern "C" {

rg_status rg_match_blocks(rg_ctx* ctx, const uint32_t* left, int lw, int lh, const uint32_t* right,
                          int rw, int rh, const int32_t* points_xy, const int64_t* offsets,
                          const rg_search_range* ranges, int n_blocks, int mode, double tau_v,
                          rg_match_result* out) {
  RG_NVTX("rg_match_blocks");
  return match_blocks_common(ctx, left, lw, lh, right, rw, rh, points_xy, offsets, ranges, n_blocks, mode,
                             tau_v, out);
}

// 9x7 extension: same matcher over 64-bit codes
rg_status rg_match_blocks64(rg_ctx* ctx, const uint64_t* left, int lw, int lh, const uint64_t* right,
                            int rw, int rh, const int32_t* points_xy, const int64_t* offsets,
                            const rg_search_range* ranges, int n_blocks, int mode, double tau_v,
                            rg_match_result* out) {
  using u64 = unsigned long long;
  return match_blocks_common(ctx, reinterpret_cast<const u64*>(left), lw, lh,
                             reinterpret_cast<const u64*>(right), rw, rh, points_xy, offsets, ranges,
                             n_blocks, mode, tau_v, out);
}

// 9x7 extension: full / nearest-downscaled 64-bit census of one image
rg_status rg_census_transform64(rg_ctx* ctx, const uint8_t* img, int w, int h, int ow, int oh,
                                uint64_t* codes) {
  TRY(bind(ctx));
  if (!img || !codes || w < 1 || h < 1) return set_err(ctx, RG_EINVAL, "census_transform64: bad image");
  if (ow > w || oh > h) return set_err(ctx, RG_EINVAL, "census_transform64: output dims exceed source");
  if (ow < 1 || oh < 1) return set_err(ctx, RG_EINVAL, "census_transform64: empty output");
  using u64 = unsigned long long;
  uint8_t* d = nullptr;
  TRY(upload_image(ctx, B_IMG_L, img, w, h, &d));
  u64* full = DBUF(u64, ctx, B_TMP0, (size_t)w * h);
  NEED(full);
  u64* red = nullptr;
  if (ow != w || oh != h) {
    red = DBUF(u64, ctx, B_TMP1, (size_t)ow * oh);
    NEED(red);
  }
  int32_t *ix = nullptr, *iy = nullptr;
  TRY(upload_inverse_maps(ctx, w, h, ow, oh, ctx->stream, &ix, &iy));
  RG_CUDA(ctx, launch_census64_frames(d, nullptr, 1, 0, w, w, h, full, nullptr, make_geom(w, h, 0, 0), red,
                                      nullptr, make_geom(ow, oh, 0, 0), ix, iy, nullptr, ctx->stream));
  count_launch(ctx, ST_CENSUS);
  RG_CUDA(ctx, cudaMemcpyAsync(codes, red ? red : full, sizeof(u64) * (size_t)ow * oh, cudaMemcpyDeviceToHost,
                               ctx->stream));
  RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return RG_OK;
}

// =========================================================== object ranger helpers
rg_status rg_validate_ranger_config(rg_ctx* ctx, const rg_ranger_config* cfg) {
  return check_cfg(ctx, cfg);
}

static rg_status upload_dets(rg_ctx* ctx, const rg_detection* dets, int n, rg_detection** out) {
  rg_detection* d = DBUF(rg_detection, ctx, B_DETS, std::max(n, 1));
  NEED(d);
  if (n > 0)
    RG_CUDA(ctx, cudaMemcpyAsync(d, dets, sizeof(rg_detection) * n, cudaMemcpyHostToDevice, ctx->stream));
  *out = d;
  return RG_OK;
}

rg_status rg_select_objects(rg_ctx* ctx, const rg_detection* dets, int n, const rg_ranger_config* cfg,
                            int32_t* out_idx, int* n_out) {
  TRY(bind(ctx));
  if (!cfg || !n_out || n < 0 || (n > 0 && (!dets || !out_idx)))
    return set_err(ctx, RG_EINVAL, "select_objects: bad arguments");
  *n_out = 0;
  if (n == 0 || cfg->max_objects <= 0) return RG_OK;
  rg_detection* d = nullptr;
  TRY(upload_dets(ctx, dets, n, &d));
  int32_t* idx = DBUF(int32_t, ctx, B_TMP0, n + 1);
  NEED(idx);
  RG_CUDA(ctx, launch_select_objects(d, n, *cfg, idx, idx + n, ctx->stream));
  count_launch(ctx, ST_PLAN);
  std::vector<int32_t> h(static_cast<size_t>(n + 1));
  RG_CUDA(ctx, cudaMemcpyAsync(h.data(), idx, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *n_out = h[n];
  std::copy(h.begin(), h.begin() + h[n], out_idx);
  return RG_OK;
}

rg_status rg_find_occluders(rg_ctx* ctx, const rg_detection* dets, int n, int32_t* occ_offsets,
                            int32_t* occ_idx) {
  TRY(bind(ctx));
  if (n < 0 || !occ_offsets || (n > 0 && (!dets || !occ_idx)))
    return set_err(ctx, RG_EINVAL, "find_occluders: bad arguments");
  occ_offsets[0] = 0;
  if (n == 0) return RG_OK;
  rg_detection* d = nullptr;
  TRY(upload_dets(ctx, dets, n, &d));
  int32_t* cnt = DBUF(int32_t, ctx, B_TMP0, n);
  int32_t* lists = DBUF(int32_t, ctx, B_TMP1, (size_t)n * n);
  NEED(cnt);
  NEED(lists);
  RG_CUDA(ctx, launch_find_occluders(d, n, cnt, lists, ctx->stream));
  count_launch(ctx, ST_PLAN);
  std::vector<int32_t> hc(static_cast<size_t>(n)), hl((size_t)n * n);
  RG_CUDA(ctx, cudaMemcpyAsync(hc.data(), cnt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaMemcpyAsync(hl.data(), lists, sizeof(int32_t) * n * n, cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  int k = 0;
  for (int i = 0; i < n; ++i) {
    occ_offsets[i] = k;
    for (int t = 0; t < hc[i]; ++t) occ_idx[k++] = hl[(size_t)i * n + t];
  }
  occ_offsets[n] = k;
  return RG_OK;
}

rg_status rg_sample_query_points(rg_ctx* ctx, const rg_detection* det, int kind,
                                 const double* occluder_boxes, int n_occ, const rg_ranger_config* cfg,
                                 int img_w, int img_h, int64_t* block_offsets, int32_t* points_xy,
                                 rg_search_range* ranges, int cap_blocks, int64_t cap_points,
                                 int* n_blocks) {
  TRY(bind(ctx));
  if (!det || !cfg || !block_offsets || !n_blocks || n_occ < 0 || (n_occ > 0 && !occluder_boxes))
    return set_err(ctx, RG_EINVAL, "sample_query_points: bad arguments");
  *n_blocks = 0;
  block_offsets[0] = 0;
  if (cfg->close_scale < 1 || cfg->max_total_points < 0 || cfg->tau_s <= 0)
    return set_err(ctx, RG_EINVAL, "sample_query_points: bad config");
  // grid of sub-blocks (template_match.hpp:189-194), same IEEE ops as the device
  int rows = 1, cols = 1;
  if (kind != RG_KIND_FAR) {
    const double bx0 = (det->cx - det->w / 2) * img_w, bx1 = (det->cx + det->w / 2) * img_w;
    const double by0 = (det->cy - det->h / 2) * img_h, by1 = (det->cy + det->h / 2) * img_h;
    const double half_tau = cfg->tau_s / 2;
    cols = std::max(2, int((bx1 - bx0) / half_tau));
    rows = std::max(2, int((by1 - by0) / half_tau));
  }
  const int cap = std::max(1, int(std::sqrt(double(cfg->max_total_points))));
  const int q = kind == RG_KIND_FAR ? std::min(cfg->grid_side_points, cap)
                                    : std::min(cfg->close_block_side_points, cap);
  const int per_block = std::max(q * q, 1);
  const int nb = rows * cols;
  rg_detection* d = nullptr;
  TRY(upload_dets(ctx, det, 1, &d));
  double* docc = DBUF(double, ctx, B_TMP2, 4 * std::max(n_occ, 1));
  int32_t* pts = DBUF(int32_t, ctx, B_TMP0, 2 * (size_t)nb * per_block);
  int32_t* cnt = DBUF(int32_t, ctx, B_TMP1, nb);
  NEED(docc);
  NEED(pts);
  NEED(cnt);
  if (n_occ > 0)
    RG_CUDA(ctx, cudaMemcpyAsync(docc, occluder_boxes, sizeof(double) * 4 * n_occ, cudaMemcpyHostToDevice, ctx->stream));
  RG_CUDA(ctx, launch_sample_blocks(d, kind, docc, n_occ, *cfg, img_w, img_h, rows, cols, pts, cnt,
                                    per_block, ctx->stream));
  count_launch(ctx, ST_PLAN);
  std::vector<int32_t> hp(2 * (size_t)nb * per_block), hcnt(static_cast<size_t>(nb));
  RG_CUDA(ctx, cudaMemcpyAsync(hp.data(), pts, sizeof(int32_t) * hp.size(), cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaMemcpyAsync(hcnt.data(), cnt, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  const int s = cfg->close_scale;
  int out_b = 0;
  int64_t np = 0;
  for (int b = 0; b < nb; ++b) {
    if (hcnt[b] < 4) continue;  // template_match.hpp:185, 219
    if (out_b >= cap_blocks || np + hcnt[b] > cap_points)
      return set_err(ctx, RG_EOVERFLOW, "sample_query_points: output capacity");
    for (int k = 0; k < hcnt[b]; ++k) {
      points_xy[2 * (np + k)] = hp[2 * ((size_t)b * per_block + k)];
      points_xy[2 * (np + k) + 1] = hp[2 * ((size_t)b * per_block + k) + 1];
    }
    np += hcnt[b];
    ranges[out_b] = kind == RG_KIND_FAR ? rg_search_range{0, cfg->dx_max_far, -1, 1}
                                        : rg_search_range{0, (cfg->dx_max_close + s - 1) / s, -1, 1};
    block_offsets[++out_b] = np;
  }
  *n_blocks = out_b;
  return RG_OK;
}

rg_status rg_aggregate_close_disparities(rg_ctx* ctx, const double* disps, int n, double tau_d,
                                         int n_min, int32_t* valid, double* disparity,
                                         int32_t* run_length) {
  TRY(bind(ctx));
  if (n < 0 || (n > 0 && !disps) || !valid || !disparity || !run_length)
    return set_err(ctx, RG_EINVAL, "aggregate_close_disparities: bad arguments");
  double* dv = DBUF(double, ctx, B_TMP2, std::max(n, 1));
  double* scratch = DBUF(double, ctx, B_TMP3, std::max(n, 1));
  int32_t* oi = DBUF(int32_t, ctx, B_TMP0, 2);
  double* od = DBUF(double, ctx, B_TMP1, 1);
  NEED(dv);
  NEED(scratch);
  NEED(oi);
  NEED(od);
  if (n > 0) RG_CUDA(ctx, cudaMemcpyAsync(dv, disps, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  RG_CUDA(ctx, launch_aggregate_values(dv, n, tau_d, n_min, scratch, oi, od, ctx->stream));
  count_launch(ctx, ST_AGG);
  int32_t hi[2];
  double hd;
  RG_CUDA(ctx, cudaMemcpyAsync(hi, oi, sizeof(hi), cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaMemcpyAsync(&hd, od, sizeof(hd), cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *valid = hi[0];
  *run_length = hi[1];
  *disparity = hd;
  return RG_OK;
}

// =========================================================== estimate_object_disparities
rg_status rg_estimate_object_disparities(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w,
                                         int h, const rg_detection* dets, int n_dets,
                                         const rg_ranger_config* cfg, rg_census_cache* cache,
                                         double focal_px, double baseline_m, rg_object_disparity* out,
                                         int* n_out, rg_ranger_stats* stats) {
  RG_NVTX("rg_estimate_object_disparities");
  TRY(bind(ctx));
  TRY(check_cfg(ctx, cfg));
  if (cfg->census_9x7 && cache)  // caches hold 5x5 codes
    return set_err(ctx, RG_EINVAL, "estimate_object_disparities: census_9x7 cannot use a CensusCache");
  if (!left || !right || !n_out || w < 1 || h < 1 || n_dets < 0 || (n_dets > 0 && (!dets || !out)))
    return set_err(ctx, RG_EINVAL, "estimate_object_disparities: bad arguments");
  *n_out = 0;
  if (stats) {
    stats->query_points = 0;
    stats->image_pixels = (int64_t)w * h;
    stats->n_far = stats->n_close = 0;
  }
  if (n_dets == 0) return RG_OK;  // template_match.hpp:275
  if (n_dets > 4096) return set_err(ctx, RG_EINVAL, "estimate_object_disparities: > 4096 detections per frame");
  const int s = cfg->close_scale, cw = w / s, ch = h / s;
  cudaStream_t st = ctx->stream;
  uint8_t *dl = nullptr, *dr = nullptr;
  TRY(upload_image(ctx, B_IMG_L, left, w, h, &dl));
  TRY(upload_image(ctx, B_IMG_R, right, w, h, &dr));
  rg_detection* dd = nullptr;
  TRY(upload_dets(ctx, dets, n_dets, &dd));
  int32_t* doff = DBUF(int32_t, ctx, B_DET_OFF, 2);
  const int out_stride = std::max(1, std::min(n_dets, cfg->max_objects));
  rg_object_disparity* dout = DBUF(rg_object_disparity, ctx, B_OUT, out_stride);
  int32_t* dcnt = DBUF(int32_t, ctx, B_OUT_CNT, 1);
  rg_ranger_stats* dstats = DBUF(rg_ranger_stats, ctx, B_STATS, 1);
  NEED(doff);
  NEED(dout);
  NEED(dcnt);
  NEED(dstats);
  const int32_t hoff[2] = {0, n_dets};
  RG_CUDA(ctx, cudaMemcpyAsync(doff, hoff, sizeof(hoff), cudaMemcpyHostToDevice, st));
  FrameJob J = {dl, dr, 1, w, h, w, (int64_t)w * h, dd, doff, out_stride, dout, dcnt, dstats,
                focal_px, baseline_m};
  // a pre-filled cache is used as-is (template_match.hpp:312, 317); its host
  // codes are copied straight into the padded device rasters
  if (cache && cache->has_full) {
    J.full_l = cache->full_left;
    J.full_r = cache->full_right;
  }
  if (cache && cache->has_scaled && cw > 0 && ch > 0) {
    J.scaled_l = cache->scaled_left;
    J.scaled_r = cache->scaled_right;
  }
  PipelineBufs pb;
  TRY(run_pipeline(ctx, J, *cfg, st, &pb));
  int32_t hcnt = 0;
  RG_CUDA(ctx, cudaMemcpyAsync(&hcnt, dcnt, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RG_CUDA(ctx, cudaStreamSynchronize(st));
  RG_CUDA(ctx, cudaMemcpyAsync(out, dout, sizeof(rg_object_disparity) * hcnt, cudaMemcpyDeviceToHost, st));
  rg_ranger_stats hs;
  RG_CUDA(ctx, cudaMemcpyAsync(&hs, dstats, sizeof(hs), cudaMemcpyDeviceToHost, st));
  RG_CUDA(ctx, cudaStreamSynchronize(st));
  *n_out = hcnt;
  if (stats) *stats = hs;

  // fill an empty cache with ROI-masked codes (template_match.hpp:304-321)
  if (cache && (!cache->has_full || !cache->has_scaled)) {
    const int nslots = pb.capacity;  // CLOSE slots sit at the top of the list
    std::vector<ObjEntry> objs(static_cast<size_t>(hcnt));
    std::vector<rg_match_result> res(static_cast<size_t>(std::max(nslots, 1)));
    if (hcnt > 0)
      RG_CUDA(ctx, cudaMemcpyAsync(objs.data(), pb.objs, sizeof(ObjEntry) * hcnt, cudaMemcpyDeviceToHost, st));
    if (nslots > 0)
      RG_CUDA(ctx, cudaMemcpyAsync(res.data(), pb.res, sizeof(rg_match_result) * nslots, cudaMemcpyDeviceToHost, st));
    RG_CUDA(ctx, cudaStreamSynchronize(st));
    bool any_far = false, any_close = false;
    std::vector<rg_rect> far_rois, sc_rois;
    const int dxs = (cfg->dx_max_close + s - 1) / s;
    for (const ObjEntry& e : objs) {
      bool has_block = false;
      for (int t = 0; t < e.n_slots; ++t) has_block |= res[e.slot_base + t].n_points >= 4;
      const rg_detection& dt = dets[e.det];
      const double bx0 = (dt.cx - dt.w / 2) * w, bx1 = (dt.cx + dt.w / 2) * w;
      const double by0 = (dt.cy - dt.h / 2) * h, by1 = (dt.cy + dt.h / 2) * h;
      auto add_roi = [](std::vector<rg_rect>& v, double x0, double y0, double x1, double y1,
                        double sx, double sy, int dilx, int dily, int ww, int hh) {
        rg_rect r;  // template_match.hpp:245-253
        r.x0 = std::max(0, int(std::floor(x0 * sx)) - dilx);
        r.x1 = std::min(ww, int(std::ceil(x1 * sx)) + dilx + 1);
        r.y0 = std::max(0, int(std::floor(y0 * sy)) - dily);
        r.y1 = std::min(hh, int(std::ceil(y1 * sy)) + dily + 1);
        v.push_back(r);
      };
      if (e.kind == RG_KIND_FAR) {
        any_far |= has_block;
        add_roi(far_rois, bx0, by0, bx1, by1, 1, 1, cfg->dx_max_far + 2, 3, w, h);
      } else {
        any_close |= has_block;
        add_roi(sc_rois, bx0, by0, bx1, by1, double(cw) / w, double(ch) / h, dxs + 2, 3, cw, ch);
      }
    }
    auto fill = [&](const uint32_t* src, const PadGeom& g, const std::vector<rg_rect>& rois,
                    uint32_t* host) -> rg_status {
      const int ww = g.w, hh = g.h;
      uint32_t* tmp = DBUF(uint32_t, ctx, B_TMP1, (size_t)ww * hh);
      rg_rect* dro = DBUF(rg_rect, ctx, B_ROIS, std::max<size_t>(rois.size(), 1));
      NEED(tmp);
      NEED(dro);
      RG_CUDA(ctx, cudaMemcpy2DAsync(tmp, 4 * (size_t)ww, src + g.origin, 4 * (size_t)g.pitch, 4 * (size_t)ww, hh,
                                     cudaMemcpyDeviceToDevice, st));
      if (!rois.empty())
        RG_CUDA(ctx, cudaMemcpyAsync(dro, rois.data(), sizeof(rg_rect) * rois.size(), cudaMemcpyHostToDevice, st));
      RG_CUDA(ctx, launch_roi_mask(tmp, ww, hh, dro, (int)rois.size(), st));
      count_launch(ctx, ST_CENSUS);
      RG_CUDA(ctx, cudaMemcpyAsync(host, tmp, 4 * (size_t)ww * hh, cudaMemcpyDeviceToHost, st));
      RG_CUDA(ctx, cudaStreamSynchronize(st));
      return RG_OK;
    };
    if (!cache->has_full && any_far) {
      TRY(fill(pb.fl, pb.gf, far_rois, cache->full_left));
      TRY(fill(pb.fr, pb.gf, far_rois, cache->full_right));
      cache->has_full = 1;
    }
    if (!cache->has_scaled && any_close) {
      TRY(fill(pb.sl, pb.gs, sc_rois, cache->scaled_left));
      TRY(fill(pb.sr, pb.gs, sc_rois, cache->scaled_right));
      cache->has_scaled = 1;
    }
  }
  return RG_OK;
}

// =========================================================== batched frames
rg_status rg_range_frames(rg_ctx* ctx, const rg_frame_batch* b, const rg_ranger_config* cfg,
                          void* stream) {
  RG_NVTX("rg_range_frames");
  TRY(bind(ctx, false));
  TRY(check_cfg(ctx, cfg));
  if (!b || b->n_frames < 0 || b->width < 1 || b->height < 1 || b->pitch < b->width)
    return set_err(ctx, RG_EINVAL, "range_frames: bad batch");
  if (b->n_frames == 0) return RG_OK;
  if (b->max_dets_per_frame > 4096) return set_err(ctx, RG_EINVAL, "range_frames: > 4096 detections per frame");
  if (b->out_stride < std::min(b->max_dets_per_frame, cfg->max_objects))
    return set_err(ctx, RG_EINVAL, "range_frames: out_stride too small");
  FrameJob J = {b->d_left, b->d_right, b->n_frames, b->width, b->height, b->pitch, b->frame_stride,
                b->d_dets, b->d_det_offsets, b->out_stride, b->d_out, b->d_out_count, nullptr,
                b->focal_px, b->baseline_m};
  J.left_shift = b->d_left_shift;
  J.out_index = b->d_out_index;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (ctx->sync_mode || ctx->profiling || ctx->overlap) {  // blocking schedules (per-stage events, chunk joins)
    TRY(rg_sync(ctx));
    return run_pipeline_overlapped(ctx, J, *cfg, s);
  }
  return run_pipeline_async(ctx, J, *cfg, s);
}

rg_status rg_sync(rg_ctx* ctx) {  // (see also rg::wait_async)
  TRY(bind(ctx));
  TRY(retire_pending(ctx, true));
  ctx->last_stream = nullptr;
  if (ctx->overflowed) {
    const int n = ctx->overflowed;
    ctx->overflowed = 0;
    return set_err(ctx, RG_EOVERFLOW,
                   std::to_string(n) + " batch(es) overflowed the device block list and produced no results; "
                   "the list has grown: submit them again");
  }
  return RG_OK;
}

rg_status rg_set_sync_mode(rg_ctx* ctx, int on) {
  if (!ctx) return RG_EINVAL;
  TRY(rg_sync(ctx));
  ctx->sync_mode = on != 0;
  return RG_OK;
}

rg_status rg_range_frames_host(rg_ctx* ctx, const rg_frame_batch* b, const rg_ranger_config* cfg,
                               int chunk, void* stream) {
  RG_NVTX("rg_range_frames_host");
  TRY(bind(ctx));
  TRY(check_cfg(ctx, cfg));
  if (!b || b->n_frames < 0 || b->width < 1 || b->height < 1 || b->pitch < b->width)
    return set_err(ctx, RG_EINVAL, "range_frames_host: bad batch");
  if (b->n_frames == 0) return RG_OK;
  if (b->max_dets_per_frame > 4096) return set_err(ctx, RG_EINVAL, "range_frames_host: > 4096 detections per frame");
  if (b->out_stride < std::min(b->max_dets_per_frame, cfg->max_objects))
    return set_err(ctx, RG_EINVAL, "range_frames_host: out_stride too small");
  if (b->d_out_index) return set_err(ctx, RG_EINVAL, "range_frames_host: d_out_index is a device-batch output");
  if (chunk < 1) chunk = 16;
  const int F = b->n_frames;
  // compute on `stream` (or the context stream), H2D staging on copy_stream
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  cudaStream_t cs = ctx->copy_stream;
  const size_t img_bytes = (size_t)b->pitch * b->height;
  const int32_t* hoff = b->d_det_offsets;  // host pointers in this variant
  int max_chunk_dets = 1;
  for (int c0 = 0; c0 < F; c0 += chunk)
    max_chunk_dets = std::max(max_chunk_dets, hoff[std::min(F, c0 + chunk)] - hoff[c0]);
  // double-buffered device staging: images, detections, offsets, results
  uint8_t* st_l = DBUF(uint8_t, ctx, B_STAGE_L, 2 * img_bytes * chunk);
  uint8_t* st_r = DBUF(uint8_t, ctx, B_STAGE_R, 2 * img_bytes * chunk);
  rg_detection* st_d = DBUF(rg_detection, ctx, B_DETS, 2 * (size_t)max_chunk_dets);
  int32_t* st_o = DBUF(int32_t, ctx, B_DET_OFF, 2 * (size_t)(chunk + 1));
  rg_object_disparity* st_out = DBUF(rg_object_disparity, ctx, B_OUT, 2 * (size_t)chunk * b->out_stride);
  int32_t* st_cnt = DBUF(int32_t, ctx, B_OUT_CNT, 2 * (size_t)chunk);
  int32_t* counters = DBUF(int32_t, ctx, B_COUNTERS, kCounterInts);
  int32_t* hoffs = static_cast<int32_t*>(host_buf(ctx, 1, sizeof(int32_t) * 2 * (chunk + 1)));
  int32_t* hc = static_cast<int32_t*>(host_buf(ctx, 0, kCounterInts * sizeof(int32_t)));
  NEED(st_l);
  NEED(st_r);
  NEED(st_d);
  NEED(st_o);
  NEED(st_out);
  NEED(st_cnt);
  NEED(counters);
  NEED(hoffs);
  NEED(hc);
  // per-frame left shifts (host array in this variant): one upload
  int32_t* d_shift = nullptr;
  if (b->d_left_shift) {
    d_shift = DBUF(int32_t, ctx, B_SHIFT, F);
    NEED(d_shift);
    RG_CUDA(ctx, cudaMemcpyAsync(d_shift, b->d_left_shift, sizeof(int32_t) * F, cudaMemcpyHostToDevice, s));
  }
  cudaEvent_t ready[2] = {ctx->ev[6], ctx->ev[7]}, done[2] = {ctx->ev[8], ctx->ev[9]};
  auto stage = [&](int c0, int k) -> rg_status {  // H2D of one chunk into slot k
    const int n = std::min(chunk, F - c0);
    int32_t* ho = hoffs + k * (chunk + 1);
    for (int i = 0; i <= n; ++i) ho[i] = hoff[c0 + i] - hoff[c0];
    const size_t stride = (size_t)b->frame_stride;
    uint8_t* dl = st_l + (size_t)k * img_bytes * chunk;
    uint8_t* dr = st_r + (size_t)k * img_bytes * chunk;
    if (stride == img_bytes) {
      RG_CUDA(ctx, cudaMemcpyAsync(dl, b->d_left + c0 * stride, img_bytes * n, cudaMemcpyHostToDevice, cs));
      RG_CUDA(ctx, cudaMemcpyAsync(dr, b->d_right + c0 * stride, img_bytes * n, cudaMemcpyHostToDevice, cs));
    } else {
      for (int i = 0; i < n; ++i) {
        RG_CUDA(ctx, cudaMemcpyAsync(dl + i * img_bytes, b->d_left + (c0 + i) * stride, img_bytes, cudaMemcpyHostToDevice, cs));
        RG_CUDA(ctx, cudaMemcpyAsync(dr + i * img_bytes, b->d_right + (c0 + i) * stride, img_bytes, cudaMemcpyHostToDevice, cs));
      }
    }
    if (ho[n] > 0)
      RG_CUDA(ctx, cudaMemcpyAsync(st_d + (size_t)k * max_chunk_dets, b->d_dets + hoff[c0],
                                   sizeof(rg_detection) * ho[n], cudaMemcpyHostToDevice, cs));
    RG_CUDA(ctx, cudaMemcpyAsync(st_o + k * (chunk + 1), ho, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, cs));
    RG_CUDA(ctx, cudaEventRecord(ready[k], cs));
    return RG_OK;
  };
  TRY(stage(0, 0));
  for (int c0 = 0, it = 0; c0 < F; c0 += chunk, ++it) {
    const int k = it & 1, n = std::min(chunk, F - c0);
    RG_CUDA(ctx, cudaStreamWaitEvent(s, ready[k], 0));
    FrameJob J = {st_l + (size_t)k * img_bytes * chunk, st_r + (size_t)k * img_bytes * chunk, n, b->width,
                  b->height, b->pitch, (int64_t)img_bytes, st_d + (size_t)k * max_chunk_dets,
                  st_o + k * (chunk + 1), b->out_stride, st_out + (size_t)k * chunk * b->out_stride,
                  st_cnt + (size_t)k * chunk, nullptr, b->focal_px, b->baseline_m};
    if (d_shift) J.left_shift = d_shift + c0;
    TRY(enqueue_pipeline(ctx, J, *cfg, s, counters, nullptr));
    RG_CUDA(ctx, cudaEventRecord(done[k], s));
    // prefetch the next chunk into the other slot once its previous user is done
    if (c0 + chunk < F) {
      if (it >= 1) RG_CUDA(ctx, cudaStreamWaitEvent(cs, done[k ^ 1], 0));
      TRY(stage(c0 + chunk, k ^ 1));
    }
    TRY(finish_pipeline(ctx, J, *cfg, s, counters, hc, nullptr));
    RG_CUDA(ctx, cudaMemcpyAsync(b->d_out + (size_t)c0 * b->out_stride, J.out,
                                 sizeof(rg_object_disparity) * (size_t)n * b->out_stride,
                                 cudaMemcpyDeviceToHost, s));
    RG_CUDA(ctx, cudaMemcpyAsync(b->d_out_count + c0, J.out_count, sizeof(int32_t) * n,
                                 cudaMemcpyDeviceToHost, s));
  }
  RG_CUDA(ctx, cudaStreamSynchronize(s));
  RG_CUDA(ctx, cudaStreamSynchronize(cs));
  return RG_OK;
}

// =========================================================== BM / autorect
rg_status rg_validate_bm_params(rg_ctx* ctx, const rg_bm_params* p) { return check_bm(ctx, p); }

// bm_disparity on device images (w x h, packed) into device raw (w x h)
static rg_status bm_device(rg_ctx* ctx, const uint8_t* dl, const uint8_t* dr, int w, int h,
                           const rg_bm_params& p, int16_t* draw, cudaStream_t st) {
  const int s = p.downscale;
  if (s == 1) {
    RG_CUDA(ctx, launch_bm(dl, dr, 1, 0, w, h, w, h, 0, 0, 0, 1, p, draw, nullptr, st));
    count_launch(ctx, ST_RECT);
    return RG_OK;
  }
  const int ow = w / s, oh = h / s;  // image.hpp:98-105
  if (ow < 1 || oh < 1) return set_err(ctx, RG_EINVAL, "downscale: output would be empty");
  rg_bm_params q = p;  // bm.hpp:121-125
  q.downscale = 1;
  q.min_disparity = (p.min_disparity + s - 1) / s;
  q.num_disparities = std::max(1, (p.min_disparity + p.num_disparities) / s - q.min_disparity);
  uint8_t* ql = DBUF(uint8_t, ctx, B_TMP0, (size_t)ow * oh);
  uint8_t* qr = DBUF(uint8_t, ctx, B_TMP1, (size_t)ow * oh);
  int16_t* qm = DBUF(int16_t, ctx, B_TMP2, (size_t)ow * oh);
  NEED(ql);
  NEED(qr);
  NEED(qm);
  RG_CUDA(ctx, launch_downscale(dl, w, h, s, ql, st));
  RG_CUDA(ctx, launch_downscale(dr, w, h, s, qr, st));
  RG_CUDA(ctx, launch_bm(ql, qr, 1, 0, ow, oh, ow, oh, 0, 0, 0, 1, q, qm, nullptr, st));
  RG_CUDA(ctx, launch_upscale(qm, ow, oh, s, q.min_disparity * 16 * s, draw, w, h, st));
  count_launch(ctx, ST_RECT, 4);
  return RG_OK;
}

rg_status rg_bm_disparity(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                          const rg_bm_params* p, int16_t* out_raw) {
  TRY(bind(ctx));
  TRY(check_bm(ctx, p));
  if (!left || !right || !out_raw || w < 1 || h < 1)
    return set_err(ctx, RG_EINVAL, "bm_disparity: bad arguments");
  uint8_t *dl = nullptr, *dr = nullptr;
  TRY(upload_image(ctx, B_BM_L, left, w, h, &dl));
  TRY(upload_image(ctx, B_BM_R, right, w, h, &dr));
  int16_t* draw = DBUF(int16_t, ctx, B_BM_OUT, (size_t)w * h);
  NEED(draw);
  TRY(bm_device(ctx, dl, dr, w, h, *p, draw, ctx->stream));
  RG_CUDA(ctx, cudaMemcpyAsync(out_raw, draw, sizeof(int16_t) * w * h, cudaMemcpyDeviceToHost, ctx->stream));
  RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return RG_OK;
}

// raw value range of bm_disparity's output (bm.hpp:113-135: the downscale
// path matches over q and upscales raw by s)
static void bm_raw_range(const rg_bm_params& p, int* lo, int* hi) {
  const int s = p.downscale;
  if (s <= 1) {
    *lo = p.min_disparity * 16;
    *hi = (p.min_disparity + p.num_disparities) * 16 - 1;
    return;
  }
  const int qlo = (p.min_disparity + s - 1) / s;
  const int qnd = std::max(1, (p.min_disparity + p.num_disparities) / s - qlo);
  const int a = qlo * 16 * s, b = ((qlo + qnd) * 16 - 1) * s;
  *lo = std::min(a, b);
  *hi = std::max(a, b);
}

static rg_status box_stats_device(rg_ctx* ctx, const int16_t* draw, int w, int h, const rg_detection* ddets,
                                  const std::vector<int32_t>& idx, int raw_lo, int raw_hi, double sigma_obs2,
                                  double gamma, double sigma_sys2, std::vector<rg_box_stats>& res) {
  const int nb = (int)idx.size();
  res.assign(static_cast<size_t>(nb), rg_box_stats{});
  if (nb == 0) return RG_OK;
  const int nbins = raw_hi - raw_lo + 1;
  if (nbins < 1 || nbins > 49152) return set_err(ctx, RG_EINVAL, "box_disparity: raw range too wide");
  int32_t* didx = DBUF(int32_t, ctx, B_BOX_IDX, nb);
  rg_box_stats* dout = DBUF(rg_box_stats, ctx, B_BOX_OUT, nb);
  NEED(didx);
  NEED(dout);
  cudaStream_t st = ctx->stream;
  RG_CUDA(ctx, cudaMemcpyAsync(didx, idx.data(), sizeof(int32_t) * nb, cudaMemcpyHostToDevice, st));
  RG_CUDA(ctx, launch_box_disparity(draw, w, h, 0, ddets, didx, nullptr, nb, raw_lo, nbins, sigma_obs2, gamma,
                                    sigma_sys2, dout, st));
  count_launch(ctx, ST_AGG);
  RG_CUDA(ctx, cudaMemcpyAsync(res.data(), dout, sizeof(rg_box_stats) * nb, cudaMemcpyDeviceToHost, st));
  RG_CUDA(ctx, cudaStreamSynchronize(st));
  for (const auto& r : res)
    if (r.valid < 0) return set_err(ctx, RG_EINVAL, "box_disparity: raw value outside [raw_lo, raw_hi]");
  return RG_OK;
}

rg_status rg_box_disparity(rg_ctx* ctx, const int16_t* raw, int w, int h, const rg_detection* dets, int n,
                           int raw_lo, int raw_hi, double sigma_obs2, double gamma, double sigma_sys2,
                           rg_box_stats* out) {
  TRY(bind(ctx));
  if (!raw || w < 1 || h < 1 || n < 0 || (n > 0 && (!dets || !out)))
    return set_err(ctx, RG_EINVAL, "box_disparity: bad arguments");
  if (n == 0) return RG_OK;
  int16_t* draw = DBUF(int16_t, ctx, B_BM_OUT, (size_t)w * h);
  NEED(draw);
  RG_CUDA(ctx, cudaMemcpyAsync(draw, raw, sizeof(int16_t) * w * h, cudaMemcpyHostToDevice, ctx->stream));
  rg_detection* dd = nullptr;
  TRY(upload_dets(ctx, dets, n, &dd));
  std::vector<int32_t> idx(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::vector<rg_box_stats> res;
  TRY(box_stats_device(ctx, draw, w, h, dd, idx, raw_lo, raw_hi, sigma_obs2, gamma, sigma_sys2, res));
  std::copy(res.begin(), res.end(), out);
  return RG_OK;
}

rg_status rg_radar_refine_step(rg_ctx* ctx, int16_t* d_raw, int w, int h, const rg_radar_detection* radar, int n,
                               rg_vote_state* st, const rg_calibration* calib, double* applied) {
  RG_NVTX("rg_radar_refine_step");
  TRY(bind(ctx));
  if (!d_raw || !st || !calib || w < 1 || h < 1 || n < 0 || (n > 0 && !radar))
    return set_err(ctx, RG_EINVAL, "radar_refine_step: bad arguments");
  std::vector<int32_t> boxes(4 * (size_t)std::max(n, 1));
  std::vector<double> dr(std::max(n, 1));
  int nb = 0;
  if (rg_radar_boxes(radar, n, calib, w, h, boxes.data(), dr.data(), &nb) != RG_OK)
    return set_err(ctx, RG_EINVAL, "radar_refine_step: bad radar detections");
  std::vector<double> best(std::max(nb, 1), 0.0);
  std::vector<int32_t> found(std::max(nb, 1), 0);
  if (nb > 0) {  // the closest-offset search of every box on the device
    int32_t* db = DBUF(int32_t, ctx, B_TMP0, 4 * (size_t)nb);
    double* dd = DBUF(double, ctx, B_TMP1, 2 * (size_t)nb);
    int32_t* df = DBUF(int32_t, ctx, B_TMP2, (size_t)nb);
    NEED(db);
    NEED(dd);
    NEED(df);
    RG_CUDA(ctx, cudaMemcpyAsync(db, boxes.data(), sizeof(int32_t) * 4 * nb, cudaMemcpyHostToDevice, ctx->stream));
    RG_CUDA(ctx, cudaMemcpyAsync(dd, dr.data(), sizeof(double) * nb, cudaMemcpyHostToDevice, ctx->stream));
    RG_CUDA(ctx, launch_radar_votes(d_raw, w, db, dd, nb, dd + nb, df, ctx->stream));
    count_launch(ctx, ST_RECT);
    RG_CUDA(ctx, cudaMemcpyAsync(best.data(), dd + nb, sizeof(double) * nb, cudaMemcpyDeviceToHost, ctx->stream));
    RG_CUDA(ctx, cudaMemcpyAsync(found.data(), df, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, ctx->stream));
    RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  double a = 0.0;
  int raw_off = 0;
  if (rg_radar_vote_update(st, best.data(), found.data(), nb, &a, &raw_off) != RG_OK)
    return set_err(ctx, RG_EINVAL, "radar_refine_step: vote state not initialised");
  if (raw_off != 0) {
    RG_CUDA(ctx, launch_raw_offset(d_raw, (int64_t)w * h, raw_off, ctx->stream));
    count_launch(ctx, ST_RECT);
  }
  if (applied) *applied = a;
  return RG_OK;
}

rg_status rg_dense_objects_refined(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                                   const rg_detection* dets, int n, const rg_ranger_config* cfg,
                                   const rg_bm_params* bm, double sigma_obs2, double gamma, double sigma_sys2,
                                   const rg_radar_detection* radar, int n_radar, rg_vote_state* st,
                                   const rg_calibration* calib, rg_object_disparity* out, rg_box_stats* box_out,
                                   int* n_out, int16_t* raw_out, double* radar_applied) {
  RG_NVTX("rg_dense_objects");
  TRY(bind(ctx));
  TRY(check_cfg(ctx, cfg));
  TRY(check_bm(ctx, bm));
  if (!left || !right || !n_out || w < 1 || h < 1 || n < 0 || (n > 0 && (!dets || !out)))
    return set_err(ctx, RG_EINVAL, "dense_objects: bad arguments");
  if (st && (!calib || n_radar < 0 || (n_radar > 0 && !radar)))
    return set_err(ctx, RG_EINVAL, "dense_objects: radar refiner needs a calibration and the radar list");
  *n_out = 0;
  if (radar_applied) *radar_applied = 0.0;
  // pipeline.hpp:140-141: the selected detections in input order
  std::vector<int32_t> sel(static_cast<size_t>(std::max(n, 1)));
  int ns = 0;
  if (n > 0) TRY(rg_select_objects(ctx, dets, n, cfg, sel.data(), &ns));
  sel.resize(static_cast<size_t>(ns));
  std::sort(sel.begin(), sel.end());
  // primary depth: the dense BM map on the device (pipeline.hpp:284-286)
  uint8_t *dl = nullptr, *dr = nullptr;
  TRY(upload_image(ctx, B_BM_L, left, w, h, &dl));
  TRY(upload_image(ctx, B_BM_R, right, w, h, &dr));
  int16_t* draw = DBUF(int16_t, ctx, B_BM_OUT, (size_t)w * h);
  NEED(draw);
  TRY(bm_device(ctx, dl, dr, w, h, *bm, draw, ctx->stream));
  // the radar refiner on the dense map (pipeline.hpp:182-183)
  if (st) TRY(rg_radar_refine_step(ctx, draw, w, h, radar, n_radar, st, calib, radar_applied));
  if (raw_out)
    RG_CUDA(ctx, cudaMemcpyAsync(raw_out, draw, sizeof(int16_t) * w * h, cudaMemcpyDeviceToHost, ctx->stream));
  rg_detection* dd = nullptr;
  if (n > 0) TRY(upload_dets(ctx, dets, n, &dd));
  int lo = 0, hi = 0;
  bm_raw_range(*bm, &lo, &hi);
  if (st) lo = std::max(-32767, lo - 48), hi = std::min(32767, hi + 48);  // the refiner's offset is within +-3 px
  std::vector<rg_box_stats> res;
  TRY(box_stats_device(ctx, draw, w, h, dd, sel, lo, hi, sigma_obs2, gamma, sigma_sys2, res));
  // pipeline.hpp:218-224
  for (int k = 0; k < ns; ++k) {
    const rg_detection& d = dets[sel[k]];
    rg_object_disparity o{};
    o.det_id = d.id;
    const double side = std::max(d.w * w, d.h * h);  // classify_far_close, template_match.hpp:63-67
    o.kind = side < cfg->tau_s ? RG_KIND_FAR : RG_KIND_CLOSE;
    o.valid = res[k].valid > 0;
    o.disparity = o.valid ? res[k].median : 0.0;
    o.n_blocks_used = o.valid ? res[k].count : 0;
    out[k] = o;
    if (box_out) box_out[k] = res[k];
  }
  *n_out = ns;
  return RG_OK;
}

rg_status rg_dense_objects(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                           const rg_detection* dets, int n, const rg_ranger_config* cfg, const rg_bm_params* bm,
                           double sigma_obs2, double gamma, double sigma_sys2, rg_object_disparity* out,
                           rg_box_stats* box_out, int* n_out, int16_t* raw_out) {
  return rg_dense_objects_refined(ctx, left, right, w, h, dets, n, cfg, bm, sigma_obs2, gamma, sigma_sys2, nullptr,
                                  0, nullptr, nullptr, out, box_out, n_out, raw_out, nullptr);
}

static rg_status check_rect(rg_ctx* ctx, int w, int h, const rg_rect* roi, int dmin, int dmax,
                            const rg_bm_params* p) {  // autorect.hpp:25-32
  if (!roi || !p) return set_err(ctx, RG_EINVAL, "auto_rect_search: null argument");
  if (roi->x1 - roi->x0 < p->block_size || roi->y1 - roi->y0 < p->block_size)
    return set_err(ctx, RG_EINVAL, "auto_rect_search: ROI smaller than the match window");
  if (roi->x0 < 0 || roi->y0 < 0 || roi->x1 > w || roi->y1 > h)
    return set_err(ctx, RG_EINVAL, "auto_rect_search: ROI leaves the image");
  if (dmin > dmax) return set_err(ctx, RG_EINVAL, "auto_rect_search: empty delta range");
  return check_bm(ctx, p);
}

rg_status rg_auto_rect_search(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                              const rg_rect* roi, int delta_min, int delta_max, const rg_bm_params* p,
                              int32_t* best_delta, int64_t* counts) {
  TRY(bind(ctx));
  if (!left || !right || !best_delta || w < 1 || h < 1)
    return set_err(ctx, RG_EINVAL, "auto_rect_search: bad arguments");
  TRY(check_rect(ctx, w, h, roi, delta_min, delta_max, p));
  uint8_t *dl = nullptr, *dr = nullptr;
  TRY(upload_image(ctx, B_BM_L, left, w, h, &dl));
  TRY(upload_image(ctx, B_BM_R, right, w, h, &dr));
  const int nd = delta_max - delta_min + 1;
  int64_t* dc = DBUF(int64_t, ctx, B_BM_CNT, nd);
  int32_t* db = DBUF(int32_t, ctx, B_TMP3, 1);
  NEED(dc);
  NEED(db);
  cudaStream_t st = ctx->stream;
  RG_CUDA(ctx, cudaMemsetAsync(dc, 0, sizeof(int64_t) * nd, st));
  const int rw = roi->x1 - roi->x0, rh = roi->y1 - roi->y0;
  if (p->downscale == 1) {
    RG_CUDA(ctx, launch_bm(dl, dr, 1, 0, w, h, rw, rh, roi->x0, roi->y0, delta_min, nd, *p, nullptr, dc, st));
    count_launch(ctx, ST_RECT);
  } else {  // per delta: shifted crop -> bm_disparity (downscale path) -> count
    std::vector<int64_t> hc(static_cast<size_t>(nd));
    std::vector<int16_t> raw((size_t)rw * rh);
    std::vector<uint8_t> lc((size_t)rw * rh), rc((size_t)rw * rh);
    for (int y = 0; y < rh; ++y) std::memcpy(&rc[(size_t)y * rw], right + (size_t)(roi->y0 + y) * w + roi->x0, rw);
    uint8_t *cl = nullptr, *cr = nullptr;
    TRY(upload_image(ctx, B_STAGE_R, rc.data(), rw, rh, &cr));
    int16_t* draw = DBUF(int16_t, ctx, B_BM_OUT, (size_t)rw * rh);
    NEED(draw);
    for (int k = 0; k < nd; ++k) {
      const int delta = delta_min + k;
      for (int y = 0; y < rh; ++y) {
        int sy = roi->y0 + y - delta;
        sy = sy < 0 ? 0 : (sy >= h ? h - 1 : sy);
        std::memcpy(&lc[(size_t)y * rw], left + (size_t)sy * w + roi->x0, rw);
      }
      TRY(upload_image(ctx, B_STAGE_L, lc.data(), rw, rh, &cl));
      TRY(bm_device(ctx, cl, cr, rw, rh, *p, draw, st));
      RG_CUDA(ctx, cudaMemcpyAsync(raw.data(), draw, sizeof(int16_t) * raw.size(), cudaMemcpyDeviceToHost, st));
      RG_CUDA(ctx, cudaStreamSynchronize(st));
      int64_t c = 0;
      const int lo = p->min_disparity * 16;
      for (int16_t v : raw) c += (v != -32768 && v > lo);
      hc[k] = c;
    }
    RG_CUDA(ctx, cudaMemcpyAsync(dc, hc.data(), sizeof(int64_t) * nd, cudaMemcpyHostToDevice, st));
  }
  RG_CUDA(ctx, launch_autorect_pick(dc, 1, delta_min, nd, db, st));
  count_launch(ctx, ST_RECT);
  RG_CUDA(ctx, cudaMemcpyAsync(best_delta, db, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (counts) RG_CUDA(ctx, cudaMemcpyAsync(counts, dc, sizeof(int64_t) * nd, cudaMemcpyDeviceToHost, st));
  RG_CUDA(ctx, cudaStreamSynchronize(st));
  return RG_OK;
}

rg_status rg_auto_rect_frames(rg_ctx* ctx, const uint8_t* d_left, const uint8_t* d_right, int n_frames,
                              int64_t frame_stride, int pitch, int w, int h, const rg_rect* roi,
                              int delta_min, int delta_max, const rg_bm_params* p, int32_t* d_best,
                              int64_t* d_counts, void* stream) {
  RG_NVTX("rg_auto_rect_frames");
  TRY(bind(ctx));
  if (!d_left || !d_right || !d_best || n_frames < 0 || w < 1 || h < 1 || pitch < w)
    return set_err(ctx, RG_EINVAL, "auto_rect_frames: bad arguments");
  TRY(check_rect(ctx, w, h, roi, delta_min, delta_max, p));
  if (p->downscale != 1) return set_err(ctx, RG_EINVAL, "auto_rect_frames: downscale must be 1 (use rg_auto_rect_search)");
  if (n_frames == 0) return RG_OK;
  const int nd = delta_max - delta_min + 1;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  int64_t* dc = d_counts;
  if (!dc) {
    dc = DBUF(int64_t, ctx, B_BM_CNT, (size_t)n_frames * nd);
    NEED(dc);
  }
  if (ctx->profiling) RG_CUDA(ctx, cudaEventRecord(ctx->ev[10], st));
  RG_CUDA(ctx, cudaMemsetAsync(dc, 0, sizeof(int64_t) * n_frames * nd, st));
  RG_CUDA(ctx, launch_bm(d_left, d_right, n_frames, frame_stride, pitch, h, roi->x1 - roi->x0,
                         roi->y1 - roi->y0, roi->x0, roi->y0, delta_min, nd, *p, nullptr, dc, st));
  RG_CUDA(ctx, launch_autorect_pick(dc, n_frames, delta_min, nd, d_best, st));
  count_launch(ctx, ST_RECT, 2);
  if (ctx->profiling) {
    RG_CUDA(ctx, cudaEventRecord(ctx->ev[11], st));
    RG_CUDA(ctx, cudaEventSynchronize(ctx->ev[11]));
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ctx->ev[10], ctx->ev[11]) == cudaSuccess) ctx->stage_ms[ST_RECT] += ms;
  }
  return RG_OK;
}

}  // extern "C"

namespace rg {
// for entry points outside api.cu: wait for the context's asynchronous batches
rg_status wait_async(rg_ctx* ctx) {
  if (!ctx || !ctx->pend_n) return RG_OK;
  const rg_status st = retire_pending(ctx, true);
  ctx->last_stream = nullptr;
  return st;
}
}  // namespace rg
