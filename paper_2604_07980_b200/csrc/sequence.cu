// sequence.cu -- host orchestration of the TEMPLATE_MATCHER frame loop.
//
// Pipeline::process_frame (pipeline.hpp:124-178) ranges frame t on
// shift_vertical(left_t, lround(current)) where `current` is the rectification
// offset filtered over the offset searches of frames < t; the search itself
// runs on the UNCORRECTED pair (pipeline.hpp:144-149).  That dependency is only
// through the cheap host-side filter, so a batch of frames runs as two device
// passes around one host scan (SURVEY.md 8(e) "two-pass schedule"):
//   pass A  rg_auto_rect_frames: delta*_t for every frame (K5/K6, batched)
//   host    for t in order: shift_t = lround(current); filter_offset(delta*_t)
//   pass B  rg_range_frames with d_left_shift = shift_t (K1 row remap)
// Both passes are the batched kernels; frames never leave the device.
#include <algorithm>
#include <cmath>
#include <vector>

#include "rg_common.cuh"

using namespace rg;

namespace {

rg_status fail(rg_ctx* ctx, rg_status st, const char* msg) { return set_err(ctx, st, msg); }

}  // namespace

extern "C" {

rg_status rg_rect_state_init(rg_rect_state* st, int window, double rate) {  // autorect.hpp:69-72
  if (!st || window < 1 || window > RG_RECT_MAX_WINDOW) return RG_EINVAL;
  *st = rg_rect_state{};
  st->window = window;
  st->delta_max = rate;
  st->current = 0.0;
  return RG_OK;
}

rg_status rg_filter_offset(rg_rect_state* st, int delta_star, double* applied) {  // autorect.hpp:77-90
  if (!st || st->window < 1 || st->window > RG_RECT_MAX_WINDOW || st->n_hist < 0 || st->n_hist > st->window)
    return RG_EINVAL;
  if (st->n_hist < st->window) {
    st->history[st->n_hist++] = delta_star;
  } else {
    st->history[st->next] = delta_star;
    st->next = (st->next + 1) % st->n_hist;
  }
  int v[RG_RECT_MAX_WINDOW];
  std::copy(st->history, st->history + st->n_hist, v);
  std::sort(v, v + st->n_hist);
  const double candidate = v[(st->n_hist - 1) / 2];  // lower median
  const double step = std::clamp(candidate - st->current, -st->delta_max, st->delta_max);
  st->current += step;
  if (applied) *applied = st->current;
  return RG_OK;
}

rg_status rg_range_sequence(rg_ctx* ctx, const rg_frame_batch* b, const rg_ranger_config* cfg,
                            const rg_rect_search_config* rect, rg_rect_state* st, int32_t* out_shift,
                            int32_t* out_delta, double* out_rect_applied, void* stream) {
  RG_NVTX("rg_range_sequence");
  if (!ctx) return RG_EINVAL;
  if (cudaSetDevice(ctx->device) != cudaSuccess || wait_async(ctx) != RG_OK) return RG_ECUDA;
  if (!b || !cfg || !rect || !st) return fail(ctx, RG_EINVAL, "range_sequence: null argument");
  if (b->n_frames < 0 || b->width < 1 || b->height < 1)
    return fail(ctx, RG_EINVAL, "range_sequence: bad batch");
  const int F = b->n_frames, w = b->width, h = b->height;
  if (F == 0) return RG_OK;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  std::vector<int32_t> delta(F, 0), shift(F, 0);
  std::vector<double> applied(F, 0.0);
  if (rect->enabled) {
    if (rect->delta_min > rect->delta_max) return fail(ctx, RG_EINVAL, "range_sequence: empty offset range");
    if (st->window < 1 || st->window > RG_RECT_MAX_WINDOW)
      return fail(ctx, RG_EINVAL, "range_sequence: rect state not initialised");
    // rect_search_roi: the central half, grown to one block (pipeline.hpp:268-275)
    rg_rect roi = {w / 4, h / 4, w * 3 / 4, h * 3 / 4};
    const int need = rect->bm.block_size;
    roi.x1 = std::max(roi.x1, std::min(w, roi.x0 + need));
    roi.y1 = std::max(roi.y1, std::min(h, roi.y0 + need));
    // pass A: the offset search on the uncorrected pairs of every frame
    int32_t* d_best = static_cast<int32_t*>(dev_buf(ctx, B_SEQ, sizeof(int32_t) * F));
    if (!d_best) return fail(ctx, RG_ENOMEM, "device allocation failed");
    rg_status e = rg_auto_rect_frames(ctx, b->d_left, b->d_right, F, b->frame_stride, b->pitch, w, h, &roi,
                                      rect->delta_min, rect->delta_max, &rect->bm, d_best, nullptr, s);
    if (e != RG_OK) return e;
    RG_CUDA(ctx, cudaMemcpyAsync(delta.data(), d_best, sizeof(int32_t) * F, cudaMemcpyDeviceToHost, s));
    RG_CUDA(ctx, cudaStreamSynchronize(s));
    // host scan in frame order: the shift applied to frame t is the filter
    // state before frame t's own search result is pushed
    for (int t = 0; t < F; ++t) {
      applied[t] = st->current;  // RefinerLogRecord::rect_delta (pipeline.hpp:134, 264)
      shift[t] = (int32_t)std::lround(st->current);
      if ((e = rg_filter_offset(st, delta[t], nullptr)) != RG_OK)
        return fail(ctx, e, "range_sequence: filter_offset");
    }
  }
  // pass B: ranging with the per-frame left shifts
  rg_frame_batch bb = *b;
  bb.d_left_shift = nullptr;
  if (rect->enabled) {
    int32_t* d_shift = static_cast<int32_t*>(dev_buf(ctx, B_SHIFT, sizeof(int32_t) * F));
    if (!d_shift) return fail(ctx, RG_ENOMEM, "device allocation failed");
    RG_CUDA(ctx, cudaMemcpyAsync(d_shift, shift.data(), sizeof(int32_t) * F, cudaMemcpyHostToDevice, s));
    bb.d_left_shift = d_shift;
  }
  const rg_status e = rg_range_frames(ctx, &bb, cfg, s);
  if (e != RG_OK) return e;
  if (out_shift) std::copy(shift.begin(), shift.end(), out_shift);
  if (out_delta) std::copy(delta.begin(), delta.end(), out_delta);
  if (out_rect_applied) std::copy(applied.begin(), applied.end(), out_rect_applied);
  // (the pageable shift upload is staged before cudaMemcpyAsync returns, so
  // the host vector may go; pass B stays asynchronous on s)
  return RG_OK;
}

}  // extern "C"
