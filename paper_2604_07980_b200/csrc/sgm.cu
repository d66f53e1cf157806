// sgm.cu -- census semi-global matching on sm_100a.
//
// Reference: sgm.hpp:37-155.  Stages, all on the device:
//   K1  census of both images (census.cu, reference layout)
//   S1  cost volume C[y][x][i] = popcount(cl(x,y) ^ cr(x-d,y)), d = d_min + i,
//       27 (kSgmNoData) where x-d leaves the frame (sgm.hpp:37-56)
//   S2  one kernel per path direction (sgm.hpp:60-110): a WARP walks one
//       path, lanes own disparities (d = lane + 32k); each step takes the
//       predecessor's L from registers, d+-1 by shuffles, the path minimum by a
//       warp reduction, and adds L into the int32 accumulator.  Paths of one
//       direction are independent, so the grid is one warp per path start.
//   S3  winner-take-all over evaluable disparities, parabolic sub-pixel in
//       the reference's FP64 operation order, lround, clamp (sgm.hpp:121-153).
// Integer arithmetic is identical to the reference's int32 recurrence; the
// only FP is S3's sub-pixel step (-fmad=false + explicit _rn intrinsics).
#include <climits>

#include "rg_common.cuh"

namespace rg {
namespace {

constexpr int kNoData = 27;         // detail::kSgmNoData, sgm.hpp:35
constexpr int kBig = INT_MAX / 4;   // sgm.hpp:63
constexpr int kInvalidRaw = -32768; // DisparityMap::kInvalid

__global__ void sgm_cost_kernel(const uint32_t* __restrict__ cl, const uint32_t* __restrict__ cr, int w, int h,
                                int nd, int d_lo, uint8_t* __restrict__ cost) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)w * h * nd;
  if (idx >= total) return;
  const int i = (int)(idx % nd);
  const int64_t px = idx / nd;
  const int x = (int)(px % w), y = (int)(px / w);
  const int rx = x - (d_lo + i);
  uint8_t c = (uint8_t)kNoData;
  if (rx >= 0 && rx < w) c = (uint8_t)__popc(cl[(int64_t)y * w + x] ^ cr[(int64_t)y * w + rx]);
  cost[idx] = c;
}

// one warp per path of direction (sx, sy); path starts = pixels whose
// predecessor p - (sx, sy) is outside the image
template <int NDW>
__global__ void __launch_bounds__(128) sgm_pass_kernel(const uint8_t* __restrict__ cost, int w, int h, int nd,
                                                       int p1, int p2, int sx, int sy, int32_t* __restrict__ acc,
                                                       int n_starts, int row_starts) {
  const int lane = threadIdx.x & 31;
  const int path = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (path >= n_starts) return;
  int x, y;
  if (path < row_starts) {  // starts on the first row of the walk (sy != 0)
    x = path;
    y = sy > 0 ? 0 : h - 1;
  } else {                  // starts on the first column of the walk (sx != 0)
    const int k = path - row_starts + (sy != 0 ? 1 : 0);
    x = sx > 0 ? 0 : w - 1;
    y = sy >= 0 ? k : h - 1 - k;
  }
  int L[NDW];
  int pmin = 0;
  bool first = true;
  // the next step's costs are loaded one step ahead (they do not depend on L)
  int cn[NDW];
  auto load_cost = [&](int xx, int yy) {
    const uint8_t* c = cost + ((int64_t)yy * w + xx) * nd;
#pragma unroll
    for (int k = 0; k < NDW; ++k) {
      const int d = lane + 32 * k;
      cn[k] = d < nd ? (int)__ldg(c + d) : 0;
    }
  };
  load_cost(x, y);
  while (x >= 0 && x < w && y >= 0 && y < h) {
    int32_t* a = acc + ((int64_t)y * w + x) * nd;
    int cv[NDW];
#pragma unroll
    for (int k = 0; k < NDW; ++k) cv[k] = cn[k];
    {
      const int xn = x + sx, yn = y + sy;
      if (xn >= 0 && xn < w && yn >= 0 && yn < h) load_cost(xn, yn);
    }
    int mn = kBig;
    if (first) {
#pragma unroll
      for (int k = 0; k < NDW; ++k) L[k] = (lane + 32 * k < nd) ? cv[k] : kBig;
      first = false;
    } else {
      int Ln[NDW];
#pragma unroll
      for (int k = 0; k < NDW; ++k) {
        // predecessor L at d-1 and d+1 (kBig outside [0, nd): the reference
        // skips those terms, sgm.hpp:94-95)
        int lm = __shfl_up_sync(0xffffffffu, L[k], 1);
        int lp = __shfl_down_sync(0xffffffffu, L[k], 1);
        const int lm_prev = __shfl_sync(0xffffffffu, L[k > 0 ? k - 1 : 0], 31);
        const int lp_next = __shfl_sync(0xffffffffu, L[k + 1 < NDW ? k + 1 : k], 0);
        if (lane == 0) lm = k > 0 ? lm_prev : kBig;
        if (lane == 31) lp = k + 1 < NDW ? lp_next : kBig;
        const int d = lane + 32 * k;
        if (d + 1 >= nd) lp = kBig;
        int best = L[k];
        if (lm != kBig) best = min(best, lm + p1);
        if (lp != kBig) best = min(best, lp + p1);
        best = min(best, pmin + p2);
        Ln[k] = d < nd ? cv[k] + best - pmin : kBig;
      }
#pragma unroll
      for (int k = 0; k < NDW; ++k) L[k] = Ln[k];
    }
#pragma unroll
    for (int k = 0; k < NDW; ++k) {
      mn = min(mn, L[k]);
      const int d = lane + 32 * k;
      if (d < nd) a[d] += L[k];
    }
    pmin = __reduce_min_sync(0xffffffffu, mn);
    x += sx;
    y += sy;
  }
}

__device__ __forceinline__ double subpix(double cm, double c0, double cp) {  // census.hpp:167-171
  const double denom = __dsub_rn(__dadd_rn(cm, cp), __dmul_rn(2.0, c0));
  if (denom <= 0.0) return 0.0;
  return __ddiv_rn(-__dsub_rn(cp, cm), __dmul_rn(2.0, denom));
}

__global__ void sgm_wta_kernel(const int32_t* __restrict__ acc, int w, int h, int nd, int d_lo,
                               int16_t* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w || y >= h) return;
  const int32_t* a = acc + ((int64_t)y * w + x) * nd;
  int best_i = -1, best = INT_MAX;
  for (int i = 0; i < nd; ++i) {
    const int rx = x - (d_lo + i);
    if (rx < 0 || rx >= w) continue;  // winner must be evaluable
    const int v = a[i];
    if (v < best) {
      best = v;
      best_i = i;
    }
  }
  int r = kInvalidRaw;
  if (best_i >= 0) {
    double d_hat = (double)(d_lo + best_i);
    if (best_i > 0 && best_i + 1 < nd && x - (d_lo + best_i + 1) >= 0)
      d_hat = __dadd_rn(d_hat, subpix((double)a[best_i - 1], (double)best, (double)a[best_i + 1]));
    long long v = llround(__dmul_rn(d_hat, 16.0));
    const long long lo = (long long)d_lo * 16, hi = (long long)(d_lo + nd) * 16 - 1;
    v = v < lo ? lo : (v > hi ? hi : v);
    r = (int)v;
  }
  out[(int64_t)y * w + x] = (int16_t)r;
}

}  // namespace

cudaError_t launch_sgm_cost(const uint32_t* cl, const uint32_t* cr, int w, int h, int nd, int d_lo, uint8_t* cost,
                            cudaStream_t s) {
  const int64_t total = (int64_t)w * h * nd;
  if (total <= 0) return cudaSuccess;
  sgm_cost_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(cl, cr, w, h, nd, d_lo, cost);
  return cudaGetLastError();
}

cudaError_t launch_sgm_pass(const uint8_t* cost, int w, int h, int nd, int p1, int p2, int sx, int sy,
                            int32_t* acc, cudaStream_t s) {
  if (w <= 0 || h <= 0 || nd <= 0 || (sx == 0 && sy == 0)) return cudaSuccess;
  const int row_starts = sy != 0 ? w : 0;
  const int col_starts = sx != 0 ? (sy != 0 ? h - 1 : h) : 0;
  const int n = row_starts + col_starts;
  const int grid = (n + 3) / 4;
  const int ndw = (nd + 31) / 32;
#define RG_SGM_CASE(K) \
  case K: sgm_pass_kernel<K><<<grid, 128, 0, s>>>(cost, w, h, nd, p1, p2, sx, sy, acc, n, row_starts); break;
  switch (ndw) {
    RG_SGM_CASE(1) RG_SGM_CASE(2) RG_SGM_CASE(3) RG_SGM_CASE(4)
    RG_SGM_CASE(5) RG_SGM_CASE(6) RG_SGM_CASE(7) RG_SGM_CASE(8)
    default: return cudaErrorInvalidValue;
  }
#undef RG_SGM_CASE
  return cudaGetLastError();
}

cudaError_t launch_sgm_wta(const int32_t* acc, int w, int h, int nd, int d_lo, int16_t* out, cudaStream_t s) {
  if (w <= 0 || h <= 0) return cudaSuccess;
  dim3 grid((w + 127) / 128, h);
  sgm_wta_kernel<<<grid, 128, 0, s>>>(acc, w, h, nd, d_lo, out);
  return cudaGetLastError();
}

}  // namespace rg

// ------------------------------------------------------------------ C ABI
using namespace rg;

namespace {

rg_status sgm_bind(rg_ctx* ctx) {
  if (!ctx) return RG_EINVAL;
  cudaError_t e = cudaSetDevice(ctx->device);
  return e == cudaSuccess ? RG_OK : cuda_err(ctx, e, "cudaSetDevice");
}

rg_status sgm_check(rg_ctx* ctx, const rg_sgm_params* p) {  // sgm.hpp:21-28
  if (!p) return set_err(ctx, RG_EINVAL, "SgmParams: null");
  if (p->num_disparities < 1) return set_err(ctx, RG_EINVAL, "SgmParams: num_disparities must be >= 1");
  if (p->p1 < 0 || p->p2 < p->p1) return set_err(ctx, RG_EINVAL, "SgmParams: need 0 <= P1 <= P2");
  if (p->num_disparities > 256) return set_err(ctx, RG_EINVAL, "SgmParams: num_disparities > 256 unsupported");
  return RG_OK;
}

#define SG_TRY(expr)                  \
  do {                                \
    rg_status _s = (expr);            \
    if (_s != RG_OK) return _s;       \
  } while (0)
#define SG_NEED(ptr)                                                      \
  do {                                                                    \
    if (!(ptr)) return set_err(ctx, RG_ENOMEM, "device allocation failed"); \
  } while (0)

// census (reference layout) -> cost -> 4 passes -> WTA on device images
rg_status sgm_device(rg_ctx* ctx, const uint8_t* dl, const uint8_t* dr, int w, int h, int pitch,
                     const rg_sgm_params* p, int16_t* d_out, cudaStream_t s) {
  const int nd = p->num_disparities;
  const size_t px = (size_t)w * h;
  uint32_t* cl = static_cast<uint32_t*>(dev_buf(ctx, B_TMP0, sizeof(uint32_t) * px));
  uint32_t* cr = static_cast<uint32_t*>(dev_buf(ctx, B_TMP1, sizeof(uint32_t) * px));
  uint8_t* cost = static_cast<uint8_t*>(dev_buf(ctx, B_SGM_COST, px * nd));
  int32_t* acc = static_cast<int32_t*>(dev_buf(ctx, B_SGM_ACC, sizeof(int32_t) * px * nd));
  SG_NEED(cl);
  SG_NEED(cr);
  SG_NEED(cost);
  SG_NEED(acc);
  const PadGeom g = make_geom(w, h, 0, 0);
  RG_CUDA(ctx, launch_census_frames(dl, dr, 1, (int64_t)pitch * h, pitch, w, h, cl, cr, g, nullptr, nullptr, g,
                                    nullptr, nullptr, nullptr, false, s));
  count_launch(ctx, 0);
  RG_CUDA(ctx, launch_sgm_cost(cl, cr, w, h, nd, p->min_disparity, cost, s));
  RG_CUDA(ctx, cudaMemsetAsync(acc, 0, sizeof(int32_t) * px * nd, s));
  const int dirs[4][2] = {{1, 0}, {0, 1}, {1, 1}, {-1, 1}};  // sgm.hpp:130
  for (const auto& d : dirs) RG_CUDA(ctx, launch_sgm_pass(cost, w, h, nd, p->p1, p->p2, d[0], d[1], acc, s));
  RG_CUDA(ctx, launch_sgm_wta(acc, w, h, nd, p->min_disparity, d_out, s));
  count_launch(ctx, 4, 6);
  return RG_OK;
}

}  // namespace

extern "C" {

rg_status rg_validate_sgm_params(rg_ctx* ctx, const rg_sgm_params* p) {
  SG_TRY(sgm_bind(ctx));
  return sgm_check(ctx, p);
}

rg_status rg_sgm_disparity(rg_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                           const rg_sgm_params* p, int16_t* out_raw) {
  SG_TRY(sgm_bind(ctx));
  SG_TRY(sgm_check(ctx, p));
  if (!left || !right || !out_raw || w < 1 || h < 1) return set_err(ctx, RG_EINVAL, "sgm_disparity: bad image");
  cudaStream_t s = ctx->stream;
  const size_t px = (size_t)w * h;
  uint8_t* dl = static_cast<uint8_t*>(dev_buf(ctx, B_IMG_L, px));
  uint8_t* dr = static_cast<uint8_t*>(dev_buf(ctx, B_IMG_R, px));
  int16_t* dout = static_cast<int16_t*>(dev_buf(ctx, B_BM_OUT, sizeof(int16_t) * px));
  SG_NEED(dl);
  SG_NEED(dr);
  SG_NEED(dout);
  RG_CUDA(ctx, cudaMemcpyAsync(dl, left, px, cudaMemcpyHostToDevice, s));
  RG_CUDA(ctx, cudaMemcpyAsync(dr, right, px, cudaMemcpyHostToDevice, s));
  SG_TRY(sgm_device(ctx, dl, dr, w, h, w, p, dout, s));
  RG_CUDA(ctx, cudaMemcpyAsync(out_raw, dout, sizeof(int16_t) * px, cudaMemcpyDeviceToHost, s));
  RG_CUDA(ctx, cudaStreamSynchronize(s));
  return RG_OK;
}

rg_status rg_sgm_frames(rg_ctx* ctx, const uint8_t* d_left, const uint8_t* d_right, int n_frames,
                        int64_t frame_stride, int pitch, int w, int h, const rg_sgm_params* p, int16_t* d_raw,
                        void* stream) {
  SG_TRY(sgm_bind(ctx));
  SG_TRY(sgm_check(ctx, p));
  if (!d_left || !d_right || !d_raw || n_frames < 0 || w < 1 || h < 1 || pitch < w)
    return set_err(ctx, RG_EINVAL, "sgm_frames: bad arguments");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  for (int f = 0; f < n_frames; ++f)
    SG_TRY(sgm_device(ctx, d_left + f * frame_stride, d_right + f * frame_stride, w, h, pitch, p,
                      d_raw + (int64_t)f * w * h, s));
  return RG_OK;
}

rg_status rg_sgm_cost_volume(rg_ctx* ctx, const uint32_t* left_codes, const uint32_t* right_codes, int w, int h,
                             const rg_sgm_params* p, uint8_t* cost) {
  SG_TRY(sgm_bind(ctx));
  SG_TRY(sgm_check(ctx, p));
  if (!left_codes || !right_codes || !cost || w < 1 || h < 1)
    return set_err(ctx, RG_EINVAL, "sgm_cost_volume: bad arguments");
  cudaStream_t s = ctx->stream;
  const size_t px = (size_t)w * h, nd = (size_t)p->num_disparities;
  uint32_t* cl = static_cast<uint32_t*>(dev_buf(ctx, B_TMP0, sizeof(uint32_t) * px));
  uint32_t* cr = static_cast<uint32_t*>(dev_buf(ctx, B_TMP1, sizeof(uint32_t) * px));
  uint8_t* dc = static_cast<uint8_t*>(dev_buf(ctx, B_SGM_COST, px * nd));
  SG_NEED(cl);
  SG_NEED(cr);
  SG_NEED(dc);
  RG_CUDA(ctx, cudaMemcpyAsync(cl, left_codes, sizeof(uint32_t) * px, cudaMemcpyHostToDevice, s));
  RG_CUDA(ctx, cudaMemcpyAsync(cr, right_codes, sizeof(uint32_t) * px, cudaMemcpyHostToDevice, s));
  RG_CUDA(ctx, launch_sgm_cost(cl, cr, w, h, (int)nd, p->min_disparity, dc, s));
  count_launch(ctx, 4);
  RG_CUDA(ctx, cudaMemcpyAsync(cost, dc, px * nd, cudaMemcpyDeviceToHost, s));
  RG_CUDA(ctx, cudaStreamSynchronize(s));
  return RG_OK;
}

rg_status rg_sgm_direction_pass(rg_ctx* ctx, const uint8_t* cost, int w, int h, int nd, int p1, int p2, int sx,
                                int sy, int32_t* acc) {
  SG_TRY(sgm_bind(ctx));
  if (!cost || !acc || w < 1 || h < 1 || nd < 1 || nd > 256 || sx < -1 || sx > 1 || sy < -1 || sy > 1)
    return set_err(ctx, RG_EINVAL, "sgm_direction_pass: bad arguments");
  cudaStream_t s = ctx->stream;
  const size_t n = (size_t)w * h * nd;
  uint8_t* dc = static_cast<uint8_t*>(dev_buf(ctx, B_SGM_COST, n));
  int32_t* da = static_cast<int32_t*>(dev_buf(ctx, B_SGM_ACC, sizeof(int32_t) * n));
  SG_NEED(dc);
  SG_NEED(da);
  RG_CUDA(ctx, cudaMemcpyAsync(dc, cost, n, cudaMemcpyHostToDevice, s));
  RG_CUDA(ctx, cudaMemcpyAsync(da, acc, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  RG_CUDA(ctx, launch_sgm_pass(dc, w, h, nd, p1, p2, sx, sy, da, s));
  count_launch(ctx, 4);
  RG_CUDA(ctx, cudaMemcpyAsync(acc, da, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  RG_CUDA(ctx, cudaStreamSynchronize(s));
  return RG_OK;
}

}  // extern "C"
