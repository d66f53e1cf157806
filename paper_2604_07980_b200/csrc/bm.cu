// bm.cu -- K5: SAD block matcher and the auto-rectification offset search.
//
// Replaces bm_disparity_at_scale / bm_disparity (reference bm.hpp:37-135),
// downscale / upscale_disparity (image.hpp:98-141) and the per-delta body of
// auto_rect_search (autorect.hpp:37-44).  The vertical offset delta is a grid
// dimension: CTA (tile, frame*n_delta + k) matches the ROI crop of the left
// image shifted by delta_min + k rows (edge-row clamp, image.hpp:145-154)
// against the unshifted right crop, entirely in crop-local coordinates
// (bm.hpp:47-61).  Per disparity the 9x9 SAD is a separable box sum:
// column sums staged in shared memory, then a running row sum per thread.
// The per-pixel winner is tracked in streaming form over increasing d:
// first minimum, its two neighbours, and the second best over |i-best| > 1
// (via the prefix minimum lagging two indices behind) -- exactly the
// reference's rules (bm.hpp:75-92).  Valid counts (raw > 16*d_min) are
// reduced per CTA and added with one integer atomic (deterministic).
#include <cstdlib>

#include <algorithm>
#include <cstdlib>

#include "rg_common.cuh"

namespace rg {
namespace {

constexpr int BT = 256;  // threads
constexpr int TXB = 64;  // tile columns (8 threads x 8 pixels)
constexpr int TYB = 32;  // tile rows
constexpr int kInvalid = -32768;
constexpr int kBig = 0x7fffffff;

__device__ __forceinline__ double subpix(double cm, double c0, double cp) {  // census.hpp:167-171
  const double denom = __dsub_rn(__dadd_rn(cm, cp), __dmul_rn(2.0, c0));
  if (denom <= 0.0) return 0.0;
  return __ddiv_rn(-__dsub_rn(cp, cm), __dmul_rn(2.0, denom));
}

// Dynamic smem: L tile [(TYB+2hw) x LW], R tile [(TYB+2hw) x RW], column sums
// [TYB x CW] ints.
__global__ void __launch_bounds__(BT) bm_kernel(const uint8_t* __restrict__ left,
                                                const uint8_t* __restrict__ right, int64_t stride,
                                                int pitch, int img_h, int W, int H, int x0c,
                                                int y0c, int delta_min, int n_delta, int bs,
                                                int d_lo, int nd, double tex, double uniq,
                                                int16_t* __restrict__ raw,
                                                int64_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int hw = bs / 2;
  const int frame = blockIdx.z / n_delta, kd = blockIdx.z - frame * n_delta;
  const int delta = delta_min + kd;
  const uint8_t* Limg = left + (int64_t)frame * stride;
  const uint8_t* Rimg = right + (int64_t)frame * stride;
  const int tx0 = blockIdx.x * TXB, ty0 = blockIdx.y * TYB;
  const int d_hi = d_lo + nd;
  const int TR = TYB + 2 * hw;              // tile rows incl. halo
  const int LW = TXB + 2 * hw;              // left tile columns
  const int lx0 = tx0 - hw;                 // crop column of L tile col 0
  const int rx0 = tx0 - hw - (d_hi - 1);    // crop column of R tile col 0
  const int RW = TXB + 2 * hw + nd - 1;
  const int CW = LW;                        // column sums per row
  uint8_t* Lt = smem;
  uint8_t* Rt = Lt + TR * LW;
  int* cs = reinterpret_cast<int*>(smem + (((TR * (LW + RW)) + 15) & ~15));

  // stage crops: left rows shifted by delta with edge clamp, right unshifted;
  // values outside the crop are never used by a defined pixel
  for (int i = threadIdx.x; i < TR * LW; i += BT) {
    const int r = i / LW, c = i - r * LW;
    const int cy = ty0 - hw + r, cx = lx0 + c;
    uint8_t v = 0;
    if (cy >= 0 && cy < H && cx >= 0 && cx < W) {
      int sy = y0c + cy - delta;
      sy = sy < 0 ? 0 : (sy >= img_h ? img_h - 1 : sy);
      v = Limg[(int64_t)sy * pitch + x0c + cx];
    }
    Lt[i] = v;
  }
  for (int i = threadIdx.x; i < TR * RW; i += BT) {
    const int r = i / RW, c = i - r * RW;
    const int cy = ty0 - hw + r, cx = rx0 + c;
    uint8_t v = 0;
    if (cy >= 0 && cy < H && cx >= 0 && cx < W) v = Rimg[(int64_t)(y0c + cy) * pitch + x0c + cx];
    Rt[i] = v;
  }
  __syncthreads();

  // this thread's 8 pixels: one row, 8 consecutive columns
  const int seg = threadIdx.x & 7, row = threadIdx.x >> 3;
  const int y = ty0 + row;
  const int xs = tx0 + seg * 8;
  // per-pixel streaming state
  int best[8], bi[8], second[8], cmv[8], cpv[8], last[8], pm2[8], neval[8];
  bool defined[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int x = xs + p;
    defined[p] = x >= hw && x < W - hw && y >= hw && y < H - hw;
    if (defined[p]) {  // texture gate, bm.hpp:50-56
      long grad = 0;
      const int lc = x - lx0;
      for (int j = -hw; j <= hw; ++j) {
        const uint8_t* r = Lt + (row + hw + j) * LW + lc;
        for (int i = -hw; i < hw; ++i) grad += abs((int)r[i + 1] - (int)r[i]);
      }
      if ((double)grad < tex) defined[p] = false;
    }
    best[p] = kBig;
    bi[p] = -1;
    second[p] = kBig;
    cmv[p] = -1;
    cpv[p] = -1;
    last[p] = -1;
    pm2[p] = kBig;
    neval[p] = 0;
  }

  for (int idx = 0; idx < nd; ++idx) {
    const int d = d_lo + idx;
    // column sums: cs[r][c] = sum_j |L(r+j, c) - R(r+j, c - d)|, c over L tile
    const int roff = (lx0 - d) - rx0;  // R tile column of L tile column 0
    for (int it = threadIdx.x; it < CW * (TYB / 8); it += BT) {
      const int c = it % CW, g = it / CW;
      const int r0 = g * 8;
      int s = 0;
      for (int j = 0; j < bs; ++j)
        s += abs((int)Lt[(r0 + j) * LW + c] - (int)Rt[(r0 + j) * RW + c + roff]);
      cs[r0 * CW + c] = s;
      for (int r = r0 + 1; r < r0 + 8; ++r) {
        s += abs((int)Lt[(r + bs - 1) * LW + c] - (int)Rt[(r + bs - 1) * RW + c + roff]) -
             abs((int)Lt[(r - 1) * LW + c] - (int)Rt[(r - 1) * RW + c + roff]);
        cs[r * CW + c] = s;
      }
    }
    __syncthreads();
    // row sums over bs columns and the streaming winner update
    const int* csr = cs + row * CW + seg * 8;  // cs col of pixel xs - hw
    int sad = 0;
    for (int i = 0; i < bs; ++i) sad += csr[i];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      if (p > 0) sad += csr[p - 1 + bs] - csr[p - 1];
      const int x = xs + p;
      const bool ev = defined[p] && (x - d - hw >= 0) && (x - d + hw < W);  // bm.hpp:61-64
      const int v = ev ? sad : -1;
      if (v >= 0) {
        ++neval[p];
        if (v < best[p]) {  // new first minimum at idx
          second[p] = pm2[p];  // min over indices <= idx-2
          best[p] = v;
          bi[p] = idx;
          cmv[p] = last[p];
          cpv[p] = -1;
        } else {
          if (idx == bi[p] + 1)
            cpv[p] = v;
          else if (idx > bi[p] + 1 && v < second[p])
            second[p] = v;
        }
      } else if (idx == bi[p] + 1) {
        cpv[p] = -1;
      }
      // advance the lagged prefix minimum: pm2(idx+1) = min(pm2(idx), sad[idx-1])
      if (last[p] >= 0 && last[p] < pm2[p]) pm2[p] = last[p];
      last[p] = v;
    }
    __syncthreads();
  }

  // epilogue: uniqueness, sub-pixel, raw (bm.hpp:74-100)
  int valid_count = 0;
  const int lo = d_lo * 16;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int x = xs + p;
    if (x >= W || y >= H) continue;
    int out = kInvalid;
    if (defined[p] && neval[p] > 0) {
      bool ok = true;
      if (second[p] != kBig &&
          __dmul_rn((double)best[p], __dadd_rn(1.0, __ddiv_rn(uniq, 100.0))) >= (double)second[p])
        ok = false;
      if (ok) {
        double d_hat = (double)(d_lo + bi[p]);
        if (bi[p] > 0 && bi[p] + 1 < nd && cmv[p] >= 0 && cpv[p] >= 0)
          d_hat = __dadd_rn(d_hat, subpix((double)cmv[p], (double)best[p], (double)cpv[p]));
        long long r = llround(__dmul_rn(d_hat, 16.0));
        const long long rlo = (long long)d_lo * 16, rhi = (long long)d_hi * 16 - 1;
        r = r < rlo ? rlo : (r > rhi ? rhi : r);
        out = (int)r;
      }
    }
    if (raw) raw[((int64_t)frame * n_delta + kd) * W * H + (int64_t)y * W + x] = (int16_t)out;
    if (out != kInvalid && out > lo) ++valid_count;
  }
  if (counts) {
    for (int o = 16; o > 0; o >>= 1) valid_count += __shfl_xor_sync(0xffffffffu, valid_count, o);
    __shared__ int wsum[BT / 32];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = valid_count;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int q = 0; q < BT / 32; ++q) t += wsum[q];
      if (t) atomicAdd((unsigned long long*)&counts[(int64_t)frame * n_delta + kd], (unsigned long long)t);
    }
  }
}

// ---------------------------------------------------------------------------
// Fast SAD matcher: disparities in lanes.  A warp owns a band of 32 output
// columns and a strip of rows of one (frame, delta) crop; lane l owns the
// disparities d_lo + l + 32k (k < DPL).  Per lane the column sums of |L - R|
// over the 2HW+1 window rows live in registers for the band plus halo and
// are updated by one row in / one row out per output row; the 9-wide row sum
// slides along the band.  Per pixel the argmin over d is a warp reduction:
// __reduce_min_sync on (SAD << 7 | d) gives the first minimum (ties -> the
// smaller d, bm.hpp:75-82), a second reduction the best over |i - best| > 1
// (bm.hpp:84-89), two shuffles the neighbours; the FP64 epilogue then runs
// lane-parallel over the band's 32 pixels.  Texture gate (bm.hpp:50-56):
// column sums of horizontal |diffs| per lane column, window sum by shuffles.
constexpr int LBW = 32;   // band width (output columns)
constexpr int LRS = 32;   // strip rows
constexpr int LWPB = 4;   // warps (bands) per CTA

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

template <int HW, int DPL>
__global__ void __launch_bounds__(LWPB * 32) bm_lanes_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t stride, int pitch, int img_h,
    int W, int H, int x0c, int y0c, int delta_min, int n_delta, int d_lo, int nd, double tex, double uniq,
    int16_t* __restrict__ raw, int64_t* __restrict__ counts, int skip0, int skip1) {
  constexpr int NC = LBW + 2 * HW;  // column sums per lane
  // column sums in smem, lane-major so every access is conflict-free
  __shared__ int css[LWPB][DPL][NC][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int band = blockIdx.x * LWPB + warp;
  const int xb = band * LBW;
  if (xb >= W || (band >= skip0 && band < skip1)) return;  // warp-uniform; no block-level sync below
  const int yb = blockIdx.y * LRS;
  const int frame = blockIdx.z / n_delta, kd = blockIdx.z - frame * n_delta;
  const int delta = delta_min + kd;
  const uint8_t* Limg = left + (int64_t)frame * stride + x0c;
  const uint8_t* Rimg = right + (int64_t)frame * stride + x0c;
  const int d_hi = d_lo + nd;
  int(*cs)[NC][32] = css[warp];
  // crop row -> image row (left shifted by delta with edge clamp, image.hpp:145-154)
  auto lrow = [&](int yr) { return Limg + (int64_t)clampi(y0c + clampi(yr, 0, H - 1) - delta, 0, img_h - 1) * pitch; };
  auto rrow = [&](int yr) { return Rimg + (int64_t)(y0c + clampi(yr, 0, H - 1)) * pitch; };
  // this lane's disparity offsets into the right row (clamped: out-of-crop
  // samples only reach non-evaluable (x, d) pairs)
  int dd[DPL];
#pragma unroll
  for (int k = 0; k < DPL; ++k) dd[k] = d_lo + lane + 32 * k;
  for (int c = 0; c < NC; ++c) {
    const int xc = clampi(xb - HW + c, 0, W - 1);
    int acc[DPL];
#pragma unroll
    for (int k = 0; k < DPL; ++k) acc[k] = 0;
    for (int j = -HW; j <= HW; ++j) {
      const uint8_t* lr = lrow(yb + j);
      const uint8_t* rr = rrow(yb + j);
      const int lv = lr[xc];
#pragma unroll
      for (int k = 0; k < DPL; ++k) acc[k] += abs(lv - (int)rr[clampi(xb - HW + c - dd[k], 0, W - 1)]);
    }
#pragma unroll
    for (int k = 0; k < DPL; ++k) cs[k][c][lane] = acc[k];
  }
  // texture column sums: lane holds columns xb-HW+lane and xb-HW+32+lane
  int tv0 = 0, tv1 = 0;
  const int tc0 = xb - HW + lane, tc1 = tc0 + 32;
  auto hd = [&](const uint8_t* lr, int c) {
    return abs((int)lr[clampi(c + 1, 0, W - 1)] - (int)lr[clampi(c, 0, W - 1)]);
  };
  for (int j = -HW; j <= HW; ++j) {
    const uint8_t* lr = lrow(yb + j);
    tv0 += hd(lr, tc0);
    tv1 += hd(lr, tc1);
  }
  int valid_count = 0;
  const int lo_raw = d_lo * 16;
  const int yend = min(yb + LRS, H);
  for (int y = yb; y < yend; ++y) {
    if (y > yb) {  // slide the column sums down one row
      const uint8_t* ln = lrow(y + HW);
      const uint8_t* rn = rrow(y + HW);
      const uint8_t* lo = lrow(y - HW - 1);
      const uint8_t* ro = rrow(y - HW - 1);
#pragma unroll 4
      for (int c = 0; c < NC; ++c) {
        const int xc = clampi(xb - HW + c, 0, W - 1);
        const int lnv = ln[xc], lov = lo[xc];
#pragma unroll
        for (int k = 0; k < DPL; ++k) {
          const int xr = clampi(xb - HW + c - dd[k], 0, W - 1);
          cs[k][c][lane] += abs(lnv - (int)rn[xr]) - abs(lov - (int)ro[xr]);
        }
      }
      tv0 += hd(ln, tc0) - hd(lo, tc0);
      tv1 += hd(ln, tc1) - hd(lo, tc1);
    }
    __syncwarp();
    // texture gate of this lane's pixel x = xb + lane: columns x-HW .. x+HW-1
    int grad = 0;
#pragma unroll
    for (int t = 0; t < 2 * HW; ++t) {
      const int src = lane + t;
      const int a = __shfl_sync(0xffffffffu, tv0, src & 31);
      const int b = __shfl_sync(0xffffffffu, tv1, src & 31);
      grad += src < 32 ? a : b;
    }
    // per-pixel argmin over d (results land in lane == pixel index)
    int my_best = 0, my_bi = -1, my_second = 0x7fffffff, my_cm = -1, my_cp = -1;
    int sad[DPL];
#pragma unroll
    for (int k = 0; k < DPL; ++k) {
      sad[k] = 0;
#pragma unroll
      for (int c = 0; c < 2 * HW + 1; ++c) sad[k] += cs[k][c][lane];
    }
#pragma unroll 2
    for (int xi = 0; xi < LBW; ++xi) {
      if (xi > 0) {
#pragma unroll
        for (int k = 0; k < DPL; ++k) sad[k] += cs[k][xi + 2 * HW][lane] - cs[k][xi - 1][lane];
      }
      const int x = xb + xi;
      int key = 0x7fffffff;
      bool ev[DPL];
#pragma unroll
      for (int k = 0; k < DPL; ++k) {
        ev[k] = (lane + 32 * k < nd) && (x - dd[k] - HW >= 0) && (x - dd[k] + HW < W);  // bm.hpp:61-64
        if (ev[k]) key = min(key, (sad[k] << 7) | (lane + 32 * k));
      }
      const int bk = __reduce_min_sync(0xffffffffu, key);
      if (bk != 0x7fffffff) {  // warp-uniform
        const int bi = bk & 127;
        int sec = 0x7fffffff, vm = -1, vp = -1;
#pragma unroll
        for (int k = 0; k < DPL; ++k) {
          const int i = lane + 32 * k;
          if (ev[k] && abs(i - bi) > 1) sec = min(sec, sad[k]);
          if (bi >= 1 && k == ((bi - 1) >> 5)) vm = ev[k] ? sad[k] : -1;
          if (k == ((bi + 1) >> 5)) vp = ev[k] ? sad[k] : -1;
        }
        sec = __reduce_min_sync(0xffffffffu, sec);
        const int cm = __shfl_sync(0xffffffffu, vm, (bi - 1) & 31);
        const int cp = __shfl_sync(0xffffffffu, vp, (bi + 1) & 31);
        if (lane == xi) {
          my_best = bk >> 7;
          my_bi = bi;
          my_second = sec;
          my_cm = bi >= 1 ? cm : -1;
          my_cp = bi + 1 < nd ? cp : -1;
        }
      }
    }
    // lane-parallel epilogue for pixel (xb + lane, y) (bm.hpp:47-100)
    const int x = xb + lane;
    if (x < W) {
      int out = kInvalid;
      const bool defined = x >= HW && x < W - HW && y >= HW && y < H - HW && !((double)grad < tex);
      if (defined && my_bi >= 0) {
        bool ok = true;
        if (my_second != 0x7fffffff &&
            __dmul_rn((double)my_best, __dadd_rn(1.0, __ddiv_rn(uniq, 100.0))) >= (double)my_second)
          ok = false;
        if (ok) {
          double d_hat = (double)(d_lo + my_bi);
          if (my_bi > 0 && my_bi + 1 < nd && my_cm >= 0 && my_cp >= 0)
            d_hat = __dadd_rn(d_hat, subpix((double)my_cm, (double)my_best, (double)my_cp));
          long long r = llround(__dmul_rn(d_hat, 16.0));
          const long long rlo = (long long)d_lo * 16, rhi = (long long)d_hi * 16 - 1;
          r = r < rlo ? rlo : (r > rhi ? rhi : r);
          out = (int)r;
        }
      }
      if (raw) raw[((int64_t)frame * n_delta + kd) * W * H + (int64_t)y * W + x] = (int16_t)out;
      if (out != kInvalid && out > lo_raw) ++valid_count;
    }
    __syncwarp();
  }
  if (counts) {
    valid_count = __reduce_add_sync(0xffffffffu, valid_count);
    if (lane == 0 && valid_count)
      atomicAdd((unsigned long long*)&counts[(int64_t)frame * n_delta + kd], (unsigned long long)valid_count);
  }
}

template <int HW, int DPL>
static cudaError_t launch_lanes(const uint8_t* left, const uint8_t* right, int n_frames, int64_t stride, int pitch,
                                int img_h, int w, int h, int x0, int y0, int delta_min, int n_delta, rg_bm_params p,
                                int16_t* raw, int64_t* counts, cudaStream_t s, int skip0 = 0, int skip1 = 0) {
  const int bands = (w + LBW - 1) / LBW;
  if (skip0 <= 0 && skip1 >= bands) return cudaSuccess;
  dim3 grid((bands + LWPB - 1) / LWPB, (h + LRS - 1) / LRS, n_frames * n_delta);
  bm_lanes_kernel<HW, DPL><<<grid, LWPB * 32, 0, s>>>(left, right, stride, pitch, img_h, w, h, x0, y0, delta_min,
                                                       n_delta, p.min_disparity, p.num_disparities,
                                                       p.texture_threshold, p.uniqueness_ratio, raw, counts,
                                                       skip0, skip1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Byte-SIMD SAD matcher for num_disparities <= 32, block_size <= 9 (the
// autorect search and the common dense configs).  Same band/strip tiling as
// bm_lanes_kernel (warp = 32 output columns x SB_RS rows of one (frame, delta)
// crop, lane = disparity), but every stage runs packed:
//   * |L - R| of 4 columns is one VABSDIFF4 (__vabsdiffu4) on 32-bit words:
//     the lane's right-row bytes x - d are realigned by a funnel shift;
//   * the 2HW+1-row column sums V are 16-bit pairs (c, c+1) updated by one
//     IADD3 per pair (V + new - old is exact lane-wise: both lanes' results
//     are window sums in [0, 2^16), so no borrow crosses the halves); the
//     absolute differences of the last 2HW+1 rows live in a shared-memory ring;
//   * the row-direction box sum slides over (x, x+16) pairs, one IADD3 per
//     two output pixels;
//   * the per-pixel argmin is transposed: lane d writes key = SAD << 5 | d for
//     its 32 pixels into a [pixel][d] tile and lane x then reduces its own
//     32 keys with 3-input mins (first minimum = smallest d, bm.hpp:75-82);
//     the second best (|i - best| > 1, bm.hpp:84-89) is a second pass after
//     masking the three neighbours in the tile.
// Texture gate (bm.hpp:50-56): sum of 8 adjacent |diffs| per window row with
// two VABSDIFF4.ACC (__vsadu4) per row, slid over rows.
// Only bands whose byte reads stay inside the image rows are run here (the
// launcher computes that range); the others run bm_lanes_kernel.
constexpr int SB_W = 4;     // warps (bands) per CTA
#ifndef RG_BM_RS
#define RG_BM_RS 32
#endif
constexpr int SB_RS = RG_BM_RS;  // rows per warp strip
constexpr int SB_NCW = 10;  // AD words per row: columns xb-4 .. xb+35
constexpr int SB_TP = 36;   // transpose tile pitch (words)
constexpr uint32_t SB_INF = 0xFFFFFFFFu;

#ifndef RG_BM_RING
#define RG_BM_RING 0  // 1: |L-R| of the window rows kept in a smem ring; 0: recompute the leaving row
#endif
constexpr int SB_RINGW = RG_BM_RING ? SB_NCW : 0;

template <int HW>
constexpr size_t sb_smem() {
  return sizeof(uint32_t) * SB_W * ((2 * HW + 1) * (SB_RINGW + 1) * 32 + 32 * SB_TP);
}

#ifndef RG_BM_MINB
#define RG_BM_MINB 8
#endif
template <int HW, bool LA>  // LA: the band's left columns are word-aligned (x0 % 4 == 0)
__global__ void __launch_bounds__(SB_W * 32, RG_BM_MINB) bm_simd_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t stride, int pitch, int img_h,
    int W, int H, int x0c, int y0c, int delta_min, int n_delta, int d_lo, int nd, double tex, double uniq,
    int16_t* __restrict__ raw, int64_t* __restrict__ counts, int band0, int band1) {
  constexpr int NR = 2 * HW + 1;
  extern __shared__ __align__(16) uint32_t sbm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int band = band0 + blockIdx.x * SB_W + warp;
  if (band >= band1) return;  // warp-uniform; warps never synchronise with each other
  uint32_t* ring = sbm + warp * (NR * (SB_RINGW + 1) * 32 + 32 * SB_TP);  // [NR][NCW][32]
  int* tring = reinterpret_cast<int*>(ring + NR * SB_RINGW * 32);           // [NR][32] texture rows
  uint32_t* tile = ring + NR * (SB_RINGW + 1) * 32;                        // [32 pixels][SB_TP]
  const int xb = band * 32;
  const int yb = blockIdx.y * SB_RS;
  if (yb >= H) return;
  const int frame = blockIdx.z / n_delta, kd = blockIdx.z - frame * n_delta;
  const int delta = delta_min + kd;
  const uint8_t* Lf = left + (int64_t)frame * stride;
  const uint8_t* Rf = right + (int64_t)frame * stride;
  // crop row -> image row pointers (left shifted by delta with edge clamp,
  // image.hpp:145-154; crop rows clamped like the reference's reads never need)
  auto lrow = [&](int yr) {
    return reinterpret_cast<const uint32_t*>(
        Lf + (int64_t)clampi(y0c + clampi(yr, 0, H - 1) - delta, 0, img_h - 1) * pitch);
  };
  auto rrow = [&](int yr) {
    return reinterpret_cast<const uint32_t*>(Rf + (int64_t)(y0c + clampi(yr, 0, H - 1)) * pitch);
  };
  const int k = lane;
  const int dk = d_lo + min(k, nd - 1);      // idle lanes (k >= nd) read valid bytes
  const int lcol = x0c + xb - 4;             // image column of AD column 0
  const int lw0 = lcol >> 2, lsh = (lcol & 3) * 8;
  const int rcol = lcol - dk;                // this lane's right column for AD column 0
  const int rw0 = rcol >> 2, rsh = (rcol & 3) * 8;
  // |L - R| words of one crop row: columns xb-4+4g .. +3 of this lane's d
  auto ad_row = [&](int yr, uint32_t (&a)[SB_NCW]) {
    const uint32_t* lp = lrow(yr) + lw0;
    const uint32_t* rp = rrow(yr) + rw0;
    uint32_t lv[SB_NCW + 1], rv[SB_NCW + 1];
#pragma unroll
    for (int g = 0; g <= SB_NCW; ++g) {
      if (!LA || g < SB_NCW) lv[g] = __ldg(lp + g);
      rv[g] = __ldg(rp + g);
    }
#pragma unroll
    for (int g = 0; g < SB_NCW; ++g)
      a[g] = __vabsdiffu4(LA ? lv[g] : __funnelshift_r(lv[g], lv[g + 1], lsh),
                          __funnelshift_r(rv[g], rv[g + 1], rsh));
  };
  // texture: 8 adjacent |diffs| of row yr around pixel x = xb + lane (columns
  // x-4 .. x+4), window columns x-HW .. x+HW only
  const int tcol = x0c + xb + lane - 4;
  const int tw0 = tcol >> 2, tsh = (tcol & 3) * 8;
  constexpr uint32_t TM0 = HW >= 4 ? 0xFFFFFFFFu : (0xFFFFFFFFu << (8 * (4 - HW)));   // i = -4..-1
  constexpr uint32_t TM1 = HW >= 4 ? 0xFFFFFFFFu : (0xFFFFFFFFu >> (8 * (4 - HW)));   // i = 0..3
  auto tex_row = [&](int yr) -> int {
    const uint32_t* lp = lrow(yr) + tw0;
    const uint32_t u0 = __ldg(lp), u1 = __ldg(lp + 1), u2 = __ldg(lp + 2);
    const uint32_t a0 = __funnelshift_r(u0, u1, tsh), a1 = __funnelshift_r(u1, u2, tsh);  // x-4..x-1, x..x+3
    const uint32_t b0 = __funnelshift_r(a0, a1, 8), b1 = __funnelshift_r(a1, __funnelshift_r(u2, u2, tsh), 8);
    return (int)__vsadu4(a0 & TM0, b0 & TM0) + (int)__vsadu4(a1 & TM1, b1 & TM1);
  };
  // ---- initial window rows yb-HW .. yb+HW
  uint32_t V[SB_NCW * 2];
#pragma unroll
  for (int i = 0; i < SB_NCW * 2; ++i) V[i] = 0u;
  int grad = 0;
  for (int r = 0; r < NR; ++r) {
    uint32_t a[SB_NCW];
    ad_row(yb - HW + r, a);
#pragma unroll
    for (int g = 0; g < SB_NCW; ++g) {
      if (RG_BM_RING) ring[(r * SB_RINGW + g) * 32 + lane] = a[g];
      V[2 * g] += __byte_perm(a[g], 0u, 0x4140);
      V[2 * g + 1] += __byte_perm(a[g], 0u, 0x4342);
    }
    const int tr = tex_row(yb - HW + r);
    tring[r * 32 + lane] = tr;
    grad += tr;
  }
  // evaluable pixels of this lane's d: x - d - HW >= 0 && x - d + HW < W (bm.hpp:61-64)
  const int xlo = dk + HW - xb, xhi = W - 1 - HW + dk - xb;  // band-relative
  const bool all_ev = __all_sync(0xffffffffu, k >= nd || (xlo <= 0 && xhi >= 31));
  const int x = xb + lane;
  const int lo_raw = d_lo * 16;
  int valid_count = 0;
  const int yend = min(yb + SB_RS, H);
  for (int y = yb; y < yend; ++y) {
    if (y > yb) {  // slide the window down one row: + row y+HW, - row y-HW-1
      const int slot = (y - yb - 1) % NR;
      uint32_t a[SB_NCW], ao[SB_NCW];
      ad_row(y + HW, a);
      if (!RG_BM_RING) ad_row(y - HW - 1, ao);
#pragma unroll
      for (int g = 0; g < SB_NCW; ++g) {
        uint32_t o;
        if (RG_BM_RING) {
          uint32_t* rs = ring + (slot * SB_RINGW + g) * 32 + lane;
          o = *rs;
          *rs = a[g];
        } else {
          o = ao[g];
        }
        V[2 * g] = V[2 * g] + __byte_perm(a[g], 0u, 0x4140) - __byte_perm(o, 0u, 0x4140);
        V[2 * g + 1] = V[2 * g + 1] + __byte_perm(a[g], 0u, 0x4342) - __byte_perm(o, 0u, 0x4342);
      }
      const int tr = tex_row(y + HW);
      grad += tr - tring[slot * 32 + lane];
      tring[slot * 32 + lane] = tr;
    }
    // ---- row box sums over (x, x+16) pairs; AD column c = x + 4 (+16)
    uint32_t Vh[16 + 2 * HW];  // Vh[j] = (V(j - HW + 4), V(j - HW + 20))
#pragma unroll
    for (int j = 0; j < 16 + 2 * HW; ++j) {
      const int c = j - HW + 4;
      Vh[j] = __byte_perm(V[c >> 1], V[(c >> 1) + 8], (c & 1) ? 0x7632 : 0x5410);
    }
    uint32_t S = 0;
#pragma unroll
    for (int j = 0; j < 2 * HW + 1; ++j) S += Vh[j];
    const uint32_t kbits = (k < nd) ? (uint32_t)k : SB_INF;
    if (all_ev) {  // every (pixel, d) of the band is evaluable: no masks
#pragma unroll
      for (int xi = 0; xi < 16; ++xi) {
        if (xi > 0) S = S + Vh[xi + 2 * HW] - Vh[xi - 1];
        tile[xi * SB_TP + k] = ((S << 5) & 0x1FFFE0u) | kbits;           // pixel xi
        tile[(xi + 16) * SB_TP + k] = ((S >> 11) & 0x1FFFE0u) | kbits;   // pixel xi + 16
      }
    } else {
#pragma unroll
      for (int xi = 0; xi < 16; ++xi) {
        if (xi > 0) S = S + Vh[xi + 2 * HW] - Vh[xi - 1];
        uint32_t k0 = ((S << 5) & 0x1FFFE0u) | kbits;
        uint32_t k1 = ((S >> 11) & 0x1FFFE0u) | kbits;
        if (xi < xlo || xi > xhi) k0 = SB_INF;
        if (xi + 16 < xlo || xi + 16 > xhi) k1 = SB_INF;
        tile[xi * SB_TP + k] = k0;
        tile[(xi + 16) * SB_TP + k] = k1;
      }
    }
    __syncwarp();
    // ---- per-pixel argmin: lane = pixel xb + lane
    uint32_t* row = tile + lane * SB_TP;
    uint32_t bk = SB_INF;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + 4 * q);
      bk = min(min(bk, v.x), min(v.y, min(v.z, v.w)));
    }
    int out = kInvalid;
    const bool defined = x < W && x >= HW && x < W - HW && y >= HW && y < H - HW && !((double)grad < tex);
    if (bk != SB_INF) {
      const int bi = (int)(bk & 31u);
      const uint32_t vm = bi >= 1 ? row[bi - 1] : SB_INF;
      const uint32_t vp = bi + 1 < 32 ? row[bi + 1] : SB_INF;
      // second best over |i - bi| > 1
      if (bi >= 1) row[bi - 1] = SB_INF;
      row[bi] = SB_INF;
      if (bi + 1 < 32) row[bi + 1] = SB_INF;
      uint32_t sk = SB_INF;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(row + 4 * q);
        sk = min(min(sk, v.x), min(v.y, min(v.z, v.w)));
      }
      if (defined) {
        const int best = (int)(bk >> 5);
        bool ok = true;
        if (sk != SB_INF && __dmul_rn((double)best, __dadd_rn(1.0, __ddiv_rn(uniq, 100.0))) >= (double)(sk >> 5))
          ok = false;
        if (ok && !raw) {
          // count-only (autorect): raw > d_lo*16 <=> bi >= 1, since the
          // parabolic offset of a minimum lies in [-1/2, 1/2] (no FP64 needed)
          if (bi >= 1) ++valid_count;
        } else if (ok) {
          double d_hat = (double)(d_lo + bi);
          if (bi > 0 && bi + 1 < nd && vm != SB_INF && vp != SB_INF)
            d_hat = __dadd_rn(d_hat, subpix((double)(vm >> 5), (double)best, (double)(vp >> 5)));
          long long r = llround(__dmul_rn(d_hat, 16.0));
          const long long rlo = (long long)d_lo * 16, rhi = (long long)(d_lo + nd) * 16 - 1;
          r = r < rlo ? rlo : (r > rhi ? rhi : r);
          out = (int)r;
        }
      }
    }
    if (x < W && raw) {
      raw[((int64_t)frame * n_delta + kd) * W * H + (int64_t)y * W + x] = (int16_t)out;
      if (out != kInvalid && out > lo_raw) ++valid_count;
    }
    __syncwarp();
  }
  if (counts) {
    valid_count = __reduce_add_sync(0xffffffffu, valid_count);
    if (lane == 0 && valid_count)
      atomicAdd((unsigned long long*)&counts[(int64_t)frame * n_delta + kd], (unsigned long long)valid_count);
  }
}

template <int HW, bool LA>
static cudaError_t launch_simd(const uint8_t* left, const uint8_t* right, int n_frames, int64_t stride, int pitch,
                               int img_h, int w, int h, int x0, int y0, int delta_min, int n_delta, rg_bm_params p,
                               int16_t* raw, int64_t* counts, cudaStream_t s) {
  // bands whose reads stay in [row start, row start + pitch): left edge of the
  // widest disparity, right edge of the smallest one (+ realignment slack)
  const int bands = (w + 31) / 32;
  const int d_lo = p.min_disparity, d_max = p.min_disparity + p.num_disparities - 1;
  auto in_row = [&](int b) {
    const int lcol = x0 + 32 * b - 4;
    const int lo = std::min(lcol, lcol - d_max), hi = std::max(lcol, lcol - d_lo);
    return lo >= 0 && ((hi >> 2) + SB_NCW) * 4 + 3 <= pitch - 1;
  };
  int b0 = 0;
  while (b0 < bands && !in_row(b0)) ++b0;
  int b1 = b0;
  while (b1 < bands && in_row(b1)) ++b1;
  cudaError_t e = launch_lanes<HW, 1>(left, right, n_frames, stride, pitch, img_h, w, h, x0, y0, delta_min, n_delta,
                                      p, raw, counts, s, b0, b1);
  if (e != cudaSuccess || b1 <= b0) return e;
  static SmemAttr attr;
  if ((e = attr.ensure((const void*)bm_simd_kernel<HW, LA>, sb_smem<HW>())) != cudaSuccess) return e;
  dim3 grid((b1 - b0 + SB_W - 1) / SB_W, (h + SB_RS - 1) / SB_RS, n_frames * n_delta);
  bm_simd_kernel<HW, LA><<<grid, SB_W * 32, sb_smem<HW>(), s>>>(left, right, stride, pitch, img_h, w, h, x0, y0,
                                                             delta_min, n_delta, d_lo, p.num_disparities,
                                                             p.texture_threshold, p.uniqueness_ratio, raw, counts,
                                                             b0, b1);
  return cudaGetLastError();
}

__global__ void downscale_kernel(const uint8_t* __restrict__ in, int w, int h, int s,
                                 uint8_t* __restrict__ out) {  // image.hpp:98-116
  const int ow = w / s, oh = h / s;
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= ow || y >= oh) return;
  int sum = 0;
  for (int j = 0; j < s; ++j)
    for (int i = 0; i < s; ++i) sum += in[(int64_t)(y * s + j) * w + x * s + i];
  out[(int64_t)y * ow + x] = (uint8_t)llround(__ddiv_rn((double)sum, (double)(s * s)));
}

__global__ void upscale_kernel(const int16_t* __restrict__ in, int w, int h, int s, int lo,
                               int16_t* __restrict__ out, int ow, int oh) {  // image.hpp:122-141
  // out is ow x oh (the original dims); cells past the upscaled extent stay invalid
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= ow || y >= oh) return;
  int16_t v = (int16_t)kInvalid;
  const int sx = x / s, sy = y / s;
  if (sx < w && sy < h) {
    const int r = in[(int64_t)sy * w + sx];
    if (r != kInvalid) {
      const int scaled = r * s;
      if (scaled >= lo && scaled <= 32767) v = (int16_t)scaled;
    }
  }
  out[(int64_t)y * ow + x] = v;
}

__global__ void autorect_pick_kernel(const int64_t* __restrict__ counts, int n_frames,
                                     int delta_min, int n_delta, int32_t* __restrict__ best) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;  // autorect.hpp:35-57
  if (f >= n_frames) return;
  int bd = 0;
  long long bc = -1;
  for (int k = 0; k < n_delta; ++k) {
    const int delta = delta_min + k;
    const long long c = counts[(int64_t)f * n_delta + k];
    bool better = c > bc;
    if (c == bc) better = abs(delta) < abs(bd) || (abs(delta) == abs(bd) && delta < bd);
    if (better) {
      bc = c;
      bd = delta;
    }
  }
  best[f] = bd;
}

// autorect with downscale > 1 (autorect.hpp:36-44): crop(shift_vertical(img,
// delta), roi) as one gather (image.hpp:75-82, 145-154) ...
__global__ void crop_shift_kernel(const uint8_t* __restrict__ src, int w, int h, int x0, int y0, int rw, int rh,
                                  int delta, uint8_t* __restrict__ dst) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= rw || y >= rh) return;
  const int sy = min(max(y0 + y - delta, 0), h - 1);
  dst[(int64_t)y * rw + x] = src[(int64_t)sy * w + x0 + x];
}

// ... and the count of raw values that are valid and above 16 d_min
__global__ void count_above_kernel(const int16_t* __restrict__ raw, int64_t n, int lo, int64_t* __restrict__ count) {
  int c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = raw[i];
    c += (v != -32768 && v > lo) ? 1 : 0;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(reinterpret_cast<unsigned long long*>(count), (unsigned long long)c);
}

}  // namespace

cudaError_t launch_bm(const uint8_t* left, const uint8_t* right, int n_frames, int64_t stride,
                      int pitch, int img_h, int w, int h, int x0, int y0, int delta_min,
                      int n_delta, rg_bm_params p, int16_t* raw, int64_t* counts, cudaStream_t s) {
  if (n_frames <= 0 || n_delta <= 0) return cudaSuccess;
  const int hw = p.block_size / 2;
  const int dpl = (p.num_disparities + 31) / 32;
  const bool aligned = pitch % 4 == 0 && stride % 4 == 0 && reinterpret_cast<uintptr_t>(left) % 4 == 0 &&
                       reinterpret_cast<uintptr_t>(right) % 4 == 0;
  if (getenv("RG_BM_LEGACY") == nullptr && getenv("RG_BM_NOSIMD") == nullptr && aligned && hw >= 1 && hw <= 4 &&
      p.num_disparities <= 32) {
#define RG_BM_SIMD(HW)                                                                                          \
  if (hw == HW)                                                                                                 \
    return x0 % 4 == 0 ? launch_simd<HW, true>(left, right, n_frames, stride, pitch, img_h, w, h, x0, y0,       \
                                               delta_min, n_delta, p, raw, counts, s)                           \
                       : launch_simd<HW, false>(left, right, n_frames, stride, pitch, img_h, w, h, x0, y0,      \
                                                delta_min, n_delta, p, raw, counts, s);
    RG_BM_SIMD(1) RG_BM_SIMD(2) RG_BM_SIMD(3) RG_BM_SIMD(4)
#undef RG_BM_SIMD
  }
  if (getenv("RG_BM_LEGACY") == nullptr && hw >= 1 && hw <= 4 && dpl <= 2) {
#define RG_BM_CASE(HW, DPL)                                                                             \
  if (hw == HW && dpl == DPL)                                                                            \
    return launch_lanes<HW, DPL>(left, right, n_frames, stride, pitch, img_h, w, h, x0, y0, delta_min, n_delta, \
                                 p, raw, counts, s);
    RG_BM_CASE(1, 1) RG_BM_CASE(2, 1) RG_BM_CASE(3, 1) RG_BM_CASE(4, 1)
    RG_BM_CASE(1, 2) RG_BM_CASE(2, 2) RG_BM_CASE(3, 2) RG_BM_CASE(4, 2)
#undef RG_BM_CASE
  }
  const int TR = TYB + 2 * hw, LW = TXB + 2 * hw, RW = TXB + 2 * hw + p.num_disparities - 1;
  const size_t smem = (((size_t)TR * (LW + RW)) + 15) / 16 * 16 + sizeof(int) * TYB * LW;
  cudaError_t e = cudaFuncSetAttribute(bm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((w + TXB - 1) / TXB, (h + TYB - 1) / TYB, n_frames * n_delta);
  bm_kernel<<<grid, BT, smem, s>>>(left, right, stride, pitch, img_h, w, h, x0, y0, delta_min,
                                   n_delta, p.block_size, p.min_disparity, p.num_disparities,
                                   p.texture_threshold, p.uniqueness_ratio, raw, counts);
  return cudaGetLastError();
}

cudaError_t launch_downscale(const uint8_t* in, int w, int h, int s, uint8_t* out, cudaStream_t st) {
  dim3 grid((w / s + 127) / 128, h / s);
  downscale_kernel<<<grid, 128, 0, st>>>(in, w, h, s, out);
  return cudaGetLastError();
}

cudaError_t launch_upscale(const int16_t* in, int w, int h, int s, int lo, int16_t* out, int ow,
                           int oh, cudaStream_t st) {
  dim3 grid((ow + 127) / 128, oh);
  upscale_kernel<<<grid, 128, 0, st>>>(in, w, h, s, lo, out, ow, oh);
  return cudaGetLastError();
}

cudaError_t launch_crop_shift(const uint8_t* src, int w, int h, int x0, int y0, int rw, int rh, int delta,
                              uint8_t* dst, cudaStream_t st) {
  dim3 grid((rw + 255) / 256, rh);
  crop_shift_kernel<<<grid, 256, 0, st>>>(src, w, h, x0, y0, rw, rh, delta, dst);
  return cudaGetLastError();
}

cudaError_t launch_count_above(const int16_t* raw, int64_t n, int lo, int64_t* count, cudaStream_t st) {
  count_above_kernel<<<148, 256, 0, st>>>(raw, n, lo, count);
  return cudaGetLastError();
}

cudaError_t launch_autorect_pick(const int64_t* counts, int n_frames, int delta_min, int n_delta,
                                 int32_t* best, cudaStream_t s) {
  autorect_pick_kernel<<<(n_frames + 127) / 128, 128, 0, s>>>(counts, n_frames, delta_min, n_delta,
                                                               best);
  return cudaGetLastError();
}

}  // namespace rg
