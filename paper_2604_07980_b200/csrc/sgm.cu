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

// Fast path of sgm_disparity: the same recurrence, but
//  * the census costs are computed on the fly (lane d loads cr(x - d_lo - d,
//    y): consecutive codes) and prefetched SGM_PF steps ahead of the
//    recurrence (L2 latency is far longer than one step);
//  * each direction writes its L_r to its own buffer (LT = uint8/uint16 when
//    27 + P2 fits), so no step waits on a read-modify-write; the WTA kernel
//    sums the four buffers (sgm.hpp:129-131 adds them into acc);
//  * the four directions are independent, so ONE launch walks all their
//    paths (direction from the path index): ~w + 3h + 2w warps per frame.
#ifndef RG_SGM_PF
#define RG_SGM_PF 4
#endif
constexpr int SGM_PF = RG_SGM_PF;

struct SgmDirs {
  int sx[4], sy[4], first[5], rows[4];  // path index ranges and row-start counts per direction
};

template <int NDW, typename LT>
__global__ void __launch_bounds__(128) sgm_pass_fast_kernel(const uint32_t* __restrict__ cl,
                                                            const uint32_t* __restrict__ cr, int w, int h, int nd,
                                                            int d_lo, int p1, int p2, LT* __restrict__ Lbase,
                                                            int64_t dstride, SgmDirs dirs) {
  // lane owns the NDW ADJACENT disparities d = NDW*lane + j, so the d-1 / d+1
  // neighbours need only two shuffles per step
  const int lane = threadIdx.x & 31;
  const int gpath = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (gpath >= dirs.first[4]) return;
  int di = 0;
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (gpath >= dirs.first[k]) di = k;
  const int sx = dirs.sx[di], sy = dirs.sy[di];
  const int path = gpath - dirs.first[di];
  int x, y;
  if (path < dirs.rows[di]) {
    x = path;
    y = sy > 0 ? 0 : h - 1;
  } else {
    const int k = path - dirs.rows[di] + (sy != 0 ? 1 : 0);
    x = sx > 0 ? 0 : w - 1;
    y = sy >= 0 ? k : h - 1 - k;
  }
  int len = INT_MAX;
  if (sx > 0) len = min(len, w - x);
  if (sx < 0) len = min(len, x + 1);
  if (sy > 0) len = min(len, h - y);
  if (sy < 0) len = min(len, y + 1);
  const int d0 = NDW * lane;  // first disparity index of this lane
  const int64_t pstep = (int64_t)sy * w + sx;  // pixel-index step along the path
  const int64_t pix0 = (int64_t)y * w + x;
  LT* __restrict__ o = Lbase + di * dstride + pix0 * nd + d0;
  const int64_t ostep = pstep * nd;
  // rx = xx - d_lo - d0 - j must lie in [0, w): with xr = xx - d_lo - d0 the
  // test is (unsigned)(xr - j) < w
  const uint32_t* clp = cl + pix0;          // cl at the prefetch position
  const uint32_t* crow = cr + (pix0 - x);   // row start at the prefetch position
  int xr = x - d_lo - d0;
  int tp = 0;                               // step index of the next prefetch
  auto prefetch = [&](int (&c)[NDW]) {      // costs of step tp (clamped to the path end)
    const uint32_t lc = __ldg(clp);
#pragma unroll
    for (int j = 0; j < NDW; ++j) {
      const int rx = xr - j;
      const bool ok = (unsigned)rx < (unsigned)w && d0 + j < nd;
      c[j] = ok ? __popc(lc ^ __ldg(crow + rx)) : kNoData;
    }
    if (tp + 1 < len) {
      clp += pstep;
      crow += (int64_t)sy * w;
      xr += sx;
    }
    ++tp;
  };
  int q[SGM_PF][NDW];
#pragma unroll
  for (int t = 0; t < SGM_PF; ++t) prefetch(q[t]);
  int L[NDW];
  int pmin = 0;
  auto step = [&](int t, int (&c)[NDW]) {
    int cv[NDW];
#pragma unroll
    for (int j = 0; j < NDW; ++j) cv[j] = c[j];
    prefetch(c);  // refill this slot SGM_PF steps ahead (clamped re-reads at the end are unused)
    if (t == 0) {
#pragma unroll
      for (int j = 0; j < NDW; ++j) L[j] = (d0 + j < nd) ? cv[j] : kBig;
    } else {
      // neighbours across the lane boundary (kBig outside [0, nd))
      int lm = __shfl_up_sync(0xffffffffu, L[NDW - 1], 1);
      int lp = __shfl_down_sync(0xffffffffu, L[0], 1);
      if (lane == 0) lm = kBig;
      if (lane == 31) lp = kBig;
      int Ln[NDW];
#pragma unroll
      for (int j = 0; j < NDW; ++j) {
        const int dm = j > 0 ? L[j - 1] : lm;
        const int dp = j + 1 < NDW ? L[j + 1] : lp;
        // kBig + p1 stays below INT_MAX for the validated p1 <= p2 < 2^29
        int best = min(L[j], pmin + p2);
        best = min(best, min(dm, dp) + p1);
        Ln[j] = (d0 + j < nd) ? cv[j] + best - pmin : kBig;
      }
#pragma unroll
      for (int j = 0; j < NDW; ++j) L[j] = Ln[j];
    }
    int mn = L[0];
#pragma unroll
    for (int j = 1; j < NDW; ++j) mn = min(mn, L[j]);
    if (d0 < nd) {
      if (sizeof(LT) == 1 && NDW == 2 && nd % 2 == 0) {  // aligned u16 pair (d0 + 1 < nd since nd even)
        *reinterpret_cast<uint16_t*>(o) = (uint16_t)(L[0] | (L[1] << 8));
      } else if (sizeof(LT) == 1 && NDW == 4 && nd % 4 == 0) {
        *reinterpret_cast<uint32_t*>(o) = (uint32_t)(L[0] | (L[1] << 8) | (L[2] << 16) | (L[3] << 24));
      } else {
#pragma unroll
        for (int j = 0; j < NDW; ++j)
          if (d0 + j < nd) o[j] = (LT)L[j];
      }
    }
    o += ostep;
    pmin = __reduce_min_sync(0xffffffffu, mn);
  };
  int t0 = 0;
  for (; t0 + SGM_PF <= len; t0 += SGM_PF) {
#pragma unroll
    for (int u = 0; u < SGM_PF; ++u) step(t0 + u, q[u]);
  }
#pragma unroll
  for (int u = 0; u < SGM_PF; ++u)
    if (t0 + u < len) step(t0 + u, q[u]);
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

// WTA over the sum of the four directional buffers (dir stride = w*h*nd):
// one warp per pixel, lanes over d, first minimum by one reduction of
// (sum << 9 | i) (sum <= 4 * (27 + P2) fits above the 9 index bits for the
// LT = uint8 case; wider LT use a 64-bit key via two reductions)
template <typename LT>
__global__ void __launch_bounds__(256) sgm_wta4_kernel(const LT* __restrict__ Lb, int64_t dstride, int w, int h,
                                                      int nd, int d_lo, int16_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t pix = blockIdx.x * 8LL + (threadIdx.x >> 5);
  if (pix >= (int64_t)w * h) return;
  const int x = (int)(pix % w);
  const int64_t base = pix * nd;
  unsigned long long key = ~0ull;
  for (int i = lane; i < nd; i += 32) {
    const int rx = x - (d_lo + i);
    if (rx < 0 || rx >= w) continue;  // winner must be evaluable
    const long long v = (long long)Lb[base + i] + Lb[dstride + base + i] + Lb[2 * dstride + base + i] +
                        Lb[3 * dstride + base + i];
    const unsigned long long kk = ((unsigned long long)v << 9) | (unsigned)i;
    key = kk < key ? kk : key;
  }
  const uint32_t hi = __reduce_min_sync(0xffffffffu, (uint32_t)(key >> 32));
  const uint32_t lo = __reduce_min_sync(0xffffffffu, (uint32_t)(key >> 32) == hi ? (uint32_t)key : 0xffffffffu);
  if (lane != 0) return;
  int r = kInvalidRaw;
  if (hi != 0xffffffffu || lo != 0xffffffffu) {
    const unsigned long long bk = ((unsigned long long)hi << 32) | lo;
    const int best_i = (int)(bk & 511ull);
    const long long best = (long long)(bk >> 9);
    double d_hat = (double)(d_lo + best_i);
    if (best_i > 0 && best_i + 1 < nd && x - (d_lo + best_i + 1) >= 0) {
      auto A = [&](int i) {
        return (long long)Lb[base + i] + Lb[dstride + base + i] + Lb[2 * dstride + base + i] +
               Lb[3 * dstride + base + i];
      };
      d_hat = __dadd_rn(d_hat, subpix((double)A(best_i - 1), (double)best, (double)A(best_i + 1)));
    }
    long long v = llround(__dmul_rn(d_hat, 16.0));
    const long long lo16 = (long long)d_lo * 16, hi16 = (long long)(d_lo + nd) * 16 - 1;
    v = v < lo16 ? lo16 : (v > hi16 ? hi16 : v);
    r = (int)v;
  }
  out[pix] = (int16_t)r;
}

// WTA for uint8 directional buffers, nd <= 64, nd % 16 == 0: one THREAD per
// pixel, 16-byte loads, sums of the four buffers in 16-bit lanes, and the
// index folded into the key: key = sum << 6 | i (sum <= 1020, i < 64, so the
// key fits 16 bits and the 16x2 unsigned min keeps the first minimum).
template <int ND>
__global__ void __launch_bounds__(128) sgm_wta4_u8_kernel(const uint8_t* __restrict__ Lb, int64_t dstride, int w,
                                                          int h, int d_lo, int16_t* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w || y >= h) return;
  const int64_t base = ((int64_t)y * w + x) * ND;
  // evaluable i: x - (d_lo + i) in [0, w)  <=>  i in [x - d_lo - w + 1, x - d_lo]
  const int ilo = max(0, x - d_lo - w + 1), ihi = min(ND - 1, x - d_lo);
  uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
  for (int c = 0; c < ND / 16; ++c) {
    uint4 v[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) v[b] = __ldg(reinterpret_cast<const uint4*>(Lb + b * dstride + base + 16 * c));
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      uint32_t lo = 0, hi = 0;  // (i, i+1), (i+2, i+3) sums for i = 16c + 4m
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t wd = m == 0 ? v[b].x : m == 1 ? v[b].y : m == 2 ? v[b].z : v[b].w;
        lo += __byte_perm(wd, 0u, 0x4140);
        hi += __byte_perm(wd, 0u, 0x4342);
      }
      const int i = 16 * c + 4 * m;
      uint32_t klo = (lo << 6) | (uint32_t)i | ((uint32_t)(i + 1) << 16);
      uint32_t khi = (hi << 6) | (uint32_t)(i + 2) | ((uint32_t)(i + 3) << 16);
      if (ilo > i || ihi < i + 3) {  // pixel near the left/right edge: mask non-evaluable i
        if (i < ilo || i > ihi) klo |= 0xFFFFu;
        if (i + 1 < ilo || i + 1 > ihi) klo |= 0xFFFF0000u;
        if (i + 2 < ilo || i + 2 > ihi) khi |= 0xFFFFu;
        if (i + 3 < ilo || i + 3 > ihi) khi |= 0xFFFF0000u;
      }
      kmin = __vminu2(kmin, __vminu2(klo, khi));
    }
  }
  const uint32_t bk = min(kmin & 0xFFFFu, kmin >> 16);
  int r = kInvalidRaw;
  if (bk != 0xFFFFu && ilo <= ihi) {
    const int best_i = (int)(bk & 63u);
    const int best = (int)(bk >> 6);
    double d_hat = (double)(d_lo + best_i);
    if (best_i > 0 && best_i + 1 < ND && x - (d_lo + best_i + 1) >= 0) {
      auto A = [&](int i) {
        return (int)Lb[base + i] + (int)Lb[dstride + base + i] + (int)Lb[2 * dstride + base + i] +
               (int)Lb[3 * dstride + base + i];
      };
      d_hat = __dadd_rn(d_hat, subpix((double)A(best_i - 1), (double)best, (double)A(best_i + 1)));
    }
    long long vv = llround(__dmul_rn(d_hat, 16.0));
    const long long lo16 = (long long)d_lo * 16, hi16 = (long long)(d_lo + ND) * 16 - 1;
    vv = vv < lo16 ? lo16 : (vv > hi16 ? hi16 : vv);
    r = (int)vv;
  }
  out[(int64_t)y * w + x] = (int16_t)r;
}

template <typename LT>
cudaError_t sgm_fast(const uint32_t* cl, const uint32_t* cr, int w, int h, int nd, int d_lo, int p1, int p2, LT* Lb,
                     int16_t* out, cudaStream_t s) {
  const int64_t dstride = (int64_t)w * h * nd;
  const int dirs[4][2] = {{1, 0}, {0, 1}, {1, 1}, {-1, 1}};  // sgm.hpp:130
  SgmDirs D;
  D.first[0] = 0;
  for (int k = 0; k < 4; ++k) {
    const int sx = dirs[k][0], sy = dirs[k][1];
    D.sx[k] = sx;
    D.sy[k] = sy;
    D.rows[k] = sy != 0 ? w : 0;
    const int cols = sx != 0 ? (sy != 0 ? h - 1 : h) : 0;
    D.first[k + 1] = D.first[k] + D.rows[k] + cols;
  }
  const int grid = (D.first[4] + 3) / 4;
  const int ndw = (nd + 31) / 32;
#define RG_SGMF_CASE(K)                                                                                 \
  case K:                                                                                               \
    sgm_pass_fast_kernel<K, LT><<<grid, 128, 0, s>>>(cl, cr, w, h, nd, d_lo, p1, p2, Lb, dstride, D); \
    break;
  switch (ndw) {
    RG_SGMF_CASE(1) RG_SGMF_CASE(2) RG_SGMF_CASE(3) RG_SGMF_CASE(4)
    RG_SGMF_CASE(5) RG_SGMF_CASE(6) RG_SGMF_CASE(7) RG_SGMF_CASE(8)
    default: return cudaErrorInvalidValue;
  }
#undef RG_SGMF_CASE
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t px = (int64_t)w * h;
  if (sizeof(LT) == 1 && nd <= 64 && nd % 16 == 0) {
    const uint8_t* lb8 = reinterpret_cast<const uint8_t*>(Lb);
    dim3 g2((w + 127) / 128, h);
    switch (nd) {
      case 16: sgm_wta4_u8_kernel<16><<<g2, 128, 0, s>>>(lb8, dstride, w, h, d_lo, out); break;
      case 32: sgm_wta4_u8_kernel<32><<<g2, 128, 0, s>>>(lb8, dstride, w, h, d_lo, out); break;
      case 48: sgm_wta4_u8_kernel<48><<<g2, 128, 0, s>>>(lb8, dstride, w, h, d_lo, out); break;
      default: sgm_wta4_u8_kernel<64><<<g2, 128, 0, s>>>(lb8, dstride, w, h, d_lo, out); break;
    }
    return cudaGetLastError();
  }
  sgm_wta4_kernel<LT><<<(unsigned)((px + 7) / 8), 256, 0, s>>>(Lb, dstride, w, h, nd, d_lo, out);
  return cudaGetLastError();
}

}  // namespace

// bytes per directional L value for penalty P2 (L <= 27 + P2, sgm.hpp:97-99)
int sgm_l_bytes(int p2) { return 27 + (long long)p2 <= 255 ? 1 : (27 + (long long)p2 <= 65535 ? 2 : 4); }

cudaError_t launch_sgm_fast(const uint32_t* cl, const uint32_t* cr, int w, int h, int nd, int d_lo, int p1, int p2,
                            void* Lbuf, int16_t* out, cudaStream_t s) {
  switch (sgm_l_bytes(p2)) {
    case 1: return sgm_fast<uint8_t>(cl, cr, w, h, nd, d_lo, p1, p2, static_cast<uint8_t*>(Lbuf), out, s);
    case 2: return sgm_fast<uint16_t>(cl, cr, w, h, nd, d_lo, p1, p2, static_cast<uint16_t*>(Lbuf), out, s);
    default: return sgm_fast<int32_t>(cl, cr, w, h, nd, d_lo, p1, p2, static_cast<int32_t*>(Lbuf), out, s);
  }
}

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
  return e == cudaSuccess ? wait_async(ctx) : cuda_err(ctx, e, "cudaSetDevice");
}

rg_status sgm_check(rg_ctx* ctx, const rg_sgm_params* p) {  // sgm.hpp:21-28
  if (!p) return set_err(ctx, RG_EINVAL, "SgmParams: null");
  if (p->num_disparities < 1) return set_err(ctx, RG_EINVAL, "SgmParams: num_disparities must be >= 1");
  if (p->p1 < 0 || p->p2 < p->p1) return set_err(ctx, RG_EINVAL, "SgmParams: need 0 <= P1 <= P2");
  if (p->num_disparities > 256) return set_err(ctx, RG_EINVAL, "SgmParams: num_disparities > 256 unsupported");
  if (p->p2 >= (1 << 29)) return set_err(ctx, RG_EINVAL, "SgmParams: P2 >= 2^29 unsupported (int32 headroom)");
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
  void* lb = dev_buf(ctx, B_SGM_ACC, (size_t)sgm_l_bytes(p->p2) * 4 * px * nd);
  SG_NEED(cl);
  SG_NEED(cr);
  SG_NEED(lb);
  const PadGeom g = make_geom(w, h, 0, 0);
  RG_CUDA(ctx, launch_census_frames(dl, dr, 1, (int64_t)pitch * h, pitch, w, h, cl, cr, g, nullptr, nullptr, g,
                                    nullptr, nullptr, nullptr, false, s));
  count_launch(ctx, 0);
  RG_CUDA(ctx, launch_sgm_fast(cl, cr, w, h, nd, p->min_disparity, p->p1, p->p2, lb, d_out, s));
  count_launch(ctx, 4, 2);
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
  RG_NVTX("rg_sgm_disparity");
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
  RG_NVTX("rg_sgm_frames");
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
