// rg_device.cuh -- device-side object-ranger geometry shared by the planner,
// the fused matcher and the aggregation kernels.
//
// Every double expression keeps the reference's operation order and is
// written with explicit _rn intrinsics, so it rounds exactly like the
// reference's x86-64 build (no FMA contraction regardless of nvcc flags).
#pragma once

#include "rg_common.cuh"

namespace rg {

struct PBox {
  double x0, y0, x1, y1;
};

// v / 2.0 of the reference, as the exactly equal multiply by 0.5 (a power-of-
// two scaling rounds the same real number: identical bits for every double)
__device__ __forceinline__ double half_of(double v) { return __dmul_rn(v, 0.5); }
// x / (double)n with the same bits: a multiply by 1/n when n is a power of two
// (1/n exact), else the IEEE division
__device__ __forceinline__ double div_n(double x, int n) {
  return (n & (n - 1)) == 0 ? __dmul_rn(x, 1.0 / (double)n) : __ddiv_rn(x, (double)n);
}
// RN(a / b) for an integer-valued divisor b given rb = RN(1 / b) (0: the IEEE
// division): q = RN(a rb) is within an ulp of a / b, r = a - b q is exact by
// FMA, and RN(q + r rb) = RN(a / b + e) with |e| <= 2^-53 ulp, while a / b
// is never a rounding midpoint (b M would need 54 significant bits) and a
// non-midpoint quotient lies >= ulp / (2 b) from one (Markstein's correction).
__device__ __forceinline__ double div_rc(double a, double b, double rb) {
  if (rb == 0.0) return __ddiv_rn(a, b);
  const double q = __dmul_rn(a, rb);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, rb, q);
}
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max

// to_pixel_box, detection.hpp:23-30
__device__ __forceinline__ PBox pixel_box(const rg_detection& d, int w, int h) {
  PBox b;
  b.x0 = __dmul_rn(__dsub_rn(d.cx, half_of(d.w)), (double)w);
  b.x1 = __dmul_rn(__dadd_rn(d.cx, half_of(d.w)), (double)w);
  b.y0 = __dmul_rn(__dsub_rn(d.cy, half_of(d.h)), (double)h);
  b.y1 = __dmul_rn(__dadd_rn(d.cy, half_of(d.h)), (double)h);
  return b;
}

// PixelBox::contains, detection.hpp:19-21
__device__ __forceinline__ bool box_contains(double x0, double y0, double x1, double y1, double x,
                                             double y) {
  return x >= x0 && x < x1 && y >= y0 && y < y1;
}

// classify_far_close, template_match.hpp:63-67
__device__ __forceinline__ int dev_classify(const rg_detection& d, int w, int h, double tau_s) {
  return dmax(__dmul_rn(d.w, (double)w), __dmul_rn(d.h, (double)h)) < tau_s ? RG_KIND_FAR
                                                                            : RG_KIND_CLOSE;
}

// find_occluders predicate, template_match.hpp:75-85: does j occlude i?
__device__ __forceinline__ bool dev_occludes(const rg_detection& di, const rg_detection& dj) {
  const double ix0 = __dsub_rn(di.cx, half_of(di.w)), ix1 = __dadd_rn(di.cx, half_of(di.w));
  const double iy0 = __dsub_rn(di.cy, half_of(di.h)), iy1 = __dadd_rn(di.cy, half_of(di.h));
  const double jx0 = __dsub_rn(dj.cx, half_of(dj.w)), jx1 = __dadd_rn(dj.cx, half_of(dj.w));
  const double jy0 = __dsub_rn(dj.cy, half_of(dj.h)), jy1 = __dadd_rn(dj.cy, half_of(dj.h));
  const double ox = __dsub_rn(dmin(ix1, jx1), dmax(ix0, jx0));
  const double oy = __dsub_rn(dmin(iy1, jy1), dmax(iy0, jy0));
  return ox > 0 && oy > 0 && jy1 > iy1;
}

// select_objects ordering, template_match.hpp:94-114: does a come before b?
// frontal (centre inside the crop) first by area desc, then the rest by
// bottom desc; ties by id, then (reference-unspecified) by index.
__device__ __forceinline__ bool dev_frontal(const rg_detection& d, const rg_ranger_config& c) {
  return d.cx >= c.crop_x0 && d.cx < c.crop_x1 && d.cy >= c.crop_y0 && d.cy < c.crop_y1;
}
__device__ __forceinline__ bool dev_precedes(const rg_detection& a, int ia, const rg_detection& b,
                                             int ib, const rg_ranger_config& c) {
  const bool fa = dev_frontal(a, c), fb = dev_frontal(b, c);
  if (fa != fb) return fa;
  if (fa) {
    const double aa = __dmul_rn(a.w, a.h), ab = __dmul_rn(b.w, b.h);
    if (aa != ab) return aa > ab;
  } else {
    const double ba = __dadd_rn(a.cy, half_of(a.h)), bb = __dadd_rn(b.cy, half_of(b.h));
    if (ba != bb) return ba > bb;
  }
  if (a.id != b.id) return a.id < b.id;
  return ia < ib;
}

// grid sizes of sample_query_points, template_match.hpp:165-168, 189-194
__device__ __forceinline__ int dev_cap(const rg_ranger_config& c) {
  const int cap = (int)__dsqrt_rn((double)c.max_total_points);
  return cap > 1 ? cap : 1;
}
__device__ __forceinline__ void dev_close_grid(const PBox& b, const rg_ranger_config& c, int* rows,
                                               int* cols) {
  const double half_tau = half_of(c.tau_s);
  const int cc = (int)__ddiv_rn(__dsub_rn(b.x1, b.x0), half_tau);
  const int rr = (int)__ddiv_rn(__dsub_rn(b.y1, b.y0), half_tau);
  *cols = cc > 2 ? cc : 2;
  *rows = rr > 2 ? rr : 2;
}

// Geometry of one (sub-)block of sample_query_points (template_match.hpp:
// 155-223) and the test of one grid point; shared by the CTA-wide sampler
// (helper API) and the warp-wide sampler of the fused matcher.
struct SampleGeom {
  PBox box;
  double bw, bh, sx0, sy0, sw, sh;
  double rn, rw, rh;  // RN(1/n), RN(1/w), RN(1/h) for div_rc (0: IEEE division)
  int n, cw, ch;
  uint32_t magic;  // ceil(2^32 / n): idx / n = umulhi(idx, magic) (0: divide)
  bool far;
};

// Per-launch integer constants of the sampler, computed once on the host
// (the divisions / square root of dev_sample_geom without the per-slot cost).
struct SampleConst {
  int cw, ch;      // reduced raster: w / close_scale, h / close_scale (:189-190)
  int nf, nc;      // grid side points of FAR blocks / CLOSE sub-blocks (:165-168, :192-194)
  uint32_t mf, mc; // ceil(2^32 / nf), ceil(2^32 / nc)
  int dxc;         // ceil(dx_max_close / close_scale) (:218)
  double rnf, rnc, rw, rh;  // RN(1/nf), RN(1/nc), RN(1/w), RN(1/h) (IEEE host divisions)
};
inline SampleConst make_sample_const(const rg_ranger_config& c, int w, int h) {
  SampleConst k;
  int cap = (int)sqrt((double)c.max_total_points);  // dev_cap
  if (cap < 1) cap = 1;
  k.cw = w / c.close_scale;
  k.ch = h / c.close_scale;
  k.nf = c.grid_side_points < cap ? c.grid_side_points : cap;
  k.nc = c.close_block_side_points < cap ? c.close_block_side_points : cap;
  // exact for idx < n^2 while n^3 < 2^32 (error idx * (magic * n - 2^32) < 2^32)
  k.mf = k.nf > 1 && k.nf <= 1024 ? (uint32_t)(0xFFFFFFFFu / (uint32_t)k.nf) + 1u : 0u;
  k.mc = k.nc > 1 && k.nc <= 1024 ? (uint32_t)(0xFFFFFFFFu / (uint32_t)k.nc) + 1u : 0u;
  k.dxc = (c.dx_max_close + c.close_scale - 1) / c.close_scale;
  k.rnf = 1.0 / (double)k.nf;
  k.rnc = 1.0 / (double)k.nc;
  k.rw = 1.0 / (double)w;
  k.rh = 1.0 / (double)h;
  return k;
}

__device__ __forceinline__ SampleGeom dev_sample_geom(const rg_detection& det, int kind, int r, int c,
                                                      int rows, int cols, const rg_ranger_config& cfg,
                                                      int w, int h) {
  SampleGeom g;
  g.box = pixel_box(det, w, h);
  g.bw = __dsub_rn(g.box.x1, g.box.x0);
  g.bh = __dsub_rn(g.box.y1, g.box.y0);
  const int cap = dev_cap(cfg);
  g.far = kind == RG_KIND_FAR;
  g.n = g.far ? min(cfg.grid_side_points, cap) : min(cfg.close_block_side_points, cap);
  g.cw = w / cfg.close_scale;
  g.ch = h / cfg.close_scale;
  g.magic = 0;
  g.rn = g.rw = g.rh = 0.0;
  g.sx0 = g.sy0 = g.sw = g.sh = 0;
  if (!g.far) {
    g.sx0 = __dadd_rn(g.box.x0, __ddiv_rn(__dmul_rn((double)c, g.bw), (double)cols));
    g.sy0 = __dadd_rn(g.box.y0, __ddiv_rn(__dmul_rn((double)r, g.bh), (double)rows));
    g.sw = __ddiv_rn(g.bw, (double)cols);
    g.sh = __ddiv_rn(g.bh, (double)rows);
  }
  return g;
}

// dev_sample_geom with the integer constants taken from k
// (rcols, rrows: RN(1/cols), RN(1/rows) or 0)
__device__ __forceinline__ SampleGeom dev_sample_geom_k(const rg_detection& det, int kind, int r, int c, int rows,
                                                        int cols, const SampleConst& k, int w, int h,
                                                        double rcols = 0.0, double rrows = 0.0) {
  SampleGeom g;
  g.box = pixel_box(det, w, h);
  g.bw = __dsub_rn(g.box.x1, g.box.x0);
  g.bh = __dsub_rn(g.box.y1, g.box.y0);
  g.far = kind == RG_KIND_FAR;
  g.n = g.far ? k.nf : k.nc;
  g.magic = g.far ? k.mf : k.mc;
  g.rn = g.far ? k.rnf : k.rnc;
  g.rw = k.rw;
  g.rh = k.rh;
  g.cw = k.cw;
  g.ch = k.ch;
  g.sx0 = g.sy0 = g.sw = g.sh = 0;
  if (!g.far) {
    g.sx0 = __dadd_rn(g.box.x0, div_rc(__dmul_rn((double)c, g.bw), (double)cols, rcols));
    g.sy0 = __dadd_rn(g.box.y0, div_rc(__dmul_rn((double)r, g.bh), (double)rows, rrows));
    g.sw = div_rc(g.bw, (double)cols, rcols);
    g.sh = div_rc(g.bh, (double)rows, rrows);
  }
  return g;
}

// Grid point idx (j-major) of the block: true + (px, py) if it survives the
// image, occlusion and reduced-raster tests.  Occluders: `occ` (n_occ boxes)
// or, when occ_all != nullptr, every detection of the frame occluding det.
__device__ __forceinline__ bool dev_sample_point(const SampleGeom& g, int idx, const rg_detection& det,
                                                 const double* occ, int n_occ, const rg_detection* occ_all,
                                                 int n_all, int self, int w, int h, int* px, int* py) {
  const int j = g.magic ? (int)__umulhi((uint32_t)idx, g.magic) : idx / g.n, i = idx - j * g.n;
  double fx, fy;
  if (g.far) {
    fy = __dadd_rn(g.box.y0, div_rc(__dmul_rn(__dadd_rn((double)j, 0.5), g.bh), (double)g.n, g.rn));
    fx = __dadd_rn(g.box.x0, div_rc(__dmul_rn(__dadd_rn((double)i, 0.5), g.bw), (double)g.n, g.rn));
    *px = (int)lround(fx);
    *py = (int)lround(fy);
    if (*px < 0 || *px >= w || *py < 0 || *py >= h) return false;
  } else {
    fy = __dadd_rn(g.sy0, div_rc(__dmul_rn(__dadd_rn((double)j, 0.5), g.sh), (double)g.n, g.rn));
    fx = __dadd_rn(g.sx0, div_rc(__dmul_rn(__dadd_rn((double)i, 0.5), g.sw), (double)g.n, g.rn));
    if (fx < 0 || fx >= w || fy < 0 || fy >= h) return false;
  }
  // occluded points drop (template_match.hpp:159-163, 181, 212)
  if (occ_all) {
    for (int k = 0; k < n_all; ++k) {
      if (k == self || !dev_occludes(det, occ_all[k])) continue;
      const PBox ob = pixel_box(occ_all[k], w, h);
      if (box_contains(ob.x0, ob.y0, ob.x1, ob.y1, fx, fy)) return false;
    }
  } else {
    for (int k = 0; k < n_occ; ++k)
      if (box_contains(occ[4 * k], occ[4 * k + 1], occ[4 * k + 2], occ[4 * k + 3], fx, fy)) return false;
  }
  if (!g.far) {  // map into the reduced raster (template_match.hpp:213-215)
    *px = (int)lround(div_rc(__dmul_rn(fx, (double)g.cw), (double)w, g.rw));
    *py = (int)lround(div_rc(__dmul_rn(fy, (double)g.ch), (double)h, g.rh));
    if (*px < 0 || *px >= g.cw || *py < 0 || *py >= g.ch) return false;
  }
  return true;
}

// CTA-wide sampler (blockDim a multiple of 32): points compacted in the
// reference's grid order with warp ballots; returns the count (CTA-uniform).
__device__ __forceinline__ int dev_sample_block(const rg_detection& det, int kind, int r, int c,
                                                int rows, int cols, const double* occ, int n_occ,
                                                const rg_detection* occ_all, int n_all, int self,
                                                const rg_ranger_config& cfg, int w, int h,
                                                int2* pts) {
  __shared__ int s_wtot[32];
  const SampleGeom g = dev_sample_geom(det, kind, r, c, rows, cols, cfg, w, h);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int base = 0;
  for (int c0 = 0; c0 < g.n * g.n; c0 += blockDim.x) {
    const int idx = c0 + threadIdx.x;
    int px = 0, py = 0;
    const bool keep = idx < g.n * g.n &&
                      dev_sample_point(g, idx, det, occ, n_occ, occ_all, n_all, self, w, h, &px, &py);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_wtot[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int q = 0; q < nw; ++q) {
      before += q < wid ? s_wtot[q] : 0;
      total += s_wtot[q];
    }
    if (keep) pts[base + before + __popc(bal & ((1u << lane) - 1u))] = make_int2(px, py);
    base += total;
    __syncthreads();
  }
  return base;
}

// Warp-wide sampler: same points, same order; returns the count (warp-uniform).
__device__ __forceinline__ int dev_sample_block_warp_g(const SampleGeom& g, const rg_detection& det,
                                                       const double* occ, int n_occ, const rg_detection* occ_all,
                                                       int n_all, int self, int w, int h, int2* pts);
__device__ __forceinline__ int dev_sample_block_warp(const rg_detection& det, int kind, int r, int c,
                                                     int rows, int cols, const double* occ, int n_occ,
                                                     const rg_detection* occ_all, int n_all, int self,
                                                     const rg_ranger_config& cfg, int w, int h,
                                                     int2* pts) {
  return dev_sample_block_warp_g(dev_sample_geom(det, kind, r, c, rows, cols, cfg, w, h), det, occ, n_occ, occ_all,
                                 n_all, self, w, h, pts);
}
__device__ __forceinline__ int dev_sample_block_warp_g(const SampleGeom& g, const rg_detection& det,
                                                       const double* occ, int n_occ, const rg_detection* occ_all,
                                                       int n_all, int self, int w, int h, int2* pts) {
  const int lane = threadIdx.x & 31;
  int base = 0;
  for (int c0 = 0; c0 < g.n * g.n; c0 += 32) {
    const int idx = c0 + lane;
    int px = 0, py = 0;
    const bool keep = idx < g.n * g.n &&
                      dev_sample_point(g, idx, det, occ, n_occ, occ_all, n_all, self, w, h, &px, &py);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) pts[base + __popc(bal & ((1u << lane) - 1u))] = make_int2(px, py);
    base += __popc(bal);
  }
  __syncwarp();
  return base;
}

// aggregate_close_disparities core (template_match.hpp:126-148) over values
// already sorted ascending; single thread.
__device__ __forceinline__ void dev_runs(const double* v, int n, double tau_d, int n_min,
                                         int* valid, double* disp, int* run_len) {
  *valid = 0;
  *disp = 0.0;
  *run_len = 0;
  if (n == 0) return;
  int best_start = -1, best_len = 0, start = 0;
  for (int i = 1; i <= n; ++i) {
    if (i == n || __dsub_rn(v[i], v[i - 1]) >= tau_d) {
      const int len = i - start;
      if (len >= best_len) {  // later run = larger disparities wins ties
        best_len = len;
        best_start = start;
      }
      start = i;
    }
  }
  if (best_len < n_min) return;
  *valid = 1;
  *run_len = best_len;
  *disp = v[best_start + best_len / 2];
}

// CTA-wide ascending bitonic sort of n <= cap doubles in shared memory
// (padded with +inf up to the next power of two <= cap).
__device__ __forceinline__ void dev_bitonic_sort(double* v, int n) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + threadIdx.x; i < m; i += blockDim.x) v[i] = __longlong_as_double(0x7ff0000000000000LL);
  __syncthreads();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;
          const double a = v[i], b = v[p];
          if ((a > b) == up) {
            v[i] = b;
            v[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// rank sort for large n (values in global scratch): out[rank(i)] = v[i]
__device__ __forceinline__ void dev_rank_sort(const double* v, int n, double* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = v[i];
    int rank = 0;
    for (int k = 0; k < n; ++k) rank += (v[k] < x) || (v[k] == x && k < i);
    out[rank] = x;
  }
  __syncthreads();
}

}  // namespace rg
