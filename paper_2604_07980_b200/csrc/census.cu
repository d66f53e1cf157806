// census.cu -- K1: 5x5 census transform on sm_100a.
//
// Replaces census_code_at / census_transform / census_transform_rois
// (reference census.hpp:43-138).  Descriptor layout is the reference's:
// sentinel bit 25, then the 25 window compares (window row -2 first, column
// -2 first), centre compare always 0, code 0 when the window leaves the
// image.  The reduced CLOSE raster is a gather of the full raster at
// (mx[x'], my[y']) with mx = lround(x' * src/out) (census.hpp:59-64), so the
// batched kernel writes it from the same registers (inverse index maps).
#include <cuda_fp16.h>

#include <cstdlib>

#include "rg_common.cuh"
#include "rg_device.cuh"

namespace rg {
namespace {

// reference census.hpp:43-56 on a byte tile: `t` points at the centre,
// `ld` is the tile row stride.
__device__ __forceinline__ uint32_t census_window(const uint8_t* t, int ld) {
  const uint32_t c = t[0];
  uint32_t code = 1u;
#pragma unroll
  for (int j = -2; j <= 2; ++j) {
#pragma unroll
    for (int i = -2; i <= 2; ++i) code = (code << 1) | (uint32_t)(t[j * ld + i] > c);
  }
  return code;
}

constexpr int TX = 128;  // output tile columns (one per thread lane-row)
constexpr int TY = 32;   // output tile rows
constexpr int TPB = 256; // threads: 128 x 2 rows at a time

// Batched full + reduced census of n_frames stereo pairs (or single images
// when right == nullptr).  grid.z = sides*frame + side.
__global__ void __launch_bounds__(TPB) census_frames_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t frame_stride,
    int pitch, int w, int h, uint32_t* __restrict__ fl, uint32_t* __restrict__ fr, PadGeom gf,
    uint32_t* __restrict__ sl, uint32_t* __restrict__ sr, PadGeom gs,
    const int32_t* __restrict__ inv_x, const int32_t* __restrict__ inv_y,
    const int32_t* __restrict__ lshift, bool s31) {
  __shared__ __align__(16) uint8_t tile[TY + 4][TX + 8];
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
  const int sh = (side == 0 && lshift) ? lshift[frame] : 0;  // shift_vertical of the left image
  const uint8_t* img = (side ? right : left) + (int64_t)frame * frame_stride;
  uint32_t* full = (side ? fr : fl) + (int64_t)frame * gf.fstride + gf.origin;
  uint32_t* red = (side ? sr : sl);
  if (red) red += (int64_t)frame * gs.fstride + gs.origin;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;

  // stage (TY+4) x (TX+4) bytes with a 2-px halo; OOB bytes are never read by
  // a defined code (their windows leave the image), zero-fill them.
  for (int idx = threadIdx.x; idx < (TY + 4) * (TX + 4); idx += TPB) {
    const int r = idx / (TX + 4), c = idx - r * (TX + 4);
    const int gx = x0 + c - 2, gy = y0 + r - 2;
    tile[r][c] = (gx >= 0 && gx < w && gy >= 0 && gy < h)
                     ? img[(int64_t)min(max(gy - sh, 0), h - 1) * pitch + gx]  // image.hpp:145-154
                     : 0;
  }
  __syncthreads();

  const int tx = threadIdx.x & (TX - 1);
  const int x = x0 + tx;
  const int ix = (red && x < w) ? inv_x[x] : -1;  // maps are only passed with a reduced raster
  for (int ty = threadIdx.x / TX; ty < TY; ty += TPB / TX) {
    const int y = y0 + ty;
    if (x >= w || y >= h) continue;
    uint32_t code = 0;
    if (x >= 2 && y >= 2 && x < w - 2 && y < h - 2) code = census_window(&tile[ty + 2][tx + 2], TX + 8);
    if (s31 && code) code = (code & 0x01FFFFFFu) | kInternalHigh;  // internal layout
    full[(int64_t)y * gf.pitch + x] = code;
    if (red && ix >= 0) {
      const int iy = inv_y[y];
      if (iy >= 0) red[(int64_t)iy * gs.pitch + ix] = code;
    }
  }
}

// any bit of rows [y0, y1) set in the row mask m (one bit per row)
__device__ __forceinline__ bool rows_any(const uint32_t* __restrict__ m, int y0, int y1) {
  for (int y = y0; y < y1;) {
    const int wd = y >> 5, b0 = y & 31, nb = min(32 - b0, y1 - y);
    const uint32_t bits = (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) << b0;
    if (__ldg(m + wd) & bits) return true;
    y += nb;
  }
  return false;
}

// ---------------------------------------------------------------------------
// Fast path (pitch % 4 == 0, W % 4 == 0, reduced raster = exact half or none):
// half2 "vertical pair" census.  Pixel rows y and y+1 ride in the two fp16
// lanes of one register, encoded exactly as 1024 + intensity.  V[r][x] holds
// (I(x, r), I(x, r+1)), so the window neighbour (i, j) of BOTH pixels of the
// pair (x, y)/(x, y+1) is the single register V[y+j][x+i]: one compare
// (HSET2 on the ALU pipe, or an exact saturated HSUB2 on the FMA pipe -- the
// two are mixed to balance the pipes) and one HFMA2 (acc = 2 acc + m) advance
// two descriptors by one bit.  The 24 compare bits go into three fp16
// accumulators initialised so each group's bits land in the low mantissa bits
// (value 1024 + B), and four byte-permute/logic ops assemble the reference's
// descriptor for both rows.  V is built once per 128 x 60 tile in shared
// memory (6 byte permutes per 4 entries from raw image words, all loads of a
// thread in flight at once); each warp then computes a 10-row strip reading
// its 5-row window straight from V (2 LDS.128 per row).
#ifndef RG_C2_MASK
#define RG_C2_MASK 0xFFFFFFFFu
#endif
#ifndef RG_C2_TX
#define RG_C2_TX 128
#endif
constexpr int C2_TX = RG_C2_TX;                   // tile columns: groups of 32 lanes x 4 pixel pairs
constexpr int C2_G = C2_TX / 128;                 // 128-column groups per warp row
static_assert(C2_TX % 128 == 0, "tile width");
#ifndef RG_C2_WARPS
#define RG_C2_WARPS 6
#endif
#ifndef RG_C2_PR
#define RG_C2_PR 5
#endif
constexpr int C2_WARPS = RG_C2_WARPS;
constexpr int C2_PR = RG_C2_PR;                          // pair rows per warp strip
constexpr int C2_TY = C2_WARPS * C2_PR * 2;       // 60 tile rows (1080, 1860 and 480 split evenly)
constexpr int C2_VW = C2_TX + 12;                 // V row stride: 4 pad + x0-2 .. x0+TX+1 + pad
constexpr int C2_VOFF = 4;                        // V index of column x0-2
constexpr int C2_WORDS = C2_TX / 4 + 2;           // image words per row (x0-4 .. x0+TX+3)
constexpr int C2_RUNS = (C2_WARPS * 32) / C2_WORDS;          // 5 runs of rows in the V build
constexpr int C2_RUN = (C2_TY + 3 + C2_RUNS - 1) / C2_RUNS;  // 13 V rows per run
constexpr int C2_VR = C2_RUNS * C2_RUN;           // V rows y0-2 .. (padded: every run is full)
constexpr size_t C2_SMEM = sizeof(uint32_t) * C2_VR * C2_VW;

__device__ __forceinline__ uint32_t c2_vpair(uint32_t a, uint32_t b, int j) {
  // entry j of the 4 columns of words a (row r) and b (row r+1): half2(1024+a_j, 1024+b_j)
  const uint32_t t = __byte_perm(a, b, j < 2 ? 0x5140 : 0x7362);  // a_j b_j a_j+1 b_j+1
  return __byte_perm(t, 0x64646464u, (j & 1) ? 0x4342 : 0x4140);
}

// The three fp16 accumulators are built so each group's compare bits sit in
// the low mantissa bits of the half (exponent fixed, value in [1024, 2048)):
// g0 = w0..w8 (init 3.0, 9 steps: mantissa = 1<<9 | B0, the sentinel rides in
// mantissa bit 9), g1 = w9..w16 (init 4.0, 8 bits incl. the centre 0),
// g2 = w17..w24 (init 4.0).  code = (1<<9 | B0) << 16 | B1 << 8 | B2 is then
// three byte permutes and a mask for both lanes (lo = row y, hi = row y+1).
template <bool S31>  // S31: internal layout, sentinel moved from bit 25 to bit 31
__device__ __forceinline__ void c2_assemble(uint32_t g0, uint32_t g1, uint32_t g2, uint32_t& lo,
                                            uint32_t& hi) {
  const uint32_t t = __byte_perm(g2, g1, 0x6240);      // [B2 lo, B1 lo, B2 hi, B1 hi]
  if (S31) {  // g0 negative: its high byte is already 0xE6|b8 (kInternalHigh | bit 24)
    lo = __byte_perm(t, g0, 0x5410) & RG_C2_MASK;
    hi = __byte_perm(t, g0, 0x7632) & RG_C2_MASK;
  } else {
    lo = __byte_perm(t, g0, 0x5410) & 0x03FFFFFFu;     // g0 lo half: 0x66|b8 -> 0x2|b8
    hi = __byte_perm(t, g0, 0x7632) & 0x03FFFFFFu;
  }
}

// Descriptors of NQ pixel pairs from the 5 V rows w[0..4] (y-2 .. y+2): the
// pair q sits at window column q * QS + 2 (QS = 1: four adjacent columns;
// QS = 2: the even columns of the stride-2 reduced census).
template <bool S31, int NQ = 4, int QS = 1>
__device__ __forceinline__ void c2_codes(const uint32_t (&w)[5][8], uint32_t lo[NQ], uint32_t hi[NQ]) {
  const __half2 two = __float2half2_rn(2.0f), four = __float2half2_rn(4.0f);
#pragma unroll
  for (int qq = 0; qq < NQ; ++qq) {
    const int q = qq * QS;
    const __half2 c = *reinterpret_cast<const __half2*>(&w[2][q + 2]);
    __half2 g[3];
    g[0] = __float2half2_rn(S31 ? -3.0f : 3.0f);  // S31: negative, so the fp16 sign lands on bit 31
    g[1] = g[2] = __float2half2_rn(4.0f);
#pragma unroll
    for (int wi = 0; wi < 25; ++wi) {
      if (wi == 12) continue;  // centre: its 0 bit is folded into w13's x4
      const int j = wi / 5, i = wi % 5;
      const __half2 v = *reinterpret_cast<const __half2*>(&w[j][q + i]);
      const __half2 m = (wi % 6 == 0) ? __hsub2_sat(v, c) : __hgt2(v, c);
      const int gi = wi < 9 ? 0 : (wi < 17 ? 1 : 2);
      g[gi] = __hfma2(g[gi], wi == 13 ? four : two, (S31 && gi == 0) ? __hneg2(m) : m);
    }
    c2_assemble<S31>(*reinterpret_cast<uint32_t*>(&g[0]), *reinterpret_cast<uint32_t*>(&g[1]),
                *reinterpret_cast<uint32_t*>(&g[2]), lo[qq], hi[qq]);
  }
}

// Phase 2 for one warp: its C2_PR pair rows of the tile whose V is in smem.
// EDGE: the strip touches the image border (codes 0 where the window leaves).
// ROI: fm / rm are the frame's full / reduced row masks; a pair row is
// computed when either raster needs it and each raster stores only its rows.
template <bool EDGE, bool S31, bool ROI = false>
__device__ __forceinline__ void c2_strip(const uint32_t* __restrict__ V, uint32_t* __restrict__ full,
                                         uint32_t* __restrict__ red, const PadGeom& gf, const PadGeom& gs,
                                         int x0, int y0, int w, int h, const uint32_t* __restrict__ fm = nullptr,
                                         const uint32_t* __restrict__ rm = nullptr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pr0 = wid * C2_PR;
  const int64_t ostep = 2 * (int64_t)gf.pitch;
#pragma unroll
  for (int g = 0; g < C2_G; ++g) {
    const int xl = x0 + 128 * g + 4 * lane;  // first column of this lane in group g
    const uint32_t* vbase = V + C2_VOFF + 128 * g + 4 * lane;  // V index of column xl - 2
    // output pointers advance by whole pair rows (no per-row 64-bit index math)
    uint32_t* o = full + (int64_t)(y0 + 2 * pr0) * gf.pitch + xl;
    uint32_t* ro = red ? red + (int64_t)((y0 >> 1) + pr0) * gs.pitch + (xl >> 1) : full;  // full: never written
#pragma unroll
    for (int p = pr0; p < pr0 + C2_PR; ++p, o += ostep, ro += gs.pitch) {
      const int y = y0 + 2 * p;
      if (EDGE && y >= h) break;
      bool wf = true, wr = true;
      if (ROI) {
        wf = (__ldg(fm + (y >> 5)) >> (y & 31)) & 3u;  // y even: y, y + 1 share a word
        wr = red && ((__ldg(rm + (y >> 6)) >> ((y >> 1) & 31)) & 1u);
        if (!wf && !wr) continue;
      }
      uint32_t win[5][8];
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const uint4* src = reinterpret_cast<const uint4*>(vbase + (2 * p + j) * C2_VW);
        const uint4 a = src[0], b = src[1];
        win[j][0] = a.x; win[j][1] = a.y; win[j][2] = a.z; win[j][3] = a.w;
        win[j][4] = b.x; win[j][5] = b.y; win[j][6] = b.z; win[j][7] = b.w;
      }
      uint32_t lo[4], hi[4];
      c2_codes<S31>(win, lo, hi);
      if (EDGE) {
        if (xl >= w) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool xin = xl + q >= 2 && xl + q <= w - 3;
          if (!(xin && y >= 2 && y <= h - 3)) lo[q] = 0u;
          if (!(xin && y + 1 >= 2 && y + 1 <= h - 3)) hi[q] = 0u;
        }
      }
      if (wf) {
        *reinterpret_cast<uint4*>(o) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        if (!EDGE || y + 1 < h) *reinterpret_cast<uint4*>(o + gf.pitch) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      }
      // reduced raster = codes at even (x, y): (x/2, y/2)
      if (red && wr) *reinterpret_cast<uint2*>(ro) = make_uint2(lo[0], lo[2]);
    }
  }
}

// RG_C2_MINB: A/B knob only.  Any explicit minimum (even 1) changes ptxas's
// register heuristic: 1 gives 88 registers and 1.54 ms per 256 C2 frames, 6
// gives 56 and 1.53 ms, the bare bound 62 registers and 1.353 ms.
#ifdef RG_C2_MINB
#define RG_C2_BOUNDS __launch_bounds__(C2_WARPS * 32, RG_C2_MINB)
#else
#define RG_C2_BOUNDS __launch_bounds__(C2_WARPS * 32)
#endif
template <bool S31>
__global__ void RG_C2_BOUNDS census_pairs_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t frame_stride,
    int pitch, int w, int h, uint32_t* __restrict__ fl, uint32_t* __restrict__ fr, PadGeom gf,
    uint32_t* __restrict__ sl, uint32_t* __restrict__ sr, PadGeom gs, const int32_t* __restrict__ lshift,
    const uint32_t* __restrict__ rmask, int mstride) {
  extern __shared__ __align__(16) uint32_t V[];  // [C2_VR][C2_VW]
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
  // ROI rows (rmask: one bit per raster row of this frame): a tile without a
  // needed row leaves before its V build, a warp strip without one after it
  const uint32_t* fm = rmask ? rmask + (int64_t)frame * mstride : nullptr;
  const uint32_t* rm = rmask ? fm + (h + 31) / 32 : nullptr;  // reduced rows follow the full rows
  if (fm && !rows_any(fm, blockIdx.y * C2_TY, min(blockIdx.y * C2_TY + C2_TY, h)) &&
      !(sl && rows_any(rm, blockIdx.y * C2_TY / 2, min(blockIdx.y * C2_TY / 2 + C2_TY / 2, gs.h))))
    return;
  // shift_vertical (image.hpp:145-154) of the left image folded into the row
  // addressing: image row y reads source row clamp(y - sh)
  const int sh = (side == 0 && lshift) ? lshift[frame] : 0;
  const uint8_t* img = (side ? right : left) + (int64_t)frame * frame_stride;
  uint32_t* full = (side ? fr : fl) + (int64_t)frame * gf.fstride + gf.origin;
  uint32_t* red = side ? sr : sl;
  if (red) red += (int64_t)frame * gs.fstride + gs.origin;
  const int x0 = blockIdx.x * C2_TX, y0 = blockIdx.y * C2_TY;

  // ---- phase 1: V rows y0-2 .. from the image words; each thread walks one
  // word column down a run of rows with every load in flight at once.
  // Out-of-image words are clamped: they only feed border codes (forced 0);
  // the first/last word columns also write harmlessly into the row padding.
  const int wk = threadIdx.x % C2_WORDS, run = threadIdx.x / C2_WORDS;
  if (run < C2_RUNS) {
    const int kw = min(max((x0 - 4) / 4 + wk, 0), (w + 3) / 4 - 1);
    const int pw = pitch / 4;
    const int r0 = run * C2_RUN, ya = y0 - 2 + r0 - sh;
    uint32_t wv[C2_RUN + 1];
    if (ya >= 0 && ya + C2_RUN <= h - 1) {  // interior run: plain strided loads
      const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + (int64_t)ya * pw + kw;
#pragma unroll
      for (int t = 0; t <= C2_RUN; ++t) wv[t] = __ldg(col + t * pw);
    } else {
      const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + kw;
#pragma unroll
      for (int t = 0; t <= C2_RUN; ++t) wv[t] = __ldg(col + (int64_t)min(max(ya + t, 0), h - 1) * pw);
    }
    uint32_t* vrow = V + r0 * C2_VW + C2_VOFF + 4 * wk - 2;  // entries of columns x0-4+4wk .. +3
#pragma unroll
    for (int t = 0; t < C2_RUN; ++t) {
      const uint32_t a = wv[t], b = wv[t + 1];
      *reinterpret_cast<uint2*>(vrow + t * C2_VW) = make_uint2(c2_vpair(a, b, 0), c2_vpair(a, b, 1));
      *reinterpret_cast<uint2*>(vrow + t * C2_VW + 2) = make_uint2(c2_vpair(a, b, 2), c2_vpair(a, b, 3));
    }
  }
  __syncthreads();
  // ---- phase 2
  const int ys = y0 + 2 * (threadIdx.x >> 5) * C2_PR;
  if (ys >= h) return;
  if (fm && !rows_any(fm, ys, min(ys + 2 * C2_PR, h)) && !(sl && rows_any(rm, ys / 2, min(ys / 2 + C2_PR, gs.h))))
    return;
  const bool edge = x0 < 2 || x0 + C2_TX + 3 > w - 3 || ys < 2 || ys + 2 * C2_PR + 1 > h - 3;
  const bool e = __any_sync(0xffffffffu, edge);  // warp-uniform (the vote lets the compiler keep one branch)
  if (fm) {
    if (e)
      c2_strip<true, S31, true>(V, full, red, gf, gs, x0, y0, w, h, fm, rm);
    else
      c2_strip<false, S31, true>(V, full, red, gf, gs, x0, y0, w, h, fm, rm);
  } else if (e) {
    c2_strip<true, S31>(V, full, red, gf, gs, x0, y0, w, h);
  } else {
    c2_strip<false, S31>(V, full, red, gf, gs, x0, y0, w, h);
  }
}

// ---------------------------------------------------------------------------
// ROI census (the reference's census_transform_rois, census.hpp:100-138, as
// estimate_object_disparities calls it, template_match.hpp:300-321): the
// full-resolution raster only inside FAR census ROIs (box dilated by
// (dx_max_far + 2, 3), detail::add_roi :245-253) and the reduced raster only
// inside CLOSE ROIs, the latter by a stride-2 kernel instead of being
// gathered from a full-frame transform -- and of each rectangle only the
// codes the matcher can read (read_rect).  Codes computed are bit-identical
// to the full transform; nothing reads the others.  At C2
// this is 931 k of the 1.28 M ROI codes (both images) of 2.59 M full-frame
// ones per frame.
//
// census_rows_kernel, per frame: the reference's ROI row masks (bit y of
// words [0, wf) = full raster row y, [wf, wf + wr) = reduced rows; only the
// A/B pair kernel uses them) and, per image, the compacted lists of the
// (4-row, 120-column) warp tiles the read sets touch.  Every detection of the
// frame contributes (a superset of the selected ones: the planner runs after
// the census).
// The rectangle [ra, re) x [ca, ce) (raster coordinates) of a detection box
// (integer bounds bx0..bx1, by0..by1, search range dxr) whose codes the
// matcher can read in image img (0 left, 1 right).  The block points lie on
// the box rows / columns (lround of coordinates inside the box); the forward
// pass reads the left image at the points and the right one at
// (x - dx, y + dy), dx in [0, dxr], |dy| <= 1; the backward pass reads the
// right image at the points shifted by (-dx*, dy*) and the left one at
// (x - dx* + dx', y), dx' in [0, dxr].  So: left = the box rows across
// [bx0 - dxr, bx1 + dxr], right = the box rows +-1 across [bx0 - dxr, bx1].
// tight 2 (default): exactly that; 1: +-1 row / +-2 column margins; 0: the
// reference's whole ROI rectangle (detail::add_roi, template_match.hpp:245-253).
__device__ __forceinline__ void read_rect(int bx0, int bx1, int by0, int by1, int dxr, int W, int H, int img,
                                          int tight, int& ra, int& re, int& ca, int& ce) {
  const int dxm = dxr + 2;
  ra = max(0, by0 - 3), re = min(H, by1 + 4), ca = max(0, bx0 - dxm), ce = min(W, bx1 + dxm + 1);
  if (tight) {
    const int mg = tight == 1;
    ra = max(ra, by0 - img - mg), re = min(re, by1 + 1 + img + mg);
    ca = max(ca, bx0 - dxr - 2 * mg);
    ce = min(ce, img ? bx1 + 1 + 2 * mg : bx1 + dxr + 1 + 2 * mg);
  }
}

constexpr int RM_T = 128;
constexpr int RW_TX = 120;  // source columns per warp tile (lanes 0..29 emit codes)
__global__ void __launch_bounds__(RM_T) census_rows_kernel(const rg_detection* __restrict__ dets,
                                                          const int32_t* __restrict__ det_off, int w, int h,
                                                          double tau_s, int cw, int ch, int wf, int wr,
                                                          uint32_t* __restrict__ mask, int dxf, int dxs, int nxt,
                                                          int tf, int tr, int rtf, int rtr, int tile_stride,
                                                          int32_t* __restrict__ tiles, int tight) {
  // row masks (wf + wr), then the 2-D tile bitmaps (bf + br) of the left and
  // of the right image
  extern __shared__ uint32_t sm_rows[];
  const int bf = (rtf * nxt + 31) / 32, br = (rtr * nxt + 31) / 32;
  uint32_t* tbm = sm_rows + wf + wr;
  __shared__ int s_pos[RM_T + 1];
  const int f = blockIdx.x;
  for (int i = threadIdx.x; i < wf + wr + 2 * (bf + br); i += RM_T) sm_rows[i] = 0u;
  __syncthreads();
  const int d0 = det_off[f], n = det_off[f + 1] - d0;
  const double sy = __ddiv_rn((double)ch, (double)h);  // template_match.hpp:305 double(ch) / h
  const double sx = __ddiv_rn((double)cw, (double)w);  // template_match.hpp:305 double(cw) / w
  auto clampi = [](double v) { return (int)fmin(fmax(v, -1.0e9), 1.0e9); };
  for (int i = threadIdx.x; i < n; i += RM_T) {
    const rg_detection d = dets[d0 + i];
    const PBox b = pixel_box(d, w, h);
    int bx0, bx1, by0, by1, dxm, W, H, rows_per_tile, cols_per_tile, ntr;
    uint32_t *m, *bm;
    if (dev_classify(d, w, h, tau_s) == RG_KIND_FAR) {  // add_roi(far_rois, box, 1, 1, dx_max_far + 2, 3, w, h)
      by0 = clampi(floor(b.y0)), by1 = clampi(ceil(b.y1));
      bx0 = clampi(floor(b.x0)), bx1 = clampi(ceil(b.x1));
      dxm = dxf + 2, W = w, H = h;
      m = sm_rows, bm = tbm, rows_per_tile = tf, cols_per_tile = RW_TX, ntr = rtf;
    } else {  // add_roi(scaled_rois, box, cw / w, ch / h, dx_scaled + 2, 3, cw, ch)
      by0 = clampi(floor(__dmul_rn(b.y0, sy))), by1 = clampi(ceil(__dmul_rn(b.y1, sy)));
      bx0 = clampi(floor(__dmul_rn(b.x0, sx))), bx1 = clampi(ceil(__dmul_rn(b.x1, sx)));
      dxm = dxs + 2, W = cw, H = ch;
      m = sm_rows + wf, bm = tbm + bf, rows_per_tile = tr, cols_per_tile = RW_TX / 2, ntr = rtr;
    }
    // the reference's ROI rows [a, e) (row masks of the A/B pair kernel)
    const int a = max(0, by0 - 3), e = min(H, by1 + 3 + 1);
    for (int y = a; y < e;) {
      const int wd = y >> 5, b0 = y & 31, nb = min(32 - b0, e - y);
      atomicOr(&m[wd], (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) << b0);
      y += nb;
    }
    // only the codes the matcher can read (read_rect)
    for (int img = 0; img < 2; ++img) {
      int ra, re, ca, ce;
      read_rect(bx0, bx1, by0, by1, dxm - 2, W, H, img, tight, ra, re, ca, ce);
      uint32_t* sbm = bm + img * (bf + br);
      if (ra < re && ca < ce)  // the warp tiles (fixed grid) the rectangle touches
        for (int rt = ra / rows_per_tile; rt <= (re - 1) / rows_per_tile && rt < ntr; ++rt)
          for (int xt = ca / cols_per_tile; xt <= (ce - 1) / cols_per_tile && xt < nxt; ++xt) {
            const int bit = rt * nxt + xt;
            atomicOr(&sbm[bit >> 5], 1u << (bit & 31));
          }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < wf + wr; i += RM_T) mask[(int64_t)f * (wf + wr) + i] = sm_rows[i];
  // compacted lists of the needed (row tile, column tile) pairs: entry =
  // (first row / 2) << 16 | column_tile; tiles[f] = {n_full_left, n_red_left,
  // n_full_right, n_red_right, then per image: full list (rtf * nxt),
  // reduced list (rtr * nxt)}
  int32_t* rec = tiles + (int64_t)f * tile_stride;
  for (int q = 0; q < 4; ++q) {
    const int img = q >> 1, side = q & 1;  // side: 0 full, 1 reduced raster
    const uint32_t* bm = tbm + img * (bf + br) + (side ? bf : 0);
    const int nw = side ? br : bf;
    int32_t* list = rec + 4 + img * (rtf + rtr) * nxt + (side ? rtf * nxt : 0);
    int base = 0;
    for (int w0 = 0; w0 < nw; w0 += RM_T) {
      const int wd = w0 + threadIdx.x;
      const uint32_t bits = wd < nw ? bm[wd] : 0u;
      s_pos[threadIdx.x] = __popc(bits);
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = 0;
        for (int t = 0; t < RM_T; ++t) {
          const int c = s_pos[t];
          s_pos[t] = acc;
          acc += c;
        }
        s_pos[RM_T] = acc;
      }
      __syncthreads();
      int pos = base + s_pos[threadIdx.x];
      for (uint32_t r = bits; r; r &= r - 1) {
        const int bit = wd * 32 + __ffs(r) - 1;
        list[pos++] = (((bit / nxt) * (side ? tr : tf) / 2) << 16) | (bit % nxt);
      }
      base += s_pos[RM_T];
      __syncthreads();
    }
    if (threadIdx.x == 0) rec[q] = base;
  }
}

// census_rows_kernel with the warp tiles placed per column instead of on a
// fixed row grid (RG_CENSUS_GREEDY, default): for every (image, raster,
// 120-column tile) the rows the read sets need, then a greedy cover by
// tiles of 2 rw_pr rows starting at the next needed row (rounded down to
// even) -- a 13-row box costs 4 tiles wherever it sits instead of 4 or 5.
// Same list layout and entry format ((first row / 2) << 16 | column tile).
__global__ void __launch_bounds__(RM_T) census_cols_kernel(const rg_detection* __restrict__ dets,
                                                          const int32_t* __restrict__ det_off, int w, int h,
                                                          double tau_s, int cw, int ch, int wf, int wr,
                                                          uint32_t* __restrict__ mask, int dxf, int dxs, int nxt,
                                                          int tf, int tr, int rtf, int rtr, int tile_stride,
                                                          int32_t* __restrict__ tiles, int tight) {
  // reference row masks (wf + wr), then per (image, column tile) the needed
  // rows of the full raster (wf words each) and of the reduced one (wr)
  extern __shared__ uint32_t sm_cols[];
  uint32_t* cf = sm_cols + wf + wr;
  uint32_t* cr = cf + 2 * nxt * wf;
  __shared__ int s_cnt[4 * 64 + 1];
  const int f = blockIdx.x;
  const int total_words = wf + wr + 2 * nxt * (wf + wr);
  for (int i = threadIdx.x; i < total_words; i += RM_T) sm_cols[i] = 0u;
  __syncthreads();
  const int d0 = det_off[f], n = det_off[f + 1] - d0;
  const double sy = __ddiv_rn((double)ch, (double)h);  // template_match.hpp:305 double(ch) / h
  const double sx = __ddiv_rn((double)cw, (double)w);  // template_match.hpp:305 double(cw) / w
  auto clampi = [](double v) { return (int)fmin(fmax(v, -1.0e9), 1.0e9); };
  auto set_rows = [](uint32_t* col, int a, int e) {
    for (int y = a; y < e;) {
      const int wd = y >> 5, b0 = y & 31, nb = min(32 - b0, e - y);
      atomicOr(&col[wd], (nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) << b0);
      y += nb;
    }
  };
  for (int i = threadIdx.x; i < n; i += RM_T) {
    const rg_detection d = dets[d0 + i];
    const PBox b = pixel_box(d, w, h);
    const bool far = dev_classify(d, w, h, tau_s) == RG_KIND_FAR;
    int bx0, bx1, by0, by1, dxm, W, H, cols_per_tile, nw;
    uint32_t *m, *cb;
    if (far) {  // add_roi(far_rois, box, 1, 1, dx_max_far + 2, 3, w, h)
      by0 = clampi(floor(b.y0)), by1 = clampi(ceil(b.y1));
      bx0 = clampi(floor(b.x0)), bx1 = clampi(ceil(b.x1));
      dxm = dxf + 2, W = w, H = h, m = sm_cols, cb = cf, cols_per_tile = RW_TX, nw = wf;
    } else {  // add_roi(scaled_rois, box, cw / w, ch / h, dx_scaled + 2, 3, cw, ch)
      by0 = clampi(floor(__dmul_rn(b.y0, sy))), by1 = clampi(ceil(__dmul_rn(b.y1, sy)));
      bx0 = clampi(floor(__dmul_rn(b.x0, sx))), bx1 = clampi(ceil(__dmul_rn(b.x1, sx)));
      dxm = dxs + 2, W = cw, H = ch, m = sm_cols + wf, cb = cr, cols_per_tile = RW_TX / 2, nw = wr;
    }
    set_rows(m, max(0, by0 - 3), min(H, by1 + 3 + 1));  // the reference's ROI rows
    for (int img = 0; img < 2; ++img) {
      int ra, re, ca, ce;
      read_rect(bx0, bx1, by0, by1, dxm - 2, W, H, img, tight, ra, re, ca, ce);
      if (ra >= re || ca >= ce) continue;
      for (int xt = ca / cols_per_tile; xt <= (ce - 1) / cols_per_tile && xt < nxt; ++xt)
        set_rows(cb + (img * nxt + xt) * nw, ra, re);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < wf + wr; i += RM_T) mask[(int64_t)f * (wf + wr) + i] = sm_cols[i];
  // greedy cover of every column (q = (img * 2 + raster) * nxt + xt): count, scan, write
  int32_t* rec = tiles + (int64_t)f * tile_stride;
  const int ncol = 4 * nxt;
  auto cover = [&](int q, int32_t* out) -> int {
    const int img = q / (2 * nxt), raster = (q / nxt) & 1, xt = q % nxt;
    const int nw = raster ? wr : wf, T = raster ? tr : tf;
    const uint32_t* col = (raster ? cr : cf) + (img * nxt + xt) * nw;
    int y = 0, cnt = 0;
    for (;;) {
      int wd = y >> 5;
      if (wd >= nw) break;
      uint32_t bits = col[wd] & (0xFFFFFFFFu << (y & 31));
      while (!bits && ++wd < nw) bits = col[wd];
      if (!bits) break;
      const int y0 = (wd * 32 + __ffs(bits) - 1) & ~1;
      if (out) out[cnt] = ((y0 >> 1) << 16) | xt;
      ++cnt;
      y = y0 + T;
    }
    return cnt;
  };
  for (int q = threadIdx.x; q < ncol; q += RM_T) s_cnt[q] = cover(q, nullptr);
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan within each (image, raster) list
    for (int l = 0; l < 4; ++l) {
      int acc = 0;
      for (int xt = 0; xt < nxt; ++xt) {
        const int c = s_cnt[l * nxt + xt];
        s_cnt[l * nxt + xt] = acc;
        acc += c;
      }
      rec[(l >> 1) * 2 + (l & 1)] = acc;  // l = img * 2 + raster -> rec[img * 2 + raster]
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < ncol; q += RM_T) {
    const int img = q / (2 * nxt), raster = (q / nxt) & 1;
    int32_t* list = rec + 4 + img * (rtf + rtr) * nxt + (raster ? rtf * nxt : 0);
    cover(q, list + s_cnt[q]);
  }
}

// Warp-tile "vertical pair" census for the ROI tiles: every warp owns a tile of
// 120 source columns x 4 output rows (2 row pairs; 120 columns + the 2-px
// halo = 32 image words, one per lane) with its own V rows in
// shared memory (no CTA barrier), so work follows the ROI rectangles at
// 4-row granularity (measured per 256 C2 frames with the matcher's read
// sets: 5 / 3 row pairs (full / reduced) 0.729 ms, 3 / 2 0.636, 2 / 2 0.627,
// 2 / 1 0.696; 128 walkers per frame and side 0.627, 256 0.631).  STRIDE 1 writes the full raster (4 codes per lane per row);
// STRIDE 2 writes the reduced raster of an exact-half CLOSE scale (reduced
// (x', y') = full (2x', 2y'), census.hpp:59-64 with lround(2i) = 2i): the V
// entry of source row s pairs rows s and s + 2, so reduced rows y', y' + 1
// (source rows 2y', 2y' + 2) advance together, and each lane emits the even
// source columns c, c + 2 of the same 8-entry window rows.
#ifndef RG_RW_WPB1
#define RG_RW_WPB1 1
#endif
#ifndef RG_RW_WPB2
#define RG_RW_WPB2 1
#endif
// warps (independent tiles) per CTA: the FAR row tiles are sparse (most warps
// leave at once), so single-warp CTAs release their slot immediately
template <int STRIDE>
__host__ __device__ constexpr int rw_wpb() { return STRIDE == 1 ? RG_RW_WPB1 : RG_RW_WPB2; }
template <int STRIDE>
#ifndef RG_RW_PR1
#define RG_RW_PR1 2
#endif
#ifndef RG_RW_PR2
#define RG_RW_PR2 2
#endif
__host__ __device__ constexpr int rw_pr() { return STRIDE == 1 ? RG_RW_PR1 : RG_RW_PR2; }  // row pairs per warp tile
constexpr int RW_VW = 136;  // V row stride: index 4 = source column x0 - 2
template <int STRIDE>
__host__ __device__ constexpr int rw_nv() { return 2 * STRIDE * (rw_pr<STRIDE>() - 1) + 5; }  // V rows (7 / 9)
template <int STRIDE>
__host__ __device__ constexpr size_t rw_smem() { return sizeof(uint32_t) * rw_wpb<STRIDE>() * rw_nv<STRIDE>() * RW_VW; }

template <bool S31, int STRIDE>
__global__ void __launch_bounds__(rw_wpb<STRIDE>() * 32) census_rowtile_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t frame_stride, int pitch, int w,
    int h, uint32_t* __restrict__ ol, uint32_t* __restrict__ orr, PadGeom g, const int32_t* __restrict__ lshift,
    const int32_t* __restrict__ tiles, int tile_stride, int list_off, int side_off) {
  constexpr int NV = rw_nv<STRIDE>(), NI = NV + STRIDE;  // V rows, image rows
  constexpr int RW_PR = rw_pr<STRIDE>();
  extern __shared__ __align__(16) uint32_t Vall[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
  // this warp walks its share of the frame's compacted list of (row tile,
  // column tile) pairs that some ROI rectangle touches (no CTA is launched
  // for an empty tile)
  const int32_t* rec = tiles + (int64_t)frame * tile_stride;
  const int n_tiles = rec[2 * side + STRIDE - 1];
  const int32_t* list = rec + list_off + side * side_off;
  uint32_t* V = Vall + wid * NV * RW_VW;
  for (int ti = blockIdx.x * rw_wpb<STRIDE>() + wid; ti < n_tiles; ti += gridDim.x * rw_wpb<STRIDE>()) {
  const int ent = list[ti];
  const int Y0 = (ent >> 16) * 2;  // first output row of this tile (even)
  const int x0 = (ent & 0xFFFF) * RW_TX;   // source column origin
  __syncwarp();  // the previous tile's window reads are done before V is rebuilt
  const int sh = (side == 0 && lshift) ? lshift[frame] : 0;  // shift_vertical of the left image
  const uint8_t* img = (side ? right : left) + (int64_t)frame * frame_stride;
  uint32_t* out = (side ? orr : ol) + (int64_t)frame * g.fstride + g.origin;
  const int S0 = STRIDE * Y0 - 2;   // source row of V row 0
  // ---- V rows: word column k of image rows S0 .. S0 + NI - 1 (clamped);
  // entry (s, c) = half2(1024 + I(c, s), 1024 + I(c, s + STRIDE))
  const int pw = pitch / 4;
  {
    const int k = lane;
    const int kw = min(max((x0 - 4) / 4 + k, 0), (w + 3) / 4 - 1);
    const int ya = S0 - sh;
    uint32_t wv[NI];
    if (ya >= 0 && ya + NI - 1 <= h - 1) {
      const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + (int64_t)ya * pw + kw;
#pragma unroll
      for (int t = 0; t < NI; ++t, col += pw) wv[t] = __ldg(col);
    } else {
      const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + kw;
#pragma unroll
      for (int t = 0; t < NI; ++t) wv[t] = __ldg(col + (int64_t)min(max(ya + t, 0), h - 1) * pw);
    }
    // word k holds source columns x0 - 4 + 4k .. + 3 = V indices 4k + 2 .. 4k + 5;
    // the 16-B group k (indices 4k .. 4k + 3) takes the last two entries of
    // word k - 1 (one lane down) and the first two of word k: one aligned
    // STS.128 per row instead of two 8-B stores at a 16-B stride (half the
    // shared-memory wavefronts of the V build; the windows read groups 1..31)
    uint4* vrow = reinterpret_cast<uint4*>(V) + k;
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      const uint32_t a = wv[t], b = wv[t + STRIDE];
      const uint32_t e2 = c2_vpair(a, b, 2), e3 = c2_vpair(a, b, 3);
      const uint32_t p2 = __shfl_up_sync(0xffffffffu, e2, 1), p3 = __shfl_up_sync(0xffffffffu, e3, 1);
      vrow[t * (RW_VW / 4)] = make_uint4(p2, p3, c2_vpair(a, b, 0), c2_vpair(a, b, 1));
    }
  }
  __syncwarp();
  // ---- codes: RW_PR row pairs (output rows y, y + 1 = source rows STRIDE y, STRIDE y + STRIDE)
  constexpr int NQ = 4 / STRIDE;
  const int xs = x0 + 4 * lane;     // source column of this lane's first output
  const int xo = xs / STRIDE;       // its output column
  if (lane >= RW_TX / 4 || xo >= g.w) continue;  // (such lanes only help build V)
  const bool edge = x0 < 2 || x0 + RW_TX + 2 > w - 3 || STRIDE * Y0 < 2 || STRIDE * (Y0 + 2 * RW_PR) > h - 3;
  const uint32_t* vbase = V + 4 + 4 * lane;  // V index of source column xs - 2
  // consecutive pairs' windows overlap by 5 - 2 STRIDE V rows (3 full, 1
  // reduced): they stay in registers, only the new rows are loaded
  // (every pair of a needed tile is computed, so the rotation is static and
  // costs no register moves)
  constexpr int KEEP = 5 - 2 * STRIDE;
  uint32_t win[5][8];
#pragma unroll
  for (int p = 0; p < RW_PR; ++p) {
    const int y = Y0 + 2 * p;
    if (y >= g.h) break;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      if (p > 0 && j < KEEP) {
#pragma unroll
        for (int q = 0; q < 8; ++q) win[j][q] = win[j + 2 * STRIDE][q];
        continue;
      }
      const uint4* src = reinterpret_cast<const uint4*>(vbase + (2 * STRIDE * p + j) * RW_VW);
      const uint4 a = src[0], b = src[1];
      win[j][0] = a.x; win[j][1] = a.y; win[j][2] = a.z; win[j][3] = a.w;
      win[j][4] = b.x; win[j][5] = b.y; win[j][6] = b.z; win[j][7] = b.w;
    }
    uint32_t lo[NQ], hi[NQ];
    c2_codes<S31, NQ, STRIDE>(win, lo, hi);
    if (edge) {
      const int sy0 = STRIDE * y, sy1 = STRIDE * y + STRIDE;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int sx = xs + STRIDE * q;
        const bool xin = sx >= 2 && sx <= w - 3;
        if (!(xin && sy0 >= 2 && sy0 <= h - 3)) lo[q] = 0u;
        if (!(xin && sy1 >= 2 && sy1 <= h - 3)) hi[q] = 0u;
      }
    }
    uint32_t* o = out + (int64_t)y * g.pitch + xo;
    const bool two = y + 1 < g.h;
    if (xo + NQ <= g.w) {
      if (STRIDE == 1) {
        *reinterpret_cast<uint4*>(o) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        if (two) *reinterpret_cast<uint4*>(o + g.pitch) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      } else {
        *reinterpret_cast<uint2*>(o) = make_uint2(lo[0], lo[NQ - 1]);
        if (two) *reinterpret_cast<uint2*>(o + g.pitch) = make_uint2(hi[0], hi[NQ - 1]);
      }
    } else {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (xo + q >= g.w) break;
        o[q] = lo[q];
        if (two) o[g.pitch + q] = hi[q];
      }
    }
  }
  }
}

// ---------------------------------------------------------------------------
// 9x7 census extension (BASELINE config 1): 64-bit descriptors, 63
// compares after the sentinel (window rows -3..3, columns -4..4, row-major,
// first compare in bit 62), 0 where the window leaves the image.  One output
// per thread from a byte tile in shared memory; the same inverse maps write
// the reduced raster.
constexpr int X_TX = 128, X_TY = 16, X_TPB = 256;

__global__ void __launch_bounds__(X_TPB) census64_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t frame_stride, int pitch,
    int w, int h, unsigned long long* __restrict__ fl, unsigned long long* __restrict__ fr, PadGeom gf,
    unsigned long long* __restrict__ sl, unsigned long long* __restrict__ sr, PadGeom gs,
    const int32_t* __restrict__ inv_x, const int32_t* __restrict__ inv_y, const int32_t* __restrict__ lshift) {
  __shared__ uint8_t tile[X_TY + 6][X_TX + 8];
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
  const int sh = (side == 0 && lshift) ? lshift[frame] : 0;
  const uint8_t* img = (side ? right : left) + (int64_t)frame * frame_stride;
  unsigned long long* full = (side ? fr : fl) + (int64_t)frame * gf.fstride + gf.origin;
  unsigned long long* red = side ? sr : sl;
  if (red) red += (int64_t)frame * gs.fstride + gs.origin;
  const int x0 = blockIdx.x * X_TX, y0 = blockIdx.y * X_TY;
  for (int idx = threadIdx.x; idx < (X_TY + 6) * (X_TX + 8); idx += X_TPB) {
    const int r = idx / (X_TX + 8), c = idx - r * (X_TX + 8);
    const int gx = x0 + c - 4, gy = y0 + r - 3;
    tile[r][c] = (gx >= 0 && gx < w && gy >= 0 && gy < h) ? img[(int64_t)min(max(gy - sh, 0), h - 1) * pitch + gx]
                                                          : 0;
  }
  __syncthreads();
  const int tx = threadIdx.x % X_TX, x = x0 + tx;
  const int ix = (red && x < w) ? inv_x[x] : -1;  // maps are only passed with a reduced raster
  for (int ty = threadIdx.x / X_TX; ty < X_TY; ty += X_TPB / X_TX) {
    const int y = y0 + ty;
    if (x >= w || y >= h) continue;
    unsigned long long code = 0ull;
    if (x >= 4 && y >= 3 && x < w - 4 && y < h - 3) {
      const uint32_t c = tile[ty + 3][tx + 4];
      code = 1ull;
#pragma unroll
      for (int j = 0; j < 7; ++j) {
        uint32_t bits = 0u;
#pragma unroll
        for (int i = 0; i < 9; ++i) bits = (bits << 1) | (uint32_t)(tile[ty + j][tx + i] > c);
        code = (code << 9) | bits;
      }
    }
    full[(int64_t)y * gf.pitch + x] = code;
    if (red && ix >= 0) {
      const int iy = inv_y[y];
      if (iy >= 0) red[(int64_t)iy * gs.pitch + ix] = code;
    }
  }
}

// 9x7 "vertical pair" census (the fast path of the 64-bit extension): the
// same half2 formulation as census_pairs_kernel -- rows y, y+1 in the two
// fp16 lanes, one compare + one HFMA2 per window tap for both rows -- with
// one fp16 accumulator per WINDOW ROW: init 2.0, 9 steps, so the row's 9
// compare bits are the low mantissa bits (1024 + B).  The window is walked
// row by row (12 V entries per lane per row: columns x-4 .. x+7 for the
// lane's 4 outputs), so registers hold one row of the window, not seven.
// Code = sentinel bit 63 | B_r << (54 - 9 r) (rows r = 0..6 = window rows
// -3..3, MSB-first; the centre compare is always 0: folded into a x4 step).
constexpr int X2_WARPS = 6, X2_PR = 5;
constexpr int X2_TX = 128, X2_TY = X2_WARPS * X2_PR * 2;       // 60 rows
constexpr int X2_VW = X2_TX + 12;                             // index 4 = column x0 - 4
constexpr int X2_WORDS = X2_TX / 4 + 2;                       // image words per row (x0-4 .. x0+TX+3)
constexpr int X2_RUNS = (X2_WARPS * 32) / X2_WORDS;            // 5
constexpr int X2_RUN = (X2_TY + 6 + X2_RUNS - 1) / X2_RUNS;    // V rows y0-3 .. y0+TY+2
constexpr int X2_VR = X2_RUNS * X2_RUN;
constexpr size_t X2_SMEM = sizeof(uint32_t) * X2_VR * X2_VW;

template <bool EDGE>
__device__ __forceinline__ void c64_strip(const uint32_t* __restrict__ V, unsigned long long* __restrict__ full,
                                          unsigned long long* __restrict__ red, const PadGeom& gf,
                                          const PadGeom& gs, int x0, int y0, int w, int h) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int xl = x0 + 4 * lane;
  const uint32_t* vbase = V + 4 + 4 * lane;  // V index of column xl - 4
  const __half2 two = __float2half2_rn(2.0f), four = __float2half2_rn(4.0f);
#pragma unroll 1
  for (int p = wid * X2_PR; p < wid * X2_PR + X2_PR; ++p) {
    const int y = y0 + 2 * p;
    if (EDGE && y >= h) break;
    uint32_t clo[4], chi[4];  // 64-bit codes of rows y (lo) and y + 1 (hi), as two 32-bit halves
    uint32_t dlo[4], dhi[4];
    __half2 cen[4];
    {
      const uint4 c4 = *reinterpret_cast<const uint4*>(vbase + (2 * p + 3) * X2_VW + 4);  // columns xl .. xl+3
      cen[0] = *reinterpret_cast<const __half2*>(&c4.x);
      cen[1] = *reinterpret_cast<const __half2*>(&c4.y);
      cen[2] = *reinterpret_cast<const __half2*>(&c4.z);
      cen[3] = *reinterpret_cast<const __half2*>(&c4.w);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) clo[q] = dlo[q] = 0u, chi[q] = dhi[q] = 0x80000000u;  // sentinel bit 63
#pragma unroll
    for (int r = 0; r < 7; ++r) {
      uint32_t e[12];
      const uint4* src = reinterpret_cast<const uint4*>(vbase + (2 * p + r) * X2_VW);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint4 a = src[k];
        e[4 * k] = a.x, e[4 * k + 1] = a.y, e[4 * k + 2] = a.z, e[4 * k + 3] = a.w;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        __half2 acc = two;
#pragma unroll
        for (int c = 0; c < 9; ++c) {
          if (r == 3 && c == 4) continue;  // centre: its 0 bit is folded into the next step's x4
          const __half2 v = *reinterpret_cast<const __half2*>(&e[q + c]);
          const __half2 m = ((r * 9 + c) % 6 == 0) ? __hsub2_sat(v, cen[q]) : __hgt2(v, cen[q]);
          acc = __hfma2(acc, (r == 3 && c == 5) ? four : two, m);
        }
        const uint32_t u = *reinterpret_cast<const uint32_t*>(&acc);
        const uint32_t bl = u & 0x1FFu, bh = (u >> 16) & 0x1FFu;
        // bit 54 - 9r of the 64-bit code: rows 0..2 in the high word, row 3
        // straddles (bits 27..35), rows 4..6 in the low word
        const int pos = 54 - 9 * r;
        if (pos >= 32) {
          chi[q] |= bl << (pos - 32);
          dhi[q] |= bh << (pos - 32);
        } else if (pos + 9 > 32) {
          clo[q] |= bl << pos, chi[q] |= bl >> (32 - pos);
          dlo[q] |= bh << pos, dhi[q] |= bh >> (32 - pos);
        } else {
          clo[q] |= bl << pos;
          dlo[q] |= bh << pos;
        }
      }
    }
    unsigned long long lo[4], hi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      lo[q] = ((unsigned long long)chi[q] << 32) | clo[q];
      hi[q] = ((unsigned long long)dhi[q] << 32) | dlo[q];
      if (EDGE) {  // 0 where the 9x7 window leaves the image
        const bool xin = xl + q >= 4 && xl + q <= w - 5;
        if (!(xin && y >= 3 && y <= h - 4)) lo[q] = 0ull;
        if (!(xin && y + 1 >= 3 && y + 1 <= h - 4)) hi[q] = 0ull;
      }
    }
    if (EDGE && xl >= w) continue;
    unsigned long long* o = full + (int64_t)y * gf.pitch + xl;
    reinterpret_cast<ulonglong2*>(o)[0] = make_ulonglong2(lo[0], lo[1]);
    reinterpret_cast<ulonglong2*>(o)[1] = make_ulonglong2(lo[2], lo[3]);
    if (!EDGE || y + 1 < h) {
      reinterpret_cast<ulonglong2*>(o + gf.pitch)[0] = make_ulonglong2(hi[0], hi[1]);
      reinterpret_cast<ulonglong2*>(o + gf.pitch)[1] = make_ulonglong2(hi[2], hi[3]);
    }
    if (red)  // reduced raster = codes at even (x, y)
      *reinterpret_cast<ulonglong2*>(red + (int64_t)(y >> 1) * gs.pitch + (xl >> 1)) = make_ulonglong2(lo[0], lo[2]);
  }
}

__global__ void __launch_bounds__(X2_WARPS * 32) census64_pairs_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t frame_stride, int pitch, int w,
    int h, unsigned long long* __restrict__ fl, unsigned long long* __restrict__ fr, PadGeom gf,
    unsigned long long* __restrict__ sl, unsigned long long* __restrict__ sr, PadGeom gs,
    const int32_t* __restrict__ lshift) {
  extern __shared__ __align__(16) uint32_t V[];  // [X2_VR][X2_VW]
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
  const int sh = (side == 0 && lshift) ? lshift[frame] : 0;
  const uint8_t* img = (side ? right : left) + (int64_t)frame * frame_stride;
  unsigned long long* full = (side ? fr : fl) + (int64_t)frame * gf.fstride + gf.origin;
  unsigned long long* red = side ? sr : sl;
  if (red) red += (int64_t)frame * gs.fstride + gs.origin;
  const int x0 = blockIdx.x * X2_TX, y0 = blockIdx.y * X2_TY;
  // ---- V rows y0-3 .. : V[r][c] = half2(1024 + I(c, r), 1024 + I(c, r + 1)), word wk at index 4 + 4 wk
  const int wk = threadIdx.x % X2_WORDS, run = threadIdx.x / X2_WORDS;
  if (run < X2_RUNS) {
    const int kw = min(max((x0 - 4) / 4 + wk, 0), (w + 3) / 4 - 1);
    const int pw = pitch / 4;
    const int r0 = run * X2_RUN, ya = y0 - 3 + r0 - sh;
    uint32_t wv[X2_RUN + 1];
    if (ya >= 0 && ya + X2_RUN <= h - 1) {
      const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + (int64_t)ya * pw + kw;
#pragma unroll
      for (int t = 0; t <= X2_RUN; ++t, col += pw) wv[t] = __ldg(col);
    } else {
      const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + kw;
#pragma unroll
      for (int t = 0; t <= X2_RUN; ++t) wv[t] = __ldg(col + (int64_t)min(max(ya + t, 0), h - 1) * pw);
    }
    uint4* vrow = reinterpret_cast<uint4*>(V + r0 * X2_VW + 4) + wk;
#pragma unroll
    for (int t = 0; t < X2_RUN; ++t) {
      const uint32_t a = wv[t], b = wv[t + 1];
      vrow[t * (X2_VW / 4)] = make_uint4(c2_vpair(a, b, 0), c2_vpair(a, b, 1), c2_vpair(a, b, 2), c2_vpair(a, b, 3));
    }
  }
  __syncthreads();
  const int ys = y0 + 2 * (threadIdx.x >> 5) * X2_PR;
  if (ys >= h) return;
  const bool edge = x0 < 4 || x0 + X2_TX + 4 > w - 5 || ys < 3 || ys + 2 * X2_PR + 2 > h - 4;
  if (__any_sync(0xffffffffu, edge))
    c64_strip<true>(V, full, red, gf, gs, x0, y0, w, h);
  else
    c64_strip<false>(V, full, red, gf, gs, x0, y0, w, h);
}

// 9x7 ROI census on the same compacted (row tile, column tile) lists as
// census_rowtile_kernel (4 output rows x 120 source columns per warp tile):
// the 64-bit codes of c64_strip (one fp16 accumulator per window row, row y
// and row y + STRIDE in the two lanes), V rows built per warp from 32 image
// words (word k = V entries 4k .. 4k + 3 = source columns x0 - 4 + 4k ..),
// so lane l reads its 12 window columns as three aligned 16-B groups.
// STRIDE 2: the reduced raster of an exact-half scale (reduced (x', y') =
// full (2x', 2y')): V entries pair source rows s and s + 2, each lane emits
// the source columns c, c + 2.
template <int STRIDE>
__host__ __device__ constexpr int c64_nv() { return 2 * STRIDE * (rw_pr<STRIDE>() - 1) + 7; }  // V rows (9 / 11)
template <int STRIDE>
__host__ __device__ constexpr size_t c64_smem() { return sizeof(uint32_t) * c64_nv<STRIDE>() * RW_VW; }

template <int STRIDE>
__global__ void __launch_bounds__(32) census64_rowtile_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t frame_stride, int pitch, int w,
    int h, unsigned long long* __restrict__ ol, unsigned long long* __restrict__ orr, PadGeom g,
    const int32_t* __restrict__ lshift, const int32_t* __restrict__ tiles, int tile_stride, int list_off,
    int side_off) {
  constexpr int NV = c64_nv<STRIDE>(), NI = NV + STRIDE;  // V rows, image rows
  constexpr int PR = rw_pr<STRIDE>();
  constexpr int NQ = 4 / STRIDE;  // codes per lane per row
  extern __shared__ __align__(16) uint32_t V[];
  const int lane = threadIdx.x & 31;
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
  const int32_t* rec = tiles + (int64_t)frame * tile_stride;
  const int n_tiles = rec[2 * side + STRIDE - 1];
  const int32_t* list = rec + list_off + side * side_off;
  const int sh = (side == 0 && lshift) ? lshift[frame] : 0;  // shift_vertical of the left image
  const uint8_t* img = (side ? right : left) + (int64_t)frame * frame_stride;
  unsigned long long* out = (side ? orr : ol) + (int64_t)frame * g.fstride + g.origin;
  const __half2 two = __float2half2_rn(2.0f), four = __float2half2_rn(4.0f);
  const int pw = pitch / 4;
  for (int ti = blockIdx.x; ti < n_tiles; ti += gridDim.x) {
    const int ent = list[ti];
    const int Y0 = (ent >> 16) * 2;  // first output row of this tile (even)
    const int x0 = (ent & 0xFFFF) * RW_TX;
    __syncwarp();  // the previous tile's window reads are done before V is rebuilt
    const int S0 = STRIDE * Y0 - 3;  // source row of V row 0
    {
      const int kw = min(max((x0 - 4) / 4 + lane, 0), (w + 3) / 4 - 1);
      const int ya = S0 - sh;
      uint32_t wv[NI];
      if (ya >= 0 && ya + NI - 1 <= h - 1) {
        const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + (int64_t)ya * pw + kw;
#pragma unroll
        for (int t = 0; t < NI; ++t, col += pw) wv[t] = __ldg(col);
      } else {
        const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + kw;
#pragma unroll
        for (int t = 0; t < NI; ++t) wv[t] = __ldg(col + (int64_t)min(max(ya + t, 0), h - 1) * pw);
      }
      uint4* vrow = reinterpret_cast<uint4*>(V) + lane;
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const uint32_t a = wv[t], b = wv[t + STRIDE];
        vrow[t * (RW_VW / 4)] = make_uint4(c2_vpair(a, b, 0), c2_vpair(a, b, 1), c2_vpair(a, b, 2),
                                           c2_vpair(a, b, 3));
      }
    }
    __syncwarp();
    const int xs = x0 + 4 * lane;  // source column of this lane's first output
    const int xo = xs / STRIDE;
    if (lane >= RW_TX / 4 || xo >= g.w) continue;  // (such lanes only help build V)
    const bool edge = x0 < 4 || x0 + RW_TX + 4 > w - 5 || STRIDE * Y0 < 3 || STRIDE * (Y0 + 2 * PR) > h - 4;
    const uint32_t* vbase = V + 4 * lane;  // V index of source column xs - 4
#pragma unroll 1
    for (int p = 0; p < PR; ++p) {
      const int y = Y0 + 2 * p;
      if (y >= g.h) break;
      uint32_t clo[NQ], chi[NQ], dlo[NQ], dhi[NQ];
      __half2 cen[NQ];
      {
        const uint4 c4 = *reinterpret_cast<const uint4*>(vbase + (2 * STRIDE * p + 3) * RW_VW + 4);  // xs .. xs+3
        const uint32_t cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int q = 0; q < NQ; ++q) cen[q] = *reinterpret_cast<const __half2*>(&cc[STRIDE * q]);
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) clo[q] = dlo[q] = 0u, chi[q] = dhi[q] = 0x80000000u;  // sentinel bit 63
#pragma unroll
      for (int r = 0; r < 7; ++r) {
        uint32_t e[12];
        const uint4* src = reinterpret_cast<const uint4*>(vbase + (2 * STRIDE * p + r) * RW_VW);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const uint4 a = src[k];
          e[4 * k] = a.x, e[4 * k + 1] = a.y, e[4 * k + 2] = a.z, e[4 * k + 3] = a.w;
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          __half2 acc = two;
#pragma unroll
          for (int c = 0; c < 9; ++c) {
            if (r == 3 && c == 4) continue;  // centre: its 0 bit is folded into the next step's x4
            const __half2 v = *reinterpret_cast<const __half2*>(&e[STRIDE * q + c]);
            const __half2 m = ((r * 9 + c) % 6 == 0) ? __hsub2_sat(v, cen[q]) : __hgt2(v, cen[q]);
            acc = __hfma2(acc, (r == 3 && c == 5) ? four : two, m);
          }
          const uint32_t u = *reinterpret_cast<const uint32_t*>(&acc);
          const uint32_t bl = u & 0x1FFu, bh = (u >> 16) & 0x1FFu;
          const int pos = 54 - 9 * r;  // bit 54 - 9r of the 64-bit code (c64_strip)
          if (pos >= 32) {
            chi[q] |= bl << (pos - 32);
            dhi[q] |= bh << (pos - 32);
          } else if (pos + 9 > 32) {
            clo[q] |= bl << pos, chi[q] |= bl >> (32 - pos);
            dlo[q] |= bh << pos, dhi[q] |= bh >> (32 - pos);
          } else {
            clo[q] |= bl << pos;
            dlo[q] |= bh << pos;
          }
        }
      }
      unsigned long long lo[NQ], hi[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        lo[q] = ((unsigned long long)chi[q] << 32) | clo[q];
        hi[q] = ((unsigned long long)dhi[q] << 32) | dlo[q];
        if (edge) {  // 0 where the 9x7 window leaves the image
          const int sx = xs + STRIDE * q, sy0 = STRIDE * y, sy1 = STRIDE * y + STRIDE;
          const bool xin = sx >= 4 && sx <= w - 5;
          if (!(xin && sy0 >= 3 && sy0 <= h - 4)) lo[q] = 0ull;
          if (!(xin && sy1 >= 3 && sy1 <= h - 4)) hi[q] = 0ull;
        }
      }
      unsigned long long* o = out + (int64_t)y * g.pitch + xo;
      const bool two_rows = y + 1 < g.h;
      if (xo + NQ <= g.w) {
#pragma unroll
        for (int q = 0; q < NQ; q += 2) {
          reinterpret_cast<ulonglong2*>(o)[q / 2] = make_ulonglong2(lo[q], lo[q + 1]);
          if (two_rows) reinterpret_cast<ulonglong2*>(o + g.pitch)[q / 2] = make_ulonglong2(hi[q], hi[q + 1]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          if (xo + q >= g.w) break;
          o[q] = lo[q];
          if (two_rows) o[g.pitch + q] = hi[q];
        }
      }
    }
  }
}

// Host-fed batches (rg_range_frames_host): the image bytes the ROI census
// reads for the matcher, fetched straight from the caller's pinned frames
// over PCIe (zero-copy) instead of copy-engine transfers of whole frames.
// Per detection and image the rectangle of census_rows_kernel (tight: the
// matcher's read set; else the reference's ROI rectangle), in source pixels
// and dilated by the census window (RX columns, RY rows each side) plus one
// pixel, at 16-B granularity.  One warp per (image row, side, frame): it
// marks the row's needed 16-B segments from every detection of the frame,
// then copies them.  Bytes moved are added to bytes[frame & 63].
constexpr int GR_WARPS = 4;
constexpr int GR_SEGW = 8;  // mask words per row: <= 4096 columns
template <int RX, int RY>
__global__ void __launch_bounds__(GR_WARPS * 32) gather_rows_kernel(
    const uint8_t* __restrict__ hl, const uint8_t* __restrict__ hr, int64_t src_stride, int src_pitch,
    uint8_t* __restrict__ dl, uint8_t* __restrict__ dr, int64_t dst_stride, int dst_pitch, int w, int h,
    const rg_detection* __restrict__ dets, const int32_t* __restrict__ det_off, double tau_s, int cw, int ch,
    int dxf, int dxs, int tight, const int32_t* __restrict__ lshift, unsigned long long* __restrict__ bytes,
    int n_frames) {
  __shared__ uint32_t mask[GR_WARPS][GR_SEGW];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // a persistent grid (a few CTAs per SM, resident while the previous
  // chunk's compute kernels run): warps stride over (row, side, frame)
  for (int item = blockIdx.x * GR_WARPS + wid; item < h * 2 * n_frames; item += gridDim.x * GR_WARPS) {
  const int r = item % h, side = (item / h) & 1, f = item / (2 * h);
  __syncwarp();
  if (lane < GR_SEGW) mask[wid][lane] = 0u;
  __syncwarp();
  const int sh = (side == 0 && lshift) ? lshift[f] : 0;
  const double sy = __ddiv_rn((double)ch, (double)h), sx = __ddiv_rn((double)cw, (double)w);
  auto clampi = [](double v) { return (int)fmin(fmax(v, -1.0e9), 1.0e9); };
  const int d0 = det_off[f], n = det_off[f + 1] - d0;
  for (int i = lane; i < n; i += 32) {
    const rg_detection d = dets[d0 + i];
    const PBox b = pixel_box(d, w, h);
    const bool far = dev_classify(d, w, h, tau_s) == RG_KIND_FAR;
    int bx0, bx1, by0, by1, dxm, W, H, s;
    if (far) {
      by0 = clampi(floor(b.y0)), by1 = clampi(ceil(b.y1)), bx0 = clampi(floor(b.x0)), bx1 = clampi(ceil(b.x1));
      dxm = dxf + 2, W = w, H = h, s = 1;
    } else {
      by0 = clampi(floor(__dmul_rn(b.y0, sy))), by1 = clampi(ceil(__dmul_rn(b.y1, sy)));
      bx0 = clampi(floor(__dmul_rn(b.x0, sx))), bx1 = clampi(ceil(__dmul_rn(b.x1, sx)));
      dxm = dxs + 2, W = cw, H = ch, s = 2;
    }
    int ra, re, c0, ce;
    read_rect(bx0, bx1, by0, by1, dxm - 2, W, H, side, tight, ra, re, c0, ce);
    if (ra >= re || c0 >= ce) continue;
    // raster rows [ra, re) -> image rows read by their windows (left image:
    // shifted by sh and clamped like the census row loads); the margin-less
    // read sets (tight 2) take no extra pixel either
    const int gm = tight == 2 ? 0 : 1;
    int ya = s * ra - RY - gm, ye = s * (re - 1) + RY + gm;
    ya = min(max(ya - sh, 0), h - 1), ye = min(max(ye - sh, 0), h - 1);
    if (r < ya || r > ye) continue;
    const int xa = max(0, s * c0 - RX - gm), xe = min(w - 1, s * (ce - 1) + RX + gm);
    const int sa = xa >> 4, sb = xe >> 4;  // segments [sa, sb]: one atomic per mask word
    for (int wd = sa >> 5; wd <= (sb >> 5); ++wd) {
      const int lo = max(sa - 32 * wd, 0), hi = min(sb - 32 * wd, 31);
      atomicOr(&mask[wid][wd], (hi == 31 ? 0xFFFFFFFFu : ((2u << hi) - 1u)) & ~((1u << lo) - 1u));
    }
  }
  __syncwarp();
  const uint8_t* src = (side ? hr : hl) + (int64_t)f * src_stride + (int64_t)r * src_pitch;
  uint8_t* dst = (side ? dr : dl) + (int64_t)f * dst_stride + (int64_t)r * dst_pitch;
  const int nseg = (w + 15) >> 4;
  // every load of the lane in flight before the first store (PCIe latency)
  uint4 v[GR_SEGW];
  int moved = 0;
#pragma unroll
  for (int t = 0; t < GR_SEGW; ++t) {
    const int sg = lane + 32 * t;
    if (sg < nseg && ((mask[wid][t] >> lane) & 1u)) v[t] = __ldcs(reinterpret_cast<const uint4*>(src + 16 * sg));
  }
#pragma unroll
  for (int t = 0; t < GR_SEGW; ++t) {
    const int sg = lane + 32 * t;
    if (sg < nseg && ((mask[wid][t] >> lane) & 1u)) {
      *reinterpret_cast<uint4*>(dst + 16 * sg) = v[t];
      ++moved;
    }
  }
  moved = __reduce_add_sync(0xffffffffu, moved);
  if (lane == 0 && moved) atomicAdd(bytes + (f & 63), 16ull * (unsigned long long)moved);
  }
}

// census_transform_rois mask (census.hpp:111-136): keep codes inside the
// union of the clipped rectangles, zero elsewhere.  Kept codes leave in the
// reference layout (sentinel bit 25) whichever layout they were computed in.
__global__ void roi_mask_kernel(uint32_t* __restrict__ codes, int w, int h,
                                const rg_rect* __restrict__ rois, int n_rois) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w || y >= h) return;
  bool in = false;
  for (int r = 0; r < n_rois && !in; ++r) {
    const rg_rect q = rois[r];
    in = x >= max(0, q.x0) && x < min(w, q.x1) && y >= max(0, q.y0) && y < min(h, q.y1);
  }
  uint32_t& c = codes[(int64_t)y * w + x];
  if (!in)
    c = 0u;
  else if (c)
    c = (c & 0x01FFFFFFu) | 0x02000000u;
}

}  // namespace


cudaError_t launch_census_frames(const uint8_t* left, const uint8_t* right, int n_frames,
                                 int64_t frame_stride, int pitch, int w, int h, uint32_t* fl,
                                 uint32_t* fr, const PadGeom& gf, uint32_t* sl, uint32_t* sr,
                                 const PadGeom& gs, const int32_t* inv_x, const int32_t* inv_y,
                                 const int32_t* lshift, bool internal, cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  const int sides = right ? 2 : 1;
  const bool aligned = (pitch % 4 == 0) && (w % 4 == 0) && (frame_stride % 4 == 0) &&
                       (reinterpret_cast<uintptr_t>(left) % 4 == 0) &&
                       (!right || reinterpret_cast<uintptr_t>(right) % 4 == 0) && gf.pitch % 4 == 0 &&
                       gf.origin % 4 == 0 && w >= 8 && h >= 8;
  const bool half = !sl || (gs.w * 2 == w && gs.h * 2 == h && gs.pitch % 2 == 0 && gs.origin % 2 == 0);
  if (aligned && half) {
    auto kern = internal ? census_pairs_kernel<true> : census_pairs_kernel<false>;
    static SmemAttr attr[2];
    const cudaError_t e = attr[internal].ensure((const void*)kern, C2_SMEM);
    if (e != cudaSuccess) return e;
    dim3 grid((w + C2_TX - 1) / C2_TX, (h + C2_TY - 1) / C2_TY, sides * n_frames);
    kern<<<grid, C2_WARPS * 32, C2_SMEM, s>>>(left, right, frame_stride, pitch, w, h, fl, fr, gf, sl, sr, gs,
                                              lshift, nullptr, 0);
    return cudaGetLastError();
  }
  dim3 grid((w + TX - 1) / TX, (h + TY - 1) / TY, sides * n_frames);
  census_frames_kernel<<<grid, TPB, 0, s>>>(left, right, frame_stride, pitch, w, h, fl, fr, gf, sl,
                                            sr, gs, inv_x, inv_y, lshift, internal);
  return cudaGetLastError();
}

// 32-bit words of the row masks + tile lists of launch_census_rois
size_t census_rois_scratch_words(int n_frames, int w, int h, int ch) {
  const int tf = 2 * rw_pr<1>(), tr = 2 * rw_pr<2>(), nxt = (w + RW_TX - 1) / RW_TX;
  return (size_t)n_frames * ((h + 31) / 32 + (ch + 31) / 32 + 4 + 2 * ((h + tf - 1) / tf + (ch + tr - 1) / tr) * nxt);
}

// ROI census of a batch (see census_rows_kernel): the tile lists, the full
// raster on the FAR tiles and the reduced raster on the CLOSE tiles.
// cudaErrorNotSupported when the fast layout does not apply (the caller then
// runs the full-frame launch_census_frames).
namespace {
// census_rows_kernel over a batch: row masks + per-image compacted tile lists
// of the warp tiles (RW_TX columns x 2 rw_pr rows; reduced: RW_TX / 2) the
// ROI rectangles touch.  Returns the list geometry for the tile kernels.
struct RoiLists {
  int32_t* tiles;
  int tile_stride, side_off, red_off;
};
cudaError_t roi_lists(int n_frames, int w, int h, const PadGeom& gs, const rg_detection* dets,
                      const int32_t* det_off, double tau_s, int dx_far, int dx_close_scaled, uint32_t* masks,
                      cudaStream_t s, RoiLists* out) {
  const int wf = (h + 31) / 32, wr = (gs.h + 31) / 32;
  const int tf = 2 * rw_pr<1>(), tr = 2 * rw_pr<2>();  // output rows per warp tile
  const int nxt = (w + RW_TX - 1) / RW_TX;              // column tiles (reduced: RW_TX / 2 columns)
  const int rtf = (h + tf - 1) / tf, rtr = (gs.h + tr - 1) / tr;
  const int side_off = (rtf + rtr) * nxt;
  const int tile_stride = 4 + 2 * side_off;
  int32_t* tiles = reinterpret_cast<int32_t*>(masks + (size_t)n_frames * (wf + wr));
  const int bmw = 2 * ((rtf * nxt + 31) / 32 + (rtr * nxt + 31) / 32);
  // A/B knob: RG_CENSUS_TIGHT=0 computes the reference's whole ROI rectangles
  // on both images; default: only the part of each the matcher reads
  static const int tight = [] {
    const char* v = getenv("RG_CENSUS_TIGHT");
    return v ? atoi(v) : 2;
  }();
  static const bool greedy = [] { const char* v = getenv("RG_CENSUS_GREEDY"); return v ? atoi(v) != 0 : true; }();
  *out = {tiles, tile_stride, side_off, 4 + rtf * nxt};
  if (greedy && nxt <= 64) {
    const size_t smem = sizeof(uint32_t) * (size_t)(wf + wr + 2 * nxt * (wf + wr));
    static SmemAttr attr;
    const cudaError_t e = attr.ensure((const void*)census_cols_kernel, smem);
    if (e != cudaSuccess) return e;
    census_cols_kernel<<<n_frames, RM_T, smem, s>>>(dets, det_off, w, h, tau_s, gs.w, gs.h, wf, wr, masks, dx_far,
                                                    dx_close_scaled, nxt, tf, tr, rtf, rtr, tile_stride, tiles,
                                                    tight);
    return cudaGetLastError();
  }
  census_rows_kernel<<<n_frames, RM_T, sizeof(uint32_t) * (wf + wr + bmw), s>>>(
      dets, det_off, w, h, tau_s, gs.w, gs.h, wf, wr, masks, dx_far, dx_close_scaled, nxt, tf, tr, rtf, rtr,
      tile_stride, tiles, tight);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_census_rois(const uint8_t* left, const uint8_t* right, int n_frames, int64_t frame_stride,
                               int pitch, int w, int h, uint32_t* fl, uint32_t* fr, const PadGeom& gf, uint32_t* sl,
                               uint32_t* sr, const PadGeom& gs, const int32_t* lshift, bool internal,
                               const rg_detection* dets, const int32_t* det_off, double tau_s, int dx_far,
                               int dx_close_scaled, uint32_t* masks, cudaStream_t s, cudaEvent_t full_done,
                               cudaStream_t side, cudaEvent_t ev_lists, cudaEvent_t ev_red) {
  if (n_frames <= 0) return cudaSuccess;
  const int sides = right ? 2 : 1;
  const bool aligned = (pitch % 4 == 0) && (w % 4 == 0) && (frame_stride % 4 == 0) &&
                       (reinterpret_cast<uintptr_t>(left) % 4 == 0) &&
                       (!right || reinterpret_cast<uintptr_t>(right) % 4 == 0) && gf.pitch % 4 == 0 &&
                       gf.origin % 4 == 0 && w >= 8 && h >= 8;
  const bool half = sl && gs.w * 2 == w && gs.h * 2 == h && gs.pitch % 2 == 0 && gs.origin % 2 == 0 &&
                    gs.w >= 4 && gs.h >= 4;
  if (!aligned || !half || !masks || !dets) return cudaErrorNotSupported;
  RoiLists rl;
  cudaError_t e = roi_lists(n_frames, w, h, gs, dets, det_off, tau_s, dx_far, dx_close_scaled, masks, s, &rl);
  if (e != cudaSuccess) return e;
  int32_t* tiles = rl.tiles;
  const int tile_stride = rl.tile_stride, side_off = rl.side_off;
  const int wf = (h + 31) / 32, wr = (gs.h + 31) / 32;
  static const int mode = [] {
    // A/B knob: 1 warp row tiles (default), 0 the full-frame pair tiles storing
    // only ROI rows (measured: no faster than storing every row -- K1 is
    // bound by its compares and V builds, not by its stores)
    const char* v = getenv("RG_CENSUS_MODE");
    return v ? atoi(v) : 1;
  }();
  if (mode == 0) {
    auto kern = internal ? census_pairs_kernel<true> : census_pairs_kernel<false>;
    static SmemAttr pattr[2];
    e = pattr[internal].ensure((const void*)kern, C2_SMEM);
    if (e != cudaSuccess) return e;
    dim3 grid((w + C2_TX - 1) / C2_TX, (h + C2_TY - 1) / C2_TY, sides * n_frames);
    kern<<<grid, C2_WARPS * 32, C2_SMEM, s>>>(left, right, frame_stride, pitch, w, h, fl, fr, gf, sl, sr, gs, lshift,
                                              masks, wf + wr);
    return cudaGetLastError();
  }
  // a fixed number of single-warp CTAs per (frame, side) walk the compacted
  // 2-D tile lists
  auto rowtile = [&](auto kern, size_t smem, SmemAttr& attr, uint32_t* a, uint32_t* b, const PadGeom& g,
                     int walkers, int list_off, int wpb, cudaStream_t ks) -> cudaError_t {
    cudaError_t e2 = attr.ensure((const void*)kern, smem);
    if (e2 != cudaSuccess) return e2;
    dim3 grid(walkers, 1, sides * n_frames);
    kern<<<grid, wpb * 32, smem, ks>>>(left, right, frame_stride, pitch, w, h, a, b, g, lshift, tiles,
                                       tile_stride, list_off, side_off);
    return cudaGetLastError();
  };
  // par (side stream + two events): the reduced-raster tiles run on the side
  // stream alongside the full-raster ones, s waits for them at the end
  const bool par = side && ev_lists && ev_red && !full_done;
  if (par) {
    e = cudaEventRecord(ev_lists, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev_lists, 0);
    if (e != cudaSuccess) return e;
  }
  static const int walk_f = [] { const char* v = getenv("RG_ROWTILE_WALK1"); return v ? atoi(v) : 128; }();
  static const int walk_r = [] { const char* v = getenv("RG_ROWTILE_WALK2"); return v ? atoi(v) : 128; }();
  static SmemAttr attr[4];
  if (par) {
    e = internal ? rowtile(census_rowtile_kernel<true, 2>, rw_smem<2>(), attr[2], sl, sr, gs, walk_r, rl.red_off,
                           rw_wpb<2>(), side)
                 : rowtile(census_rowtile_kernel<false, 2>, rw_smem<2>(), attr[3], sl, sr, gs, walk_r, rl.red_off,
                           rw_wpb<2>(), side);
    if (e == cudaSuccess) e = cudaEventRecord(ev_red, side);
    if (e != cudaSuccess) return e;
  }
  e = internal ? rowtile(census_rowtile_kernel<true, 1>, rw_smem<1>(), attr[0], fl, fr, gf, walk_f, 4, rw_wpb<1>(), s)
               : rowtile(census_rowtile_kernel<false, 1>, rw_smem<1>(), attr[1], fl, fr, gf, walk_f, 4, rw_wpb<1>(),
                         s);
  if (e != cudaSuccess) return e;
  if (par) return cudaStreamWaitEvent(s, ev_red, 0);
  if (full_done) {  // the full raster is complete (the FAR matcher may start)
    e = cudaEventRecord(full_done, s);
    if (e != cudaSuccess) return e;
  }
  e = internal ? rowtile(census_rowtile_kernel<true, 2>, rw_smem<2>(), attr[2], sl, sr, gs, walk_r, rl.red_off,
                         rw_wpb<2>(), s)
               : rowtile(census_rowtile_kernel<false, 2>, rw_smem<2>(), attr[3], sl, sr, gs, walk_r, rl.red_off,
                         rw_wpb<2>(), s);
  return e;
}

cudaError_t launch_census64_frames(const uint8_t* left, const uint8_t* right, int n_frames, int64_t frame_stride,
                                   int pitch, int w, int h, unsigned long long* fl, unsigned long long* fr,
                                   const PadGeom& gf, unsigned long long* sl, unsigned long long* sr,
                                   const PadGeom& gs, const int32_t* inv_x, const int32_t* inv_y,
                                   const int32_t* lshift, cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  static const bool scalar = getenv("RG_CENSUS64_SCALAR") != nullptr;  // A/B knob: the per-pixel kernel
  const bool aligned = (pitch % 4 == 0) && (w % 4 == 0) && (frame_stride % 4 == 0) &&
                       (reinterpret_cast<uintptr_t>(left) % 4 == 0) &&
                       (!right || reinterpret_cast<uintptr_t>(right) % 4 == 0) && gf.pitch % 2 == 0 &&
                       gf.origin % 2 == 0 && w >= 12 && h >= 8;
  const bool half = !sl || (gs.w * 2 == w && gs.h * 2 == h && gs.pitch % 2 == 0 && gs.origin % 2 == 0);
  if (aligned && half && !scalar) {
    static SmemAttr attr;
    const cudaError_t e = attr.ensure((const void*)census64_pairs_kernel, X2_SMEM);
    if (e != cudaSuccess) return e;
    dim3 grid((w + X2_TX - 1) / X2_TX, (h + X2_TY - 1) / X2_TY, (right ? 2 : 1) * n_frames);
    census64_pairs_kernel<<<grid, X2_WARPS * 32, X2_SMEM, s>>>(left, right, frame_stride, pitch, w, h, fl, fr, gf,
                                                               sl, sr, gs, lshift);
    return cudaGetLastError();
  }
  dim3 grid((w + X_TX - 1) / X_TX, (h + X_TY - 1) / X_TY, (right ? 2 : 1) * n_frames);
  census64_kernel<<<grid, X_TPB, 0, s>>>(left, right, frame_stride, pitch, w, h, fl, fr, gf, sl, sr, gs, inv_x,
                                         inv_y, lshift);
  return cudaGetLastError();
}

// 9x7 ROI census of a batch: census_rows_kernel's lists, the full raster on
// the FAR tiles and the reduced raster on the CLOSE tiles
// (census64_rowtile_kernel).  cudaErrorNotSupported when the layout does not
// apply (the caller then runs launch_census64_frames).
cudaError_t launch_census64_rois(const uint8_t* left, const uint8_t* right, int n_frames, int64_t frame_stride,
                                 int pitch, int w, int h, unsigned long long* fl, unsigned long long* fr,
                                 const PadGeom& gf, unsigned long long* sl, unsigned long long* sr,
                                 const PadGeom& gs, const int32_t* lshift, const rg_detection* dets,
                                 const int32_t* det_off, double tau_s, int dx_far, int dx_close_scaled,
                                 uint32_t* masks, cudaStream_t s, cudaStream_t side, cudaEvent_t ev_lists,
                                 cudaEvent_t ev_red) {
  if (n_frames <= 0) return cudaSuccess;
  const bool aligned = (pitch % 4 == 0) && (w % 4 == 0) && (frame_stride % 4 == 0) &&
                       (reinterpret_cast<uintptr_t>(left) % 4 == 0) &&
                       (!right || reinterpret_cast<uintptr_t>(right) % 4 == 0) && gf.pitch % 2 == 0 &&
                       gf.origin % 2 == 0 && w >= 12 && h >= 8;
  const bool half = sl && gs.w * 2 == w && gs.h * 2 == h && gs.pitch % 2 == 0 && gs.origin % 2 == 0 &&
                    gs.w >= 4 && gs.h >= 4;
  if (!aligned || !half || !masks || !dets) return cudaErrorNotSupported;
  RoiLists rl;
  cudaError_t e = roi_lists(n_frames, w, h, gs, dets, det_off, tau_s, dx_far, dx_close_scaled, masks, s, &rl);
  if (e != cudaSuccess) return e;
  static SmemAttr attr[2];
  static const int walkers = [] { const char* v = getenv("RG_ROWTILE_WALK64"); return v ? atoi(v) : 128; }();
  const dim3 grid(walkers, 1, (right ? 2 : 1) * n_frames);
  e = attr[0].ensure((const void*)census64_rowtile_kernel<1>, c64_smem<1>());
  if (e != cudaSuccess) return e;
  const bool par0 = side && ev_lists && ev_red;
  if (par0) {  // the lists are done: the reduced tiles may start on the side stream
    e = cudaEventRecord(ev_lists, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev_lists, 0);
    if (e != cudaSuccess) return e;
  }
  census64_rowtile_kernel<1><<<grid, 32, c64_smem<1>(), s>>>(left, right, frame_stride, pitch, w, h, fl, fr, gf,
                                                             lshift, rl.tiles, rl.tile_stride, 4, rl.side_off);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = attr[1].ensure((const void*)census64_rowtile_kernel<2>, c64_smem<2>());
  if (e != cudaSuccess) return e;
  // par: the reduced-raster tiles on the side stream alongside the full ones
  const bool par = par0;
  census64_rowtile_kernel<2><<<grid, 32, c64_smem<2>(), par ? side : s>>>(
      left, right, frame_stride, pitch, w, h, sl, sr, gs, lshift, rl.tiles, rl.tile_stride, rl.red_off, rl.side_off);
  e = cudaGetLastError();
  if (e != cudaSuccess || !par) return e;
  e = cudaEventRecord(ev_red, side);
  return e == cudaSuccess ? cudaStreamWaitEvent(s, ev_red, 0) : e;
}

// Zero-copy gather of the census read sets of n_frames pinned host frames
// (see gather_rows_kernel); cudaErrorNotSupported when the layout does not
// allow 16-B segments (the caller then copies whole frames).
cudaError_t launch_gather_rows(const uint8_t* hl, const uint8_t* hr, int64_t src_stride, int src_pitch, uint8_t* dl,
                               uint8_t* dr, int64_t dst_stride, int dst_pitch, int w, int h, int n_frames,
                               const rg_detection* dets, const int32_t* det_off, double tau_s, int close_scale,
                               int dx_far, int dx_close_scaled, bool wide, const int32_t* lshift,
                               unsigned long long* bytes, cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  const auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  if (src_pitch % 16 || dst_pitch % 16 || src_stride % 16 || dst_stride % 16 || !al(hl) || !al(hr) || !al(dl) ||
      !al(dr) || w > 32 * GR_SEGW * 16 || w % 16)
    return cudaErrorNotSupported;
  static const int tight = [] {
    const char* v = getenv("RG_CENSUS_TIGHT");
    return v ? atoi(v) : 2;
  }();
  static const int ctas = [] { const char* v = getenv("RG_GATHER_CTAS"); return v ? atoi(v) : 4 * 148; }();
  const int items = h * 2 * n_frames;
  const int grid = std::max(1, std::min(ctas, (items + GR_WARPS - 1) / GR_WARPS));
  const int cw = w / close_scale, ch = h / close_scale;
  if (wide)
    gather_rows_kernel<4, 3><<<grid, GR_WARPS * 32, 0, s>>>(hl, hr, src_stride, src_pitch, dl, dr, dst_stride,
                                                            dst_pitch, w, h, dets, det_off, tau_s, cw, ch, dx_far,
                                                            dx_close_scaled, tight, lshift, bytes, n_frames);
  else
    gather_rows_kernel<2, 2><<<grid, GR_WARPS * 32, 0, s>>>(hl, hr, src_stride, src_pitch, dl, dr, dst_stride,
                                                            dst_pitch, w, h, dets, det_off, tau_s, cw, ch, dx_far,
                                                            dx_close_scaled, tight, lshift, bytes, n_frames);
  return cudaGetLastError();
}

cudaError_t launch_roi_mask(uint32_t* codes, int w, int h, const rg_rect* rois, int n_rois,
                            cudaStream_t s) {
  dim3 grid((w + 255) / 256, h);
  roi_mask_kernel<<<grid, 256, 0, s>>>(codes, w, h, rois, n_rois);
  return cudaGetLastError();
}

}  // namespace rg
