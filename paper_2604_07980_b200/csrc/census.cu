// census.cu -- K1: 5x5 census transform on sm_100a.
//
// Replaces census_code_at / census_transform / census_transform_rois
// (reference census.hpp:43-138).  Descriptor layout is the reference's:
// sentinel bit 25, then the 25 window compares (window row -2 first, column
// -2 first), centre compare always 0, code 0 when the window leaves the
// image.  The reduced CLOSE raster is a gather of the full raster at
// (mx[x'], my[y']) with mx = lround(x' * src/out) (census.hpp:59-64), so the
// batched kernel writes it from the same registers (inverse index maps).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "rg_common.cuh"

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
    const int32_t* __restrict__ inv_x, const int32_t* __restrict__ inv_y) {
  __shared__ __align__(16) uint8_t tile[TY + 4][TX + 8];
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
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
    tile[r][c] = (gx >= 0 && gx < w && gy >= 0 && gy < h) ? img[(int64_t)gy * pitch + gx] : 0;
  }
  __syncthreads();

  const int tx = threadIdx.x & (TX - 1);
  const int x = x0 + tx;
  const int ix = (x < w) ? inv_x[x] : -1;
  for (int ty = threadIdx.x / TX; ty < TY; ty += TPB / TX) {
    const int y = y0 + ty;
    if (x >= w || y >= h) continue;
    uint32_t code = 0;
    if (x >= 2 && y >= 2 && x < w - 2 && y < h - 2) code = census_window(&tile[ty + 2][tx + 2], TX + 8);
    full[(int64_t)y * gf.pitch + x] = code;
    if (red && ix >= 0) {
      const int iy = inv_y[y];
      if (iy >= 0) red[(int64_t)iy * gs.pitch + ix] = code;
    }
  }
}

// ---------------------------------------------------------------------------
// Fast path (pitch % 4 == 0, W % 4 == 0, reduced raster = exact half or none):
// half2 "vertical pair" census.  Pixel rows y and y+1 ride in the two fp16
// lanes of one register, encoded exactly as 1024 + intensity.  V[r][x] holds
// (I(x, r), I(x, r+1)), so the window neighbour (i, j) of BOTH pixels of the
// pair (x, y)/(x, y+1) is the single register V[y+j][x+i]: one HSET2 (n > c,
// 1.0/0.0 per lane) and one HFMA2 (acc = 2 acc + m) advance two descriptors
// by one bit.  24 compares go into three fp16 accumulators (1+10, 1+10, 1+5
// bits, each exact below 2048) that are unpacked into the reference's bit
// layout at the end; the centre compare (always 0) is folded into a x4 step.
// V is built once per CTA in shared memory (6 PRMT per 4 entries from the
// raw image words); each warp then streams a 16-row strip keeping a rolling
// 5-row window of V in registers (2 new rows per pixel-pair row).
constexpr int C2_LANES_PAIRS = 4;                 // pixel pairs per lane
constexpr int C2_TX = 32 * C2_LANES_PAIRS;        // 128 tile columns
constexpr int C2_WARPS = 8;
constexpr int C2_PR = 4;                          // pair rows per warp strip
constexpr int C2_TY = C2_WARPS * C2_PR * 2;       // 64 tile rows
constexpr int C2_VW = C2_TX + 4;                  // V entries per row (x0-2 .. x0+TX+1)
constexpr int C2_VR = C2_TY + 3;                  // V rows (y0-2 .. y0+TY)
constexpr int C2_WORDS = C2_TX / 4 + 2;           // image words per row (x0-4 .. x0+TX+3)
constexpr size_t C2_SMEM = sizeof(uint32_t) * C2_VR * C2_VW;

__device__ __forceinline__ uint32_t c2_vpair(uint32_t a, uint32_t b, int j) {
  // entry j of the 4 columns of words a (row r) and b (row r+1): half2(1024+a_j, 1024+b_j)
  const uint32_t t = __byte_perm(a, b, j < 2 ? 0x5140 : 0x7362);  // a_j b_j a_j+1 b_j+1
  return __byte_perm(t, 0x64646464u, (j & 1) ? 0x4342 : 0x4140);
}

// The three fp16 accumulators are built so each group's compare bits sit in
// the low bits of the half's mantissa (value 1024 + B, exponent fixed):
// g0 = w0..w7 (init 4.0, 8 steps), g1 = w8..w16 (init 2.0, 9 bits incl. the
// centre 0), g2 = w17..w24 (init 4.0).  code = 1<<25 | B0<<17 | B1<<8 | B2,
// assembled with byte permutes for both lanes (lo = row y, hi = row y+1).
__device__ __forceinline__ void c2_assemble(uint32_t g0, uint32_t g1, uint32_t g2, uint32_t& lo,
                                            uint32_t& hi) {
  const uint32_t xl = __byte_perm(g2, g1, 0x0540);  // [B2, B1 lo8, 0x64|B1b8, 0]
  const uint32_t xh = __byte_perm(g2, g1, 0x0762);  // same from the high halves
  lo = (((xl & 0x1FFFFu) | ((g0 << 17) & 0x1FE0000u)) & 0x1FFFFFFu) | 0x2000000u;
  hi = (((xh & 0x1FFFFu) | ((g0 << 1) & 0x1FE0000u)) & 0x1FFFFFFu) | 0x2000000u;
}

// Phase 2 for one warp: its C2_PR pair rows of the tile whose V is in smem.
__device__ __forceinline__ void c2_strip(const uint32_t* __restrict__ V, uint32_t* __restrict__ full,
                                         uint32_t* __restrict__ red, const PadGeom& gf, const PadGeom& gs,
                                         int x0, int y0, int w, int h) {
  // ---- phase 2: warp strip of C2_PR pair rows, lane = 4 pixel pairs
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int xl = x0 + 4 * lane;  // first column of this lane
  if (xl >= w) return;
  const __half2 two = __float2half2_rn(2.0f), four = __float2half2_rn(4.0f);
  uint32_t win[5][8];
  const int pr0 = wid * C2_PR;
  auto load_row = [&](int slot, int vr) {
    const uint4* src = reinterpret_cast<const uint4*>(V + vr * C2_VW + 4 * lane);
    const uint4 p = src[0], q = src[1];
    win[slot][0] = p.x; win[slot][1] = p.y; win[slot][2] = p.z; win[slot][3] = p.w;
    win[slot][4] = q.x; win[slot][5] = q.y; win[slot][6] = q.z; win[slot][7] = q.w;
  };
  if (y0 + 2 * pr0 >= h) return;
#pragma unroll
  for (int j = 0; j < 5; ++j) load_row(j, 2 * pr0 + j);
  const bool xedge = xl < 2 || xl + 3 > w - 3;
#pragma unroll
  for (int p = pr0; p < pr0 + C2_PR; ++p) {
    const int y = y0 + 2 * p;
    if (y >= h) break;
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const __half2 c = *reinterpret_cast<const __half2*>(&win[2][q + 2]);
      __half2 g[3];
      g[0] = g[2] = __float2half2_rn(4.0f);
      g[1] = __float2half2_rn(2.0f);
#pragma unroll
      for (int wi = 0; wi < 25; ++wi) {
        if (wi == 12) continue;  // centre: its 0 bit is folded into w13's x4
        const int j = wi / 5, i = wi % 5;
        // compare on the ALU pipe (HSET2) for 2/3 of the taps and on the FMA
        // pipe (saturated (1024+n)-(1024+c), exact) for the rest, so the two
        // pipes stay balanced with the HFMA2 packing
        const __half2 v = *reinterpret_cast<const __half2*>(&win[j][q + i]);
        const __half2 m = (wi % 3 == 0) ? __hsub2_sat(v, c) : __hgt2(v, c);
        const int gi = wi < 8 ? 0 : (wi < 17 ? 1 : 2);
        g[gi] = __hfma2(g[gi], wi == 13 ? four : two, m);
      }
      c2_assemble(*reinterpret_cast<uint32_t*>(&g[0]), *reinterpret_cast<uint32_t*>(&g[1]),
                  *reinterpret_cast<uint32_t*>(&g[2]), lo[q], hi[q]);
    }
    // border: codes are 0 where the window leaves the image (census.hpp:44)
    if (xedge || y < 2 || y + 1 > h - 3) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool xin = xl + q >= 2 && xl + q <= w - 3;
        if (!(xin && y >= 2 && y <= h - 3)) lo[q] = 0u;
        if (!(xin && y + 1 >= 2 && y + 1 <= h - 3)) hi[q] = 0u;
      }
    }
    uint32_t* o = full + (int64_t)y * gf.pitch + xl;
    *reinterpret_cast<uint4*>(o) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    if (y + 1 < h) *reinterpret_cast<uint4*>(o + gf.pitch) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    if (red) {  // reduced raster = codes at even (x, y): (x/2, y/2)
      uint32_t* ro = red + (int64_t)(y >> 1) * gs.pitch + (xl >> 1);
      *reinterpret_cast<uint2*>(ro) = make_uint2(lo[0], lo[2]);
    }
    // roll the window down two V rows
    if (p + 1 < pr0 + C2_PR) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        win[0][k] = win[2][k];
        win[1][k] = win[3][k];
        win[2][k] = win[4][k];
      }
      load_row(3, 2 * (p + 1) + 3);
      load_row(4, 2 * (p + 1) + 4);
    }
  }
}

__global__ void __launch_bounds__(C2_WARPS * 32) census_pairs_kernel(
    const uint8_t* __restrict__ left, const uint8_t* __restrict__ right, int64_t frame_stride,
    int pitch, int w, int h, uint32_t* __restrict__ fl, uint32_t* __restrict__ fr, PadGeom gf,
    uint32_t* __restrict__ sl, uint32_t* __restrict__ sr, PadGeom gs) {
  extern __shared__ __align__(16) uint32_t V[];  // [C2_VR][C2_VW]
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
  const uint8_t* img = (side ? right : left) + (int64_t)frame * frame_stride;
  uint32_t* full = (side ? fr : fl) + (int64_t)frame * gf.fstride + gf.origin;
  uint32_t* red = side ? sr : sl;
  if (red) red += (int64_t)frame * gs.fstride + gs.origin;
  const int x0 = blockIdx.x * C2_TX, y0 = blockIdx.y * C2_TY;
  // ---- phase 1: V rows y0-2 .. y0+TY from the image words; each thread walks
  // one word column down a run of rows, so every image word is loaded once.
  // Out-of-image words are clamped: they only feed border codes (forced to 0).
  const int wmax = (w + 3) / 4 - 1;
  constexpr int RUNS = (C2_WARPS * 32) / C2_WORDS;         // 7 runs of rows
  constexpr int RUN_LEN = (C2_VR + RUNS - 1) / RUNS;       // 19 rows per run
  const int wk = threadIdx.x % C2_WORDS, run = threadIdx.x / C2_WORDS;
  if (run < RUNS) {
    const int kw = min(max((x0 - 4) / 4 + wk, 0), wmax);
    const uint32_t* col = reinterpret_cast<const uint32_t*>(img) + kw;
    const int pw = pitch / 4;
    const int r0 = run * RUN_LEN, n = min(RUN_LEN, C2_VR - r0);
    uint32_t wv[RUN_LEN + 1];  // all loads of the run in flight at once
#pragma unroll
    for (int t = 0; t <= RUN_LEN; ++t)
      if (t <= n) wv[t] = __ldg(col + (int64_t)min(max(y0 - 2 + r0 + t, 0), h - 1) * pw);
#pragma unroll
    for (int t = 0; t < RUN_LEN; ++t) {
      if (t < n) {
        const uint32_t a = wv[t], b = wv[t + 1];
        uint32_t* vrow = V + (r0 + t) * C2_VW + 4 * wk - 2;  // entries 4wk-2 .. 4wk+1
        if (wk > 0) *reinterpret_cast<uint2*>(vrow) = make_uint2(c2_vpair(a, b, 0), c2_vpair(a, b, 1));
        if (wk < C2_WORDS - 1)
          *reinterpret_cast<uint2*>(vrow + 2) = make_uint2(c2_vpair(a, b, 2), c2_vpair(a, b, 3));
      }
    }
  }
  __syncthreads();

  c2_strip(V, full, red, gf, gs, x0, y0, w, h);
}

// ---------------------------------------------------------------------------
// Persistent TMA-pipelined variant of the fast path.  Each CTA walks tiles
// t = blockIdx.x, +gridDim.x, ...; the raw bytes of tile t+1 (160 x 68 box,
// out-of-image bytes zero-filled by the TMA unit) stream into the other smem
// buffer with cp.async.bulk.tensor while tile t builds V and computes, so the
// HBM read latency is off the critical path.
// the innermost TMA box coordinate must be a multiple of 16 bytes (measured:
// x = -8 or 8 raises an illegal-instruction fault, -16/16 work), so the raw
// box starts 16 columns left of the tile
constexpr int T_RW = 160;                 // raw box columns: x0-16 .. x0+TX+16
constexpr int T_RH = C2_TY + 4;           // raw box rows:    y0-2 .. y0+TY+1
constexpr int T_RAW = T_RW * T_RH;        // bytes per raw buffer (10880)
constexpr int T_RAW_PAD = (T_RAW + 127) / 128 * 128;
constexpr size_t T_SMEM = 2 * T_RAW_PAD + C2_SMEM + 2 * sizeof(uint64_t) + 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void tma_load_tile(const CUtensorMap* tm, uint32_t dst, uint32_t bar, int cx,
                                              int cy, int cz) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(T_RAW)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(tm), "r"(cx), "r"(cy), "r"(cz), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_issue(const CUtensorMap* const* tmaps, int t, int b, int per_img, int tx,
                                          int sides, unsigned char* raw, uint64_t* bar) {
  const int img = t / per_img, rem = t - img * per_img;
  const int yy = rem / tx, xx = rem - yy * tx;
  const int frame = img / sides, side = img - frame * sides;
  tma_load_tile(tmaps[side], smem_u32(raw + b * T_RAW_PAD), smem_u32(&bar[b]), xx * C2_TX - 16, yy * C2_TY - 2,
                frame);
}

__global__ void __launch_bounds__(C2_WARPS * 32, 4) census_tma_kernel(
    const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmR, int sides,
    int n_frames, int w, int h, uint32_t* __restrict__ fl, uint32_t* __restrict__ fr, PadGeom gf,
    uint32_t* __restrict__ sl, uint32_t* __restrict__ sr, PadGeom gs) {
  extern __shared__ __align__(128) unsigned char tsm[];
  unsigned char* raw = tsm;                                            // 2 raw buffers
  uint32_t* V = reinterpret_cast<uint32_t*>(tsm + 2 * T_RAW_PAD);      // [C2_VR][C2_VW]
  uint64_t* bar = reinterpret_cast<uint64_t*>(tsm + 2 * T_RAW_PAD + C2_SMEM);
  const int tx = (w + C2_TX - 1) / C2_TX, ty = (h + C2_TY - 1) / C2_TY;
  const int per_img = tx * ty, total = per_img * sides * n_frames;
  // (the tensor maps are addressed in param space: never copy them locally)
  const CUtensorMap* tmaps[2] = {&tmL, &tmR};
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && (int)blockIdx.x < total)
    tma_issue(tmaps, blockIdx.x, 0, per_img, tx, sides, raw, bar);
  uint32_t phase[2] = {0u, 0u};
  constexpr int RUNS = (C2_WARPS * 32) / C2_WORDS;
  constexpr int RUN_LEN = (C2_VR + RUNS - 1) / RUNS;
  const int wk = threadIdx.x % C2_WORDS, run = threadIdx.x / C2_WORDS;
  int it = 0;
  for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
    const int b = it & 1;
    // prefetch the next tile into the other buffer (its last reader finished
    // before the barrier that closed the previous iteration)
    if (threadIdx.x == 0 && t + (int)gridDim.x < total)
      tma_issue(tmaps, t + gridDim.x, b ^ 1, per_img, tx, sides, raw, bar);
    mbar_wait(smem_u32(&bar[b]), phase[b]);
    phase[b] ^= 1u;
    // V from the raw tile: raw word m+3 covers image columns x0-4+4m .. +3
    const unsigned char* rb = raw + b * T_RAW_PAD;
    if (run < RUNS) {
      const int r0 = run * RUN_LEN, n = min(RUN_LEN, C2_VR - r0);
      const uint32_t* col = reinterpret_cast<const uint32_t*>(rb) + (wk + 3);
      uint32_t a = col[r0 * (T_RW / 4)];
      for (int q = 0; q < n; ++q) {
        const uint32_t bb = col[(r0 + q + 1) * (T_RW / 4)];
        uint32_t* vrow = V + (r0 + q) * C2_VW + 4 * wk - 2;
        if (wk > 0) *reinterpret_cast<uint2*>(vrow) = make_uint2(c2_vpair(a, bb, 0), c2_vpair(a, bb, 1));
        if (wk < C2_WORDS - 1)
          *reinterpret_cast<uint2*>(vrow + 2) = make_uint2(c2_vpair(a, bb, 2), c2_vpair(a, bb, 3));
        a = bb;
      }
    }
    __syncthreads();
    const int img = t / per_img, rem = t - img * per_img;
    const int yy = rem / tx, xx = rem - yy * tx;
    const int frame = img / sides, side = img - frame * sides;
    uint32_t* full = (side ? fr : fl) + (int64_t)frame * gf.fstride + gf.origin;
    uint32_t* red = side ? sr : sl;
    if (red) red += (int64_t)frame * gs.fstride + gs.origin;
    c2_strip(V, full, red, gf, gs, xx * C2_TX, yy * C2_TY, w, h);
    __syncthreads();
  }
}

// census_transform_rois mask (census.hpp:111-136): keep codes inside the
// union of the clipped rectangles, zero elsewhere.
__global__ void roi_mask_kernel(uint32_t* __restrict__ codes, int w, int h,
                                const rg_rect* __restrict__ rois, int n_rois) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w || y >= h) return;
  bool in = false;
  for (int r = 0; r < n_rois && !in; ++r) {
    const rg_rect q = rois[r];
    in = x >= max(0, q.x0) && x < min(w, q.x1) && y >= max(0, q.y0) && y < min(h, q.y1);
  }
  if (!in) codes[(int64_t)y * w + x] = 0u;
}

}  // namespace


// Tensor maps for the raw frames (uint8, 3-D: columns x rows x frames).
static cudaError_t make_tmap(CUtensorMap* tm, const uint8_t* base, int w, int h, int n_frames, int pitch,
                             int64_t frame_stride) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return cudaErrorNotSupported;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n_frames};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)frame_stride};
  const cuuint32_t box[3] = {(cuuint32_t)T_RW, (cuuint32_t)T_RH, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorNotSupported;
}

static cudaError_t launch_census_tma(const uint8_t* left, const uint8_t* right, int n_frames,
                                     int64_t frame_stride, int pitch, int w, int h, uint32_t* fl, uint32_t* fr,
                                     const PadGeom& gf, uint32_t* sl, uint32_t* sr, const PadGeom& gs,
                                     cudaStream_t s) {
  CUtensorMap tmL, tmR;
  cudaError_t e = make_tmap(&tmL, left, w, h, n_frames, pitch, frame_stride);
  if (e != cudaSuccess) return e;
  e = make_tmap(&tmR, right ? right : left, w, h, n_frames, pitch, frame_stride);
  if (e != cudaSuccess) return e;
  static int n_sm = 0, per_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaFuncSetAttribute(census_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T_SMEM);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, census_tma_kernel, C2_WARPS * 32, T_SMEM);
    if (per_sm < 1) per_sm = 1;
  }
  const int sides = right ? 2 : 1;
  const long long tiles = (long long)((w + C2_TX - 1) / C2_TX) * ((h + C2_TY - 1) / C2_TY) * sides * n_frames;
  const int grid = (int)std::min<long long>(tiles, (long long)n_sm * per_sm);
  census_tma_kernel<<<grid, C2_WARPS * 32, T_SMEM, s>>>(tmL, tmR, sides, n_frames, w, h, fl, fr, gf, sl, sr, gs);
  return cudaGetLastError();
}

cudaError_t launch_census_frames(const uint8_t* left, const uint8_t* right, int n_frames,
                                 int64_t frame_stride, int pitch, int w, int h, uint32_t* fl,
                                 uint32_t* fr, const PadGeom& gf, uint32_t* sl, uint32_t* sr,
                                 const PadGeom& gs, const int32_t* inv_x, const int32_t* inv_y,
                                 cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  const int sides = right ? 2 : 1;
  const bool aligned = (pitch % 4 == 0) && (w % 4 == 0) && (frame_stride % 4 == 0) &&
                       (reinterpret_cast<uintptr_t>(left) % 4 == 0) &&
                       (!right || reinterpret_cast<uintptr_t>(right) % 4 == 0) && gf.pitch % 4 == 0 &&
                       gf.origin % 4 == 0 && w >= 8 && h >= 8;
  const bool half = !sl || (gs.w * 2 == w && gs.h * 2 == h && gs.pitch % 2 == 0 && gs.origin % 2 == 0);
  const bool tma_ok = aligned && half && pitch % 16 == 0 && frame_stride % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(left) % 16 == 0 &&
                      (!right || reinterpret_cast<uintptr_t>(right) % 16 == 0) && getenv("RG_CENSUS_TMA") != nullptr;
  if (tma_ok) {
    cudaError_t e = launch_census_tma(left, right, n_frames, frame_stride, pitch, w, h, fl, fr, gf, sl, sr, gs, s);
    if (e != cudaErrorNotSupported) return e;
  }
  if (aligned && half) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(census_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C2_SMEM);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    dim3 grid((w + C2_TX - 1) / C2_TX, (h + C2_TY - 1) / C2_TY, sides * n_frames);
    census_pairs_kernel<<<grid, C2_WARPS * 32, C2_SMEM, s>>>(left, right, frame_stride, pitch, w, h, fl, fr,
                                                             gf, sl, sr, gs);
    return cudaGetLastError();
  }
  dim3 grid((w + TX - 1) / TX, (h + TY - 1) / TY, sides * n_frames);
  census_frames_kernel<<<grid, TPB, 0, s>>>(left, right, frame_stride, pitch, w, h, fl, fr, gf, sl,
                                            sr, gs, inv_x, inv_y);
  return cudaGetLastError();
}

cudaError_t launch_roi_mask(uint32_t* codes, int w, int h, const rg_rect* rois, int n_rois,
                            cudaStream_t s) {
  dim3 grid((w + 255) / 256, h);
  roi_mask_kernel<<<grid, 256, 0, s>>>(codes, w, h, rois, n_rois);
  return cudaGetLastError();
}

}  // namespace rg
