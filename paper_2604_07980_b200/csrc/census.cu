// census.cu -- K1: 5x5 census transform on sm_100a.
//
// Replaces census_code_at / census_transform / census_transform_rois
// (reference census.hpp:43-138).  Descriptor layout is the reference's:
// sentinel bit 25, then the 25 window compares (window row -2 first, column
// -2 first), centre compare always 0, code 0 when the window leaves the
// image.  The reduced CLOSE raster is a gather of the full raster at
// (mx[x'], my[y']) with mx = lround(x' * src/out) (census.hpp:59-64), so the
// batched kernel writes it from the same registers (inverse index maps).
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
    int pitch, int w, int h, uint32_t* __restrict__ fl, uint32_t* __restrict__ fr,
    uint32_t* __restrict__ sl, uint32_t* __restrict__ sr, int cw, int ch,
    const int32_t* __restrict__ inv_x, const int32_t* __restrict__ inv_y) {
  __shared__ __align__(16) uint8_t tile[TY + 4][TX + 8];
  const int sides = right ? 2 : 1;
  const int frame = blockIdx.z / sides, side = blockIdx.z - frame * sides;
  const uint8_t* img = (side ? right : left) + (int64_t)frame * frame_stride;
  uint32_t* full = (side ? fr : fl) + (int64_t)frame * w * h;
  uint32_t* red = (side ? sr : sl);
  if (red) red += (int64_t)frame * cw * ch;
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
    full[(int64_t)y * w + x] = code;
    if (red && ix >= 0) {
      const int iy = inv_y[y];
      if (iy >= 0) red[(int64_t)iy * cw + ix] = code;
    }
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

cudaError_t launch_census_frames(const uint8_t* left, const uint8_t* right, int n_frames,
                                 int64_t frame_stride, int pitch, int w, int h, uint32_t* fl,
                                 uint32_t* fr, uint32_t* sl, uint32_t* sr, int cw, int ch,
                                 const int32_t* inv_x, const int32_t* inv_y, cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  dim3 grid((w + TX - 1) / TX, (h + TY - 1) / TY, (right ? 2 : 1) * n_frames);
  census_frames_kernel<<<grid, TPB, 0, s>>>(left, right, frame_stride, pitch, w, h, fl, fr, sl, sr,
                                            cw, ch, inv_x, inv_y);
  return cudaGetLastError();
}

cudaError_t launch_roi_mask(uint32_t* codes, int w, int h, const rg_rect* rois, int n_rois,
                            cudaStream_t s) {
  dim3 grid((w + 255) / 256, h);
  roi_mask_kernel<<<grid, 256, 0, s>>>(codes, w, h, rois, n_rois);
  return cudaGetLastError();
}

}  // namespace rg
