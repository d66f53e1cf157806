// render.cu -- device frame source: render_stereo_pair (reference
// synth.hpp:142-230) for a batch of scenes, straight into HBM.
//
// Byte-identical to the host renderer (synth.cpp), which is pinned to the
// reference by frame hashes.  Three stages per batch:
//   1. host: prepare_scene (projection, far-to-near order, spans) and the
//      256-entry radiometric map for every frame (O(objects), synth_scene.h);
//   2. render_body_kernel: one thread per (x, y) of a frame renders the left
//      pixel and the right pixel, the right one already radiometrically mapped
//      and vertically shifted (synth.hpp:212-220 fold into the addressing:
//      right(x, y) = lut[body(x, clamp(y - dy))]);
//   3. noise_kernel (noise_sigma > 0): the reference draws one
//      normal_distribution<double>(0, sigma) sample per pixel, left image then
//      right, from one std::mt19937_64(seed) (synth.hpp:221-228).  That stream
//      is sequential, so one CTA per frame walks it: the MT19937-64 recurrence
//      X[j] = X[j-156] ^ twist(X[j-312], X[j-311]) yields 156 outputs per
//      step in parallel; consecutive output pairs are the polar method's
//      (x, y) attempts (libstdc++ normal_distribution::operator()), a block
//      scan of the accept flags numbers the accepted pairs, and accepted pair
//      p perturbs pixels 2p (y * mult) and 2p + 1 (x * mult, the saved value).
//
// FP64 rules as everywhere in the library (-fmad=false, reference operation
// order).  The one libm call whose device result may differ is log() in the
// polar transform (CUDA: <= 1 ulp; glibc: < 1 ulp); a 1-ulp change of a
// normal moves a pixel only when v + sigma * n lies within ~1e-13 of a
// half-integer, so frames are byte-identical in practice -- tests compare
// whole frames against the host renderer.
#include <cstring>
#include <vector>

#include "rg_common.cuh"
#include "synth_scene.h"

namespace rg {
namespace {

using rg_synth::RenderObj;

struct FrameScene {  // per frame, device copy
  double bg_contrast, cell, bias, sigma;
  uint64_t bg_seed, seed;
  int32_t quant, dy, obj0, n_obj;
  uint8_t lut[256];
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // synth.hpp:56-61
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// ValueNoise::sample (synth.hpp:65-89), same operation order as synth.cpp.
__device__ __forceinline__ double noise_node(uint64_t seed, long long gx, long long gy) {
  const uint64_t k = uint64_t(gx) * 0x100000001B3ull ^ uint64_t(gy);
  return __ull2double_rn(mix64(seed ^ mix64(k)) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ uint8_t noise_byte(uint64_t seed, double cell, double contrast, int quant, double x,
                                              double y) {
  const double u = __ddiv_rn(x, cell), v = __ddiv_rn(y, cell);
  const long long iu = (long long)floor(u), iv = (long long)floor(v);
  const double tu = __dsub_rn(u, (double)iu), tv = __dsub_rn(v, (double)iv);
  const double a = noise_node(seed, iu, iv), b = noise_node(seed, iu + 1, iv);
  const double c = noise_node(seed, iu, iv + 1), d = noise_node(seed, iu + 1, iv + 1);
  const double top = __dadd_rn(__dmul_rn(a, __dsub_rn(1.0, tu)), __dmul_rn(b, tu));
  const double bot = __dadd_rn(__dmul_rn(c, __dsub_rn(1.0, tu)), __dmul_rn(d, tu));
  const double mixv = __dadd_rn(__dmul_rn(top, __dsub_rn(1.0, tv)), __dmul_rn(bot, tv));
  double val = __dadd_rn(128.0, __dmul_rn(contrast, __dsub_rn(__dmul_rn(2.0, mixv), 1.0)));
  if (quant > 1) val = __dmul_rn(round(__ddiv_rn(val, (double)quant)), (double)quant);
  val = val < 0.0 ? 0.0 : (val > 255.0 ? 255.0 : val);
  return (uint8_t)llround(val);  // lround: half away from zero
}

// Body of one left pixel (lx) and of the right pixel (rx) of image row y.
__device__ __forceinline__ void body_pixels(const FrameScene& fs, const RenderObj* __restrict__ ob, int x, int yl,
                                            int yr, uint8_t& lv, uint8_t& rv) {
  bool lset = false, rset = false;
  // paint order is far to near: scanning near to far, the first hit is the
  // pixel's final value
  for (int t = fs.n_obj - 1; t >= 0 && !(lset && rset); --t) {
    const RenderObj& s = ob[t];
    if (!lset && yl >= s.ly0 && yl <= s.ly1 && x >= s.lx0 && x <= s.lx1) {
      lv = noise_byte(s.tex_seed, fs.cell, s.contrast, fs.quant, __dsub_rn((double)x, s.u0),
                      __dsub_rn((double)yl, s.v0));
      lset = true;
    }
    if (!rset && yr >= s.ly0 && yr <= s.ly1 && x >= s.rx0 && x <= s.rx1) {
      const double u = __ddiv_rn(__dadd_rn((double)x, s.c0), s.k);
      if (!(u < s.u0 || u > s.u1)) {
        rv = noise_byte(s.tex_seed, fs.cell, s.contrast, fs.quant, __dsub_rn(u, s.u0), __dsub_rn((double)yr, s.v0));
        rset = true;
      }
    }
  }
  if (!lset) lv = noise_byte(fs.bg_seed, fs.cell, fs.bg_contrast, fs.quant, (double)x, (double)yl);
  if (!rset) rv = noise_byte(fs.bg_seed, fs.cell, fs.bg_contrast, fs.quant, __dadd_rn((double)x, fs.bias), (double)yr);
}

constexpr int kBodyTx = 128;

__global__ void __launch_bounds__(kBodyTx) render_body_kernel(const FrameScene* __restrict__ scenes,
                                                              const RenderObj* __restrict__ objs, int w, int h,
                                                              uint8_t* __restrict__ left, uint8_t* __restrict__ right,
                                                              int64_t frame_stride) {
  const int frame = blockIdx.z, y = blockIdx.y;
  const int x = blockIdx.x * kBodyTx + threadIdx.x;
  if (x >= w) return;
  const FrameScene& fs = scenes[frame];
  const int yr = min(max(y - fs.dy, 0), h - 1);  // shift_vertical, image.hpp:145-154
  uint8_t lv, rv;
  body_pixels(fs, objs + fs.obj0, x, y, yr, lv, rv);
  const int64_t o = (int64_t)frame * frame_stride + (int64_t)y * w + x;
  left[o] = lv;
  right[o] = fs.lut[rv];
}

// ---- noise: std::mt19937_64 + std::normal_distribution<double> (libstdc++)
constexpr int kMtN = 312, kMtM = 156, kRing = 512;
constexpr int kNoiseThreads = 160;  // 156 generators + 4 idle lanes of the 5th warp
constexpr int kNoiseWarps = kNoiseThreads / 32;

__device__ __forceinline__ uint64_t mt_temper(uint64_t z) {  // mersenne_twister_engine::operator()
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  return z ^ (z >> 43);
}

__device__ __forceinline__ double canonical(uint64_t z) {  // generate_canonical<double, 53>, k = 1
  const double r = __dmul_rn(__ull2double_rn(z), 0x1.0p-64);
  return r >= 1.0 ? 0x1.fffffffffffffp-1 : r;  // nextafter(1, 0)
}

__device__ __forceinline__ uint8_t add_noise(uint8_t v, double n, double sigma) {
  const double s = __dadd_rn(__dmul_rn(n, sigma), 0.0);  // ret * stddev + mean
  const long long r = llround(__dadd_rn((double)v, s));
  return (uint8_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
}

__global__ void __launch_bounds__(kNoiseThreads) noise_kernel(const FrameScene* __restrict__ scenes, int w, int h,
                                                              uint8_t* __restrict__ left, uint8_t* __restrict__ right,
                                                              int64_t frame_stride) {
  __shared__ uint64_t ring[kRing];
  __shared__ int warp_acc[2][kNoiseWarps];
  const FrameScene& fs = scenes[blockIdx.x];
  if (!(fs.sigma > 0)) return;
  const double sigma = fs.sigma;
  uint8_t* L = left + (int64_t)blockIdx.x * frame_stride;
  uint8_t* R = right + (int64_t)blockIdx.x * frame_stride;
  const int64_t npx = (int64_t)w * h, pairs = npx;  // 2 * npx normals = npx accepted pairs
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  if (tid == 0) {  // mersenne_twister_engine::seed
    uint64_t x = fs.seed;
    ring[0] = x;
    for (int i = 1; i < kMtN; ++i) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
      ring[i] = x;
    }
  }
  __syncthreads();

  int64_t done = 0;  // accepted pairs so far (uniform)
  for (int64_t j0 = kMtN, step = 0; done < pairs; j0 += kMtM, ++step) {
    bool accept = false;
    double u = 0.0;
    if (tid < kMtM) {
      const int64_t j = j0 + tid;
      const uint64_t a = ring[(j - kMtN) & (kRing - 1)], b = ring[(j - kMtN + 1) & (kRing - 1)];
      const uint64_t yv = (a & 0xFFFFFFFF80000000ull) | (b & 0x7FFFFFFFull);
      const uint64_t xj = ring[(j - kMtM) & (kRing - 1)] ^ (yv >> 1) ^ ((yv & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
      ring[j & (kRing - 1)] = xj;
      u = __dsub_rn(__dmul_rn(2.0, canonical(mt_temper(xj))), 1.0);
    }
    // draw d = j - 312; attempt (d, d + 1), d even -> (x, y) of the polar method
    const double px = u, py = __shfl_down_sync(0xffffffffu, u, 1);
    if (tid < kMtM && (tid & 1) == 0) {
      const double r2 = __dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py));
      accept = !(r2 > 1.0 || r2 == 0.0);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, accept);
    if (lane == 0) warp_acc[step & 1][wid] = __popc(bal);
    __syncthreads();  // ring writes and warp counts visible
    int before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kNoiseWarps; ++k) {
      const int c = warp_acc[step & 1][k];
      before += k < wid ? c : 0;
      total += c;
    }
    if (accept) {
      const int64_t p = done + before + __popc(bal & ((1u << lane) - 1u));
      if (p < pairs) {
        const double r2 = __dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py));
        const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
        const int64_t n0 = 2 * p;  // normal 2p = y * mult, normal 2p + 1 = x * mult
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t n = n0 + e;
          const double nv = __dmul_rn(e ? px : py, mult);
          uint8_t* img = n < npx ? L : R;
          const int64_t i = n < npx ? n : n - npx;
          img[i] = add_noise(img[i], nv, sigma);
        }
      }
    }
    done += total;
  }
}

}  // namespace

rg_status render_frames_device(rg_ctx* ctx, const rg_scene_config* cfgs, const rg_scene_object* objs,
                               const int32_t* obj_offsets, int n_frames, uint8_t* d_left, uint8_t* d_right,
                               int64_t frame_stride, cudaStream_t s) {
  const int w = cfgs[0].width, h = cfgs[0].height;
  if ((int64_t)w * h > frame_stride) return set_err(ctx, RG_EINVAL, "render_frames_device: frame_stride < w*h");
  std::vector<FrameScene> fs(static_cast<size_t>(n_frames));
  std::vector<RenderObj> all, one;
  for (int f = 0; f < n_frames; ++f) {
    const rg_scene_config& c = cfgs[f];
    if (c.width != w || c.height != h)
      return set_err(ctx, RG_EINVAL, "render_frames_device: every frame must share width and height");
    const int n = obj_offsets[f + 1] - obj_offsets[f];
    if (rg_synth::prepare_scene(c, objs + obj_offsets[f], n, one) != RG_OK)
      return set_err(ctx, RG_EINVAL, "render_frames_device: invalid scene");
    FrameScene& q = fs[f];
    q.bg_contrast = c.background_contrast;
    q.cell = c.texture_cell_px;
    q.bias = c.disparity_bias_px;
    q.sigma = c.noise_sigma;
    q.bg_seed = c.background_seed;
    q.seed = c.seed;
    q.quant = c.texture_quant;
    q.dy = c.vertical_offset_px;
    q.obj0 = (int32_t)all.size();
    q.n_obj = (int32_t)one.size();
    rg_synth::radiometric_lut(c, q.lut);
    all.insert(all.end(), one.begin(), one.end());
  }
  const size_t sb = sizeof(FrameScene) * fs.size(), ob = sizeof(RenderObj) * std::max<size_t>(all.size(), 1);
  uint8_t* d = static_cast<uint8_t*>(dev_buf(ctx, B_SYNTH, sb + ob));
  if (!d) return set_err(ctx, RG_ENOMEM, "render_frames_device: scratch");
  // scene tables staged through a pinned buffer (the previous call's copy
  // must have left it): the call returns with the kernels enqueued
  if (!ctx->ev_stage) RG_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_stage, cudaEventDisableTiming));
  RG_CUDA(ctx, cudaEventSynchronize(ctx->ev_stage));
  uint8_t* hb = static_cast<uint8_t*>(host_buf(ctx, 2, sb + ob));
  if (!hb) return set_err(ctx, RG_ENOMEM, "render_frames_device: pinned staging");
  memcpy(hb, fs.data(), sb);
  if (!all.empty()) memcpy(hb + sb, all.data(), sizeof(RenderObj) * all.size());
  RG_CUDA(ctx, cudaMemcpyAsync(d, hb, sb + ob, cudaMemcpyHostToDevice, s));
  RG_CUDA(ctx, cudaEventRecord(ctx->ev_stage, s));
  const FrameScene* dfs = reinterpret_cast<const FrameScene*>(d);
  const RenderObj* dob = reinterpret_cast<const RenderObj*>(d + sb);
  dim3 grid((w + kBodyTx - 1) / kBodyTx, h, n_frames);
  render_body_kernel<<<grid, kBodyTx, 0, s>>>(dfs, dob, w, h, d_left, d_right, frame_stride);
  RG_CUDA(ctx, cudaGetLastError());
  noise_kernel<<<n_frames, kNoiseThreads, 0, s>>>(dfs, w, h, d_left, d_right, frame_stride);
  RG_CUDA(ctx, cudaGetLastError());
  count_launch(ctx, 4, 2);
  return RG_OK;
}

}  // namespace rg

using namespace rg;

extern "C" rg_status rg_render_frames_device(rg_ctx* ctx, const rg_scene_config* cfgs, const rg_scene_object* objs,
                                             const int32_t* obj_offsets, int n_frames, uint8_t* d_left,
                                             uint8_t* d_right, int64_t frame_stride, void* stream) {
  RG_NVTX("rg_render_frames_device");
  if (!ctx) return RG_EINVAL;
  if (!cfgs || !obj_offsets || !d_left || !d_right || n_frames < 1 || frame_stride < 1)
    return set_err(ctx, RG_EINVAL, "render_frames_device: bad arguments");
  const cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_err(ctx, e, "cudaSetDevice");
  if (const rg_status w = wait_async(ctx)) return w;
  for (int f = 0; f < n_frames; ++f)
    if (obj_offsets[f + 1] < obj_offsets[f] || (obj_offsets[f + 1] > obj_offsets[f] && !objs))
      return set_err(ctx, RG_EINVAL, "render_frames_device: bad object offsets");
  const rg_status st = render_frames_device(ctx, cfgs, objs, obj_offsets, n_frames, d_left, d_right, frame_stride,
                                            stream ? static_cast<cudaStream_t>(stream) : ctx->stream);
  if (st == RG_OK && !stream) RG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // NULL stream: blocking call
  return st;
}
