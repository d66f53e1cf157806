// dense.cu -- per-box statistics of a dense disparity map (SURVEY.md 8(f)
// row 3: the STEREO_BM primary method feeding Pipeline::box_disparity,
// pipeline.hpp:304-328).
//
// One CTA per box: the box's valid raw values (int16, 1/16 px) go into a
// shared-memory histogram; a block scan over the bins gives the median (rank
// (n-1)/2 of the sorted samples), the near subset (ranks >= 3(n-1)/4) and the
// sums that dynamic_disparity_variance (geometry.hpp:162-178) needs.  Every
// sample is raw/16, so all partial sums are exact dyadic rationals: the means
// equal the reference's std::accumulate for any summation order, and the FP64
// tail runs in the reference's operation order.
#include <cmath>

#include "rg_common.cuh"

namespace rg {
namespace {

constexpr int kBoxThreads = 256;
constexpr int kInvalidRaw = -32768;

__global__ void __launch_bounds__(kBoxThreads) box_disparity_kernel(
    const int16_t* __restrict__ raw, int w, int h, int64_t frame_stride, const rg_detection* __restrict__ dets,
    const int32_t* __restrict__ box_det, const int32_t* __restrict__ box_frame, int raw_lo, int nbins,
    double sigma_obs2, double gamma, double sigma_sys2, rg_box_stats* __restrict__ out) {
  extern __shared__ int hist[];
  __shared__ long long s_cnt[kBoxThreads], s_sum[kBoxThreads];
  __shared__ int bad;
  const int b = blockIdx.x, tid = threadIdx.x;
  const rg_detection d = dets[box_det[b]];
  const int16_t* m = raw + (box_frame ? (int64_t)box_frame[b] * frame_stride : 0);
  // pipeline.hpp:308-313 with to_pixel_box, detection.hpp:23-30
  const double bx0 = __dmul_rn(__dsub_rn(d.cx, __ddiv_rn(d.w, 2.0)), (double)w);
  const double bx1 = __dmul_rn(__dadd_rn(d.cx, __ddiv_rn(d.w, 2.0)), (double)w);
  const double by0 = __dmul_rn(__dsub_rn(d.cy, __ddiv_rn(d.h, 2.0)), (double)h);
  const double by1 = __dmul_rn(__dadd_rn(d.cy, __ddiv_rn(d.h, 2.0)), (double)h);
  const int y0 = max(0, (int)floor(by0)), y1 = min(h, (int)ceil(by1));
  const int x0 = max(0, (int)floor(bx0)), x1 = min(w, (int)ceil(bx1));
  for (int i = tid; i < nbins; i += kBoxThreads) hist[i] = 0;
  if (tid == 0) bad = 0;
  __syncthreads();
  const int bw = max(0, x1 - x0), bh = max(0, y1 - y0);
  for (int k = tid; k < bw * bh; k += kBoxThreads) {
    const int y = y0 + k / bw, x = x0 + k % bw;
    const int v = m[(int64_t)y * w + x];
    if (v == kInvalidRaw) continue;  // DisparityMap::valid, image.hpp:66
    const int bi = v - raw_lo;
    if (bi < 0 || bi >= nbins) {
      bad = 1;
      continue;
    }
    atomicAdd(&hist[bi], 1);
  }
  __syncthreads();
  // per-thread contiguous chunk of bins: count and raw sum
  const int per = (nbins + kBoxThreads - 1) / kBoxThreads;
  const int b0 = tid * per, b1 = min(nbins, b0 + per);
  long long c = 0, sm = 0;
  for (int i = b0; i < b1; ++i) {
    c += hist[i];
    sm += (long long)hist[i] * (raw_lo + i);
  }
  s_cnt[tid] = c;
  s_sum[tid] = sm;
  __syncthreads();
  if (tid == 0) {
    rg_box_stats r{};
    long long n = 0, sum_all = 0;
    for (int t = 0; t < kBoxThreads; ++t) {
      n += s_cnt[t];
      sum_all += s_sum[t];
    }
    r.count = (int)n;
    if (bad) {
      r.valid = -1;  // a raw value outside [raw_lo, raw_lo + nbins): caller error
    } else if (n > 0) {
      // rank -> value over the chunks, then the bins of one chunk
      auto value_at = [&](long long rank, long long* below_sum) {
        long long acc = 0, accs = 0;
        for (int t = 0; t < kBoxThreads; ++t) {
          if (acc + s_cnt[t] > rank) {
            const int c0 = t * per, c1 = min(nbins, c0 + per);
            for (int i = c0; i < c1; ++i) {
              const long long hc = hist[i];
              const int v = raw_lo + i;
              if (acc + hc > rank) {
                *below_sum = accs + (rank - acc) * (long long)v;  // sum of the samples of rank < `rank`
                return v;
              }
              acc += hc;
              accs += hc * v;
            }
          }
          acc += s_cnt[t];
          accs += s_sum[t];
        }
        *below_sum = accs;
        return raw_lo;
      };
      long long unused = 0, below = 0;
      const int med = value_at((n - 1) / 2, &unused);
      const long long near_from = (3 * (n - 1)) / 4;  // pipeline.hpp:319
      value_at(near_from, &below);
      const long long n_near = n - near_from;
      const long long near_sum = sum_all - below;
      // geometry.hpp:168-177: accumulate(samples) / size; raw/16 sums are exact
      const double mean_near = __ddiv_rn((double)near_sum / 16.0, (double)n_near);
      const double mean_all = __ddiv_rn((double)sum_all / 16.0, (double)n);
      const double diff = __dsub_rn(mean_near, mean_all);
      r.variance = __dadd_rn(__dadd_rn(__ddiv_rn(sigma_obs2, (double)n_near), __dmul_rn(__dmul_rn(gamma, diff), diff)),
                             sigma_sys2);
      r.median = (double)med / 16.0;  // DisparityMap::disparity, image.hpp:67
      r.valid = 1;
    }
    out[b] = r;
  }
}

// radar_refine_step's vote search (radar_refiner.hpp:117-131): per radar
// detection, the valid map pixel of its projected extent box whose offset
// d_radar - disparity is closest to zero (ties: the smaller offset).  The key
// (|off|, off) is a total order, so the block reduction is order-free; the
// offsets are exact FP64 (raw / 16 is exact).
constexpr int kVoteThreads = 256;
__global__ void __launch_bounds__(kVoteThreads) radar_vote_kernel(const int16_t* __restrict__ raw, int w,
                                                                 const int32_t* __restrict__ boxes,
                                                                 const double* __restrict__ d_radar,
                                                                 double* __restrict__ best_off,
                                                                 int32_t* __restrict__ found) {
  __shared__ double s_off[kVoteThreads];
  __shared__ int s_ok[kVoteThreads];
  const int b = blockIdx.x;
  const int x0 = boxes[4 * b], y0 = boxes[4 * b + 1], x1 = boxes[4 * b + 2], y1 = boxes[4 * b + 3];
  const double dr = d_radar[b];
  const int bw = x1 - x0 + 1, n = bw * (y1 - y0 + 1);
  double best = 0.0;
  int ok = 0;
  for (int i = threadIdx.x; i < n; i += kVoteThreads) {
    const int y = y0 + i / bw, x = x0 + i % bw;
    const int r = raw[(int64_t)y * w + x];
    if (r == kInvalidRaw) continue;
    const double off = __dsub_rn(dr, __dmul_rn((double)r, 0.0625));  // raw / 16.0 (DisparityMap::disparity)
    if (!ok || fabs(off) < fabs(best) || (fabs(off) == fabs(best) && off < best)) best = off, ok = 1;
  }
  s_off[threadIdx.x] = best;
  s_ok[threadIdx.x] = ok;
  __syncthreads();
  for (int st = kVoteThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      const double a = s_off[threadIdx.x], c = s_off[threadIdx.x + st];
      const int oa = s_ok[threadIdx.x], oc = s_ok[threadIdx.x + st];
      if (oc && (!oa || fabs(c) < fabs(a) || (fabs(c) == fabs(a) && c < a))) {
        s_off[threadIdx.x] = c;
        s_ok[threadIdx.x] = 1;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    best_off[b] = s_off[0];
    found[b] = s_ok[0];
  }
}

// radar_refine_step's map update (radar_refiner.hpp:157-165): every valid raw
// value + raw_off, clamped to [INT16_MIN + 1, INT16_MAX].
__global__ void raw_offset_kernel(int16_t* __restrict__ raw, int64_t n, int raw_off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = raw[i];
    if (r == kInvalidRaw) continue;
    raw[i] = (int16_t)min(max(r + raw_off, -32767), 32767);
  }
}

}  // namespace

cudaError_t launch_radar_votes(const int16_t* raw, int w, const int32_t* boxes, const double* d_radar, int n,
                               double* best_off, int32_t* found, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  radar_vote_kernel<<<n, kVoteThreads, 0, s>>>(raw, w, boxes, d_radar, best_off, found);
  return cudaGetLastError();
}

cudaError_t launch_raw_offset(int16_t* raw, int64_t n, int raw_off, cudaStream_t s) {
  if (n <= 0 || raw_off == 0) return cudaSuccess;
  raw_offset_kernel<<<592, 256, 0, s>>>(raw, n, raw_off);
  return cudaGetLastError();
}

cudaError_t launch_box_disparity(const int16_t* raw, int w, int h, int64_t frame_stride, const rg_detection* dets,
                                 const int32_t* box_det, const int32_t* box_frame, int n_boxes, int raw_lo,
                                 int nbins, double sigma_obs2, double gamma, double sigma_sys2,
                                 rg_box_stats* out, cudaStream_t s) {
  if (n_boxes <= 0) return cudaSuccess;
  const size_t smem = sizeof(int) * (size_t)nbins;
  static SmemAttr attr;
  if (smem > 48 * 1024) {
    const cudaError_t e = attr.ensure((const void*)box_disparity_kernel, smem);
    if (e != cudaSuccess) return e;
  }
  box_disparity_kernel<<<n_boxes, kBoxThreads, smem, s>>>(raw, w, h, frame_stride, dets, box_det, box_frame, raw_lo,
                                                         nbins, sigma_obs2, gamma, sigma_sys2, out);
  return cudaGetLastError();
}

}  // namespace rg
