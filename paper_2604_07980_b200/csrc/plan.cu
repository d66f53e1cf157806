// plan.cu -- K3 (object selection / work planning) and K4 (aggregation +
// range) of the batched object ranger, plus the single-shot kernels behind
// the reference's helper functions (select_objects, find_occluders,
// sample_query_points, aggregate_close_disparities).
//
// K3, one CTA per frame (template_match.hpp:277-310): priority rank of every
// detection (select_objects :94-114, as an O(n^2) rank count so the CTA
// needs no sort), selected set in input order, FAR/CLOSE classification
// (:63-67), and one "slot" per potential QueryBlock -- FAR objects get one,
// CLOSE objects rows x cols (:192-197).  Slots are appended to a global list
// with one atomic per object; the list order does not matter because results
// are addressed by slot and each object keeps its slot range.
//
// K4, one CTA per selected object (template_match.hpp:332-361): FAR takes its
// single verified block, CLOSE sorts the verified sub-block disparities
// (x close_scale, :353) and keeps the longest tight run (:126-148); the range
// z = f / ((1/b) d) is the canonical reprojection (geometry.hpp:124-146).
#include <cstdlib>

#include "rg_common.cuh"
#include "rg_device.cuh"

namespace rg {
namespace {

constexpr int PT = 256;
constexpr int kMaxDetsPerFrame = 4096;
constexpr int kKeyCap = 1024;  // detections per frame ranked from shared-memory keys

__global__ void __launch_bounds__(PT) plan_frames_kernel(
    const rg_detection* __restrict__ dets, const int32_t* __restrict__ det_off, int w, int h,
    rg_ranger_config cfg, int out_stride, ObjEntry* __restrict__ objs,
    rg_object_disparity* __restrict__ out, int32_t* __restrict__ out_count,
    Slot* __restrict__ slots, int slot_capacity, int32_t* __restrict__ counters,
    rg_ranger_stats* __restrict__ stats, int32_t* __restrict__ out_index) {
  __shared__ unsigned char sel[kMaxDetsPerFrame];
  __shared__ int warp_tot[PT / 32];
  __shared__ int warp_sf[PT / 32], warp_sc[PT / 32], chunk_base[2];
  __shared__ double s_key[kKeyCap];
  __shared__ int s_id[kKeyCap];
  __shared__ bool s_front[kKeyCap];
  const int f = blockIdx.x;
  const int d0 = det_off[f], n = det_off[f + 1] - d0;
  const rg_detection* D = dets + d0;
  // rank of every detection in the priority order; selected iff rank < budget
  if (n <= kKeyCap) {
    // dev_precedes on precomputed keys: frontal flag, then area (frontal) or
    // box bottom (else), then id, then index -- the same doubles, so the same
    // order, without re-deriving both keys for every pair
    for (int i = threadIdx.x; i < n; i += PT) {
      const rg_detection d = D[i];
      const bool f = dev_frontal(d, cfg);
      s_front[i] = f;
      s_key[i] = f ? __dmul_rn(d.w, d.h) : __dadd_rn(d.cy, half_of(d.h));
      s_id[i] = d.id;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += PT) {
      const bool fi = s_front[i];
      const double ki = s_key[i];
      const int idi = s_id[i];
      int rank = 0;
#pragma unroll 8
      for (int j = 0; j < n; ++j) {  // no early exit: independent iterations overlap their smem loads
        const bool fj = s_front[j];
        const double kj = s_key[j];
        const bool prec = fj != fi ? fj : kj != ki ? kj > ki : s_id[j] != idi ? s_id[j] < idi : j < i;
        rank += (j != i && prec) ? 1 : 0;
      }
      sel[i] = rank < cfg.max_objects;
    }
  } else {
    for (int i = threadIdx.x; i < n; i += PT) {
      const rg_detection di = D[i];
      int rank = 0;
      for (int j = 0; j < n && rank < cfg.max_objects; ++j)
        if (j != i && dev_precedes(D[j], j, di, i, cfg)) ++rank;
      sel[i] = rank < cfg.max_objects;
    }
  }
  __syncthreads();
  // selected objects in input order: block-wide exclusive scan over chunks
  int base_k = 0, n_far = 0, n_close = 0;
  for (int c0 = 0; c0 < n; c0 += PT) {
    const int i = c0 + threadIdx.x;
    const int flag = (i < n) ? sel[i] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int q = 0; q < PT / 32; ++q) {
      if (q < wid) before += warp_tot[q];
      total += warp_tot[q];
    }
    // kind and sub-block grid of this thread's object, then one block-wide
    // exclusive scan of the slot counts per kind and ONE atomic per kind and
    // chunk (per-object atomics on the same two counters serialised the
    // planner: 23 -> ~10 us for one C2 frame)
    int kind = RG_KIND_FAR, rows = 1, cols = 1;
    rg_detection di{};
    if (flag) {
      di = D[i];
      kind = dev_classify(di, w, h, cfg.tau_s);
      if (kind == RG_KIND_CLOSE) dev_close_grid(pixel_box(di, w, h), cfg, &rows, &cols);
    }
    const int ns = flag ? rows * cols : 0;
    int incf = kind == RG_KIND_FAR ? ns : 0, incc = kind == RG_KIND_CLOSE ? ns : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int uf = __shfl_up_sync(0xffffffffu, incf, o), uc = __shfl_up_sync(0xffffffffu, incc, o);
      if (lane >= o) incf += uf, incc += uc;
    }
    if (lane == 31) warp_sf[wid] = incf, warp_sc[wid] = incc;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tf = 0, tc = 0;
      for (int q = 0; q < PT / 32; ++q) tf += warp_sf[q], tc += warp_sc[q];
      // FAR blocks fill the slot list from the bottom, CLOSE sub-blocks from
      // the top: the matcher's CTAs then hold slots of one kind, whose costs
      // are alike (a FAR block is ~5x a CLOSE sub-block at C2), instead of a
      // few FAR warps holding a whole CTA of finished CLOSE warps; the
      // heavier FAR CTAs are also dispatched first (shorter tail)
      chunk_base[0] = tf ? atomicAdd(&counters[0], tf) : 0;
      chunk_base[1] = tc ? atomicAdd(&counters[4], tc) : 0;
    }
    __syncthreads();
    if (flag) {
      const int k = base_k + before + __popc(bal & ((1u << lane) - 1u));
      int pf = 0, pc = 0;
      for (int q = 0; q < wid; ++q) pf += warp_sf[q], pc += warp_sc[q];
      const int sb = kind == RG_KIND_FAR ? chunk_base[0] + pf + incf - ns
                                         : slot_capacity - (chunk_base[1] + pc + incc);
      ObjEntry e;
      e.det = d0 + i;
      e.kind = kind;
      e.slot_base = sb;
      e.n_slots = ns;
      e.rows = rows;
      e.cols = cols;
      e.frame = f;
      const int g = f * out_stride + k;
      e.occ_n = -1;  // occluders_kernel lists them (else the matcher scans per slot)
      objs[g] = e;
      rg_object_disparity od;
      od.det_id = di.id;
      od.kind = kind;
      od.n_blocks_used = 0;
      od.valid = 0;
      od.disparity = 0.0;
      od.z_cam = 0.0;
      out[g] = od;
      if (out_index) out_index[g] = i;
      if (sb < 0 || sb + ns > slot_capacity) {
        counters[1] = 1;  // overflow: the host grows the list and re-runs
      } else {
        // pad = sub-block row << 16 | column (the matcher skips the division)
        const int cq = max(cols, 1);
        for (int t = 0, r = 0, c = 0; t < ns; ++t) {
          slots[sb + t] = Slot{f, g, t, (r << 16) | c};
          if (++c == cq) c = 0, ++r;
        }
      }
      if (kind == RG_KIND_FAR)
        ++n_far;
      else
        ++n_close;
    }
    base_k += total;
    __syncthreads();
  }
  // per-frame counters
  for (int o = 16; o > 0; o >>= 1) {
    n_far += __shfl_xor_sync(0xffffffffu, n_far, o);
    n_close += __shfl_xor_sync(0xffffffffu, n_close, o);
  }
  __shared__ int tf[PT / 32], tc[PT / 32];
  if ((threadIdx.x & 31) == 0) {
    tf[threadIdx.x >> 5] = n_far;
    tc[threadIdx.x >> 5] = n_close;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, b = 0;
    for (int q = 0; q < PT / 32; ++q) {
      a += tf[q];
      b += tc[q];
    }
    out_count[f] = base_k;
    if (stats) {
      stats[f].query_points = 0;
      stats[f].image_pixels = (int64_t)w * h;
      stats[f].n_far = a;
      stats[f].n_close = b;
    }
  }
}

// Occluders of every selected object among its frame's detections
// (find_occluders, template_match.hpp:71-89), once per object instead of once
// per slot: a warp per object (grid over frames x objects, after K3), lanes
// over the detections, frame-local indices in detection order; more than
// kOccMax -> occ_n = -1 (the matcher then scans every detection itself).
constexpr int OC_WARPS = 8;
__global__ void __launch_bounds__(OC_WARPS * 32) occluders_kernel(
    const rg_detection* __restrict__ dets, const int32_t* __restrict__ det_off, int out_stride,
    const int32_t* __restrict__ out_count, ObjEntry* __restrict__ objs, int16_t* __restrict__ occ_list) {
  const int f = blockIdx.y, k = blockIdx.x * OC_WARPS + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= out_count[f]) return;  // warp-uniform
  const int d0 = det_off[f], n = det_off[f + 1] - d0;
  const int g = f * out_stride + k;
  const int self = objs[g].det - d0;
  const rg_detection di = dets[d0 + self];
  int16_t* ol = occ_list + (int64_t)g * kOccMax;
  int no = 0;
  for (int j0 = 0; j0 < n && no <= kOccMax; j0 += 32) {
    const int j = j0 + lane;
    const bool occl = j < n && j != self && dev_occludes(di, dets[d0 + j]);
    const unsigned bal = __ballot_sync(0xffffffffu, occl);
    const int pos = no + __popc(bal & ((1u << lane) - 1u));
    if (occl && pos < kOccMax) ol[pos] = (int16_t)j;
    no += __popc(bal);
  }
  if (lane == 0) objs[g].occ_n = no <= kOccMax ? no : -1;
}

__global__ void __launch_bounds__(128) aggregate_kernel(
    const ObjEntry* __restrict__ objs, const int32_t* __restrict__ out_count, int out_stride,
    const rg_match_result* __restrict__ res, int slot_capacity, rg_ranger_config cfg,
    double focal, double baseline, double* __restrict__ scratch,
    rg_object_disparity* __restrict__ out, const int32_t* __restrict__ counters) {
  __shared__ double vals[kAggCapacity];
  __shared__ int cnt;
  const int g = blockIdx.x;
  const int f = g / out_stride, k = g - f * out_stride;
  if (k >= out_count[f]) return;
  if (counters[1]) return;  // overflowed plan: the host re-runs the batch
  const ObjEntry e = objs[g];
  if (e.slot_base + e.n_slots > slot_capacity) return;  // overflowed batch, re-run follows
  int valid = 0, used = 0;
  double disp = 0.0;
  if (e.kind == RG_KIND_FAR) {
    // template_match.hpp:338-347: the single FAR block, verified or invalid
    const rg_match_result r = res[e.slot_base];
    if (r.n_points >= 4 && r.has_value && r.verified) {
      valid = 1;
      disp = r.dx_subpix;
      used = 1;
    }
  } else {
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const bool big = e.n_slots > kAggCapacity;
    double* dst = big ? scratch + e.slot_base : vals;
    for (int t = threadIdx.x; t < e.n_slots; t += blockDim.x) {
      const rg_match_result r = res[e.slot_base + t];
      if (r.n_points >= 4 && r.has_value && r.verified)
        dst[atomicAdd(&cnt, 1)] = __dmul_rn(r.dx_subpix, (double)cfg.close_scale);
    }
    __syncthreads();
    const int m = cnt;
    if (!big) {
      dev_bitonic_sort(vals, m);
    } else {
      // more CLOSE blocks than fit in smem: values sit in this object's
      // scratch region [slot_base, +n_slots); rank-sort them into the mirror
      // region at +slot_capacity (scratch holds 2 * slot_capacity doubles)
      dev_rank_sort(dst, m, scratch + slot_capacity + e.slot_base);
      dst = scratch + slot_capacity + e.slot_base;
    }
    if (threadIdx.x == 0) dev_runs(big ? dst : vals, m, cfg.tau_d, cfg.n_min, &valid, &disp, &used);
  }
  if (threadIdx.x == 0) {
    rg_object_disparity od = out[g];
    od.valid = valid;
    od.disparity = disp;
    od.n_blocks_used = used;
    od.z_cam = 0.0;
    if (valid && disp > 0 && focal > 0 && baseline > 0)
      od.z_cam = __ddiv_rn(focal, __dmul_rn(__ddiv_rn(1.0, baseline), disp));
    out[g] = od;
  }
}

// ---------------------------------------------------------------- helpers
__global__ void select_objects_kernel(const rg_detection* __restrict__ dets, int n,
                                      rg_ranger_config cfg, int32_t* __restrict__ out_idx,
                                      int32_t* __restrict__ n_out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < n; ++j)
      if (j != i && dev_precedes(dets[j], j, dets[i], i, cfg)) ++rank;
    if (rank < cfg.max_objects) out_idx[rank] = i;
  }
  if (threadIdx.x == 0) *n_out = n < cfg.max_objects ? n : cfg.max_objects;
}

__global__ void find_occluders_kernel(const rg_detection* __restrict__ dets, int n,
                                      int32_t* __restrict__ counts, int32_t* __restrict__ lists) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  for (int j = 0; j < n; ++j)
    if (j != i && dev_occludes(dets[i], dets[j])) lists[(int64_t)i * n + c++] = j;
  counts[i] = c;
}

__global__ void sample_blocks_kernel(const rg_detection* __restrict__ det, int kind,
                                     const double* __restrict__ occ, int n_occ, rg_ranger_config cfg,
                                     int w, int h, int rows, int cols, int32_t* __restrict__ pts,
                                     int32_t* __restrict__ counts, int per_block) {
  extern __shared__ double occ_s[];
  for (int i = threadIdx.x; i < 4 * n_occ; i += blockDim.x) occ_s[i] = occ[i];
  __syncthreads();
  const int b = blockIdx.x;
  int2* out = reinterpret_cast<int2*>(pts) + (int64_t)b * per_block;
  const int np = dev_sample_block(*det, kind, b / cols, b % cols, rows, cols, occ_s, n_occ,
                                  nullptr, 0, -1, cfg, w, h, out);
  if (threadIdx.x == 0) counts[b] = np;
}

__global__ void aggregate_values_kernel(const double* __restrict__ v, int n, double tau_d,
                                        int n_min, double* __restrict__ scratch,
                                        int32_t* __restrict__ out_i, double* __restrict__ out_d) {
  __shared__ double vals[kAggCapacity];
  const bool big = n > kAggCapacity;
  if (!big) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) vals[i] = v[i];
    __syncthreads();
    dev_bitonic_sort(vals, n);
  } else {
    dev_rank_sort(v, n, scratch);
  }
  if (threadIdx.x == 0) {
    int valid, len;
    double d;
    dev_runs(big ? scratch : vals, n, tau_d, n_min, &valid, &d, &len);
    out_i[0] = valid;
    out_i[1] = len;
    out_d[0] = d;
  }
}

// K4, warp per object (the default): FAR reads its one block; CLOSE
// gathers its verified sub-block disparities (x close_scale) into a per-warp
// shared-memory array of up to 64 (ballot compaction), sorts them with a
// warp bitonic network (two elements per lane) and lane 0 runs the
// longest-run scan (template_match.hpp:116-148).  Objects with more than 64
// CLOSE blocks use the global scratch and a warp rank sort.  One launch of
// F * out_stride warps instead of as many 128-thread CTAs.
constexpr int kAggWarps = 8, kAggWarpCap = 64;
__global__ void __launch_bounds__(kAggWarps * 32) aggregate_warp_kernel(
    const ObjEntry* __restrict__ objs, const int32_t* __restrict__ out_count, int out_stride, int n_obj,
    const rg_match_result* __restrict__ res, int slot_capacity, rg_ranger_config cfg, double focal,
    double baseline, double* __restrict__ scratch, rg_object_disparity* __restrict__ out,
    const int32_t* __restrict__ counters) {
  __shared__ double vals[kAggWarps][kAggWarpCap];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = blockIdx.x * kAggWarps + wid;
  if (g >= n_obj) return;
  const int f = g / out_stride, k = g - f * out_stride;
  if (k >= out_count[f] || counters[1]) return;  // no object / overflowed plan (re-run follows)
  const ObjEntry e = objs[g];
  if (e.slot_base + e.n_slots > slot_capacity) return;
  int valid = 0, used = 0;
  double disp = 0.0;
  if (e.kind == RG_KIND_FAR) {
    if (lane == 0) {  // template_match.hpp:338-347: the single FAR block, verified or invalid
      const rg_match_result r = res[e.slot_base];
      if (r.n_points >= 4 && r.has_value && r.verified) valid = 1, disp = r.dx_subpix, used = 1;
    }
  } else if (e.n_slots <= 32) {
    // up to 32 sub-blocks (every CLOSE object at C2): one value per lane,
    // bitonic sort by shuffles, runs by ballots -- aggregate_close_disparities
    // (template_match.hpp:126-148) without shared memory or a serial scan
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    double x = inf;
    bool ok = false;
    if (lane < e.n_slots) {
      const rg_match_result r = res[e.slot_base + lane];
      ok = r.n_points >= 4 && r.has_value && r.verified;
      if (ok) x = __dmul_rn(r.dx_subpix, (double)cfg.close_scale);  // template_match.hpp:353
    }
    const int m = __popc(__ballot_sync(0xffffffffu, ok));
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, x, j);
        const bool keep_min = ((lane & j) == 0) == ((lane & kk) == 0);
        x = keep_min ? (y < x ? y : x) : (x < y ? y : x);
      }
    // runs of the ascending values: a new run where v[i] - v[i-1] >= tau_d
    // (dev_runs); the longest wins, ties to the later run
    const double xp = __shfl_up_sync(0xffffffffu, x, 1);
    const bool start = lane < m && (lane == 0 || __dsub_rn(x, xp) >= cfg.tau_d);
    const unsigned sm = __ballot_sync(0xffffffffu, start);
    unsigned key = 0;
    if (start) {
      const unsigned later = sm & ~((2u << lane) - 1u);
      const int next = later ? __ffs(later) - 1 : m;
      key = ((unsigned)(next - lane) << 8) | (unsigned)lane;
    }
    key = __reduce_max_sync(0xffffffffu, key);
    const int blen = (int)(key >> 8), bstart = (int)(key & 0xFFu);
    const double med = __shfl_sync(0xffffffffu, x, (bstart + blen / 2) & 31);
    if (m > 0 && blen >= cfg.n_min) valid = 1, disp = med, used = blen;
  } else {
    const bool big = e.n_slots > kAggWarpCap;
    double* dst = big ? scratch + e.slot_base : vals[wid];
    int m = 0;
    for (int t0 = 0; t0 < e.n_slots; t0 += 32) {
      const int t = t0 + lane;
      bool ok = false;
      double v = 0.0;
      if (t < e.n_slots) {
        const rg_match_result r = res[e.slot_base + t];
        ok = r.n_points >= 4 && r.has_value && r.verified;
        v = __dmul_rn(r.dx_subpix, (double)cfg.close_scale);  // template_match.hpp:353
      }
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      if (ok) dst[m + __popc(bal & ((1u << lane) - 1u))] = v;
      m += __popc(bal);
    }
    __syncwarp();
    if (!big) {  // bitonic sort of 64 (padded with +inf), two elements per lane
      const double inf = __longlong_as_double(0x7ff0000000000000LL);
      for (int i = m + lane; i < kAggWarpCap; i += 32) dst[i] = inf;
      __syncwarp();
      for (int kk = 2; kk <= kAggWarpCap; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
          // compare-exchange pair p of 32: (i, i ^ j) with i the lower index
          const int i = ((lane & ~(j - 1)) << 1) | (lane & (j - 1));
          const int q = i ^ j;
          const bool up = (i & kk) == 0;
          const double a = dst[i], b = dst[q];
          __syncwarp();
          if ((a > b) == up) dst[i] = b, dst[q] = a;
          __syncwarp();
        }
    } else {  // rank sort into the mirror region (scratch holds 2 * slot_capacity doubles)
      double* o = scratch + slot_capacity + e.slot_base;
      for (int i = lane; i < m; i += 32) {
        const double x = dst[i];
        int rank = 0;
        for (int q = 0; q < m; ++q) rank += (dst[q] < x) || (dst[q] == x && q < i);
        o[rank] = x;
      }
      __syncwarp();
      dst = o;
    }
    if (lane == 0) dev_runs(dst, m, cfg.tau_d, cfg.n_min, &valid, &disp, &used);
  }
  if (lane == 0) {
    rg_object_disparity od = out[g];
    od.valid = valid;
    od.disparity = disp;
    od.n_blocks_used = used;
    od.z_cam = 0.0;
    if (valid && disp > 0 && focal > 0 && baseline > 0)
      od.z_cam = __ddiv_rn(focal, __dmul_rn(__ddiv_rn(1.0, baseline), disp));
    out[g] = od;
  }
}

}  // namespace

cudaError_t launch_plan_frames(const rg_detection* dets, const int32_t* det_off, int n_frames, int w,
                               int h, rg_ranger_config cfg, int out_stride, ObjEntry* objs,
                               rg_object_disparity* out, int32_t* out_count, Slot* slots,
                               int slot_capacity, int32_t* counters, rg_ranger_stats* stats,
                               int32_t* out_index, int16_t* occ_list, bool list_occluders, cudaStream_t s) {
  if (n_frames <= 0) return cudaSuccess;
  plan_frames_kernel<<<n_frames, PT, 0, s>>>(dets, det_off, w, h, cfg, out_stride, objs, out,
                                             out_count, slots, slot_capacity, counters, stats, out_index);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || out_stride <= 0 || !list_occluders) return e;
  occluders_kernel<<<dim3((out_stride + OC_WARPS - 1) / OC_WARPS, n_frames), OC_WARPS * 32, 0, s>>>(
      dets, det_off, out_stride, out_count, objs, occ_list);
  return cudaGetLastError();
}

cudaError_t launch_aggregate(const ObjEntry* objs, const int32_t* out_count, int n_frames,
                             int out_stride, const rg_match_result* res, int slot_capacity,
                             rg_ranger_config cfg, double focal, double baseline, double* scratch,
                             rg_object_disparity* out, const int32_t* counters, cudaStream_t s) {
  if (n_frames <= 0 || out_stride <= 0) return cudaSuccess;
  static const bool cta = getenv("RG_AGG_CTA") != nullptr;  // A/B knob: the CTA-per-object kernel
  const int n_obj = n_frames * out_stride;
  if (!cta) {
    aggregate_warp_kernel<<<(n_obj + kAggWarps - 1) / kAggWarps, kAggWarps * 32, 0, s>>>(
        objs, out_count, out_stride, n_obj, res, slot_capacity, cfg, focal, baseline, scratch, out, counters);
    return cudaGetLastError();
  }
  aggregate_kernel<<<n_obj, 128, 0, s>>>(objs, out_count, out_stride, res, slot_capacity, cfg, focal, baseline,
                                         scratch, out, counters);
  return cudaGetLastError();
}

cudaError_t launch_select_objects(const rg_detection* dets, int n, rg_ranger_config cfg,
                                  int32_t* out_idx, int32_t* n_out, cudaStream_t s) {
  select_objects_kernel<<<1, 256, 0, s>>>(dets, n, cfg, out_idx, n_out);
  return cudaGetLastError();
}

cudaError_t launch_find_occluders(const rg_detection* dets, int n, int32_t* counts, int32_t* lists,
                                  cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  find_occluders_kernel<<<(n + 127) / 128, 128, 0, s>>>(dets, n, counts, lists);
  return cudaGetLastError();
}

cudaError_t launch_sample_blocks(const rg_detection* det, int kind, const double* occ, int n_occ,
                                 rg_ranger_config cfg, int w, int h, int rows, int cols,
                                 int32_t* pts, int32_t* counts, int per_block, cudaStream_t s) {
  const size_t smem = sizeof(double) * 4 * (size_t)(n_occ > 0 ? n_occ : 1);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sample_blocks_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  sample_blocks_kernel<<<rows * cols, 128, smem, s>>>(det, kind, occ, n_occ, cfg, w, h, rows, cols,
                                                      pts, counts, per_block);
  return cudaGetLastError();
}

cudaError_t launch_aggregate_values(const double* v, int n, double tau_d, int n_min,
                                    double* scratch, int32_t* out_i, double* out_d,
                                    cudaStream_t s) {
  aggregate_values_kernel<<<1, 256, 0, s>>>(v, n, tau_d, n_min, scratch, out_i, out_d);
  return cudaGetLastError();
}

}  // namespace rg
