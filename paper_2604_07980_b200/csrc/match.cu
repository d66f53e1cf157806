// match.cu -- K2: per-block census template matcher on sm_100a.
//
// Replaces block_match / forward_backward_match / batch_match (reference
// census.hpp:178-315) for arbitrary caller-supplied blocks and rasters (the
// C-ABI rg_match_blocks path; the fused planner path lives in
// match_warp.cu).  One CTA (256 threads) per QueryBlock:
//   2. keep points with a defined left descriptor (census.hpp:195-201).
//   3. stage the right-census window the block can reach into shared memory
//      (zero outside the raster -> "undefined", exactly like the reference's
//      inside() && code != 0 test), then sweep all (dx, dy) candidates with
//      XOR + POPC, lanes over consecutive dx so window reads are
//      conflict-free; a window without zero codes takes the branch-free path
//      where every point contributes (n = #valid points).
//   4. exact argmin of (sum/n, |dx|, dy, dx) by rational cross-multiplication
//      (equivalent to the reference's double compare for these magnitudes,
//      SURVEY.md Appendix A.3), warp-shuffle + smem reduction.
//   5. FP64 mean, neighbour costs and the parabolic sub-pixel step in the
//      reference's operation order (-fmad=false).
//   6. backward pass over ALL points shifted by (-dx_f, +dy_f), searching the
//      left raster over the negated dx range with dy pinned (census.hpp:288-301).
#include <climits>

#include "rg_common.cuh"
#include "rg_device.cuh"

namespace rg {
namespace {

constexpr int NT = kMatchThreads;
constexpr int NWARP = NT / 32;

struct Best {
  int sum, n, dx, dy;  // n == 0: no contributing point (infinite cost)
};

// strict "a beats b" on the key (sum/n, |dx|, dy, dx); census.hpp:225-252
__device__ __forceinline__ bool better(const Best& a, const Best& b) {
  if (a.n == 0) return false;
  if (b.n == 0) return true;
  const long long l = (long long)a.sum * b.n, r = (long long)b.sum * a.n;
  if (l != r) return l < r;
  const int aa = abs(a.dx), ab = abs(b.dx);
  if (aa != ab) return aa < ab;
  if (a.dy != b.dy) return a.dy < b.dy;
  return a.dx < b.dx;
}

__device__ __forceinline__ Best shfl_best(const Best& v, int src_lane_xor) {
  Best o;
  o.sum = __shfl_xor_sync(0xffffffffu, v.sum, src_lane_xor);
  o.n = __shfl_xor_sync(0xffffffffu, v.n, src_lane_xor);
  o.dx = __shfl_xor_sync(0xffffffffu, v.dx, src_lane_xor);
  o.dy = __shfl_xor_sync(0xffffffffu, v.dy, src_lane_xor);
  return o;
}

// census.hpp:167-171 in the reference's operation order
__device__ __forceinline__ double subpixel(double cm, double c0, double cp) {
  const double denom = __dsub_rn(__dadd_rn(cm, cp), __dmul_rn(2.0, c0));
  if (denom <= 0.0) return 0.0;
  return __ddiv_rn(-__dsub_rn(cp, cm), __dmul_rn(2.0, denom));
}

struct PassOut {
  int has;
  int dx, dy, sum, n;
  int interior;  // winner strictly inside the dx range
  int cm_sum, cm_n, cp_sum, cp_n;
};

struct Scratch {
  int nv;
  int xmin, xmax, ymin, ymax;
  int any_zero;
  Best wbest[NWARP];
  int red[2 * NWARP][2];
  PassOut pass;
};

__device__ __forceinline__ int popc(uint32_t x) { return __popc(x); }
__device__ __forceinline__ int popc(unsigned long long x) { return __popcll(x); }

template <typename CT>  // code type: uint32_t (5x5) or unsigned long long (9x7)
struct Dyn {  // dynamic shared memory views
  CT* win;      // right-census window
  CT* lc;       // left codes of the valid points
  int2* pts;    // block points (planner path); unused by the CSR path
  int* px;      // valid points after the shift
  int* py;
  int* off;     // their window offsets
};

template <typename CT>
__device__ __forceinline__ Dyn<CT> carve(void* base, int maxp, bool with_pts) {
  Dyn<CT> d;
  char* p = reinterpret_cast<char*>(base);
  d.win = reinterpret_cast<CT*>(p);
  p += sizeof(CT) * kWindowCodes;
  d.lc = reinterpret_cast<CT*>(p);
  p += sizeof(CT) * maxp;
  d.pts = reinterpret_cast<int2*>(p);
  if (with_pts) p += sizeof(int2) * maxp;
  d.px = reinterpret_cast<int*>(p);
  p += sizeof(int) * maxp;
  d.py = reinterpret_cast<int*>(p);
  p += sizeof(int) * maxp;
  d.off = reinterpret_cast<int*>(p);
  return d;
}

template <typename CT>
__device__ __forceinline__ CT sample(const RasterT<CT>& r, int x, int y) {
  return (x >= 0 && x < r.w && y >= 0 && y < r.h) ? __ldg(r.p + (int64_t)y * r.pitch + x) : CT(0);
}

// Candidate sweep over one chunk of CPT candidates per thread.
template <typename CT, int CPT, int MODE>  // MODE 0: window, no zeros; 1: window with zeros; 2: global
__device__ __forceinline__ void sweep(const Dyn<CT>& S, int nv, const RasterT<CT>& R, int c0, int nc,
                                      int ndx, int WW, const rg_search_range& rg, Best& mine,
                                      int& evals) {
  const int tid = threadIdx.x;
  int base[CPT], cdx[CPT], cdy[CPT];
  bool ok[CPT];
  int s[CPT], n[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int c = c0 + j * NT + tid;
    ok[j] = c < nc;
    const int cc = ok[j] ? c : 0;
    const int iy = cc / ndx, ix = cc - iy * ndx;
    cdx[j] = rg.dx_min + ix;
    cdy[j] = rg.dy_min + iy;
    base[j] = iy * WW + (ndx - 1 - ix);
    s[j] = 0;
    n[j] = 0;
  }
  if (MODE == 0) {
    int k = 0;
    if constexpr (sizeof(CT) == 4) for (; k + 4 <= nv; k += 4) {
      const int4 o4 = *reinterpret_cast<const int4*>(S.off + k);
      const uint4 l4 = *reinterpret_cast<const uint4*>(S.lc + k);
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        s[j] += __popc(l4.x ^ S.win[o4.x + base[j]]) + __popc(l4.y ^ S.win[o4.y + base[j]]);
        s[j] += __popc(l4.z ^ S.win[o4.z + base[j]]) + __popc(l4.w ^ S.win[o4.w + base[j]]);
      }
    }
    for (; k < nv; ++k) {
      const int o = S.off[k];
      const CT l = S.lc[k];
#pragma unroll
      for (int j = 0; j < CPT; ++j) s[j] += popc(l ^ S.win[o + base[j]]);
    }
#pragma unroll
    for (int j = 0; j < CPT; ++j) n[j] = nv;
  } else if (MODE == 1) {
    for (int k = 0; k < nv; ++k) {
      const int o = S.off[k];
      const CT l = S.lc[k];
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const CT r = S.win[o + base[j]];
        if (r != 0u) {
          s[j] += popc(l ^ r);
          ++n[j];
        }
      }
    }
  } else {
    for (int k = 0; k < nv; ++k) {
      const int x = S.px[k], y = S.py[k];
      const CT l = S.lc[k];
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const CT r = sample(R, x - cdx[j], y + cdy[j]);
        if (r != 0u) {
          s[j] += popc(l ^ r);
          ++n[j];
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    if (!ok[j] || n[j] == 0) continue;
    evals += n[j];  // Hamming evaluations, census.hpp:209-221
    const Best cand = {s[j], n[j], cdx[j], cdy[j]};
    if (better(cand, mine)) mine = cand;
  }
}

template <typename CT, int MODE>
__device__ __forceinline__ void sweep_all(const Dyn<CT>& S, int nv, const RasterT<CT>& R, int nc, int ndx,
                                          int WW, const rg_search_range& rg, Best& mine, int& evals) {
  if (nc <= NT) {
    sweep<CT, 1, MODE>(S, nv, R, 0, nc, ndx, WW, rg, mine, evals);
  } else if (nc <= 2 * NT) {
    sweep<CT, 2, MODE>(S, nv, R, 0, nc, ndx, WW, rg, mine, evals);
  } else {
    for (int c0 = 0; c0 < nc; c0 += 4 * NT) sweep<CT, 4, MODE>(S, nv, R, c0, nc, ndx, WW, rg, mine, evals);
  }
}

// Block-wide reductions ----------------------------------------------------
__device__ Best block_best(Best v, Scratch& sc) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Best u = shfl_best(v, o);
    if (better(u, v)) v = u;
  }
  if (lane == 0) sc.wbest[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < NWARP ? sc.wbest[lane] : Best{0, 0, 0, 0};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const Best u = shfl_best(v, o);
      if (better(u, v)) v = u;
    }
    if (lane == 0) sc.wbest[0] = v;
  }
  __syncthreads();
  const Best r = sc.wbest[0];
  __syncthreads();
  return r;
}

// sums (a0, a1, b0, b1) over the block
__device__ void block_sum4(int v[4], Scratch& sc) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane == 0) {
    sc.red[wid][0] = v[0];
    sc.red[wid][1] = v[1];
    sc.red[NWARP + wid][0] = v[2];
    sc.red[NWARP + wid][1] = v[3];
  }
  __syncthreads();
  int t[4] = {0, 0, 0, 0};
  for (int w = 0; w < NWARP; ++w) {
    t[0] += sc.red[w][0];
    t[1] += sc.red[w][1];
    t[2] += sc.red[NWARP + w][0];
    t[3] += sc.red[NWARP + w][1];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = t[i];
}

// One block_match pass (census.hpp:178-272).  Points come from `pts`
// (shared or global memory) shifted by (sx, sy).  Writes sc.pass.
template <typename CT>
__device__ void match_pass(const int2* pts, int np, int sx, int sy, const RasterT<CT>& L,
                           const RasterT<CT>& R, const rg_search_range& rg, const Dyn<CT>& S,
                           Scratch& sc, int& evals) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    sc.nv = 0;
    sc.xmin = INT_MAX;
    sc.ymin = INT_MAX;
    sc.xmax = INT_MIN;
    sc.ymax = INT_MIN;
  }
  __syncthreads();
  // keep points with a defined left descriptor; order is irrelevant (all
  // per-candidate quantities are integer sums over the set)
  for (int k = tid; k < np; k += NT) {
    const int2 p = pts[k];
    const int x = p.x + sx, y = p.y + sy;
    const CT c = sample(L, x, y);
    if (c != 0u) {
      const int slot = atomicAdd(&sc.nv, 1);
      S.px[slot] = x;
      S.py[slot] = y;
      S.lc[slot] = c;
      atomicMin(&sc.xmin, x);
      atomicMax(&sc.xmax, x);
      atomicMin(&sc.ymin, y);
      atomicMax(&sc.ymax, y);
    }
  }
  __syncthreads();
  const int nv = sc.nv;
  if (nv == 0) {
    if (tid == 0) sc.pass.has = 0;
    __syncthreads();
    return;
  }
  const int ndx = rg.dx_max - rg.dx_min + 1, ndy = rg.dy_max - rg.dy_min + 1;
  const int nc = ndx * ndy;
  const int xmin = sc.xmin, ymin = sc.ymin;
  const long long WWl = (long long)(sc.xmax - xmin) + ndx, WHl = (long long)(sc.ymax - ymin) + ndy;
  const bool use_win = WWl * WHl <= kWindowCodes;
  const int WW = use_win ? (int)WWl : 0;
  int any_zero = 1;
  if (use_win) {
    const int WH = (int)WHl;
    const int wx0 = xmin - rg.dx_max, wy0 = ymin + rg.dy_min;
    int zero = 0;
    for (int idx = tid; idx < WW * WH; idx += NT) {
      const int wy = idx / WW, wx = idx - wy * WW;
      const CT v = sample(R, wx0 + wx, wy0 + wy);
      S.win[idx] = v;
      zero |= (v == 0u);
    }
    for (int k = tid; k < nv; k += NT) S.off[k] = (S.py[k] - ymin) * WW + (S.px[k] - xmin);
    any_zero = __syncthreads_or(zero);
  }
  Best mine = {0, 0, 0, 0};
  if (use_win && !any_zero)
    sweep_all<CT, 0>(S, nv, R, nc, ndx, WW, rg, mine, evals);
  else if (use_win)
    sweep_all<CT, 1>(S, nv, R, nc, ndx, WW, rg, mine, evals);
  else
    sweep_all<CT, 2>(S, nv, R, nc, ndx, WW, rg, mine, evals);
  const Best b = block_best(mine, sc);
  if (b.n == 0) {  // no offset had a contributing point
    if (tid == 0) sc.pass.has = 0;
    __syncthreads();
    return;
  }
  const int bix = b.dx - rg.dx_min;
  const int interior = bix > 0 && bix + 1 < ndx;
  int v[4] = {0, 0, 0, 0};
  if (interior) {  // costs of (dx-1, dy) and (dx+1, dy)
    for (int k = tid; k < nv; k += NT) {
      const int x = S.px[k], y = S.py[k] + b.dy;
      const CT l = S.lc[k];
      const CT rm = sample(R, x - (b.dx - 1), y);
      const CT rp = sample(R, x - (b.dx + 1), y);
      if (rm) {
        v[0] += popc(l ^ rm);
        v[1] += 1;
      }
      if (rp) {
        v[2] += popc(l ^ rp);
        v[3] += 1;
      }
    }
  }
  block_sum4(v, sc);
  if (tid == 0) {
    PassOut& o = sc.pass;
    o.has = 1;
    o.dx = b.dx;
    o.dy = b.dy;
    o.sum = b.sum;
    o.n = b.n;
    o.interior = interior;
    o.cm_sum = v[0];
    o.cm_n = v[1];
    o.cp_sum = v[2];
    o.cp_n = v[3];
  }
  __syncthreads();
}

// FP64 epilogue of a pass: cost, neighbour costs, sub-pixel (census.hpp:255-270)
__device__ void finish_pass(const PassOut& p, rg_match_result& r) {
  r.has_value = 1;
  r.dx_int = p.dx;
  r.dy_int = p.dy;
  r.cost = __ddiv_rn((double)p.sum, (double)p.n);
  r.valid_points = p.n;
  r.dx_subpix = (double)p.dx;
  r.cost_minus = -1.0;
  r.cost_plus = -1.0;
  if (p.interior && p.cm_n > 0 && p.cp_n > 0) {
    const double cm = __ddiv_rn((double)p.cm_sum, (double)p.cm_n);
    const double cp = __ddiv_rn((double)p.cp_sum, (double)p.cp_n);
    r.cost_minus = cm;
    r.cost_plus = cp;
    r.dx_subpix = __dadd_rn((double)p.dx, subpixel(cm, r.cost, cp));
  }
}

// block_match / forward_backward_match of one block; result written by tid 0.
template <typename CT>
__device__ void match_block(const int2* pts, int np, const RasterT<CT>& L, const RasterT<CT>& R,
                            const rg_search_range& rg, int mode, double tau_v, const Dyn<CT>& S,
                            Scratch& sc, rg_match_result* out, unsigned long long* eval_counter) {
  int evals = 0;
  rg_match_result r;
  r.dx_int = 0;
  r.dy_int = 0;
  r.dx_subpix = 0.0;
  r.cost = 0.0;
  r.cost_minus = -1.0;
  r.cost_plus = -1.0;
  r.valid_points = 0;
  r.verified = 0;
  r.has_value = 0;
  r.n_points = np;
  if (np > 0) {
    match_pass(pts, np, 0, 0, L, R, rg, S, sc, evals);
    if (sc.pass.has) {
      finish_pass(sc.pass, r);
      if (mode == RG_MATCH_FWD_BWD) {
        const rg_search_range brg = {-rg.dx_max, -rg.dx_min, -r.dy_int, -r.dy_int};
        match_pass(pts, np, -r.dx_int, r.dy_int, R, L, brg, S, sc, evals);
        if (sc.pass.has) {
          rg_match_result bwd;
          finish_pass(sc.pass, bwd);
          r.verified = fabs(__dadd_rn(r.dx_subpix, bwd.dx_subpix)) < tau_v;
        }
      }
    }
  }
  if (threadIdx.x == 0) *out = r;
  if (eval_counter) {  // algorithmic work of this block, one atomic per CTA
    for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
    if ((threadIdx.x & 31) == 0 && evals) atomicAdd(eval_counter, (unsigned long long)evals);
  }
}

// ---------------------------------------------------------------- CSR path
template <typename CT>
__global__ void __launch_bounds__(NT) match_blocks_kernel(RasterT<CT> L, RasterT<CT> R,
                                                          const int32_t* __restrict__ pts,
                                                          const int64_t* __restrict__ offs,
                                                          const rg_search_range* __restrict__ ranges,
                                                          int mode, double tau_v, int maxp,
                                                          rg_match_result* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ Scratch sc;
  const int b = blockIdx.x;
  const Dyn<CT> S = carve<CT>(dyn, maxp, false);
  const int64_t o0 = offs[b];
  const int np = (int)(offs[b + 1] - o0);
  match_block(reinterpret_cast<const int2*>(pts) + o0, np, L, R, ranges[b], mode, tau_v, S, sc,
              &out[b], nullptr);
}

template <typename CT>
size_t dyn_bytes(int maxp, bool with_pts) {
  return sizeof(CT) * ((size_t)kWindowCodes + maxp) + (with_pts ? sizeof(int2) * maxp : 0) +
         3 * sizeof(int) * (size_t)maxp;
}

template <typename CT>
cudaError_t launch_csr(RasterT<CT> L, RasterT<CT> R, const int32_t* pts, const int64_t* offs,
                       const rg_search_range* ranges, int n_blocks, int mode, double tau_v,
                       rg_match_result* out, int max_points, cudaStream_t s) {
  if (n_blocks <= 0) return cudaSuccess;
  const int maxp = (max_points + 3) & ~3;
  const size_t smem = dyn_bytes<CT>(maxp, false);
  cudaError_t e = cudaFuncSetAttribute(match_blocks_kernel<CT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  match_blocks_kernel<CT><<<n_blocks, NT, smem, s>>>(L, R, pts, offs, ranges, mode, tau_v, maxp, out);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_match_blocks(Raster L, Raster R, const int32_t* pts, const int64_t* offs,
                                const rg_search_range* ranges, int n_blocks, int mode,
                                double tau_v, rg_match_result* out, int max_points,
                                cudaStream_t s) {
  return launch_csr<uint32_t>(L, R, pts, offs, ranges, n_blocks, mode, tau_v, out, max_points, s);
}

cudaError_t launch_match_blocks64(Raster64 L, Raster64 R, const int32_t* pts, const int64_t* offs,
                                  const rg_search_range* ranges, int n_blocks, int mode,
                                  double tau_v, rg_match_result* out, int max_points,
                                  cudaStream_t s) {
  return launch_csr<unsigned long long>(L, R, pts, offs, ranges, n_blocks, mode, tau_v, out, max_points,
                                        s);
}

}  // namespace rg
