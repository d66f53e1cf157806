// match_warp.cu -- K2 of the batched object ranger: fused query-point sampler
// + forward/backward census block matcher, one WARP per QueryBlock.
//
// Replaces, per slot planned by K3: sample_query_points (template_match.hpp:
// 155-223), forward_backward_match (census.hpp:281-303) and its two
// block_match passes (census.hpp:178-272).  Design (B200):
//   * warp-local: every stage (occluders, sampling, point filter, sweep,
//     argmin, neighbours, sub-pixel) is done by one warp with ballots and
//     shuffles -- no CTA barriers; a CTA carries 4 independent slots.
//   * the census rasters are zero-padded (PadGeom) so a sample at any offset
//     the search range reaches is a plain load; an out-of-image sample reads a
//     0 code, which is exactly the reference's "inside() && code != 0" drop.
//   * lanes own consecutive dx; each lane sweeps up to 9 chunks of 32 dx for
//     every point: one LDG (L1-resident row segment, immediate offsets) +
//     LOP3 + POPC + IADD per Hamming evaluation.  Points are visited in
//     grid order so each row segment stays L1-hot across the 8 points of a
//     row and the 3 dy.
//   * a block whose whole search window lies where the computed census is
//     defined takes the branch-free path (every point contributes, n = #points);
//     border blocks and caller-supplied rasters take the checked path.
//   * argmin of (sum/n, |dx|, dy, dx) by exact rational compare and warp
//     shuffles; FP64 epilogue in the reference's operation order.
#include <climits>
#include <cstdlib>

#include "rg_common.cuh"
#include "rg_device.cuh"

namespace rg {
namespace {

#ifndef RG_MW_CMAX
#define RG_MW_CMAX 4
#endif
#ifndef RG_MW_TAIL
#define RG_MW_TAIL 4
#endif
#ifndef RG_MW_PIPE
#define RG_MW_PIPE 1
#endif
#ifndef RG_MW_PIPE_UNROLL
#define RG_MW_PIPE_UNROLL 2
#endif
#ifndef RG_MW_NOINLINE
#define RG_MW_NOINLINE 0
#endif
#ifndef RG_MW_DY2  // two row offsets per FAST point pass (sweep2): measured 0.98 vs 0.895 ms per
#define RG_MW_DY2 0  // 256 C2 frames (1.30 vs 1.00 at 8 warps x 4 CTAs) -- an A/B knob
#endif
#ifndef RG_MW_CSA  // carry-save groups of 3 points in FAST sweeps: measured 1.22 vs 0.90 ms (loses the
#define RG_MW_CSA 0  // one-point-ahead load pipelining; at 40 registers it spills) -- kept as an A/B knob
#endif
constexpr int kPipeUnroll = RG_MW_PIPE_UNROLL;
#ifndef RG_MW_OCC
#define RG_MW_OCC 32
#endif
constexpr int kWarpOcc = RG_MW_OCC;  // occluder boxes per warp in smem (more: the per-point scan of every detection)
constexpr int kLatencyFrames = 4;  // batches up to this size use the latency-mode matcher      // occluder boxes per warp kept in smem
constexpr int CMAX = RG_MW_CMAX;  // 32-wide dx chunks per sweep (balanced groups)
constexpr int TAIL = RG_MW_TAIL;  // a last chunk with <= TAIL candidates goes point-parallel

struct Cand {
  int sum, n, dx, dy;  // n == 0: infinite cost
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {  // census.hpp:225-252
  if (a.n == 0) return false;
  if (b.n == 0) return true;
  const long long l = (long long)a.sum * b.n, r = (long long)b.sum * a.n;
  if (l != r) return l < r;
  const int aa = abs(a.dx), ab = abs(b.dx);
  if (aa != ab) return aa < ab;
  if (a.dy != b.dy) return a.dy < b.dy;
  return a.dx < b.dx;
}

// Correctly rounded a / b for the small non-negative integers of a pass
// (Hamming sums and valid-point counts): Markstein's correction on the
// correctly rounded reciprocal y = RN(1/b) from a per-device table --
// q = RN(a y), r = a - b q (exact by FMA), RN(q + r y) = RN(a / b) -- instead
// of the __ddiv_rn sequence.  Checked against __ddiv_rn for every b <= kRecip
// and 0 <= a <= 64 b (rg_selftest_division; a pass's sums are <= 63 b).
constexpr int kRecip = 4096;
__constant__ double c_recip[kRecip + 1];
// RN(1/b) for div_rc (0 outside the table: the IEEE division)
__device__ __forceinline__ double recip(int b) { return b >= 1 && b <= kRecip ? c_recip[b] : 0.0; }
__device__ __forceinline__ double div_int(int a, int b) {
  if (b >= 1 && b <= kRecip) {
    const double y = c_recip[b], da = (double)a, db = (double)b;
    const double q = __dmul_rn(da, y);
    const double r = __fma_rn(-q, db, da);
    return __fma_rn(r, y, q);
  }
  return __ddiv_rn((double)a, (double)b);
}

__global__ void selftest_div_kernel(int b_max, unsigned long long* bad) {
  const int b = blockIdx.x + 1;
  if (b > b_max) return;
  unsigned long long n = 0;
  for (int a = threadIdx.x; a <= 64 * b; a += blockDim.x) {
    const double x = div_int(a, b), y = __ddiv_rn((double)a, (double)b);
    n += __double_as_longlong(x) != __double_as_longlong(y);
  }
  // div_rc with arbitrary numerators (the sampler's coordinates): 64 b
  // pseudo-random doubles of magnitude 2^-12 .. 2^20 (either sign) per b
  const double rb = recip(b);
  for (int t = threadIdx.x; t <= 64 * b; t += blockDim.x) {
    unsigned long long z = (unsigned long long)b * 0x9E3779B97F4A7C15ull + (unsigned long long)t * 0xBF58476D1CE4E5B9ull;
    z ^= z >> 31;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 29;
    const int ex = (int)((z >> 53) % 33) - 12;
    const double a = ldexp(1.0 + (double)(z & 0xFFFFFFFFFFFFFull) * 0x1p-52, ex) * ((z >> 52) & 1 ? -1.0 : 1.0);
    const double x = div_rc(a, (double)b, rb), y = __ddiv_rn(a, (double)b);
    n += __double_as_longlong(x) != __double_as_longlong(y);
  }
  if (n) atomicAdd(bad, n);
}

__device__ __forceinline__ double subpixel(double cm, double c0, double cp) {  // census.hpp:167-171
  const double denom = __dsub_rn(__dadd_rn(cm, cp), __dmul_rn(2.0, c0));
  if (denom <= 0.0) return 0.0;
  return __ddiv_rn(-__dsub_rn(cp, cm), __dmul_rn(2.0, denom));
}

struct Pass {
  int has, dx, dy, sum, n, interior, cm_sum, cm_n, cp_sum, cp_n;
};

// a valid point of a pass: BYTE offset into the raster + left code (32-bit
// 5x5 or 64-bit 9x7).  Byte offsets keep the per-point address a single
// 64-bit add.
template <typename CT>
struct VPoint;
template <>
struct __align__(8) VPoint<uint32_t> {
  uint32_t off;
  uint32_t code;
};
template <>
struct __align__(16) VPoint<unsigned long long> {
  uint32_t off;
  uint32_t pad;
  unsigned long long code;
};
__device__ __forceinline__ int popc(uint32_t x) { return __popc(x); }
__device__ __forceinline__ int popc(unsigned long long x) { return __popcll(x); }
// all ones for a defined code of the internal layout (sentinel = top bit), 0 for undefined
__device__ __forceinline__ uint32_t defined_mask(uint32_t r) { return (uint32_t)((int32_t)r >> 31); }
__device__ __forceinline__ unsigned long long defined_mask(unsigned long long r) {
  return (unsigned long long)((long long)r >> 63);
}
template <typename CT>
__device__ __forceinline__ CT ld_at(const CT* base, uint32_t byte_off) {
  return __ldg(reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + byte_off));
}

// Sweep modes.  FAST: every sample is a defined code (n = #points).  SIGN:
// samples may be undefined, rasters in the internal layout (sentinel in the
// top bit): mask by the sign.  GENERIC: caller-supplied codes, test r != 0.
enum { M_FAST = 0, M_SIGN = 1, M_GENERIC = 2 };

// FAST-mode argmin key: all candidates of a FAST pass share n, so the
// reference order (sum/n, |dx|, dy, dx) (census.hpp:225-252) is the order of
// (sum, |dx|, dy, dx >= 0) packed into 64 bits (|dx| < 2^15, |dy| < 2^15).
__device__ __forceinline__ unsigned long long fast_key(int sum, int dx, int dy) {
  const uint32_t lo = ((uint32_t)abs(dx) << 17) | ((uint32_t)(dy + 0x8000) << 1) | (dx >= 0 ? 1u : 0u);
  return ((unsigned long long)(uint32_t)sum << 32) | lo;
}

// One sweep over K dx-chunks for one dy: `base` = this lane's sample pointer
// for chunk c0 at offset 0; chunk c reads 32*c codes to the left.
// PF > 0 (latency mode): the lines of point k+1+PF are prefetched into L1
// while point k is consumed -- a small batch leaves most SMs idle and each
// warp's point loop then waits on L2 latency, not on issue.
template <typename CT, int MODE, int K, int PF = 0>
__device__ __forceinline__ void sweep(const VPoint<CT>* __restrict__ vp, int nv, const CT* base,
                                      int lane, int c0, int ndx, int dx_min, int dy, Cand& best,
                                      unsigned long long& bkey, int& evals) {
  int s[K], n[K];
#pragma unroll
  for (int c = 0; c < K; ++c) s[c] = n[c] = 0;
  const int nv_all = nv;
#if RG_MW_CSA
  // FAST sweeps take the points three at a time through a carry-save adder:
  // popc(a) + popc(b) + popc(c) = popc(a ^ b ^ c) + 2 popc(maj(a, b, c)), so
  // 2 POPC per 3 evaluations -- the point loop is POPC-bound (a warp POPC
  // occupies its pipe 8 cycles; tools/hamming_probe.cu: 15.4 -> 21.5
  // evaluations / clk / SM); the remaining nv % 3 points take the loop below
  if (MODE == M_FAST && sizeof(CT) == 4 && PF == 0) {
    int s2[K];
#pragma unroll
    for (int c = 0; c < K; ++c) s2[c] = 0;
    const int n3 = nv - nv % 3;
    int k = 0;
    for (; k < n3; k += 3) {
      const VPoint<CT> qa = vp[k], qb = vp[k + 1], qc = vp[k + 2];
      const CT* pa = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qa.off);
      const CT* pb = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qb.off);
      const CT* pc = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qc.off);
      CT ra[K], rb[K], rc[K];
#pragma unroll
      for (int c = 0; c < K; ++c) ra[c] = __ldg(pa - 32 * c), rb[c] = __ldg(pb - 32 * c), rc[c] = __ldg(pc - 32 * c);
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const uint32_t x = (uint32_t)(qa.code ^ ra[c]), y = (uint32_t)(qb.code ^ rb[c]),
                       z = (uint32_t)(qc.code ^ rc[c]);
        s[c] += __popc(x ^ y ^ z);
        s2[c] += __popc((x & y) | (z & (x | y)));
      }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] += 2 * s2[c];
    vp += n3;
    nv -= n3;
  }
#endif
#if RG_MW_PIPE
  // software-pipelined: the samples of point k+1 are in flight while point k
  // is consumed (the last prefetch re-reads point nv-1, harmless)
  VPoint<CT> qn = vp[0];
  CT rn[K];
  {
    const CT* a = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qn.off);
#pragma unroll
    for (int c = 0; c < K; ++c) rn[c] = __ldg(a - 32 * c);
  }
#if RG_MW_PIPE == 2  // distance 2: points k+1 and k+2 in flight
  VPoint<CT> qm = vp[min(1, nv - 1)];
  CT rm[K];
  {
    const CT* a = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qm.off);
#pragma unroll
    for (int c = 0; c < K; ++c) rm[c] = __ldg(a - 32 * c);
  }
#endif
#pragma unroll kPipeUnroll
  for (int k = 0; k < nv; ++k) {
    const CT l = qn.code;
    CT rc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) rc[c] = rn[c];
#if RG_MW_PIPE == 2
    qn = qm;
#pragma unroll
    for (int c = 0; c < K; ++c) rn[c] = rm[c];
    qm = vp[min(k + 2, nv - 1)];
    const CT* a = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qm.off);
#pragma unroll
    for (int c = 0; c < K; ++c) rm[c] = __ldg(a - 32 * c);
#else
    qn = vp[k + 1];  // vp[nv] duplicates vp[nv - 1] (warp_pass), so no clamp
    const CT* a = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qn.off);
#pragma unroll
    for (int c = 0; c < K; ++c) rn[c] = __ldg(a - 32 * c);
    if (PF > 0) {
      const CT* pa = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + vp[min(k + 1 + PF, nv)].off);
#pragma unroll
      for (int c = 0; c < K; ++c) asm volatile("prefetch.global.L1 [%0];" ::"l"(pa - 32 * c));
    }
#endif
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const CT r = rc[c];
#else
  for (int k = 0; k < nv; ++k) {
    const VPoint<CT> q = vp[k];
    const CT* a = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + q.off);
    const CT l = q.code;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const CT r = __ldg(a - 32 * c);
#endif
      if (MODE == M_FAST) {
        s[c] += popc(l ^ r);
      } else if (MODE == M_SIGN) {
        const CT m = defined_mask(r);
        s[c] += popc((l ^ r) & m);
        n[c] -= (int)m;
      } else if (r != 0u) {
        s[c] += popc(l ^ r);
        ++n[c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < K; ++c) {
    const int ix = lane + 32 * (c0 + c);
    if (MODE == M_FAST) {
      if (ix < ndx) {
        evals += nv_all;  // Hamming evaluations, census.hpp:209-221
        const unsigned long long key = fast_key(s[c], dx_min + ix, dy);
        bkey = key < bkey ? key : bkey;
      }
    } else if (ix < ndx && n[c] > 0) {
      evals += n[c];
      const Cand cd = {s[c], n[c], dx_min + ix, dy};
      if (better(cd, best)) best = cd;
    }
  }
}

// FAST sweep of K dx-chunks for TWO row offsets dy, dy + 1 in one pass over
// the points: one point record and one address per point feed 2K samples, and
// twice as many independent loads are in flight (the point loop is bound by
// the L1 latency of its one-point-ahead pipeline, ncu: long-scoreboard).
template <typename CT, int K>
__device__ __forceinline__ void sweep2(const VPoint<CT>* __restrict__ vp, int nv, const CT* base, int64_t pitch_b,
                                       int lane, int c0, int ndx, int dx_min, int dy, unsigned long long& bkey,
                                       int& evals) {
  int s0[K], s1[K];
#pragma unroll
  for (int c = 0; c < K; ++c) s0[c] = s1[c] = 0;
  VPoint<CT> qn = vp[0];
  CT rn0[K], rn1[K];
  {
    const CT* a = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qn.off);
    const CT* b = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(a) + pitch_b);
#pragma unroll
    for (int c = 0; c < K; ++c) rn0[c] = __ldg(a - 32 * c), rn1[c] = __ldg(b - 32 * c);
  }
#pragma unroll 2
  for (int k = 0; k < nv; ++k) {
    const CT l = qn.code;
    CT r0[K], r1[K];
#pragma unroll
    for (int c = 0; c < K; ++c) r0[c] = rn0[c], r1[c] = rn1[c];
    qn = vp[k + 1];  // vp[nv] duplicates vp[nv - 1] (warp_pass)
    const CT* a = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(base) + qn.off);
    const CT* b = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(a) + pitch_b);
#pragma unroll
    for (int c = 0; c < K; ++c) rn0[c] = __ldg(a - 32 * c), rn1[c] = __ldg(b - 32 * c);
#pragma unroll
    for (int c = 0; c < K; ++c) {
      s0[c] += popc(l ^ r0[c]);
      s1[c] += popc(l ^ r1[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < K; ++c) {
    const int ix = lane + 32 * (c0 + c);
    if (ix < ndx) {
      evals += 2 * nv;  // Hamming evaluations, census.hpp:209-221
      const unsigned long long k0 = fast_key(s0[c], dx_min + ix, dy), k1 = fast_key(s1[c], dx_min + ix, dy + 1);
      bkey = k0 < bkey ? k0 : bkey;
      bkey = k1 < bkey ? k1 : bkey;
    }
  }
}

template <typename CT>
__device__ __forceinline__ void sweep2_chunks(const VPoint<CT>* vp, int nv, const CT* base, int64_t pitch_b,
                                              int lane, int c0, int k, int ndx, int dx_min, int dy,
                                              unsigned long long& bkey, int& evals) {
  switch (k) {
    case 1: sweep2<CT, 1>(vp, nv, base, pitch_b, lane, c0, ndx, dx_min, dy, bkey, evals); break;
    case 2: sweep2<CT, 2>(vp, nv, base, pitch_b, lane, c0, ndx, dx_min, dy, bkey, evals); break;
    case 3: sweep2<CT, 3>(vp, nv, base, pitch_b, lane, c0, ndx, dx_min, dy, bkey, evals); break;
    default: sweep2<CT, 4>(vp, nv, base, pitch_b, lane, c0, ndx, dx_min, dy, bkey, evals); break;
  }
}

template <typename CT, int MODE, int PF = 0>
__device__ __forceinline__ void sweep_chunks(const VPoint<CT>* vp, int nv, const CT* base, int lane,
                                             int c0, int k, int ndx, int dx_min, int dy, Cand& best,
                                             unsigned long long& bkey, int& evals) {
  static_assert(CMAX >= 1 && CMAX <= 9, "chunk cap");
#define RG_SWEEP_CASE(K)                                                                                 \
  case K:                                                                                                \
    if (K <= CMAX)                                                                                       \
      sweep<CT, MODE, (K <= CMAX ? K : 1), PF>(vp, nv, base, lane, c0, ndx, dx_min, dy, best, bkey, evals); \
    break;
  switch (k) {
    RG_SWEEP_CASE(1)
    RG_SWEEP_CASE(2)
    RG_SWEEP_CASE(3)
    RG_SWEEP_CASE(4)
    RG_SWEEP_CASE(5)
    RG_SWEEP_CASE(6)
    RG_SWEEP_CASE(7)
    RG_SWEEP_CASE(8)
    RG_SWEEP_CASE(9)
    default:
      break;
  }
#undef RG_SWEEP_CASE
}

// The last m (<= TAIL) candidates of a range that is not a multiple of 32:
// lanes split the points instead of the candidates, so the warp does not
// evaluate 32 - m dead lanes for every point.
template <typename CT, int MODE>
__device__ __forceinline__ void sweep_tail(const VPoint<CT>* vp, int nv, const CT* rdy, int dx0, int m,
                                           int dy, int lane, Cand& best, unsigned long long& bkey,
                                           int& evals) {
  for (int j = 0; j < m; ++j) {
    const int dx = dx0 + j;
    const CT* rd = rdy - dx;
    int sum = 0, n = 0;
    for (int k = lane; k < nv; k += 32) {
      const VPoint<CT> q = vp[k];
      const CT r = ld_at(rd, q.off);
      if (MODE == M_FAST) {
        sum += popc(q.code ^ r);
      } else if (MODE == M_SIGN) {
        const CT mk = defined_mask(r);
        sum += popc((q.code ^ r) & mk);
        n -= (int)mk;
      } else if (r != 0u) {
        sum += popc(q.code ^ r);
        ++n;
      }
    }
    sum = __reduce_add_sync(0xffffffffu, sum);
    n = MODE == M_FAST ? nv : __reduce_add_sync(0xffffffffu, n);
    if (lane == 0 && n > 0) {
      evals += n;
      if (MODE == M_FAST) {
        const unsigned long long key = fast_key(sum, dx, dy);
        bkey = key < bkey ? key : bkey;
      } else {
        const Cand cd = {sum, n, dx, dy};
        if (better(cd, best)) best = cd;
      }
    }
  }
}

#ifndef RG_MW_RANGE_NOINLINE
#define RG_MW_RANGE_NOINLINE 0
#endif
#ifndef RG_MW_COOP_ITEMS  // cooperative blocks split (row offset, chunk) units, not chunks
#define RG_MW_COOP_ITEMS 1
#endif
template <typename CT, int MODE, int PF = 0>
#if RG_MW_RANGE_NOINLINE
__device__ __noinline__ void sweep_range(
#else
__device__ __forceinline__ void sweep_range(
#endif
    const VPoint<CT>* vp, int nv, const CT* R, const PadGeom& g,
                                            const rg_search_range& rg, int lane, Cand& best,
                                            unsigned long long& bkey, int& evals, int part = 0, int nparts = 1) {
#ifdef RG_MW_SKIP_SWEEP  // measurement skeleton only: everything but the sweeps (results invalid)
  if (lane == 0) best = Cand{1, 1, rg.dx_min, rg.dy_min};
  bkey = fast_key(1, rg.dx_min, rg.dy_min);
  return;
#endif
  // lane-parallel chunks in balanced groups of <= CMAX; a short tail chunk
  // goes point-parallel.  nparts > 1: this warp sweeps the chunks
  // [part * nfull / nparts, (part + 1) * nfull / nparts) of every row offset
  // and the last part the tail (cooperative FAR blocks, latency mode)
  const int ndx = rg.dx_max - rg.dx_min + 1;
  const int nch = (ndx + 31) / 32;
  const int mt = ndx & 31;
  const bool ptail = mt != 0 && mt <= TAIL;
  const int nfull = ptail ? ndx >> 5 : nch;
  if (nparts > 1 && RG_MW_COOP_ITEMS) {
    // cooperative blocks: the (row offset, chunk) units split contiguously
    // over the parts, so more warps than chunks shorten the critical path;
    // the tail of a row offset goes with its last chunk
    const int ndy = rg.dy_max - rg.dy_min + 1;
    const int U = ndy * nfull, u0 = part * U / nparts, u1 = (part + 1) * U / nparts;
    for (int dyi = 0; dyi < ndy; ++dyi) {
      const int dy = rg.dy_min + dyi;
      const int a = max(u0, dyi * nfull) - dyi * nfull, b = min(u1, (dyi + 1) * nfull) - dyi * nfull;
      for (int c0 = a; c0 < b;) {
        const int k = min(CMAX, b - c0);
        sweep_chunks<CT, MODE, PF>(vp, nv, R + (int64_t)dy * g.pitch - rg.dx_min - lane - 32 * c0, lane, c0, k, ndx,
                                   rg.dx_min, dy, best, bkey, evals);
        c0 += k;
      }
      const bool tail_mine = nfull ? (dyi * nfull + nfull - 1 >= u0 && dyi * nfull + nfull - 1 < u1)
                                   : (dyi % nparts == part);
      if (ptail && tail_mine)
        sweep_tail<CT, MODE>(vp, nv, R + (int64_t)dy * g.pitch, rg.dx_min + 32 * nfull, mt, dy, lane, best, bkey,
                             evals);
    }
    return;
  }
  const int cb = part * nfull / nparts, ce = (part + 1) * nfull / nparts, nmine = ce - cb;
  const int groups = (nmine + CMAX - 1) / CMAX;
  // balanced group sizes (nmine / groups without a division for 1-2 groups)
  const int gq = groups == 1 ? nmine : groups == 2 ? nmine >> 1 : groups ? nmine / groups : 0;
  const int gr = groups ? nmine - gq * groups : 0;
  for (int dy = rg.dy_min; dy <= rg.dy_max; ++dy) {
    // FAST throughput sweeps take two row offsets per pass over the points
    const bool two = RG_MW_DY2 && MODE == M_FAST && PF == 0 && nparts == 1 && sizeof(CT) == 4 &&
                     CMAX <= 4 && dy + 1 <= rg.dy_max;
    for (int gi = 0, c0 = cb; gi < groups; ++gi) {
      const int k = gq + (gi < gr ? 1 : 0);
      const CT* base = R + (int64_t)dy * g.pitch - rg.dx_min - lane - 32 * c0;
      if (two)
        sweep2_chunks<CT>(vp, nv, base, (int64_t)g.pitch * (int64_t)sizeof(CT), lane, c0, k, ndx, rg.dx_min, dy,
                          bkey, evals);
      else
        sweep_chunks<CT, MODE, PF>(vp, nv, base, lane, c0, k, ndx, rg.dx_min, dy, best, bkey, evals);
      c0 += k;
    }
    if (two && ptail && part == nparts - 1)  // the tail of row offset dy (dy + 1's follows below)
      sweep_tail<CT, MODE>(vp, nv, R + (int64_t)dy * g.pitch, rg.dx_min + 32 * nfull, mt, dy, lane, best, bkey,
                           evals);
    if (two) ++dy;
    if (ptail && part == nparts - 1)
      sweep_tail<CT, MODE>(vp, nv, R + (int64_t)dy * g.pitch, rg.dx_min + 32 * nfull, mt, dy, lane, best, bkey,
                           evals);
  }
}

// ---------------------------------------------------------------------------
// Vectorised sweep (throughput matcher: 32-bit codes in the padded internal
// layout).  Lanes own dx PAIRS: lane l of chunk c holds dx e and e + 1, e =
// E + 64 c + 2 l, and reads both samples with ONE 8-byte load at column
// x - e - 1 -- aligned iff x - E - 1 is even (raster rows start 128-B
// aligned).  So a pass's points split by the parity of x - D (D = dx_min):
// class A sweeps with E = D, class B with E = D - 1, and B's pair sums are
// realigned into A's layout by one lane shuffle per chunk.  Against one
// 4-byte load per evaluation this halves the load instructions and the L1
// wavefronts (a misaligned 128-B warp load touches two lines).
// FAST blocks (every sample defined) add groups of three points through a
// carry-save adder: popc(a) + popc(b) + popc(c) = popc(a ^ b ^ c) +
// 2 popc(maj(a, b, c)) -- 2 POPC per 3 evaluations; POPC issues at a quarter
// of the LOP3 rate (tools/hamming_probe.cu: 15.4 -> 21.5 evaluations/clk/SM).
// Per chunk group, the candidate at its last A position (lane 31, last
// chunk, dx e + 1), whose B part sits in the next group, and the final tail
// beyond the last full chunk are evaluated point-parallel (v2_fixup).
template <int NC, int MODE>
__device__ __forceinline__ void v2_class(const VPoint<uint32_t>* __restrict__ vp, int nv, const char* rb,
                                         int (&s)[NC][2], int (&n)[NC][2]) {
  int k = 0;
  if (MODE == M_FAST) {
    for (; k + 3 <= nv; k += 3) {
      const VPoint<uint32_t> a = vp[k], b = vp[k + 1], c = vp[k + 2];
      const uint2* pa = reinterpret_cast<const uint2*>(rb + a.off);
      const uint2* pb = reinterpret_cast<const uint2*>(rb + b.off);
      const uint2* pc = reinterpret_cast<const uint2*>(rb + c.off);
#pragma unroll
      for (int ch = 0; ch < NC; ++ch) {
        const uint2 va = __ldg(pa - 32 * ch), vb = __ldg(pb - 32 * ch), vc = __ldg(pc - 32 * ch);
        // element 0 (dx e) is the upper word, element 1 (dx e + 1) the lower
        const uint32_t x0 = a.code ^ va.y, y0 = b.code ^ vb.y, z0 = c.code ^ vc.y;
        const uint32_t x1 = a.code ^ va.x, y1 = b.code ^ vb.x, z1 = c.code ^ vc.x;
        const int t0 = __popc((x0 & y0) | (z0 & (x0 | y0))), t1 = __popc((x1 & y1) | (z1 & (x1 | y1)));
        s[ch][0] += __popc(x0 ^ y0 ^ z0) + 2 * t0;
        s[ch][1] += __popc(x1 ^ y1 ^ z1) + 2 * t1;
      }
    }
  }
  for (; k < nv; ++k) {
    const VPoint<uint32_t> a = vp[k];
    const uint2* pa = reinterpret_cast<const uint2*>(rb + a.off);
#pragma unroll
    for (int ch = 0; ch < NC; ++ch) {
      const uint2 v = __ldg(pa - 32 * ch);
      if (MODE == M_FAST) {
        s[ch][0] += __popc(a.code ^ v.y);
        s[ch][1] += __popc(a.code ^ v.x);
      } else {  // M_SIGN: an undefined sample (code 0 in the padded layout) drops out
        const uint32_t m0 = defined_mask(v.y), m1 = defined_mask(v.x);
        s[ch][0] += __popc((a.code ^ v.y) & m0);
        s[ch][1] += __popc((a.code ^ v.x) & m1);
        n[ch][0] -= (int)m0;
        n[ch][1] -= (int)m1;
      }
    }
  }
}

// One chunk group [c0, c0 + NC) for one dy: both classes, B realigned into A,
// then this lane's argmin over its candidates below dx_lim (the rest are fixups).
template <int NC, int MODE>
__device__ __forceinline__ void v2_group(const VPoint<uint32_t>* vpa, int na, const VPoint<uint32_t>* vpb, int nb,
                                         const char* rdy, int D, int c0, int dx_lim, int dy, int lane, int nv,
                                         Cand& best, unsigned long long& bkey, int& evals) {
  int as[NC][2], bs[NC][2], an[NC][2], bn[NC][2];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int k = 0; k < 2; ++k) as[c][k] = bs[c][k] = an[c][k] = bn[c][k] = 0;
  // lane base: element column x - e - 1 with e = E + 64 c0 + 2 lane (x enters via VPoint::off)
  const int EA = D + 64 * c0, EB = EA - 1;
  v2_class<NC, MODE>(vpa, na, rdy - 4 * (EA + 1 + 2 * lane), as, an);
  v2_class<NC, MODE>(vpb, nb, rdy - 4 * (EB + 1 + 2 * lane), bs, bn);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    // B element 1 (dx EB + 2l + 1 = EA + 2l) -> A element 0 of the same lane;
    // B element 0 of lane l + 1 (dx EA + 2l + 1) -> A element 1 of lane l; lane
    // 31 takes lane 0 of the next chunk (in the last chunk it is a fixup)
    const int nxt = __shfl_sync(0xffffffffu, bs[c][0], (lane + 1) & 31);
    int s0 = as[c][0] + bs[c][1], s1 = as[c][1] + (lane < 31 ? nxt : 0);
    int n0 = 0, n1 = 0;
    if (MODE == M_SIGN) {
      const int nnx = __shfl_sync(0xffffffffu, bn[c][0], (lane + 1) & 31);
      n0 = an[c][0] + bn[c][1];
      n1 = an[c][1] + (lane < 31 ? nnx : 0);
    }
    if (c + 1 < NC) {
      const int w = __shfl_sync(0xffffffffu, bs[c + 1][0], 0);
      if (lane == 31) s1 += w;
      if (MODE == M_SIGN) {
        const int wn = __shfl_sync(0xffffffffu, bn[c + 1][0], 0);
        if (lane == 31) n1 += wn;
      }
    }
    const int dx0 = EA + 64 * c + 2 * lane;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int dx = dx0 + k;
      if (dx >= dx_lim) continue;
      const int sum = k ? s1 : s0;
      if (MODE == M_FAST) {
        evals += nv;
        const unsigned long long key = fast_key(sum, dx, dy);
        bkey = key < bkey ? key : bkey;
      } else {
        const int nn = k ? n1 : n0;
        if (nn > 0) {
          evals += nn;
          const Cand cd = {sum, nn, dx, dy};
          if (better(cd, best)) best = cd;
        }
      }
    }
  }
}

// Fixup candidates dx in [t0, t1] (group ends and the final tail), every point
// of both classes, lanes over points.
template <int MODE>
__device__ __forceinline__ void v2_fixup(const VPoint<uint32_t>* vpa, int na, const VPoint<uint32_t>* vpb, int nb,
                                         const char* rdy, int t0, int t1, int dy, int lane, Cand& best,
                                         unsigned long long& bkey, int& evals) {
  for (int t = t0; t <= t1; ++t) {
    const char* rd = rdy - 4 * t;
    int sum = 0, n = 0;
    for (int k = lane; k < na + nb; k += 32) {
      const VPoint<uint32_t> q = k < na ? vpa[k] : vpb[k - na];
      const uint32_t r = __ldg(reinterpret_cast<const uint32_t*>(rd + q.off));
      if (MODE == M_FAST) {
        sum += __popc(q.code ^ r);
      } else {
        const uint32_t m = defined_mask(r);
        sum += __popc((q.code ^ r) & m);
        n -= (int)m;
      }
    }
    sum = __reduce_add_sync(0xffffffffu, sum);
    n = MODE == M_FAST ? na + nb : __reduce_add_sync(0xffffffffu, n);
    if (lane == 0 && n > 0) {
      evals += n;
      if (MODE == M_FAST) {
        const unsigned long long key = fast_key(sum, t, dy);
        bkey = key < bkey ? key : bkey;
      } else {
        const Cand cd = {sum, n, t, dy};
        if (better(cd, best)) best = cd;
      }
    }
  }
}

// The whole search range of one pass: chunk groups of <= 4 (balanced) per dy,
// each followed by its end fixup; the final tail after the last group.
template <int MODE>
__device__ __forceinline__ void v2_range(const VPoint<uint32_t>* vpa, int na, const VPoint<uint32_t>* vpb, int nb,
                                         const uint32_t* R, const PadGeom& g, const rg_search_range& rg, int lane,
                                         Cand& best, unsigned long long& bkey, int& evals) {
  const int D = rg.dx_min, ndx = rg.dx_max - rg.dx_min + 1;
  const int nfull = ndx >> 6, rem = ndx & 63;
  const int nch = (nfull >= 1 && rem <= 3) ? nfull : nfull + 1;
  const int groups = (nch + 3) / 4;
  const int gq = nch / groups, gr = nch - gq * groups;
  const int nv = na + nb;
  for (int dy = rg.dy_min; dy <= rg.dy_max; ++dy) {
    const char* rdy = reinterpret_cast<const char*>(R + (int64_t)dy * g.pitch);
    for (int gi = 0, c0 = 0; gi < groups; ++gi) {
      const int k = gq + (gi < gr ? 1 : 0);
      const int end = D + 64 * (c0 + k) - 1;  // this group's last A position: a fixup
      const int lim = min(end, rg.dx_max + 1);
      if (k <= 2)  // 1 or 2 chunks: the 2-chunk body (a 1-chunk group's second chunk lies past lim)
        v2_group<2, MODE>(vpa, na, vpb, nb, rdy, D, c0, lim, dy, lane, nv, best, bkey, evals);
      else
        v2_group<4, MODE>(vpa, na, vpb, nb, rdy, D, c0, lim, dy, lane, nv, best, bkey, evals);
      c0 += k;
      // the group end (and, after the last group, the tail up to dx_max)
      const int t1 = gi + 1 < groups ? end : rg.dx_max;
      if (end <= rg.dx_max) v2_fixup<MODE>(vpa, na, vpb, nb, rdy, end, t1, dy, lane, best, bkey, evals);
    }
  }
}

// One block_match pass (census.hpp:178-272) by the calling warp.
// pts: the block's points (smem), shifted by (sx, sy); L: raster of the left
// codes, R: raster sampled at (x - dx, y + dy).  Both share geometry g.
template <typename CT, int PF = 0>
#if RG_MW_NOINLINE
__device__ __noinline__ Pass warp_pass(
#else
__device__ Pass warp_pass(
#endif
    const int2* pts, int np, int sx, int sy, const CT* L, const CT* R,
                          const PadGeom& g, bool trusted, const rg_search_range& rg, VPoint<CT>* vp,
                          int lane, int& evals, int part = 0, int nparts = 1, Cand* xc = nullptr) {
  Pass o = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  int nv = 0;
  int xmin = INT_MAX, xmax = INT_MIN, ymin = INT_MAX, ymax = INT_MIN;
  for (int b = 0; b < np; b += 32) {  // keep points with a defined left code (:195-201)
    const int k = b + lane;
    int x = 0, y = 0;
    CT code = 0;
    if (k < np) {
      const int2 p = pts[k];
      x = p.x + sx;
      y = p.y + sy;
      if (x >= 0 && x < g.w && y >= 0 && y < g.h) code = L[(int64_t)y * g.pitch + x];
    }
    const bool ok = code != 0u;
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      VPoint<CT> q{};
      q.off = (uint32_t)(y * g.pitch + x) * (uint32_t)sizeof(CT);
      q.code = code;
      vp[nv + __popc(bal & ((1u << lane) - 1u))] = q;
      xmin = min(xmin, x);
      xmax = max(xmax, x);
      ymin = min(ymin, y);
      ymax = max(ymax, y);
    }
    nv += __popc(bal);
  }
  __syncwarp();
  if (nv == 0) return o;  // no contributing point anywhere: nullopt
  if (lane == 0) vp[nv] = vp[nv - 1];  // padding read by the sweeps' one-ahead prefetch
  __syncwarp();
  xmin = __reduce_min_sync(0xffffffffu, xmin);
  ymin = __reduce_min_sync(0xffffffffu, ymin);
  xmax = __reduce_max_sync(0xffffffffu, xmax);
  ymax = __reduce_max_sync(0xffffffffu, ymax);
  const int ndx = rg.dx_max - rg.dx_min + 1;
  // every sample of every real candidate lies where a computed code is defined
  // (and the candidate fits the packed FAST key)
  const bool fast = trusted && xmin - rg.dx_max >= g.sx0 && xmax - rg.dx_min <= g.sx1 &&
                    ymin + rg.dy_min >= g.sy0 && ymax + rg.dy_max <= g.sy1 && rg.dx_min > -32768 &&
                    rg.dx_max < 32768 && rg.dy_min >= -32768 && rg.dy_max < 32768;
  Cand best = {0, 0, 0, 0};
  if (fast) {
    unsigned long long bkey = ~0ull;
    sweep_range<CT, M_FAST, PF>(vp, nv, R, g, rg, lane, best, bkey, evals, part, nparts);
    // warp argmin of the packed keys (64-bit: two 32-bit reductions)
    uint32_t hi = __reduce_min_sync(0xffffffffu, (uint32_t)(bkey >> 32));
    uint32_t lo = __reduce_min_sync(0xffffffffu, (uint32_t)(bkey >> 32) == hi ? (uint32_t)bkey : ~0u);
    if (nparts > 1) {  // across the CTA's warps (same vp, same decision in every warp)
      if (lane == 0) xc[part] = Cand{(int)hi, (int)lo, 0, 0};
      __syncthreads();
      for (int q = 0; q < nparts; ++q) {
        const uint32_t h2 = (uint32_t)xc[q].sum, l2 = (uint32_t)xc[q].n;
        if (h2 < hi || (h2 == hi && l2 < lo)) hi = h2, lo = l2;
      }
      __syncthreads();
    }
    const int adx = (int)(lo >> 17);
    best.sum = (int)hi;
    best.n = nv;
    best.dx = (lo & 1u) ? adx : -adx;
    best.dy = (int)((lo >> 1) & 0xFFFFu) - 0x8000;
  } else {
    unsigned long long unused = 0;
    if (trusted)
      sweep_range<CT, M_SIGN, PF>(vp, nv, R, g, rg, lane, best, unused, evals, part, nparts);
    else
      sweep_range<CT, M_GENERIC, PF>(vp, nv, R, g, rg, lane, best, unused, evals, part, nparts);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {  // warp argmin
      Cand u;
      u.sum = __shfl_xor_sync(0xffffffffu, best.sum, off);
      u.n = __shfl_xor_sync(0xffffffffu, best.n, off);
      u.dx = __shfl_xor_sync(0xffffffffu, best.dx, off);
      u.dy = __shfl_xor_sync(0xffffffffu, best.dy, off);
      if (better(u, best)) best = u;
    }
    if (nparts > 1) {  // across the CTA's warps (a total order: any merge order)
      if (lane == 0) xc[part] = best;
      __syncthreads();
      for (int q = 0; q < nparts; ++q)
        if (better(xc[q], best)) best = xc[q];
      __syncthreads();
    }
  }
  if (best.n == 0) return o;
  const int bix = best.dx - rg.dx_min;
  o.has = 1;
  o.dx = best.dx;
  o.dy = best.dy;
  o.sum = best.sum;
  o.n = best.n;
  o.interior = bix > 0 && bix + 1 < ndx;
  if (o.interior) {  // costs at (dx - 1, dy) and (dx + 1, dy) for the parabola
    int ms = 0, mn = 0, ps = 0, pn = 0;
    for (int k = lane; k < nv; k += 32) {
      const VPoint<CT> q = vp[k];
      const CT* a = reinterpret_cast<const CT*>(reinterpret_cast<const char*>(R + (int64_t)best.dy * g.pitch - best.dx) +
                                                q.off);
      const CT rm = a[1], rp = a[-1];
      if (rm) {
        ms += popc(q.code ^ rm);
        ++mn;
      }
      if (rp) {
        ps += popc(q.code ^ rp);
        ++pn;
      }
    }
    o.cm_sum = __reduce_add_sync(0xffffffffu, ms);
    o.cm_n = __reduce_add_sync(0xffffffffu, mn);
    o.cp_sum = __reduce_add_sync(0xffffffffu, ps);
    o.cp_n = __reduce_add_sync(0xffffffffu, pn);
  }
  return o;
}

// One block_match pass with the vectorised sweep (32-bit codes, trusted
// padded rasters, one warp per block): the left-code filter writes class A
// points from the front of vp and class B points from the back (cap entries).
__device__ Pass warp_pass_v2(const int2* pts, int np, int sx, int sy, const uint32_t* L, const uint32_t* R,
                             const PadGeom& g, const rg_search_range& rg, VPoint<uint32_t>* vp, int cap, int lane,
                             int& evals) {
  Pass o = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int D = rg.dx_min;
  int na = 0, nb = 0;
  int xmin = INT_MAX, xmax = INT_MIN, ymin = INT_MAX, ymax = INT_MIN;
  const unsigned below = (1u << lane) - 1u;
  for (int b = 0; b < np; b += 32) {  // keep points with a defined left code (census.hpp:195-201)
    const int k = b + lane;
    int x = 0, y = 0;
    uint32_t code = 0;
    if (k < np) {
      const int2 p = pts[k];
      x = p.x + sx;
      y = p.y + sy;
      if (x >= 0 && x < g.w && y >= 0 && y < g.h) code = L[(int64_t)y * g.pitch + x];
    }
    const bool ok = code != 0u;
    const bool ca = ok && ((x - D) & 1);
    const unsigned ba = __ballot_sync(0xffffffffu, ca), bbm = __ballot_sync(0xffffffffu, ok && !ca);
    if (ok) {
      VPoint<uint32_t> q;
      q.off = (uint32_t)(y * g.pitch + x) * 4u;
      q.code = code;
      if (ca)
        vp[na + __popc(ba & below)] = q;
      else
        vp[cap - 1 - nb - __popc(bbm & below)] = q;
      xmin = min(xmin, x);
      xmax = max(xmax, x);
      ymin = min(ymin, y);
      ymax = max(ymax, y);
    }
    na += __popc(ba);
    nb += __popc(bbm);
  }
  __syncwarp();
  const int nv = na + nb;
  if (nv == 0) return o;  // no contributing point anywhere: nullopt
  xmin = __reduce_min_sync(0xffffffffu, xmin);
  ymin = __reduce_min_sync(0xffffffffu, ymin);
  xmax = __reduce_max_sync(0xffffffffu, xmax);
  ymax = __reduce_max_sync(0xffffffffu, ymax);
  const VPoint<uint32_t>* vpa = vp;
  const VPoint<uint32_t>* vpb = vp + cap - nb;
  const int ndx = rg.dx_max - rg.dx_min + 1;
  const bool fast = xmin - rg.dx_max >= g.sx0 && xmax - rg.dx_min <= g.sx1 && ymin + rg.dy_min >= g.sy0 &&
                    ymax + rg.dy_max <= g.sy1 && rg.dx_min > -32768 && rg.dx_max < 32768 &&
                    rg.dy_min >= -32768 && rg.dy_max < 32768;
  Cand best = {0, 0, 0, 0};
  if (fast) {
    unsigned long long bkey = ~0ull;
    v2_range<M_FAST>(vpa, na, vpb, nb, R, g, rg, lane, best, bkey, evals);
    const uint32_t hi = __reduce_min_sync(0xffffffffu, (uint32_t)(bkey >> 32));
    const uint32_t lo = __reduce_min_sync(0xffffffffu, (uint32_t)(bkey >> 32) == hi ? (uint32_t)bkey : ~0u);
    const int adx = (int)(lo >> 17);
    best.sum = (int)hi;
    best.n = nv;
    best.dx = (lo & 1u) ? adx : -adx;
    best.dy = (int)((lo >> 1) & 0xFFFFu) - 0x8000;
  } else {
    unsigned long long unused = 0;
    v2_range<M_SIGN>(vpa, na, vpb, nb, R, g, rg, lane, best, unused, evals);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {  // warp argmin (a total order)
      Cand u;
      u.sum = __shfl_xor_sync(0xffffffffu, best.sum, off);
      u.n = __shfl_xor_sync(0xffffffffu, best.n, off);
      u.dx = __shfl_xor_sync(0xffffffffu, best.dx, off);
      u.dy = __shfl_xor_sync(0xffffffffu, best.dy, off);
      if (better(u, best)) best = u;
    }
  }
  if (best.n == 0) return o;
  const int bix = best.dx - rg.dx_min;
  o.has = 1;
  o.dx = best.dx;
  o.dy = best.dy;
  o.sum = best.sum;
  o.n = best.n;
  o.interior = bix > 0 && bix + 1 < ndx;
  if (o.interior) {  // costs at (dx - 1, dy) and (dx + 1, dy) for the parabola
    int ms = 0, mn = 0, ps = 0, pn = 0;
    const char* rb = reinterpret_cast<const char*>(R + (int64_t)best.dy * g.pitch - best.dx);
    for (int k = lane; k < nv; k += 32) {
      const VPoint<uint32_t> q = k < na ? vpa[k] : vpb[k - na];
      const uint32_t* a = reinterpret_cast<const uint32_t*>(rb + q.off);
      const uint32_t rm = a[1], rp = a[-1];
      if (rm) {
        ms += __popc(q.code ^ rm);
        ++mn;
      }
      if (rp) {
        ps += __popc(q.code ^ rp);
        ++pn;
      }
    }
    o.cm_sum = __reduce_add_sync(0xffffffffu, ms);
    o.cm_n = __reduce_add_sync(0xffffffffu, mn);
    o.cp_sum = __reduce_add_sync(0xffffffffu, ps);
    o.cp_n = __reduce_add_sync(0xffffffffu, pn);
  }
  return o;
}

__device__ __forceinline__ void finish(const Pass& p, rg_match_result& r) {  // census.hpp:255-270
  r.has_value = 1;
  r.dx_int = p.dx;
  r.dy_int = p.dy;
  r.cost = div_int(p.sum, p.n);
  r.valid_points = p.n;
  r.dx_subpix = (double)p.dx;
  r.cost_minus = -1.0;
  r.cost_plus = -1.0;
  if (p.interior && p.cm_n > 0 && p.cp_n > 0) {
    const double cm = div_int(p.cm_sum, p.cm_n);
    const double cp = div_int(p.cp_sum, p.cp_n);
    r.cost_minus = cm;
    r.cost_plus = cp;
    r.dx_subpix = __dadd_rn((double)p.dx, subpixel(cm, r.cost, cp));
  }
}

// Occluders of `det` (index self) among the frame's detections [d0, d1)
// (find_occluders, template_match.hpp:71-89) into the warp's box list occ;
// returns whether any did not fit (the sampler then scans every detection).
// From the planner's list (ol, e.occ_n of them) when it has one.
__device__ __forceinline__ bool warp_occluders(const ObjEntry& e, const int16_t* ol, const rg_detection& det,
                                               int self, const rg_detection* dets, int d0, int d1, int img_w,
                                               int img_h, double* occ, int* nocc, int lane) {
  static_assert(kOccMax <= kWarpOcc, "the planner's list must fit the warp's boxes");
  if (e.occ_n >= 0) {
    if (lane < e.occ_n) {
      const PBox b = pixel_box(dets[d0 + ol[lane]], img_w, img_h);
      occ[4 * lane] = b.x0;
      occ[4 * lane + 1] = b.y0;
      occ[4 * lane + 2] = b.x1;
      occ[4 * lane + 3] = b.y1;
    }
    if (lane == 0) *nocc = e.occ_n;
    __syncwarp();
    return false;
  }
  if (lane == 0) *nocc = 0;
  __syncwarp();
  bool overflow = false;
  for (int j = d0 + lane; j < d1; j += 32) {
    if (j == self) continue;
    const rg_detection dj = dets[j];
    if (!dev_occludes(det, dj)) continue;
    const int k = atomicAdd(nocc, 1);
    if (k < kWarpOcc) {
      const PBox b = pixel_box(dj, img_w, img_h);
      occ[4 * k] = b.x0;
      occ[4 * k + 1] = b.y0;
      occ[4 * k + 2] = b.x1;
      occ[4 * k + 3] = b.y1;
    } else {
      overflow = true;
    }
  }
  __syncwarp();
  return __any_sync(0xffffffffu, overflow);
}

// K2a slot sampler: the QueryBlock points of every planned slot
// (sample_query_points, template_match.hpp:155-223, in the reference's grid
// order), one warp per slot, to pts[slot * maxp ...] with the count in
// slots[slot].pad.  Run ahead of the matcher so the FP64 geometry and the
// occluder scan execute at full occupancy instead of in front of each
// matcher warp's sweeps.  FAR slots are [0, counters[0]), CLOSE slots
// [capacity - counters[4], capacity) (plan.cu); an overflowed plan is left to
// the matcher, which flags it.
template <int WPB>
__global__ void __launch_bounds__(WPB * 32) sample_slots_kernel(
    Slot* __restrict__ slots, const int32_t* __restrict__ counters, const ObjEntry* __restrict__ objs,
    const int16_t* __restrict__ occ_list, const rg_detection* __restrict__ dets, const int32_t* __restrict__ det_off, int img_w, int img_h,
    SampleConst sk, int2* __restrict__ pts_out, rg_ranger_stats* __restrict__ stats, int maxp,
    int capacity) {
  __shared__ double occ[WPB][4 * kWarpOcc];
  __shared__ int nocc[WPB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.x * WPB + warp;
  const int n_lo = counters[0], n_hi = counters[4];
  if (n_lo + n_hi > capacity || counters[1]) return;
  if ((slot >= n_lo && slot < capacity - n_hi) || slot >= capacity) return;  // warp-uniform
  const Slot s = slots[slot];
  const ObjEntry e = objs[s.obj];
  const rg_detection det = dets[e.det];
  const int d0 = det_off[s.frame], d1 = det_off[s.frame + 1];
  const bool all = warp_occluders(e, occ_list + (int64_t)s.obj * kOccMax, det, e.det, dets, d0, d1, img_w, img_h,
                                  occ[warp], &nocc[warp], lane);
  const int np = dev_sample_block_warp_g(
      dev_sample_geom_k(det, e.kind, s.pad >> 16, s.pad & 0xFFFF, e.rows, e.cols, sk, img_w, img_h, recip(e.cols),
                        recip(e.rows)),
      det, occ[warp], min(nocc[warp], kWarpOcc), all ? dets + d0 : nullptr, d1 - d0, e.det - d0, img_w, img_h,
      pts_out + (size_t)slot * maxp);
  if (lane == 0) {
    slots[slot].pad = np;
    if (stats && np >= 4)
      atomicAdd(reinterpret_cast<unsigned long long*>(&stats[s.frame].query_points), (unsigned long long)np);
  }
}

// COOP (latency mode): a CTA per FAR block, its warps splitting the dx
// chunks of both passes (the FAR block is the critical path of a small
// batch: ~5x a CLOSE sub-block); CLOSE sub-blocks stay one per warp.
template <typename CT, int WPB, int MINB, int PF = 0, bool COOP = false, bool V2 = false, bool PRE = false>
__global__ void __launch_bounds__(WPB * 32, MINB) match_slots_warp_kernel(
    const int2* __restrict__ pre_pts, const Slot* __restrict__ slots, int32_t* __restrict__ counters,
    const ObjEntry* __restrict__ objs, const int16_t* __restrict__ occ_list,
    const rg_detection* __restrict__ dets, const int32_t* __restrict__ det_off,
    const CT* __restrict__ fl, const CT* __restrict__ fr, PadGeom gf,
    const CT* __restrict__ sl, const CT* __restrict__ sr, PadGeom gs, int img_w,
    int img_h, int trusted, rg_ranger_config cfg, SampleConst sk, rg_match_result* __restrict__ res,
    rg_ranger_stats* __restrict__ stats, int maxp, int capacity, int region) {
  extern __shared__ __align__(16) unsigned char wsm_raw[];
  __shared__ double occ[PRE ? 1 : WPB][4 * kWarpOcc];
  __shared__ int nocc[WPB];
  __shared__ Cand xc[WPB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot0 = blockIdx.x * WPB + warp;
  // an overflowed plan (counters[1], set by K3) is re-run with a bigger list:
  // skip it entirely; otherwise only planned slots inside the list exist
  // (FAR slots [0, counters[0]), CLOSE slots [capacity - counters[4], capacity);
  // the two regions meeting is an overflow too)
  const int n_lo = counters[0], n_hi = counters[4];
  if (n_lo + n_hi > capacity) {
    if (blockIdx.x == 0 && threadIdx.x == 0) counters[1] = 1;
    return;
  }
  if (counters[1]) return;
  auto run_slot = [&](const int slot, const int part, const int nparts) {
    // per warp: maxp sampled points + maxp valid points
    unsigned char* wbase = wsm_raw + (size_t)warp * (maxp * sizeof(int2) + (maxp + 1) * sizeof(VPoint<CT>));
    int2* pts = reinterpret_cast<int2*>(wbase);
    VPoint<CT>* vp = reinterpret_cast<VPoint<CT>*>(wbase + sizeof(int2) * maxp);
    const Slot s = slots[slot];
    int np;
    bool far;
    if constexpr (PRE) {  // K2a sampled the slot (FAR slots sit below n_lo)
      np = s.pad;
      far = slot < n_lo;
      pts = const_cast<int2*>(pre_pts) + (size_t)slot * maxp;
    } else {
      const ObjEntry e = objs[s.obj];
      const rg_detection det = dets[e.det];
      const int d0 = det_off[s.frame], d1 = det_off[s.frame + 1];
      const bool all = warp_occluders(e, occ_list + (int64_t)s.obj * kOccMax, det, e.det, dets, d0, d1, img_w, img_h,
                                  occ[warp], &nocc[warp], lane);
      np = dev_sample_block_warp_g(dev_sample_geom_k(det, e.kind, s.pad >> 16, s.pad & 0xFFFF, e.rows, e.cols, sk,
                                                     img_w, img_h, recip(e.cols), recip(e.rows)),
                                   det, occ[warp], min(nocc[warp], kWarpOcc), all ? dets + d0 : nullptr, d1 - d0,
                                   e.det - d0, img_w, img_h, pts);
      far = e.kind == RG_KIND_FAR;
    }
    rg_match_result r;
    r.dx_int = r.dy_int = 0;
    r.dx_subpix = r.cost = 0.0;
    r.cost_minus = r.cost_plus = -1.0;
    r.valid_points = r.verified = r.has_value = 0;
    r.n_points = np;
    int evals = 0;
    if (np >= 4) {  // blocks with < 4 points are dropped (:185, :219)
      const PadGeom& g = far ? gf : gs;
      const int64_t fo = (int64_t)s.frame * g.fstride + g.origin;
      const CT* L = (far ? fl : sl) + fo;
      const CT* R = (far ? fr : sr) + fo;
      const rg_search_range rg = far ? rg_search_range{0, cfg.dx_max_far, -1, 1}
                                     : rg_search_range{0, sk.dxc, -1, 1};
      auto pass = [&](int sx, int sy, const CT* A, const CT* B, const rg_search_range& q) -> Pass {
        if constexpr (V2 && sizeof(CT) == 4) {
          if (trusted && nparts == 1)
            return warp_pass_v2(pts, np, sx, sy, A, B, g, q, vp, maxp + 1, lane, evals);
        }
        return warp_pass<CT, PF>(pts, np, sx, sy, A, B, g, trusted != 0, q, vp, lane, evals, part, nparts, xc);
      };
      const Pass f = pass(0, 0, L, R, rg);
      if (f.has) {
        finish(f, r);
        const rg_search_range brg = {-rg.dx_max, -rg.dx_min, -f.dy, -f.dy};
        const Pass b = pass(-f.dx, f.dy, R, L, brg);
        if (b.has) {
          rg_match_result rb;
          finish(b, rb);
          r.verified = fabs(__dadd_rn(r.dx_subpix, rb.dx_subpix)) < cfg.tau_v;
        }
      }
    }
    evals = __reduce_add_sync(0xffffffffu, evals);
    if (lane == 0) {
      if (evals) atomicAdd(reinterpret_cast<unsigned long long*>(counters + 2), (unsigned long long)evals);
      if (part == 0) {
        res[slot] = r;
        if (!PRE && stats && np >= 4)
          atomicAdd(reinterpret_cast<unsigned long long*>(&stats[s.frame].query_points), (unsigned long long)np);
      }
    }
  };
  if (COOP) {
    // items: FAR slot b (b < n_lo, the whole CTA) or WPB CLOSE slots from
    // capacity - n_hi; a grid of about one wave walks them
    const int n_items = n_lo + (n_hi + WPB - 1) / WPB;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      if (it < n_lo) {
        run_slot(it, warp, WPB);
      } else {
        const int sl = capacity - n_hi + (it - n_lo) * WPB + warp;
        if (sl < capacity) run_slot(sl, 0, 1);  // no CTA barrier on this path
      }
    }
  } else if (!((slot0 >= n_lo && slot0 < capacity - n_hi) || slot0 >= capacity)) {  // warp-uniform
    // region 1: FAR slots only, 2: CLOSE slots only (split launches), 0: all
    if (region == 0 || (region == 1) == (slot0 < n_lo)) run_slot(slot0, 0, 1);
  }
}

template <typename CT, int WPB, int MINB, int PF = 0, bool COOP = false, bool V2 = false, bool PRE = false>
cudaError_t launch_variant(const int2* slot_pts, const Slot* slots, int32_t* counters, int slot_capacity,
                                  const ObjEntry* objs, const int16_t* occ_list, const rg_detection* dets,
                                  const int32_t* det_off,
                                  const void* fl, const void* fr, const PadGeom& gf, const void* sl,
                                  const void* sr, const PadGeom& gs, int img_w, int img_h, int trusted,
                                  rg_ranger_config cfg, rg_match_result* res, rg_ranger_stats* stats,
                                  int max_points, cudaStream_t s, int region = 0) {
  auto kern = match_slots_warp_kernel<CT, WPB, MINB, PF, COOP, V2, PRE>;
  max_points = (max_points + 1) & ~1;  // keeps every warp's VPoint array 16-B aligned
  const size_t smem = (sizeof(int2) * (size_t)max_points + sizeof(VPoint<CT>) * (size_t)(max_points + 1)) * WPB;
  // the opt-in covers static + dynamic shared memory (occluder boxes etc. are static)
  static const size_t static_smem = [&] {
    cudaFuncAttributes fa{};
    return cudaFuncGetAttributes(&fa, (const void*)kern) == cudaSuccess ? fa.sharedSizeBytes : (size_t)0;
  }();
  if (static_smem + smem > kSmemPerBlockOptIn) return cudaErrorInvalidConfiguration;  // caller: fewer warps
  static SmemAttr attr;  // one per instantiation
  if (static_smem + smem > 48 * 1024) {
    const cudaError_t e = attr.ensure((const void*)kern, smem);
    if (e != cudaSuccess) return e;
  }
  // COOP: about one wave of CTAs walks the work items (their count is only
  // known on the device)
  const int grid = COOP ? std::min(slot_capacity, 148 * MINB) : (slot_capacity + WPB - 1) / WPB;
  if (PRE && !slot_pts) return cudaErrorInvalidValue;
  kern<<<grid, WPB * 32, smem, s>>>(slot_pts, slots, counters, objs, occ_list, dets, det_off,
                                    static_cast<const CT*>(fl),
                                    static_cast<const CT*>(fr), gf, static_cast<const CT*>(sl),
                                    static_cast<const CT*>(sr), gs, img_w, img_h, trusted, cfg,
                                    make_sample_const(cfg, img_w, img_h), res, stats,
                                    max_points, slot_capacity, region);
  return cudaGetLastError();
}

}  // namespace

namespace {
int match_variant() {
  static const int v = [] {
    const char* e = getenv("RG_MATCH_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}
}  // namespace

bool match_presampled(int n_frames, int wide) {
  // A/B knob RG_MATCH_PRE=1: K2a ahead of the matcher.  Measured at C2
  // (256 frames): K2a 0.124 ms, the matcher 0.894 -> 0.810 ms -- a net loss
  // of 0.04 ms (the in-warp sampling overlaps other warps' sweeps; alone it
  // is ~600 instructions per slot, mostly FP64 divisions), so off by default
  static const bool on = [] {
    const char* v = getenv("RG_MATCH_PRE");
    return v ? atoi(v) != 0 : false;
  }();
  return on && match_variant() == 0 && !(n_frames > 0 && n_frames <= kLatencyFrames);
}

cudaError_t launch_sample_slots(Slot* slots, const int32_t* counters, int slot_capacity, const ObjEntry* objs,
                                const int16_t* occ_list, const rg_detection* dets, const int32_t* det_off, int img_w, int img_h,
                                rg_ranger_config cfg, int2* slot_pts, rg_ranger_stats* stats, int max_points,
                                cudaStream_t s) {
  if (slot_capacity <= 0) return cudaSuccess;
  constexpr int SW = 8;
  sample_slots_kernel<SW><<<(slot_capacity + SW - 1) / SW, SW * 32, 0, s>>>(
      slots, counters, objs, occ_list, dets, det_off, img_w, img_h, make_sample_const(cfg, img_w, img_h), slot_pts,
      stats,
      (max_points + 1) & ~1, slot_capacity);
  return cudaGetLastError();
}

cudaError_t launch_match_slots(const int2* slot_pts, const Slot* slots, int32_t* counters, int slot_capacity,
                               const ObjEntry* objs, const int16_t* occ_list, const rg_detection* dets, const int32_t* det_off,
                               const void* fl, const void* fr, const PadGeom& gf, const void* sl,
                               const void* sr, const PadGeom& gs, int img_w, int img_h, int trusted,
                               int wide, rg_ranger_config cfg, rg_match_result* res,
                               rg_ranger_stats* stats, int max_points, cudaStream_t s,
                               int n_frames, int region) {
  if (slot_capacity <= 0) return cudaSuccess;
  const int variant = match_variant();
#define RG_ARGS slot_pts, slots, counters, slot_capacity, objs, occ_list, dets, det_off, fl, fr, gf, sl, sr, gs, img_w, img_h, \
                trusted, cfg, res, stats, max_points, s, region
  // blocks too large for the default warps per CTA fall back to fewer
  // (shared memory holds every warp's points: 16 or 24 B per point)
  auto fallback = [&](cudaError_t e, auto... launchers) {
    ((e = (e == cudaErrorInvalidConfiguration ? launchers() : e)), ...);
    return e;
  };
  if (wide)  // 9x7 extension
    return fallback(slot_pts ? launch_variant<unsigned long long, 8, 2, 0, false, false, true>(RG_ARGS)
                             : launch_variant<unsigned long long, 8, 2>(RG_ARGS),
                    [&] { return launch_variant<unsigned long long, 2, 8>(RG_ARGS); },
                    [&] { return launch_variant<unsigned long long, 1, 16>(RG_ARGS); });
  auto small = [&](cudaError_t e) {
    return fallback(e, [&] { return launch_variant<uint32_t, 8, 4>(RG_ARGS); },
                    [&] { return launch_variant<uint32_t, 2, 8>(RG_ARGS); },
                    [&] { return launch_variant<uint32_t, 1, 16>(RG_ARGS); });
  };
  // latency mode (a few frames): most SMs would idle and the FAR blocks are
  // the critical path, so one CTA per FAR block splits its passes over 4
  // warps (single C2 frame: 84 -> 43 us).  The L1 prefetch of the point 4
  // ahead paid 2 us until the padded rasters got 128-B aligned rows; now it
  // costs 2 us (variant 7 keeps it); 8 or 16 warps per FAR block measured
  // 47 / 80 us (variants 5, 6).
  if (variant == 0 && n_frames > 0 && n_frames <= kLatencyFrames) {
    static const int lw = [] { const char* v = getenv("RG_LAT_WARPS"); return v ? atoi(v) : 4; }();
    switch (lw) {
      case 8: return small(launch_variant<uint32_t, 8, 6, 0, true>(RG_ARGS));
      case 12: return small(launch_variant<uint32_t, 12, 4, 0, true>(RG_ARGS));
      case 16: return small(launch_variant<uint32_t, 16, 3, 0, true>(RG_ARGS));
      default: return small(launch_variant<uint32_t, 4, 12, 0, true>(RG_ARGS));
    }
  }
  switch (variant) {  // A/B knobs; default measured best (tools/census_time.py with RG_MATCH_VARIANT)
    case 1: return launch_variant<uint32_t, 8, 4>(RG_ARGS);
    case 2: return launch_variant<uint32_t, 8, 5>(RG_ARGS);
    case 3: return launch_variant<uint32_t, 16, 4>(RG_ARGS);
    case 4: return launch_variant<uint32_t, 4, 12, 0, true>(RG_ARGS);
    case 5: return launch_variant<uint32_t, 8, 6, 4, true>(RG_ARGS);
    case 6: return launch_variant<uint32_t, 16, 3, 4, true>(RG_ARGS);
    case 7: return launch_variant<uint32_t, 4, 12, 4, true>(RG_ARGS);
    // 8-10: the vectorised carry-save sweep (warp_pass_v2), measured slower
    // (1.26-1.75 vs 0.90 ms per 256 C2 frames: long-scoreboard stalls at
    // 64 registers / 50 % occupancy, spills at 40)
    case 8: return launch_variant<uint32_t, 16, 3, 0, false, true>(RG_ARGS);
    case 9: return launch_variant<uint32_t, 8, 4, 0, false, true>(RG_ARGS);
    case 10: return launch_variant<uint32_t, 16, 2, 0, false, true>(RG_ARGS);
    default:
      return small(slot_pts ? launch_variant<uint32_t, 16, 3, 0, false, false, true>(RG_ARGS)
                                   : launch_variant<uint32_t, 16, 3>(RG_ARGS));
  }
#undef RG_ARGS
}

// c_recip of the current device: RN(1 / b) (IEEE host division), b <= kRecip
cudaError_t init_match_tables() {
  static double tab[kRecip + 1];
  static const bool filled = [] {
    tab[0] = 0.0;
    for (int b = 1; b <= kRecip; ++b) tab[b] = 1.0 / (double)b;
    return true;
  }();
  (void)filled;
  return cudaMemcpyToSymbol(c_recip, tab, sizeof(tab));
}

// div_int vs __ddiv_rn over b in [1, b_max], a in [0, 64 b]: mismatches
cudaError_t selftest_division(int b_max, unsigned long long* d_bad, cudaStream_t s) {
  b_max = std::min(std::max(b_max, 1), kRecip + 64);
  selftest_div_kernel<<<b_max, 256, 0, s>>>(b_max, d_bad);
  return cudaGetLastError();
}

}  // namespace rg
