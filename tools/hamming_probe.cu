// Measurement tool: Hamming-sum throughput of three evaluation schemes on
// this GPU (register operands, no loads), in "evaluations" = one
// popcount(l ^ r) added into a per-candidate sum, per clock per SM.
//   naive : s += popc(l ^ r)                       (LOP3 + POPC + IADD per eval)
//   csa3  : 3 evals -> (ones, twos) by a carry-save adder, 2 POPC per 3 evals
//   csa7  : 7 evals -> (ones, twos, fours), 3 POPC per 7 evals
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a hamming_probe.cu -o hamming_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

__device__ __forceinline__ unsigned maj3(unsigned a, unsigned b, unsigned c) { return (a & b) | (c & (a | b)); }

// 8 independent candidates per thread, each accumulating ITERS*NW evals
__global__ void naive_kernel(const unsigned* __restrict__ in, unsigned* out) {
  unsigned r[8], s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = in[(threadIdx.x * 3 + i) & 255], s[i] = 0;
  for (int k = 0; k < ITERS; ++k) {
    const unsigned l0 = in[k & 255] ^ k, l1 = l0 * 2654435761u, l2 = l1 ^ 0x9e3779b9u;
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] += __popc(l0 ^ r[i]) + __popc(l1 ^ r[i]) + __popc(l2 ^ r[(i + 1) & 7]);
  }
  unsigned t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void csa3_kernel(const unsigned* __restrict__ in, unsigned* out) {
  unsigned r[8], s1[8], s2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = in[(threadIdx.x * 3 + i) & 255], s1[i] = s2[i] = 0;
  for (int k = 0; k < ITERS; ++k) {
    const unsigned l0 = in[k & 255] ^ k, l1 = l0 * 2654435761u, l2 = l1 ^ 0x9e3779b9u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const unsigned x0 = l0 ^ r[i], x1 = l1 ^ r[i], x2 = l2 ^ r[(i + 1) & 7];
      s1[i] += __popc(x0 ^ x1 ^ x2);
      s2[i] += __popc(maj3(x0, x1, x2));
    }
  }
  unsigned t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += s1[i] + 2 * s2[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void csa7_kernel(const unsigned* __restrict__ in, unsigned* out) {
  unsigned r[4], s1[4], s2[4], s4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) r[i] = in[(threadIdx.x * 3 + i) & 255], s1[i] = s2[i] = s4[i] = 0;
  for (int k = 0; k < ITERS; ++k) {
    unsigned l[7];
    l[0] = in[k & 255] ^ k;
#pragma unroll
    for (int j = 1; j < 7; ++j) l[j] = l[j - 1] * 2654435761u + j;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      unsigned x[7];
#pragma unroll
      for (int j = 0; j < 7; ++j) x[j] = l[j] ^ r[(i + j) & 3];
      // CSA tree: (x0,x1,x2) -> a1,a2 ; (x3,x4,x5) -> b1,b2 ; (a1,b1,x6) -> o,c2 ; (a2,b2,c2) -> t,f
      const unsigned a1 = x[0] ^ x[1] ^ x[2], a2 = maj3(x[0], x[1], x[2]);
      const unsigned b1 = x[3] ^ x[4] ^ x[5], b2 = maj3(x[3], x[4], x[5]);
      const unsigned o = a1 ^ b1 ^ x[6], c2 = maj3(a1, b1, x[6]);
      const unsigned t = a2 ^ b2 ^ c2, f = maj3(a2, b2, c2);
      s1[i] += __popc(o);
      s2[i] += __popc(t);
      s4[i] += __popc(f);
    }
  }
  unsigned t = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) t += s1[i] + 2 * s2[i] + 4 * s4[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <typename K>
double run(K kern, const unsigned* in, unsigned* out, int sms, double evals_per_thread_iter) {
  const int blocks = sms * 8, threads = 256;
  kern<<<blocks, threads>>>(in, out);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(in, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double ev = 5.0 * blocks * threads * (double)ITERS * evals_per_thread_iter;
  return ev / (ms * 1e-3) / sms / (clk_khz * 1e3);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *in, *out;
  cudaMalloc(&in, 256 * sizeof(unsigned));
  cudaMalloc(&out, sms * 8 * 256 * sizeof(unsigned));
  cudaMemset(in, 0x5a, 256 * sizeof(unsigned));
  const double a = run(naive_kernel, in, out, sms, 24);
  const double b = run(csa3_kernel, in, out, sms, 24);
  const double c = run(csa7_kernel, in, out, sms, 28);
  printf("{\"sms\": %d, \"naive_evals_per_clk_per_sm\": %.2f, \"csa3_evals_per_clk_per_sm\": %.2f, "
         "\"csa7_evals_per_clk_per_sm\": %.2f}\n", sms, a, b, c);
  return 0;
}
