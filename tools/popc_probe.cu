// Measurement tool: per-SM throughput of the matcher's integer pipes on this
// GPU ("POPC 16/clk/SM on cc 8.x-9.0 ... confirm for cc 10.0
// with a microbenchmark").  Each thread runs long chains of independent
// POPC / LOP3 / IADD3 over 8 accumulators; results are kept live through a
// store.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a popc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void popc_kernel(const unsigned* __restrict__ in, unsigned* out) {
  unsigned a[8], s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = in[(threadIdx.x + i) & 255], s[i] = 0;
  for (int k = 0; k < ITERS; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s[i] += __popc(a[i] ^ k);  // LOP3 + POPC + IADD: the matcher's evaluation
    }
  }
  unsigned t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void popc_only_kernel(const unsigned* __restrict__ in, unsigned* out) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = in[(threadIdx.x + i) & 255];
  for (int k = 0; k < ITERS; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __popc(a[i]) + a[(i + 1) & 7];  // POPC + IADD dependent pairs
  }
  unsigned t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void lop3_kernel(const unsigned* __restrict__ in, unsigned* out) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = in[(threadIdx.x + i) & 255];
  for (int k = 0; k < ITERS; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (a[i] ^ a[(i + 1) & 7]) & (a[(i + 3) & 7] | (unsigned)k);
  }
  unsigned t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <typename K>
double run(K kern, const unsigned* in, unsigned* out, int sms, double ops_per_thread_iter) {
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
  const double ops = 5.0 * blocks * threads * (double)ITERS * ops_per_thread_iter;
  const double per_s = ops / (ms * 1e-3);
  return per_s / sms / (clk_khz * 1e3);  // per clock per SM at the max clock
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *in, *out;
  cudaMalloc(&in, 256 * sizeof(unsigned));
  cudaMemset(in, 0x5a, 256 * sizeof(unsigned));
  cudaMalloc(&out, (size_t)sms * 8 * 256 * sizeof(unsigned));
  const double evals = run(popc_kernel, in, out, sms, 8.0);      // XOR+POPC+IADD per eval
  const double popcs = run(popc_only_kernel, in, out, sms, 8.0); // POPC per op
  const double lops = run(lop3_kernel, in, out, sms, 8.0);       // ~2 logic ops fused per op
  printf("{\"sms\": %d, \"evals_per_clk_per_sm\": %.2f, \"popc_per_clk_per_sm\": %.2f, "
         "\"lop3_chains_per_clk_per_sm\": %.2f, \"note\": \"clock = cudaDevAttrClockRate (max); "
         "evals = XOR+POPC+IADD per lane\"}\n",
         sms, evals, popcs, lops);
  return 0;
}
