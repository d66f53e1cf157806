// Measurement tool: a kernel reading pinned host memory directly over PCIe
// (zero-copy, 16-B loads per thread, whole rows per warp) vs the DMA copy
// engine (cudaMemcpyAsync) for the same bytes.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a zerocopy_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void gather_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t bytes = 256ull << 20;
  void *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaMalloc(&d, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    for (int i = 0; i < 8; ++i) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("{\"dma_h2d_gbs\": %.1f", 8.0 * bytes / (ms * 1e-3) / 1e9);
  void* hd = nullptr;
  cudaHostGetDevicePointer(&hd, h, 0);
  for (int blocks : {148 * 4, 148 * 16, 148 * 64}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      for (int i = 0; i < 8; ++i)
        gather_kernel<<<blocks, 256>>>((const uint4*)hd, (uint4*)d, bytes / 16);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf(", \"zerocopy_%d_ctas_gbs\": %.1f", blocks, 8.0 * bytes / (ms * 1e-3) / 1e9);
  }
  printf("}\n");
  return 0;
}
