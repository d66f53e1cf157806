// Standalone probe of the TMA path used by census_tma_kernel (debug tool).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, int mode, int cx, int cy,
                      uint8_t* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* dst = sm + 1024;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar)));
    if (mode & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if ((mode & 4) && threadIdx.x == 0)
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(gtm) : "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(144 * 68) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(su(dst)), "l"((mode & 4) ? (const void*)gtm : (const void*)&tm), "r"(cx), "r"(cy), "r"(0), "r"(su(bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(su(bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 144 * 68; i += blockDim.x) out[i] = dst[i];
}

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 64, H = argc > 2 ? atoi(argv[2]) : 48;
  const int mode = argc > 3 ? atoi(argv[3]) : 1;
  std::vector<uint8_t> img(W * H);
  for (int i = 0; i < W * H; ++i) img[i] = (uint8_t)(i * 7 + 3);
  uint8_t *d, *o;
  cudaMalloc(&d, W * H);
  cudaMalloc(&o, 144 * 68);
  cudaMemcpy(d, img.data(), W * H, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1};
  cuuint64_t str[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
  cuuint32_t box[3] = {144, 68, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d fn=%p q=%d\n", (int)r, fn, (int)q);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 144 * 68);
  CUtensorMap* gtm;
  cudaMalloc(&gtm, sizeof(CUtensorMap));
  cudaMemcpy(gtm, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  const int cx = argc > 4 ? atoi(argv[4]) : ((mode & 2) ? 0 : -8), cy = argc > 5 ? atoi(argv[5]) : ((mode & 2) ? 0 : -2);
  probe<<<1, 128, 1024 + 144 * 68>>>(tm, gtm, mode, cx, cy, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint8_t> h(144 * 68);
  cudaMemcpy(h.data(), o, h.size(), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r0 = 0; r0 < 68; ++r0)
    for (int c = 0; c < 144; ++c) {
      const int x = c + cx, y = r0 + cy;
      const uint8_t want = (x >= 0 && x < W && y >= 0 && y < H) ? img[y * W + x] : 0;
      bad += h[r0 * 144 + c] != want;
    }
  printf("mismatches %d\n", bad);
  return 0;
}
