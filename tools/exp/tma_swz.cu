// Experiment: where does a SWIZZLE_128B TMA box land when its shared-memory
// destination is 128 B (not 1024 B) aligned?  Prints, for each destination
// row offset k, the chunk permutation observed for every landed row.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, int roff, int z0, float* out) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) sm[i] = -1.f;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(4 * 128));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su(sm + roff * 32)), "l"((uint64_t)&m), "r"(0), "r"(z0), "r"(su(&bar)) : "memory");
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(su(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) out[i] = sm[i];
}
int main() {
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  const int W = 32, Hh = 64;
  std::vector<float> h(W * Hh);
  for (int r = 0; r < Hh; ++r) for (int c = 0; c < W; ++c) h[r * W + c] = r * 100 + c;  // value = row*100 + float index
  float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 16 * 32 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap m; cuuint64_t dims[2] = {W, Hh}; cuuint64_t str[1] = {W * 4}; cuuint32_t box[2] = {32, 4}; cuuint32_t es[2] = {1, 1};
  int rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", rc);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096);
  for (int roff : {0, 1, 3, 5, 8}) {
    k<<<1, 128, 4096>>>(m, roff, 8 + roff, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> r(16 * 32); cudaMemcpy(r.data(), o, r.size() * 4, cudaMemcpyDeviceToHost);
    printf("roff %d err %s\n", roff, cudaGetErrorString(e));
    for (int row = 0; row < 16; ++row) {
      if (r[row * 32] < 0 && r[row * 32 + 4] < 0) continue;
      printf("  smem row %2d:", row);
      for (int ch = 0; ch < 8; ++ch) { float v = r[row * 32 + ch * 4]; printf(" %4.0f", v); }
      printf("\n");
    }
  }
  return 0;
}
