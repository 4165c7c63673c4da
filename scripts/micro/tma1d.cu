// Minimal 1-D TMA row-copy check (debug aid for the blur staging).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int x, int variant) {
  __shared__ __align__(128) float buf[64];
  __shared__ __align__(8) unsigned long long bar;
  unsigned b = su(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
    if (variant == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(64 * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                 ::"r"(su(buf)), "l"((unsigned long long)&tm), "r"(x), "r"(b) : "memory");
  }
  unsigned ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(b), "r"(0) : "memory");
  } while (!ok);
  if (threadIdx.x < 64) out[threadIdx.x] = buf[threadIdx.x];
}
int main() {
  float h[1000]; for (int i = 0; i < 1000; ++i) h[i] = i;
  float *d, *o; cudaMalloc(&d, 4000); cudaMalloc(&o, 256); cudaMemcpy(d, h, 4000, cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap tm; cuuint64_t gd[1] = {1000}, gs[1] = {4}; cuuint32_t bx[1] = {64}, es[1] = {1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, d, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int variant = 0; variant < 2; ++variant)
    for (int x : {0, 5, -3, 990}) {
      k<<<1, 64>>>(tm, o, x, variant);
      cudaError_t e = cudaDeviceSynchronize();
      float ho[64]; cudaMemcpy(ho, o, 256, cudaMemcpyDeviceToHost);
      printf("variant %d x=%d err=%s  first %g %g last %g\n", variant, x, cudaGetErrorString(e), ho[0], ho[1], ho[63]);
      if (e != cudaSuccess) return 1;
    }
}
