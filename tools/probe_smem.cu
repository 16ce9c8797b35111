// Probe: where does dynamic shared memory start (mod 1024) with and without static smem?
#include <cstdio>
#include <cstdint>
__global__ void k_nostatic(unsigned* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (threadIdx.x == 0) out[0] = static_cast<unsigned>(__cvta_generic_to_shared(smem_raw));
}
__global__ void k_static(unsigned* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ unsigned long long bar[3];
  if (threadIdx.x == 0) {
    bar[0] = 1;
    out[1] = static_cast<unsigned>(__cvta_generic_to_shared(smem_raw));
    out[2] = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  }
}
int main() {
  unsigned* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k_nostatic, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k_static, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  k_nostatic<<<1, 32, 200000>>>(d);
  k_static<<<1, 32, 200000>>>(d);
  unsigned h[4]; cudaMemcpy(h, d, 12, cudaMemcpyDeviceToHost);
  int maxopt = 0; cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  int resv = 0; cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, 0);
  printf("dyn base (no static) = %u (mod 1024 = %u); dyn base (static) = %u (mod 1024 = %u), static at %u; optin max %d reserved %d\n",
         h[0], h[0] % 1024, h[1], h[1] % 1024, h[2], maxopt, resv);
}
