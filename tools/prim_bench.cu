// Latency of the synchronisation primitives used by the attention kernels (1 CTA, warp 0 times).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_11101_b200/csrc tools/prim_bench.cu -o tools/prim_bench
#include <cstdio>
#include "sm100.cuh"
using namespace vlasim_dev;

__global__ void __launch_bounds__(576, 1) k_prim(unsigned long long* out, int busy) {
  __shared__ uint64_t never;
  if (threadIdx.x == 0) mbar_init(&never, 1);
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int N = 1000;
  if (warp == 0) {
    long long t0, t1;
    // (a) commit (no MMAs outstanding) + wait for its arrival
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
      if (elect_one()) umma_commit(&bar[0]);
      __syncwarp();
      mbar_wait(&bar[0], i & 1);
    }
    t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0) / N;
    // (b) commit issue only (no wait)
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
      if (elect_one()) umma_commit(&bar[1]);
      __syncwarp();
    }
    t1 = clock64();
    if (lane == 0) out[1] = (t1 - t0) / N;
    // (c) tcgen05.fence::after_thread_sync
    t0 = clock64();
    for (int i = 0; i < N; ++i) tc_fence_after();
    t1 = clock64();
    if (lane == 0) out[2] = (t1 - t0) / N;
    // (d) st16 + wait::st
    uint32_t z[16] = {0};
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
      tmem_st16(tmem + (i & 7) * 16, z);
      tmem_wait_st();
    }
    t1 = clock64();
    if (lane == 0) out[3] = (t1 - t0) / N;
    // (e) ld32 + wait::ld
    uint32_t r[32];
    unsigned acc = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
      tmem_ld32(tmem + (i & 7) * 32, r);
      tmem_wait_ld();
      acc += r[i & 31];
    }
    t1 = clock64();
    if (lane == 0) out[4] = (t1 - t0) / N;
    // (f) mbarrier arrive (1 thread) + wait by the warp (self-handshake)
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
      if (lane == 0) mbar_arrive(&bar[2]);
      mbar_wait(&bar[2], i & 1);
    }
    t1 = clock64();
    if (lane == 0) out[5] = (t1 - t0) / N;
    // (g) fence_before + syncwarp + arrive + wait
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
      tc_fence_before();
      warp_arrive(&bar[3]);
      mbar_wait(&bar[3], i & 1);
    }
    t1 = clock64();
    if (lane == 0) out[6] = (t1 - t0) / N;
    // (h) clock64 pair
    t0 = clock64();
    long long x = 0;
    for (int i = 0; i < N; ++i) x += clock64();
    t1 = clock64();
    if (lane == 0) { out[7] = (t1 - t0) / N; out[8] = acc + (x & 1); }
    if (lane == 0) mbar_arrive(&never);  // release the pollers
  } else if (busy == 2) {
    mbar_wait(&never, 0);  // poll until warp 0 is done
  } else if (busy == 1) {
    float a = threadIdx.x;
    for (int i = 0; i < 200000; ++i) a = ex2_approx(a * 0.999f);
    if (a == 1.234f) out[9] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 128);
  const char* names[] = {"commit + wait arrival", "commit issue (+syncwarp)", "tc_fence_after", "tmem st16 + wait::st",
                         "tmem ld32 + wait::ld", "arrive + wait (self)", "fence+warp_arrive+wait", "clock64"};
  for (int busy = 0; busy < 3; ++busy) {
    k_prim<<<1, 576>>>(d, busy);
    k_prim<<<1, 576>>>(d, busy);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[10];
    cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
    printf("busy=%d (%s)\n", busy, cudaGetErrorString(e));
    for (int i = 0; i < 8; ++i) printf("  %-28s %llu cycles\n", names[i], h[i]);
  }
  return 0;
}
