// Tensor-pipe microbenchmark of the dK/dV unit sequence (1 CTA):
//   dV: 4 × TS 128x128x16 (A = TMEM cols a0..), S: 8 × SS 128x64x16 → cols s0,
//   dK: 4 × TS (A = cols a1..),                 dP: 8 × SS 128x64x16 → cols s1
// alias=1: S/dP overwrite the columns dV/dK read as A (the kernel's scheme); alias=0: disjoint.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_11101_b200/csrc tools/mma_seq.cu -o tools/mma_seq
#include <cstdio>
#include "sm100.cuh"
using namespace vlasim_dev;

__global__ void __launch_bounds__(576, 1) k_seq(int iters, int alias, int commits, int variant, unsigned long long* out,
                                                 const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i == 131068 / 4 ? 0u : 0x3c003c00u;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint64_t dK = make_sdesc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t dQ = make_sdesc_sw128(smem_u32(smem + 65536), 16, 1024);
    const uint64_t dQm = make_sdesc_sw128(smem_u32(smem + 65536), 8192, 1024);
    constexpr uint32_t id_s = make_idesc_bf16(128, 64, false, false);
    constexpr uint32_t id_acc = make_idesc_bf16(128, 128, false, true);
    const long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
        const int b = it & 1;
        const uint32_t scol = b ? 64 : 0, dpcol = b ? 192 : 128;
        const uint32_t a_s = alias ? scol : 0, a_dp = alias ? dpcol : 128;  // A columns read by dV / dK
        const uint32_t w_s = alias ? scol : 64, w_dp = alias ? dpcol : 192;  // columns S/dP write
        if (variant == 2 && false) {  // all four GEMMs as SS N=128 (old 128-wide design shape)
          for (int j = 0; j < 8; ++j) umma_f16_ss(tmem + 256, sdesc_add(dK, (j % 4) * 32), sdesc_add(dQ, (j % 4) * 32), id_acc, 1);
          for (int j = 0; j < 8; ++j) umma_f16_ss(tmem, sdesc_add(dK, (j % 4) * 32), sdesc_add(dQ, (j % 4) * 32), id_acc, 1);
          for (int j = 0; j < 8; ++j) umma_f16_ts(tmem + 384, tmem + 128 + j * 8, sdesc_add(dQm, j * 2048), id_acc, 1);
          for (int j = 0; j < 8; ++j) umma_f16_ss(tmem + 128, sdesc_add(dK, (j % 4) * 32), sdesc_add(dQ, (j % 4) * 32), id_acc, 1);
          if (commits) umma_commit(&bar[0]);
          continue;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          umma_f16_ts(tmem + 256, tmem + a_s + (j >> 1) * 32 + (j & 1) * 8, sdesc_add(dQm, j * 2048), id_acc, 1);
        if (commits) umma_commit(&bar[0]);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          umma_f16_ss(tmem + w_s, sdesc_add(dK, (j / 4) * 16384 + (j % 4) * 32), sdesc_add(dQ, (j / 4) * 8192 + (j % 4) * 32), id_s, j > 0);
        if (commits) umma_commit(&bar[1]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          umma_f16_ts(tmem + 384, tmem + a_dp + (j >> 1) * 32 + (j & 1) * 8, sdesc_add(dQm, j * 2048), id_acc, 1);
        if (commits) umma_commit(&bar[2]);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          umma_f16_ss(tmem + w_dp, sdesc_add(dK, (j / 4) * 16384 + (j % 4) * 32), sdesc_add(dQ, (j / 4) * 8192 + (j % 4) * 32), id_s, j > 0);
        if (commits) umma_commit(&bar[3]);
      }
      umma_commit(&bar[0]);
    }
    __syncwarp();
    // wait for the final commit: count phases on bar[0]
    const int phases = commits ? iters + 1 : 1;
    mbar_wait(&bar[0], (phases - 1) & 1);
    const long long t1 = clock64();
    if (threadIdx.x == 0) atomicMax(&out[0], (unsigned long long)(t1 - t0));
    if (threadIdx.x == 0) *reinterpret_cast<volatile int*>(smem + 131068) = 1;  // stop flag
  } else if (warp == 1 && variant == 11) {
    // TMA-like load traffic: 32 KB bulk copies global → smem [131072, 196608) back to back
    __shared__ uint64_t lbar;
    if (threadIdx.x == 32) {
      mbar_init(&lbar, 1);
      fence_barrier_init();
      int n = 0;
      while (*reinterpret_cast<volatile int*>(smem + 131068) == 0 && n < 100000) {
        mbar_expect_tx(&lbar, 32768);
        for (int c = 0; c < 2; ++c)
          bulk_load(smem + 131072 + c * 16384, gsrc + (size_t(n % 4096) * 32768 + c * 16384), 16384, &lbar);
        mbar_wait(&lbar, n & 1);
        ++n;
      }
      out[6] = n;
    }
  } else if (warp >= 2 && variant >= 10) {
    // softmax-like ALU/MUFU load (variant 10: exp loop)
    float x = threadIdx.x * 1e-3f, acc = 0.f;
    int n = 0;
    while (*reinterpret_cast<volatile int*>(smem + 131068) == 0 && n < 4000000) {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += ex2_approx(fmaf(x, 1.0001f, -acc * 1e-6f + j));
      ++n;
    }
    if (acc == 1.2345f) out[5] = n;
  } else if (warp >= 2) {
    // softmax-like TMEM traffic: ld32 + wait, st16 + wait on this warp's lane quadrant (cols 0..63)
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t col = (warp & 4) ? 32 : 0;
    unsigned long long n = 0, lat = 0;
    while (*reinterpret_cast<volatile int*>(smem + 131068) == 0 && n < 200000) {
      const long long a = clock64();
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + 448 + col, r);
      tmem_wait_ld();
      uint32_t w[16];
      for (int j = 0; j < 16; ++j) w[j] = r[2 * j] ^ r[2 * j + 1];
      tmem_st16(tmem + lane_off + 448 + col, w);
      tmem_wait_st();
      lat += clock64() - a;
      ++n;
    }
    if ((threadIdx.x & 31) == 0) { atomicAdd(&out[1], n); atomicAdd(&out[2], lat); }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  uint8_t* g;
  cudaMalloc(&g, size_t(4096) * 32768);
  cudaMemset(g, 0, size_t(4096) * 32768);
  const int iters = 1000;
  struct { int alias, commits, variant; const char* name; } cases[] = {
      {1, 1, 0, "kernel scheme (alias, commits)"}, {1, 0, 0, "alias, no commits"},
      {0, 1, 0, "disjoint cols, commits"}, {0, 0, 0, "disjoint, no commits"},
      {1, 1, 10, "kernel scheme + 16 exp-busy warps"}, {1, 1, 11, "kernel scheme + TMA load warp"}};
  for (int blocks : {1, 148})
  for (int thr : {64, 64 + 512}) {
    for (auto& c : cases) {
      cudaMemset(d, 0, 64);
      k_seq<<<blocks, thr, 196608>>>(10, c.alias, c.commits, c.variant, d, g);
      cudaMemset(d, 0, 64);
      k_seq<<<blocks, thr, 196608>>>(iters, c.alias, c.commits, c.variant, d, g);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[8];
      cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
      if (c.variant == 11) printf("   TMA loads of 32 KB: %llu\n", h[6]);
      printf("blocks %3d ldst warps %2d  %-40s %.0f cycles/unit (model 1280)  ld+st iters %llu avg %.0f cyc  %s\n", blocks, (thr - 64) / 32,
             c.name, double(h[0]) / iters, h[1], h[1] ? double(h[2]) / h[1] : 0.0, cudaGetErrorString(e));
    }
  }
  return 0;
}
