// selftest.cu — single-CTA tcgen05 GEMM that exercises exactly the operand layouts the
// attention kernels use (K-major / MN-major SWIZZLE_128B smem operands fed by TMA, and
// an A operand staged in TMEM).  Tests compare it with a torch fp32 matmul.
#include "common.hpp"
#include "sm100.cuh"

using namespace vlasim_dev;

namespace {

constexpr int kThreads = 128;

__global__ void __launch_bounds__(kThreads, 1)
    umma_selftest_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int mode,
                         const __nv_bfloat16* __restrict__ a_glob, float* __restrict__ c, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // 64 KB
  uint8_t* sB = smem + 64 * 1024;   // 128 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  if (tid == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  // ---- loads
  if (tid == 0) {
    uint32_t bytes = 0;
    if (mode == 0 || mode == 1 || mode == 2 || mode == 4) {
      if (mode != 2) {
        for (int i = 0; i < K / 64; ++i) tma_load_2d(sA + i * 128 * 128, &tmA, i * 64, 0, &bar_load);
        bytes += 128 * K * 2;
      }
    } else {  // mode 3: A stored [K, 128]; two 64-wide MN boxes of K rows
      for (int j = 0; j < 2; ++j) tma_load_2d(sA + j * K * 128, &tmA, j * 64, 0, &bar_load);
      bytes += 128 * K * 2;
    }
    if (mode == 0) {  // B [N, K] K-major
      for (int i = 0; i < K / 64; ++i) tma_load_2d(sB + i * N * 128, &tmB, i * 64, 0, &bar_load);
    } else {          // B [K, N] MN-major
      for (int j = 0; j < N / 64; ++j) tma_load_2d(sB + j * K * 128, &tmB, j * 64, 0, &bar_load);
    }
    bytes += N * K * 2;
    mbar_expect_tx(&bar_load, bytes);
  }
  if (mode == 2) {  // stage A[row, :] in TMEM columns [256, 256 + K/2)
    const int row = tid;
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        __nv_bfloat162 v;
        v.x = a_glob[row * K + 2 * (c0 + j)];
        v.y = a_glob[row * K + 2 * (c0 + j) + 1];
        r[j] = *reinterpret_cast<uint32_t*>(&v);
      }
      tmem_st16(tmem + ((warp * 32) << 16) + 256 + c0, r);
    }
    tmem_wait_st();
  }
  mbar_wait(&bar_load, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // ---- MMA (one thread)
  if (tid == 0) {
    const bool a_mn = (mode == 3), b_mn = (mode != 0);
    const uint32_t idesc = make_idesc_bf16(128, N, a_mn, b_mn);
    const uint32_t sa = smem_u32(sA), sb = smem_u32(sB);
    if (mode == 4)  // A: TMA (K-major SW128) → smem → tcgen05.cp per 16-element K-step → TMEM [256, 256 + K/2)
      for (int s = 0; s < K / 16; ++s)
        tmem_cp_128x256b(tmem + 256 + s * 8, make_sdesc_sw128(sa + (s / 4) * 128 * 128 + (s % 4) * 32, 16, 1024));
    for (int s = 0; s < K / 16; ++s) {
      uint64_t bdesc;
      if (!b_mn)
        bdesc = make_sdesc_sw128(sb + (s / 4) * N * 128 + (s % 4) * 32, 16, 1024);
      else
        bdesc = make_sdesc_sw128(sb + s * 2048, K * 128, 1024);
      if (mode == 2 || mode == 4) {
        umma_f16_ts(tmem, tmem + 256 + s * 8, bdesc, idesc, s > 0);
      } else {
        uint64_t adesc;
        if (!a_mn)
          adesc = make_sdesc_sw128(sa + (s / 4) * 128 * 128 + (s % 4) * 32, 16, 1024);
        else
          adesc = make_sdesc_sw128(sa + s * 2048, K * 128, 1024);
        umma_f16_ss(tmem, adesc, bdesc, idesc, s > 0);
      }
    }
    umma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();

  // ---- readback: thread ↔ row
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((warp * 32) << 16) + c0, r);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) c[row * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

}  // namespace

extern "C" int vlasim_selftest_umma(int mode, const void* d_a, const void* d_b, float* d_c, int32_t N, int32_t K,
                                    vlasim_stream_t stream) {
  using namespace vlasim_host;
  if (mode < 0 || mode > 4) return set_error(VLASIM_ECONFIG, "selftest: bad mode %d", mode);
  if (N < 64 || N > 256 || N % 64 || K < 64 || K > 256 || K % 64)
    return set_error(VLASIM_ECONFIG, "selftest: N,K must be multiples of 64 in [64,256] (N=%d K=%d)", N, K);
  CUtensorMap tA{}, tB{};
  int rc;
  if (mode == 3)
    rc = encode_tmap_2d(&tA, d_a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, 128, 128 * 2, K, 64, true);
  else
    rc = encode_tmap_2d(&tA, d_a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 128, K, K * 2, 128, 64, true);
  if (rc) return rc;
  if (mode == 0)
    rc = encode_tmap_2d(&tB, d_b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, N, K, K * 2, N, 64, true);
  else
    rc = encode_tmap_2d(&tB, d_b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, N, N * 2, K, 64, true);
  if (rc) return rc;
  const size_t smem = 192 * 1024 + 1024;
  VLASIM_CUDA_TRY(cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  umma_selftest_kernel<<<1, kThreads, smem, as_stream(stream)>>>(tA, tB, mode,
                                                                 static_cast<const __nv_bfloat16*>(d_a), d_c, N, K);
  VLASIM_LAUNCH_CHECK();
  return VLASIM_OK;
}
