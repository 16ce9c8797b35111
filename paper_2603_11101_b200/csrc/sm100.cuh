// sm100.cuh — thin inline-PTX layer for Blackwell (sm_100a): mbarriers, TMA,
// tcgen05 (MMA / TMEM alloc / ld / st / commit) and the UMMA descriptors.
//
// Everything here is a direct PTX wrapper; the kernels in attn_*.cu compose
// them.  Descriptor bit layouts follow the PTX ISA "tcgen05 matrix
// descriptors" / "instruction descriptor" tables (cross-checked against the
// CuTe 4.x header layout in flashinfer/data/cutlass/include/cute/arch/
// mma_sm100_desc.hpp; no CuTe code is used).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

namespace vlasim_dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// One arrival per warp (lane 0, after the warp has converged): barriers that consumer warps
// release are initialised with a count of warps, not threads — 32× fewer serialised smem
// atomics per hand-off.  Callers issue their tcgen05 fences before this.
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2-D tiled load: box at element coords (c0 = inner, c1 = row) → smem, completes tx on bar.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* m, int32_t c0, int32_t c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void* smem_dst, const CUtensorMap* m, int32_t c0, int32_t c1,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// L2 prefetch of a 2-D box (no smem destination, no completion tracking).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* m, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1)
               : "memory");
}
// 2-D tiled store: smem box → global at element coords (c0 = inner, c1 = row); bulk-group tracked.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, int32_t c0, int32_t c1, const void* smem_src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(smem_u32(smem_src))
               : "memory");
}
// 1-D bulk copy global → smem (16-B aligned src/dst, size multiple of 16), completes tx on bar.
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 1-D bulk copy smem → global (16-B aligned, size multiple of 16), tracked by bulk groups.
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(gdst)),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Wait until the smem source of all committed bulk stores of this thread has been read.
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// Wait until all committed bulk stores of this thread have fully completed.
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- tcgen05
// TMEM address = (lane << 16) | column.
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] · B[smem]ᵀ   (kind::f16: bf16/fp16 inputs, fp32 accum)
__device__ __forceinline__ void umma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] · B[smem]
__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::f8f6f4 (e4m3 inputs, fp32 accum), both operands from smem.
__device__ __forceinline__ void umma_f8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once) on an mbarrier when all previously issued tcgen05 async ops of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes × 32b, 16 consecutive columns → 16 regs per thread (thread i ↔ lane base+i).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// ---------------------------------------------------------------- descriptors
// Shared-memory matrix descriptor, SWIZZLE_128B, version 1 (sm_100).
//  bits [0,14)  start address >> 4
//  bits [16,30) leading-dim byte offset >> 4
//  bits [32,46) stride-dim byte offset >> 4
//  bits [46,48) version = 1
//  bits [49,52) base offset (0: atoms are 1024-B aligned)
//  bits [61,64) layout: 2 = SWIZZLE_128B
// K-major SW128 (rows of 128 B, 8-row atoms):  LBO unused (=16 B), SBO = 1024 B.
// MN-major SW128 (64 MN elems × 8 K rows atoms): LBO = byte stride between 64-wide MN atoms,
//                                                 SBO = byte stride between 8-row K groups.
__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}
// Descriptor of the same layout `bytes` further on (the start address field holds addr >> 4 in
// 14 bits; smem addresses < 256 KB never carry out of it).
__device__ __forceinline__ uint64_t sdesc_add(uint64_t d, uint32_t bytes) { return d + (bytes >> 4); }
// One elected lane of a converged warp (elect.sync).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
// Instruction descriptor, kind::f16, bf16 × bf16 → f32.
//  [4,6) c_format (1=F32)  [7,10) a_format (1=BF16)  [10,13) b_format (1=BF16)
//  [15] a_major (1=MN)  [16] b_major (1=MN)  [17,23) N>>3  [24,29) M>>4
__host__ __device__ constexpr uint32_t make_idesc_bf16(uint32_t M, uint32_t N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}
// kind::f8f6f4, e4m3 × e4m3 → f32 (formats 0 = E4M3), K-major only.
__host__ __device__ constexpr uint32_t make_idesc_e4m3(uint32_t M, uint32_t N) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ---------------------------------------------------------------- misc
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// Packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2 on sm_100a) and the 3-input max (FMNMX3):
// half the issue slots of the scalar forms for the softmax's elementwise work.  Not volatile.
__device__ __forceinline__ unsigned long long f2_bits(float2 v) {
  return (static_cast<unsigned long long>(__float_as_uint(v.y)) << 32) | __float_as_uint(v.x);
}
__device__ __forceinline__ float2 f2_from(unsigned long long b) {
  return make_float2(__uint_as_float(static_cast<uint32_t>(b)), __uint_as_float(static_cast<uint32_t>(b >> 32)));
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return f2_from(r);
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(r);
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(r);
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// Not volatile: a pure function the compiler may schedule freely (MUFU.EX2).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for a pair of finite x on the FMA pipe (offloads MUFU.EX2, the softmax's binding unit):
// x = n + f with n = rint(x) by the 1.5·2^23 magic add, f ∈ [-0.5, 0.5]; 2^f by a degree-3
// polynomial fitted for relative error (max 1.0e-4, below bf16's 2^-9 rounding of P); 2^n added to
// the exponent field — t's low bits hold n, so (bits(t) << 23) ≡ n << 23 (mod 2^32): one LEA.  x is
// clamped at −126 (callers use it only where no column is masked: such results are ≤ 2^-126 of
// the row maximum, i.e. nothing after the bf16 P·V).
__device__ __forceinline__ float2 f2_ex2_poly(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 M = make_float2(12582912.f, 12582912.f), nM = make_float2(-12582912.f, -12582912.f);
  const float2 t = f2_add(x, M);
  const float2 f = f2_fma(f2_add(t, nM), make_float2(-1.f, -1.f), x);  // x − rint(x), exact
  const float2 c3 = make_float2(0.05500893f, 0.05500893f), c2 = make_float2(0.24221098f, 0.24221098f);
  const float2 c1 = make_float2(0.69328293f, 0.69328293f), one = make_float2(1.f, 1.f);
  const float2 p = f2_fma(f2_fma(f2_fma(c3, f, c2), f, c1), f, one);
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// smem → TMEM copy of a 128-row × 256-bit tile described by a UMMA smem descriptor (one A-operand
// K-step of 16 bf16): lane r ← row r, 8 columns.  Executes in issue order with tcgen05.mma.
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void red_add_v4_f32(float* gaddr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gaddr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// ---------------------------------------------------------------- profiling (VLASIM_PROF)
// Per-role wait-time accounting, compiled in only for the PROF kernel instantiations:
// accumulates clock64 cycles spent in each mbarrier wait category and flushes them to a global
// counter array (one warp-lane per role) at kernel exit.
// Event trace (timing experiments; ≤ 2000 events per role): each role appends (clock << 32 | code << 16 | unit) words to
// its own shared-memory region ([0] = count) — one STS per event; the kernel copies the regions
// of CTA 0 to global memory at exit (trace_flush).  Disabled when base is null.
struct TraceCtr {
  unsigned long long* base;
  uint32_t n;
  __device__ __forceinline__ explicit TraceCtr(unsigned long long* b) : base(b), n(0) {}
  __device__ __forceinline__ void operator()(uint32_t code, uint32_t unit) {
    if (base == nullptr || n >= 2000) return;
    base[1 + n] = (static_cast<unsigned long long>(clock()) << 32) | (code << 16) | (unit & 0xFFFFu);
    base[0] = ++n;
  }
};

template <bool ON, int N = 8>
struct WaitProf {
  unsigned long long acc[N];
  long long t_start;
  __device__ __forceinline__ WaitProf() {
    if constexpr (ON) {
#pragma unroll
      for (int i = 0; i < N; ++i) acc[i] = 0;
      t_start = clock64();
    }
  }
  template <int C>
  __device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
    if constexpr (ON) {
      const long long t0 = clock64();
      mbar_wait(bar, parity);
      acc[C] += clock64() - t0;
    } else {
      mbar_wait(bar, parity);
    }
  }
  template <int C>
  __device__ __forceinline__ void add_since(long long t0) {
    if constexpr (ON) acc[C] += clock64() - t0;
  }
  __device__ __forceinline__ long long now() const {
    if constexpr (ON) return clock64();
    return 0;
  }
  // slot N-1 receives the role's total elapsed cycles
  __device__ __forceinline__ void flush(unsigned long long* out) {
    if constexpr (ON) {
      acc[N - 1] = clock64() - t_start;
#pragma unroll
      for (int i = 0; i < N; ++i) atomicAdd(out + i, acc[i]);
    }
  }
};

// Epilogue row store without smem: thread (row = lane of a 32-row warp slab, part) holds CPT 16-B
// chunks of its row.  A butterfly over groups of CPT lanes transposes the chunks so that lane
// (g·CPT + i) holds chunk i of the group's CPT rows; CPT stores then write CPT-row × (16·CPT)-B
// segments per warp instruction (8 rows × 64 B for CPT = 4) instead of 32 scattered rows.
// dst = this lane's destination row (< 0: skip); base + dst·stride + col0 (elements) = row start.
template <int CPT>
__device__ __forceinline__ void store_rows_xpose(uint32_t (&w)[4 * CPT], int dst, __nv_bfloat16* base,
                                                 int64_t stride, int col0) {
  const int lane = threadIdx.x & 31, li = lane & (CPT - 1);
#pragma unroll
  for (int m = 1; m < CPT; m <<= 1) {  // stage: position c takes the partner's position c ^ m
    const bool hi = li & m;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if ((c & m) != 0) continue;  // handle the pair (c, c ^ m) once
      const int c1 = c | m;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // a lane with bit m clear keeps position c and receives position c1 from its partner's c;
        // a lane with bit m set keeps c1 and receives position c from its partner's c1
        const uint32_t send = hi ? w[4 * c + k] : w[4 * c1 + k];
        const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, m);
        if (hi) w[4 * c + k] = recv;
        else w[4 * c1 + k] = recv;
      }
    }
  }
  // lane (g·CPT + li) now holds chunk li of rows g·CPT + i at position i
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int src = (lane & ~(CPT - 1)) + i;
    const int d = __shfl_sync(0xffffffffu, dst, src);
    if (d >= 0)
      *reinterpret_cast<uint4*>(base + int64_t(d) * stride + col0 + li * 8) =
          make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
  }
}

}  // namespace vlasim_dev
