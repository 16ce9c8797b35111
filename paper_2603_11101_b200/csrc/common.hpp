// common.hpp — host-side plumbing shared by the C-ABI entry points:
// thread-local error state (SURVEY §8(b) status convention), CUDA checks,
// and TMA tensor-map encoding through the driver entry point (no -lcuda).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <initializer_list>
#include <string>

#include "../../include/vlasim_cuda.h"

namespace vlasim_host {

// Status codes mirror the reference's exception taxonomy (errors.hpp:8-39):
// 2 = ConfigError (bad user input), 3 = runtime (SimError family), 4 = InternalError.
std::string& last_error();
int set_error(int code, const char* fmt, ...);

#define VLASIM_CUDA_TRY(expr)                                                                          \
  do {                                                                                                 \
    cudaError_t _e = (expr);                                                                           \
    if (_e != cudaSuccess)                                                                             \
      return ::vlasim_host::set_error(VLASIM_ERUNTIME, "%s failed: %s (%s:%d)", #expr,                  \
                                      cudaGetErrorString(_e), __FILE__, __LINE__);                     \
  } while (0)

#define VLASIM_LAUNCH_CHECK()                                                                          \
  do {                                                                                                 \
    cudaError_t _e = cudaGetLastError();                                                               \
    if (_e != cudaSuccess)                                                                             \
      return ::vlasim_host::set_error(VLASIM_ERUNTIME, "kernel launch failed: %s (%s:%d)",             \
                                      cudaGetErrorString(_e), __FILE__, __LINE__);                     \
  } while (0)

// Encodes a 2-D tiled TMA map over a row-major matrix [rows, cols] of elem_bytes-wide
// elements with row pitch `row_stride_bytes`; box = [box_rows, box_cols] (box_cols*elem
// must be 128 B for SWIZZLE_128B).  Returns 0 or a status code.
int encode_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, uint64_t rows, uint64_t cols,
                   uint64_t row_stride_bytes, uint32_t box_rows, uint32_t box_cols, bool swizzle128);

inline cudaStream_t as_stream(vlasim_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();
// CTAs of a persistent attention kernel: min(work items, SMs, the caller's sm_budget when > 0)
inline int persistent_grid(int64_t max_items, int sm_budget) {
  int64_t g = max_items < num_sms() ? max_items : num_sms();
  if (sm_budget > 0 && g > sm_budget) g = sm_budget;
  return int(g < 1 ? 1 : g);
}

// Segment-aligned 128-row tiles of the packed stream, sorted by cost (attn_tiles.cu).  `buf` holds
// tiles_bytes(T, nseq) bytes; *tiles / *ntiles point into it (the count is written on device).
size_t tiles_bytes(int64_t T, int nseq);
size_t fwd_ws_bytes(const vlasim_attn_args* a);  // forward workspace: spans + tiles (attn_fwd2.cu)
int launch_build_tiles(const int32_t* cu, const int32_t* seg_src, int nseq, int64_t T, void* buf, cudaStream_t st,
                       int4** tiles, int** ntiles);

// Kernel-boundary events (vlasim_set_boundary_events): records the calling thread's next event on
// `st`; a no-op unless events were registered.
void mark_boundary(cudaStream_t st);

// VLASIM_PROF=1: kernels with wait-time accounting are launched instead and each launch prints
// (stderr) the average cycles per CTA spent in every named wait category.
bool prof_enabled();
unsigned long long* prof_buffer();  // zeroed device buffer of 64 counters
int prof_report(const char* kernel, int grid, cudaStream_t st, std::initializer_list<const char*> names);

}  // namespace vlasim_host
