// common.cu — error state, tensor-map encoding, device queries, version/selftest exports.
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.hpp"

namespace vlasim_host {

std::string& last_error() {
  static thread_local std::string msg;
  return msg;
}

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int encode_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, uint64_t rows, uint64_t cols,
                   uint64_t row_stride_bytes, uint32_t box_rows, uint32_t box_cols, bool swizzle128) {
  auto fn = get_encode_fn();
  if (!fn) return set_error(VLASIM_ERUNTIME, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(VLASIM_ERUNTIME, "cuTensorMapEncodeTiled failed (%d): rows=%llu cols=%llu stride=%llu box=%ux%u",
                     (int)r, (unsigned long long)rows, (unsigned long long)cols,
                     (unsigned long long)row_stride_bytes, box_rows, box_cols);
  return VLASIM_OK;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

bool prof_enabled() {
  static const bool on = getenv("VLASIM_PROF") != nullptr;
  return on;
}

// [0, 64) wait counters, [64, 64 + kTraceWords) event trace (trace_evt, sm100.cuh)
static constexpr size_t kTraceWords = 4 * 2001;  // 4 roles × (count + 2000 events), TraceCtr
static unsigned long long* g_prof = nullptr;
static unsigned long long* prof_buffer_peek() { return g_prof; }
unsigned long long* prof_buffer() {
  const size_t bytes = (64 + kTraceWords) * sizeof(unsigned long long);
  if (!g_prof) cudaMalloc(&g_prof, bytes);
  cudaMemset(g_prof, 0, bytes);
  return g_prof;
}

int prof_report(const char* kernel, int grid, cudaStream_t st, std::initializer_list<const char*> names) {
  unsigned long long h[64];
  VLASIM_CUDA_TRY(cudaStreamSynchronize(st));
  VLASIM_CUDA_TRY(cudaMemcpy(h, prof_buffer_peek(), sizeof(h), cudaMemcpyDeviceToHost));
  std::string line = std::string("[vlasim prof] ") + kernel + " avg cycles/CTA:";
  int i = 0;
  for (const char* n : names) {
    if (n && *n) {
      char b[96];
      snprintf(b, sizeof(b), " %s=%.0f", n, double(h[i]) / grid);
      line += b;
    }
    ++i;
  }
  fprintf(stderr, "%s\n", line.c_str());
  if (const char* path = getenv("VLASIM_TRACE")) {  // dump the CTA-0 event trace (binary, appended)
    std::vector<unsigned long long> tr(kTraceWords);
    VLASIM_CUDA_TRY(cudaMemcpy(tr.data(), prof_buffer_peek() + 64, tr.size() * 8, cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(path, "ab")) {
      for (int r = 0; r < 4; ++r) {
        const unsigned long long* b = tr.data() + r * 2001;
        const unsigned long long n = std::min<unsigned long long>(b[0], 2000);
        char tag[32] = {0};
        snprintf(tag, sizeof(tag), "%s", kernel);
        fwrite(tag, 1, 32, f);
        fwrite(&n, 8, 1, f);
        fwrite(b + 1, 8, n, f);
      }
      fclose(f);
    }
  }
  return VLASIM_OK;
}

namespace {
struct BoundaryEvents {
  cudaEvent_t ev[16];
  int n = 0, next = 0;
};
thread_local BoundaryEvents g_bev;
}  // namespace

void mark_boundary(cudaStream_t st) {
  // a bad handle must not surface as the next kernel's launch error: the hook is measurement only
  if (g_bev.next < g_bev.n && cudaEventRecord(g_bev.ev[g_bev.next++], st) != cudaSuccess) (void)cudaGetLastError();
}

}  // namespace vlasim_host

extern "C" {

int vlasim_set_boundary_events(void* const* events, int n) {
  using namespace vlasim_host;
  if (n < 0 || n > 16 || (n > 0 && !events)) return set_error(VLASIM_ECONFIG, "boundary events: 0..16 events");
  for (int i = 0; i < n; ++i) g_bev.ev[i] = static_cast<cudaEvent_t>(events[i]);
  g_bev.n = n;
  g_bev.next = 0;
  return VLASIM_OK;
}

int vlasim_boundary_count(void) { return vlasim_host::g_bev.next; }

const char* vlasim_last_error_message(void) { return vlasim_host::last_error().c_str(); }

int vlasim_version(void) { return VLASIM_ABI_VERSION; }

}  // extern "C"
