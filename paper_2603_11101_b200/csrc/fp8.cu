// fp8.cu — E4M3 per-block quantisation and the FP8 Q/K forward entry.
#include "common.hpp"

extern "C" int vlasim_fp8_quant_block_cuda(const void*, int64_t, int32_t, int32_t, uint8_t*, float*, vlasim_stream_t) {
  return vlasim_host::set_error(VLASIM_ECONFIG, "fp8 quantisation: not implemented in this build");
}
extern "C" int vlasim_fp8_dequant_block_cuda(const uint8_t*, const float*, int64_t, int32_t, int32_t, float*,
                                             vlasim_stream_t) {
  return vlasim_host::set_error(VLASIM_ECONFIG, "fp8 dequantisation: not implemented in this build");
}
extern "C" int vlasim_varlen_attn_fwd_fp8qk_cuda(const vlasim_attn_args*, void*, size_t, vlasim_stream_t) {
  return vlasim_host::set_error(VLASIM_ECONFIG, "fp8 Q/K attention: not implemented in this build");
}
extern "C" int vlasim_pack_greedy_cuda(const int32_t*, int64_t, int32_t, const vlasim_pack_out*, void*, size_t, uint32_t,
                                       vlasim_stream_t) {
  return vlasim_host::set_error(VLASIM_ECONFIG, "greedy packer: not implemented in this build");
}
