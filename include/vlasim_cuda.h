/* vlasim_cuda.h — C-ABI of the B200 (sm_100a) packing + varlen-attention path.
 *
 * This is the drop-in boundary between the reference's `vlasim` C++ entry points
 * (reconstructed in include/vlasim/packing/*.hpp) and the
 * hand-written CUDA kernels.  Plain pointers and sizes only; no torch types.
 *
 * Conventions:
 *  - Ownership: the caller owns every device buffer and the workspace; hot calls
 *    never allocate.  All calls are stream-ordered on `stream`.
 *  - Status: 0 ok; 2 bad input (the reference's ConfigError, errors.hpp:8-12);
 *    3 runtime/CUDA error (SimError family, errors.hpp:14-18); 4 violated
 *    invariant (InternalError, errors.hpp:35-39).  The message of the last
 *    failure on the calling thread is returned by vlasim_last_error_message().
 *  - Reentrant; no global mutable state on the data path ("pure functions; safe
 *    for parallel invocation on disjoint inputs").
 *
 * Each entry point names the reference operation it replaces.
 */
#ifndef VLASIM_CUDA_H_
#define VLASIM_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VLASIM_ABI_VERSION 3

enum {
  VLASIM_OK = 0,
  VLASIM_ECONFIG = 2,
  VLASIM_ERUNTIME = 3,
  VLASIM_EINTERNAL = 4
};

/* cudaStream_t-compatible opaque stream handle (NULL = legacy default stream). */
typedef struct CUstream_st* vlasim_stream_t;

const char* vlasim_last_error_message(void);
int vlasim_version(void);

/* ------------------------------------------------------------------ packing
 * Replaces vlasim::pack_ffd(lengths, capacity) together with
 * vlasim::cu_seqlens(pack) and the packed-stream layout the
 * reference's packed_attention consumes ("concatenated tensors consistent with
 * cu_seqlens").
 *
 * Ordering contract (pinned): items are placed in order of
 * (length descending, id ascending); each goes to the lowest-index open bin it
 * fits in, else a new bin is appended.  Inside a bin members keep insertion
 * order.  The packed stream is bins in index order, members in order.
 *
 * All arrays are device pointers sized for the worst case (n bins).
 */
typedef struct vlasim_pack_out {
  int32_t* bin_of;          /* [n]   bin index of sample id                               */
  int32_t* slot;            /* [n]   member index of sample id inside its bin             */
  int32_t* tok_off;         /* [n]   token offset of sample id inside its bin              */
  int32_t* bin_count;       /* [n]   members per bin            (first num_bins valid)    */
  int32_t* bin_fill;        /* [n]   tokens per bin             (first num_bins valid)    */
  int32_t* bin_member_off;  /* [n+1] exclusive scan of bin_count (CSR over members)       */
  int32_t* bin_token_off;   /* [n+1] exclusive scan of bin_fill (bin start in the stream)  */
  int32_t* member_ids;      /* [n]   sample id at packed member position m                 */
  int32_t* cu_seqlens;      /* [n+1] global segment offsets over the packed stream          */
  int32_t* cu_seqlens_bins; /* [2n]  per-bin cu_seqlens; bin b at bin_member_off[b] + b     */
  int32_t* src_off;         /* [n+1] exclusive scan of lengths in id order (+ total at [n]) */
  int32_t* num_bins;        /* [1]                                                           */
  int64_t* total_tokens;    /* [1]                                                           */
  int32_t* status;          /* [2]   {error code, offending sample id} written on device     */
} vlasim_pack_out;

/* flags of the calls that report input errors found on the device: synchronise `stream` and
   return the device status (VLASIM_ECONFIG with the offending index in the message). */
#define VLASIM_SYNC_CHECK 1u

/* Maximum capacity accepted by the GPU packer (larger → VLASIM_ECONFIG).  Bin room is held in
   16-bit counters by the greedy variant's room tree; FFD has no open-bin limit (the open-bin
   list spills from shared memory to the workspace), greedy supports up to 2^20 bins. */
#define VLASIM_PACK_MAX_CAPACITY 65535

size_t vlasim_pack_workspace_size(int64_t n, int32_t capacity);

/* flags */
#define VLASIM_PACK_SYNC_CHECK 1u /* synchronise `stream` and return the device status
                                     (oversize / non-positive length → VLASIM_ECONFIG
                                     naming the id)                         */

int vlasim_pack_ffd_cuda(const int32_t* d_len, int64_t n, int32_t capacity, const vlasim_pack_out* out,
                         void* d_workspace, size_t workspace_bytes, uint32_t flags, vlasim_stream_t stream);

/* Streaming first-fit in arrival order (SPEC.md:519 greedy variant). Same outputs. */
int vlasim_pack_greedy_cuda(const int32_t* d_len, int64_t n, int32_t capacity, const vlasim_pack_out* out,
                            void* d_workspace, size_t workspace_bytes, uint32_t flags, vlasim_stream_t stream);

/* Per packed token: position inside its sample, global segment index (packed member
 * position) and gather index (row of the sample-major source layout).  Any output
 * may be NULL.  total_tokens = Σ lengths. */
int vlasim_pack_token_ids_cuda(const int32_t* d_len, const vlasim_pack_out* out, int64_t n, int64_t total_tokens,
                               int32_t* d_pos_ids, int32_t* d_seg_ids, int32_t* d_gather_idx,
                               vlasim_stream_t stream);

/* Token-row gather / scatter between the sample-major source layout (sample id i
 * occupies rows [src_off[i], src_off[i]+len[i])) and the packed stream (segment m
 * occupies rows [cu_seqlens[m], cu_seqlens[m+1]) and holds sample member_ids[m]).
 * row_bytes must be a multiple of 16 and both bases 16-byte aligned (uint4 copies). */
int vlasim_gather_rows_cuda(const void* d_src, void* d_dst, int64_t row_bytes, const int32_t* d_len,
                            const vlasim_pack_out* out, int64_t n, vlasim_stream_t stream);
int vlasim_scatter_rows_cuda(const void* d_packed, void* d_dst, int64_t row_bytes, const int32_t* d_len,
                             const vlasim_pack_out* out, int64_t n, vlasim_stream_t stream);
/* seg_src[m] = src_off[member_ids[m]] for the n packed segments: the source row of each
 * segment's first token (vlasim_attn_args.seg_src — the gather folded into attention). */
int vlasim_pack_seg_src_cuda(const vlasim_pack_out* out, int64_t n, int32_t* d_seg_src, vlasim_stream_t stream);

/* ------------------------------------------------------------------ sharding (multi-GPU)
 * Length-balanced assignment of the packs to `world` ranks, computed identically on every rank
 * after the all-gather of the lengths (host restatement dist.py:lpt):
 * cost(bin) = Σ l² of its members; bins in (cost desc, index asc) order each go to the least-loaded
 * rank (ties: lowest rank).  Then this rank's share: its bins in index order, members in order,
 * as a packed stream (local_cu) over the rank's sample-major layout (its samples in id order:
 * local_src_off), with local_seg_src = the attention's seg_src.  Segments past *local_nseg have
 * zero length (local_cu[j] = *local_tokens).  world <= 16, bins <= 16384 (else status
 * VLASIM_ECONFIG; flags VLASIM_SYNC_CHECK synchronises and returns it).  One CTA, stream-ordered.
 */
typedef struct vlasim_shard_out {
  int32_t* bin_rank;       /* [n]    rank of bin b (first num_bins valid)                    */
  int64_t* rank_load;      /* [world] Σ l² of each rank's bins                                */
  int32_t* local_ids;      /* [n]    sample id of local segment j                             */
  int32_t* local_cu;       /* [n+1]  cu_seqlens of the rank's packed stream                   */
  int32_t* local_seg_src;  /* [n]    row of local segment j's sample in the local layout      */
  int32_t* local_src_off;  /* [n]    row of sample i in the local layout, -1 if not this rank's */
  int32_t* local_nseg;     /* [1]                                                             */
  int64_t* local_tokens;   /* [1]                                                             */
  int32_t* status;         /* [2]                                                             */
  int32_t* scratch;        /* vlasim_shard_scratch_size(n) bytes of device workspace          */
} vlasim_shard_out;

size_t vlasim_shard_scratch_size(int64_t n);
int vlasim_shard_lpt_cuda(const int32_t* d_len, const vlasim_pack_out* plan, int64_t n, int32_t world, int32_t rank,
                          const vlasim_shard_out* out, uint32_t flags, vlasim_stream_t stream);

/* ------------------------------------------------------------------ attention
 * Replaces vlasim::packed_attention(q, k, v, cu_seqlens),
 * multi-head as the reference's looped single-head op.
 *
 * Layout: q/o [T, H, d] bf16, k/v [T, Hkv, d] bf16 (row-major, token-major),
 * lse [H, T] fp32 (natural-log units), cu_seqlens [num_seqs+1] int32 over the
 * packed stream.  Block-diagonal: token t attends only to keys of its own
 * segment.  GQA/MQA: kv_head = q_head / (H / Hkv).
 *
 * mask_mode: 0 bidirectional, 1 causal, 2 prefix — key j of
 * segment [s, e) is visible to query t iff j < s + prefix_len[seg] or j <= t.
 * head_dim ∈ {64, 128, 256}.
 */
enum { VLASIM_MASK_BIDIR = 0, VLASIM_MASK_CAUSAL = 1, VLASIM_MASK_PREFIX = 2 };

typedef struct vlasim_attn_args {
  const void* q;              /* [T, H, d]   bf16 (or e4m3 codes for the fp8 entry)  */
  const void* k;              /* [T, Hkv, d] bf16 (or e4m3 codes)                    */
  const void* v;              /* [T, Hkv, d] bf16                                    */
  void* o;                    /* [T, H, d]   bf16                                    */
  float* lse;                 /* [H, T]      fp32                                    */
  const int32_t* cu_seqlens;  /* [num_seqs + 1]                                      */
  const int32_t* prefix_len;  /* [num_seqs]  (mask_mode == PREFIX only)              */
  int32_t num_seqs;
  int64_t total_tokens;       /* T: rows of the tensors (>= cu_seqlens[num_seqs]; rows past
                                 the last segment belong to none — the padded layout below)  */
  int32_t num_heads;          /* H                                                   */
  int32_t num_kv_heads;       /* Hkv (divides H)                                     */
  int32_t head_dim;           /* d                                                   */
  int32_t mask_mode;
  float softmax_scale;        /* usually 1/sqrt(d)                                   */
  /* fp8 Q/K only: per-block scales, [H, ceil(T/128), ceil(d/128)] for q and
     [Hkv, ceil(T/128), ceil(d/128)] for k                       */
  const float* q_scale;
  const float* k_scale;
  /* [num_seqs] or NULL.  NULL: q/k/v/o/lse (and dout/dq/dk/dv) are in packed-stream order.
     Set: they stay in the SOURCE (sample-major) order and segment m's packed rows
     [cu_seqlens[m], cu_seqlens[m+1]) live at source rows seg_src[m] + (t - cu_seqlens[m]);
     the lse / fp8 scale blocks are indexed by source row too.  With the packer's layout
     (seg_src[m] = src_off[member_ids[m]], vlasim_pack_seg_src_cuda) the gather into the
     packed stream and the scatter back are folded into the kernels' TMA coordinates.
     (ABI version 2; row_map must be NULL when it is set.)                                  */
  const int32_t* seg_src;
  /* 0: the persistent attention kernels take every SM.  n > 0: at most n CTAs (one per SM), so
     the remaining SMs stay free for a concurrent stream — e.g. the GPU packer of the next batch
     overlapping this batch's attention.                                                       */
  int32_t sm_budget;
} vlasim_attn_args;

typedef struct vlasim_attn_grads {
  const void* dout;          /* [T, H, d]   bf16 (packed order)                          */
  void* dq;                  /* [T, H, d]   bf16                                        */
  void* dk;                  /* [T, Hkv, d] bf16                                        */
  void* dv;                  /* [T, Hkv, d] bf16                                        */
  const int32_t* row_map;    /* [T] or NULL: packed row t → output row row_map[t].  With
                                the packer's gather index this fuses the scatter of the
                                gradients back to sample order into the kernels.         */
} vlasim_attn_grads;

/* backward: 0 forward, 1 backward, 2 FP8 Q/K backward */
size_t vlasim_varlen_attn_workspace_size(const vlasim_attn_args* a, int backward);

int vlasim_varlen_attn_fwd_cuda(const vlasim_attn_args* a, void* d_workspace, size_t workspace_bytes,
                                vlasim_stream_t stream);
int vlasim_varlen_attn_bwd_cuda(const vlasim_attn_args* a, const vlasim_attn_grads* g, void* d_workspace,
                                size_t workspace_bytes, vlasim_stream_t stream);
/* FP8 Q/K forward: q/k are e4m3 codes with per-(head,128-token,128-d) block scales. */
int vlasim_varlen_attn_fwd_fp8qk_cuda(const vlasim_attn_args* a, void* d_workspace, size_t workspace_bytes,
                                      vlasim_stream_t stream);
/* Backward of the FP8 Q/K forward: gradients of attention(deq(q), deq(k), v) (straight-through for
 * the quantiser) with the FP8 forward's o / lse.  q/k are the codes + scales of the forward; dq/dk
 * are bf16 gradients with respect to the dequantised operands.  Workspace:
 * vlasim_varlen_attn_workspace_size(a, 2). */
int vlasim_varlen_attn_bwd_fp8qk_cuda(const vlasim_attn_args* a, const vlasim_attn_grads* g, void* d_workspace,
                                      size_t workspace_bytes, vlasim_stream_t stream);

/* ------------------------------------------------------------------ fp8
 * Replaces vlasim::quantize(t, PerBlock(128,128), E4M3) applied
 * per head to x [T, heads, d] bf16: scale = fp32(amax/448) (1 if the block is all zero),
 * codes = the round-to-nearest-even E4M3 code of the REAL quotient x·448/amax (saturating
 * to ±448).  scales [heads, ceil(T/128), ceil(d/128)].
 * d_status ([2] int32 or NULL): {VLASIM_ECONFIG, flat index} when an element is non-finite
 * ("non-finite input → error"; that block's codes are not written), else {0, 0}.
 * flags VLASIM_SYNC_CHECK (needs d_status): synchronise and return the status.
 */
int vlasim_fp8_quant_block_cuda(const void* d_x, int64_t T, int32_t heads, int32_t d, uint8_t* d_codes,
                                float* d_scales, int32_t* d_status, uint32_t flags, vlasim_stream_t stream);
int vlasim_fp8_dequant_block_cuda(const uint8_t* d_codes, const float* d_scales, int64_t T, int32_t heads, int32_t d,
                                  float* d_out, vlasim_stream_t stream);
/* quant_error(original, qt) per group (head, 128-token block, 128-d block),
 * groups ordered like the scales: max relative roundtrip error over elements in E4M3's normal
 * range (|x / scale| >= 2^-6, fp32 quotient), sum of squared errors (fp64) and element count.  Global
 * metrics: max of the maxima, Σsse / Σcount. */
int vlasim_fp8_quant_error_cuda(const void* d_x, const uint8_t* d_codes, const float* d_scales, int64_t T,
                                int32_t heads, int32_t d, float* d_group_maxrel, double* d_group_sse,
                                int32_t* d_group_count, vlasim_stream_t stream);

/* ------------------------------------------------------------------ general quantizer
 * Replaces vlasim::quantize / dequantize / quant_error of the reference's quantizer module
 * (proj/CMakeLists.txt:18-21 src/quant/{fp8,tensor,quantize,compression}.cpp; contract
 * SPEC.md:539-627) on the GPU: Granularity PerTensor | PerChannel(axis) | PerBlock(128, 128 over
 * the last two dims) over an fp32 or bf16 row-major tensor of 1-8 dims.
 * Scales (fp32, RN(amax / 448), 1 for an all-zero group) are laid out per granularity:
 *   PerTensor [1];  PerChannel [shape[axis]];  PerBlock [Π shape[:-2], ⌈rows/128⌉, ⌈cols/128⌉].
 * Codes are the exact RNE E4M3 code of |x|·448/amax, one byte per element
 * in the input's layout.  Non-finite input → VLASIM_ECONFIG naming the flat index:
 * with VLASIM_SYNC_CHECK the call synchronises and returns it; otherwise d_status ({code, index},
 * optional) holds it and no codes are written. */
enum { VLASIM_GRAN_TENSOR = 0, VLASIM_GRAN_CHANNEL = 1, VLASIM_GRAN_BLOCK = 2 };
enum { VLASIM_DTYPE_F32 = 0, VLASIM_DTYPE_BF16 = 1 };

int64_t vlasim_fp8_groups(const int64_t* shape, int32_t ndim, int32_t granularity, int32_t axis);
size_t vlasim_fp8_quantize_workspace_size(const int64_t* shape, int32_t ndim, int32_t granularity, int32_t axis);
int vlasim_fp8_quantize_cuda(const void* d_x, int32_t dtype, const int64_t* shape, int32_t ndim, int32_t granularity,
                             int32_t axis, uint8_t* d_codes, float* d_scales, int32_t* d_status, void* d_workspace,
                             size_t workspace_bytes, uint32_t flags, vlasim_stream_t stream);
/* out = fp32(value(code) · scale of its group) */
int vlasim_fp8_dequantize_cuda(const uint8_t* d_codes, const float* d_scales, const int64_t* shape, int32_t ndim,
                               int32_t granularity, int32_t axis, float* d_out, vlasim_stream_t stream);
/* quant_error(original, qt) per group, reduced in a fixed order (bit-identical run
 * to run): max relative error over elements in E4M3's normal range, Σ squared error
 * (fp64), element count.  Output arrays hold vlasim_fp8_error_groups(...) entries: the groups of the
 * granularity, except PerTensor, which uses ⌈n / 65536⌉ entries of scratch and leaves the result in
 * entry 0. */
int64_t vlasim_fp8_error_groups(const int64_t* shape, int32_t ndim, int32_t granularity, int32_t axis);
int vlasim_fp8_quant_error_general_cuda(const void* d_x, int32_t dtype, const uint8_t* d_codes, const float* d_scales,
                                        const int64_t* shape, int32_t ndim, int32_t granularity, int32_t axis,
                                        float* d_group_maxrel, double* d_group_sse, int64_t* d_group_count,
                                        vlasim_stream_t stream);

/* ------------------------------------------------------------------ dynamic padding (π0.5)
 * dynamic_pad_length (PAPER.md:166-176 π0.5's per-batch max_length) on the device:
 * *d_pad_to = max(len), d_cu_seqlens [n+1] = exclusive scan of len (the valid tokens as segments),
 * d_seg_src [n] = i·pad_to.  With these, vlasim_varlen_attn_*_cuda run directly on padded
 * [n, pad_to, heads, d] storage (total_tokens = n·pad_to, seg_src set): each sample is one
 * segment, pad keys are never visible and pad queries never computed.  In that layout the
 * caller zero-initialises o and lse (their pad rows are never written and the backward reads
 * them).  A length < 1 → VLASIM_ECONFIG naming the id.
 * pad: sample-major rows (sample i at d_src_off[i]) → [n, pad_to] rows, zero fill; unpad: inverse. */
int vlasim_dynamic_pad_cuda(const int32_t* d_len, int64_t n, int32_t* d_pad_to, int32_t* d_cu_seqlens,
                            int32_t* d_seg_src, int32_t* d_status, uint32_t flags, vlasim_stream_t stream);
int vlasim_pad_rows_cuda(const void* d_src, void* d_padded, int64_t row_bytes, const int32_t* d_len,
                         const int32_t* d_src_off, const int32_t* d_pad_to, int64_t n, vlasim_stream_t stream);
int vlasim_unpad_rows_cuda(const void* d_padded, void* d_dst, int64_t row_bytes, const int32_t* d_len,
                           const int32_t* d_src_off, const int32_t* d_pad_to, int64_t n, vlasim_stream_t stream);

/* ------------------------------------------------------------------ synthetic inputs
 * Counter-based values shared with the CPU oracle:
 * x[i] = (top8(splitmix64(seed ^ i)) - 128) / 128, exactly representable in bf16. */
int vlasim_fill_synthetic_bf16(void* d_x, int64_t count, uint64_t seed, vlasim_stream_t stream);

/* Host-side sample-length generator on the reference's seeding API (rng.hpp:28-49):
 * rng = make_rng(root_seed, label, 0); dist 0 uniform_int(p1, p2); 1 truncated
 * geometric(p = p1, max = p2) by inverse CDF on uniform01; 2 GR00T-like
 * 64·uniform_int(1,2) + uniform_int(16,64); 3 π0.5 512 + uniform_int(p1, p2) + p3
 * (prefix = length − p3).  h_out is a HOST buffer of n int32. */
int vlasim_gen_lengths(uint64_t root_seed, const char* label, int dist, int64_t n, double p1, double p2, double p3,
                       int32_t* h_out);

/* ------------------------------------------------------------------ measurement hook
 * Per calling thread: the attention entry points record the registered cudaEvent_t handles, in
 * order, on their stream at every kernel boundary — forward (head_dim 64/128): start, after the
 * span + tile-table kernels, after the attention kernel; forward (256): start, after the tile
 * table, after the attention kernel; backward: start, after k_bwd_pre, after the tile table,
 * after dK/dV, after dQ.  n ≤ 16; n = 0 disables.  vlasim_boundary_count() = events recorded since
 * the last registration.  Used by bench.py for per-kernel CUDA-event times. */
int vlasim_set_boundary_events(void* const* events, int n);
int vlasim_boundary_count(void);

/* ------------------------------------------------------------------ self-test
 * Single-CTA tcgen05 GEMM used to validate the UMMA/TMA descriptor layouts the
 * attention kernels rely on.  a, b bf16 row-major, c fp32 [128, N].
 *  mode 0: C = A[128,K] · B[N,K]ᵀ   (A, B K-major)
 *  mode 1: C = A[128,K] · B[K,N]    (B MN-major)
 *  mode 2: C = A[128,K] · B[K,N]    (A staged in TMEM via tcgen05.st, B MN-major)
 *  mode 3: C = A[K,128]ᵀ · B[K,N]   (A MN-major, B MN-major)
 */
int vlasim_selftest_umma(int mode, const void* d_a, const void* d_b, float* d_c, int32_t N, int32_t K,
                         vlasim_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VLASIM_CUDA_H_ */
