"""ctypes binding of the C-ABI (include/vlasim_cuda.h) — the only way Python reaches the kernels.

There is deliberately no fallback: if libvlasim_cuda.so is missing the import of any op fails
loudly (build it with `python -m paper_2603_11101_b200.build`).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import raise_for_status

LIB_DIR = Path(__file__).resolve().parent / "lib"
LIB_PATH = Path(os.environ["VLASIM_CUDA_LIB"]) if os.environ.get("VLASIM_CUDA_LIB") else LIB_DIR / "libvlasim_cuda.so"

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f32p = C.POINTER(C.c_float)


class PackOut(C.Structure):
    _fields_ = [(name, i32p) for name in (
        "bin_of", "slot", "tok_off", "bin_count", "bin_fill", "bin_member_off", "bin_token_off",
        "member_ids", "cu_seqlens", "cu_seqlens_bins", "src_off", "num_bins")] + [
        ("total_tokens", i64p), ("status", i32p)]


class ShardOut(C.Structure):
    _fields_ = [("bin_rank", i32p), ("rank_load", i64p), ("local_ids", i32p), ("local_cu", i32p),
                ("local_seg_src", i32p), ("local_src_off", i32p), ("local_nseg", i32p), ("local_tokens", i64p),
                ("status", i32p), ("scratch", i32p)]


class AttnArgs(C.Structure):
    _fields_ = [
        ("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p), ("o", C.c_void_p), ("lse", f32p),
        ("cu_seqlens", i32p), ("prefix_len", i32p), ("num_seqs", C.c_int32), ("total_tokens", C.c_int64),
        ("num_heads", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
        ("mask_mode", C.c_int32), ("softmax_scale", C.c_float), ("q_scale", f32p), ("k_scale", f32p),
        ("seg_src", i32p), ("sm_budget", C.c_int32)]


class AttnGrads(C.Structure):
    _fields_ = [("dout", C.c_void_p), ("dq", C.c_void_p), ("dk", C.c_void_p), ("dv", C.c_void_p),
                ("row_map", i32p)]


_SIGS = {
    "vlasim_last_error_message": (C.c_char_p, []),
    "vlasim_version": (C.c_int, []),
    "vlasim_pack_workspace_size": (C.c_size_t, [C.c_int64, C.c_int32]),
    "vlasim_pack_ffd_cuda": (C.c_int, [i32p, C.c_int64, C.c_int32, C.POINTER(PackOut), C.c_void_p, C.c_size_t,
                                       C.c_uint32, C.c_void_p]),
    "vlasim_pack_greedy_cuda": (C.c_int, [i32p, C.c_int64, C.c_int32, C.POINTER(PackOut), C.c_void_p, C.c_size_t,
                                          C.c_uint32, C.c_void_p]),
    "vlasim_pack_token_ids_cuda": (C.c_int, [i32p, C.POINTER(PackOut), C.c_int64, C.c_int64, i32p, i32p, i32p,
                                             C.c_void_p]),
    "vlasim_gather_rows_cuda": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, i32p, C.POINTER(PackOut), C.c_int64,
                                          C.c_void_p]),
    "vlasim_shard_lpt_cuda": (C.c_int, [i32p, C.POINTER(PackOut), C.c_int64, C.c_int32, C.c_int32,
                                         C.POINTER(ShardOut), C.c_uint32, C.c_void_p]),
    "vlasim_shard_scratch_size": (C.c_size_t, [C.c_int64]),
    "vlasim_pack_seg_src_cuda": (C.c_int, [C.POINTER(PackOut), C.c_int64, i32p, C.c_void_p]),
    "vlasim_scatter_rows_cuda": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, i32p, C.POINTER(PackOut), C.c_int64,
                                           C.c_void_p]),
    "vlasim_varlen_attn_workspace_size": (C.c_size_t, [C.POINTER(AttnArgs), C.c_int]),
    "vlasim_varlen_attn_fwd_cuda": (C.c_int, [C.POINTER(AttnArgs), C.c_void_p, C.c_size_t, C.c_void_p]),
    "vlasim_varlen_attn_bwd_cuda": (C.c_int, [C.POINTER(AttnArgs), C.POINTER(AttnGrads), C.c_void_p, C.c_size_t,
                                              C.c_void_p]),
    "vlasim_varlen_attn_fwd_fp8qk_cuda": (C.c_int, [C.POINTER(AttnArgs), C.c_void_p, C.c_size_t, C.c_void_p]),
    "vlasim_varlen_attn_bwd_fp8qk_cuda": (C.c_int, [C.POINTER(AttnArgs), C.POINTER(AttnGrads), C.c_void_p,
                                                    C.c_size_t, C.c_void_p]),
    "vlasim_fp8_quant_block_cuda": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, f32p,
                                              i32p, C.c_uint32, C.c_void_p]),
    "vlasim_fp8_dequant_block_cuda": (C.c_int, [C.c_void_p, f32p, C.c_int64, C.c_int32, C.c_int32, f32p,
                                                C.c_void_p]),
    "vlasim_fp8_quant_error_cuda": (C.c_int, [C.c_void_p, C.c_void_p, f32p, C.c_int64, C.c_int32, C.c_int32, f32p,
                                              C.c_void_p, C.c_void_p, C.c_void_p]),
    "vlasim_fp8_groups": (C.c_int64, [i64p, C.c_int32, C.c_int32, C.c_int32]),
    "vlasim_fp8_quantize_workspace_size": (C.c_size_t, [i64p, C.c_int32, C.c_int32, C.c_int32]),
    "vlasim_fp8_quantize_cuda": (C.c_int, [C.c_void_p, C.c_int32, i64p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                           f32p, i32p, C.c_void_p, C.c_size_t, C.c_uint32, C.c_void_p]),
    "vlasim_fp8_dequantize_cuda": (C.c_int, [C.c_void_p, f32p, i64p, C.c_int32, C.c_int32, C.c_int32, f32p,
                                             C.c_void_p]),
    "vlasim_fp8_error_groups": (C.c_int64, [i64p, C.c_int32, C.c_int32, C.c_int32]),
    "vlasim_fp8_quant_error_general_cuda": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, f32p, i64p, C.c_int32,
                                                      C.c_int32, C.c_int32, f32p, C.c_void_p, i64p, C.c_void_p]),
    "vlasim_dynamic_pad_cuda": (C.c_int, [i32p, C.c_int64, i32p, i32p, i32p, i32p, C.c_uint32, C.c_void_p]),
    "vlasim_pad_rows_cuda": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, i32p, i32p, i32p, C.c_int64, C.c_void_p]),
    "vlasim_unpad_rows_cuda": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, i32p, i32p, i32p, C.c_int64,
                                         C.c_void_p]),
    "vlasim_fill_synthetic_bf16": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_void_p]),
    "vlasim_gen_lengths": (C.c_int, [C.c_uint64, C.c_char_p, C.c_int, C.c_int64, C.c_double, C.c_double,
                                     C.c_double, i32p]),
    "vlasim_set_boundary_events": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "vlasim_boundary_count": (C.c_int, []),
    "vlasim_selftest_umma": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, f32p, C.c_int32, C.c_int32, C.c_void_p]),
}

# Every symbol include/vlasim_cuda.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2603_11101_b200.build` "
                              "(there is no CPU fallback for the packing/attention path)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().vlasim_last_error_message().decode(errors="replace")
        raise_for_status(rc, f"{what}: {msg}" if what else msg)


def ptr(t, ctype=None):
    """Device pointer of a torch tensor (None → NULL) cast for ctypes."""
    if t is None:
        return None
    p = t.data_ptr()
    if ctype is None:
        return C.c_void_p(p)
    return C.cast(C.c_void_p(p), ctype)


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
