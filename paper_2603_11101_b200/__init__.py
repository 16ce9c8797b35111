"""paper_2603_11101_b200 — B200-native (sm_100a) packing + varlen attention hot path of
arxiv/paper_2603_11101 ("vlasim"), behind the reference's `vlasim` packing/attention API.

    packing    pack_ffd / cu_seqlens / token ids / row gather-scatter   (GPU packer)
    attention  packed_attention / varlen_attn_fwd / varlen_attn_bwd     (tcgen05 kernels)
    fp8        E4M3 per-block quantisation + FP8 Q/K attention
    dist       length-balanced pack sharding + NCCL metadata all-gather
All compute goes through libvlasim_cuda.so (include/vlasim_cuda.h); no CPU fallback.
"""
from .errors import ConfigError, InternalError, SimError  # noqa: F401

__all__ = ["ConfigError", "SimError", "InternalError"]
