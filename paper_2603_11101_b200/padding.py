"""π0.5 dynamic padding on the GPU — the step before packing
in the paper's π0.5 pipeline, and the layout its fixed-length baseline uses.

    dynamic_pad(lengths)              -> DynamicPad   pad_to = max(lengths) of the batch
                                                     (dynamic_pad_length), the
                                                     valid tokens' cu_seqlens and seg_src = i·pad_to
    pad_rows(x, dp) / unpad_rows(xp, dp)             sample-major rows <-> [n, pad_to, ...]
    padded_attention_fwd / _bwd                      the varlen kernels run on the padded storage:
                                                     every sample is one segment, pad keys are never
                                                     visible, pad queries never computed (no pad² work)
    prune_corpus(samples, view)                      view pruning over a batch

The fixed-length baseline of the paper's sweep pads every sample to a global cap and computes all
pad_to² pairs; attention_flops(lengths, d, pad_to) is its cost.  No CPU path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import torch

from . import _lib
from .attention import MASK_BIDIR, varlen_attn_bwd, varlen_attn_fwd
from .errors import ConfigError
from .packing import SampleLen, _as_dev_i32, prune_view


@dataclass
class DynamicPad:
    lengths: torch.Tensor     # int32 [n] (device)
    pad_to: int               # batch maximum
    pad_to_t: torch.Tensor    # int32 [1] (device copy)
    cu_seqlens: torch.Tensor  # int32 [n+1]: valid tokens, sample order (= sample-major row offsets)
    seg_src: torch.Tensor     # int32 [n]: i·pad_to

    @property
    def n(self) -> int:
        return self.lengths.numel()

    def padding_rate(self) -> float:
        """SPEC.md:456-460 at the dynamic pad length."""
        return 1.0 - int(self.cu_seqlens[-1]) / (self.n * self.pad_to)


def dynamic_pad(lengths, stream=None) -> DynamicPad:
    """Device dynamic_pad_length + the segment metadata of the padded batch (reads pad_to back to
    the host, which allocating the padded tensors needs).  Empty batch / a length < 1 → ConfigError."""
    d_len = _as_dev_i32(lengths)
    n = d_len.numel()
    if n < 1:
        raise ConfigError("dynamic_pad_length: empty batch")
    dev = d_len.device
    pad_to = torch.empty(1, dtype=torch.int32, device=dev)
    cu = torch.empty(n + 1, dtype=torch.int32, device=dev)
    seg = torch.empty(n, dtype=torch.int32, device=dev)
    status = torch.empty(2, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().vlasim_dynamic_pad_cuda(_lib.ptr(d_len, _lib.i32p), n, _lib.ptr(pad_to, _lib.i32p),
                                                  _lib.ptr(cu, _lib.i32p), _lib.ptr(seg, _lib.i32p),
                                                  _lib.ptr(status, _lib.i32p), 1, _lib.stream_ptr(stream)),
               "dynamic_pad")
    return DynamicPad(d_len, int(pad_to.item()), pad_to, cu, seg)


def _row_bytes(x: torch.Tensor) -> int:
    rb = x[0].numel() * x.element_size() if x.dim() > 1 else x.element_size()
    if rb % 16:
        raise ConfigError("pad/unpad rows must be a multiple of 16 bytes")
    return rb


def pad_rows(x: torch.Tensor, dp: DynamicPad, stream=None) -> torch.Tensor:
    """x [Σl, ...] in sample-major order → [n·pad_to, ...] (sample i at rows i·pad_to), zero fill."""
    T = int(dp.cu_seqlens[-1])
    if x.shape[0] != T or not x.is_contiguous() or not x.is_cuda:
        raise ConfigError(f"pad_rows: expected a contiguous CUDA tensor with {T} rows")
    out = torch.empty((dp.n * dp.pad_to,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    _lib.check(_lib.lib().vlasim_pad_rows_cuda(_lib.ptr(x), _lib.ptr(out), _row_bytes(x),
                                               _lib.ptr(dp.lengths, _lib.i32p), _lib.ptr(dp.cu_seqlens, _lib.i32p),
                                               _lib.ptr(dp.pad_to_t, _lib.i32p), dp.n, _lib.stream_ptr(stream)),
               "pad_rows")
    return out


def unpad_rows(xp: torch.Tensor, dp: DynamicPad, stream=None) -> torch.Tensor:
    """Inverse of pad_rows: the valid rows of [n·pad_to, ...] back to sample-major [Σl, ...]."""
    if xp.shape[0] != dp.n * dp.pad_to or not xp.is_contiguous() or not xp.is_cuda:
        raise ConfigError("unpad_rows: expected a contiguous CUDA tensor of n·pad_to rows")
    T = int(dp.cu_seqlens[-1])
    out = torch.empty((T,) + tuple(xp.shape[1:]), dtype=xp.dtype, device=xp.device)
    _lib.check(_lib.lib().vlasim_unpad_rows_cuda(_lib.ptr(xp), _lib.ptr(out), _row_bytes(xp),
                                                 _lib.ptr(dp.lengths, _lib.i32p), _lib.ptr(dp.cu_seqlens, _lib.i32p),
                                                 _lib.ptr(dp.pad_to_t, _lib.i32p), dp.n, _lib.stream_ptr(stream)),
               "unpad_rows")
    return out


def padded_attention_fwd(qp, kp, vp, dp: DynamicPad, *, mask_mode=MASK_BIDIR, prefix_len=None, softmax_scale=None,
                         stream=None):
    """Attention over padded [n·pad_to, heads, d] tensors: o (pad rows 0) and lse [H, n·pad_to] (pad 0)."""
    o = torch.zeros_like(qp)
    lse = torch.zeros(qp.shape[1], qp.shape[0], dtype=torch.float32, device=qp.device)
    return varlen_attn_fwd(qp, kp, vp, dp.cu_seqlens, mask_mode=mask_mode, prefix_len=prefix_len,
                           softmax_scale=softmax_scale, out=o, lse=lse, seg_src=dp.seg_src, stream=stream)


def padded_attention_bwd(dop, qp, kp, vp, op, lse, dp: DynamicPad, *, mask_mode=MASK_BIDIR, prefix_len=None,
                         softmax_scale=None, stream=None):
    """Gradients on the padded storage (pad rows of dq/dk/dv are 0)."""
    dq, dk, dv = torch.zeros_like(qp), torch.zeros_like(kp), torch.zeros_like(vp)
    return varlen_attn_bwd(dop, qp, kp, vp, op, lse, dp.cu_seqlens, mask_mode=mask_mode, prefix_len=prefix_len,
                           softmax_scale=softmax_scale, dq=dq, dk=dk, dv=dv, seg_src=dp.seg_src, stream=stream)


def prune_corpus(samples: Sequence[SampleLen], view: str) -> List[SampleLen]:
    """π0.5 view pruning over a batch: every sample must carry the view."""
    return [prune_view(s, view) for s in samples]
