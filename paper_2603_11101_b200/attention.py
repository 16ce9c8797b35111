"""Varlen attention API — mirror of the reference's `vlasim::packed_attention(q, k, v, cu_seqlens)`
(multi-head = the reference's looped single-head op) on the
hand-written sm_100a kernels.  Every call goes through the C-ABI; no CPU fallback.

Layout: q/o [T, H, d] bf16, k/v [T, Hkv, d] bf16, lse [H, T] fp32, cu_seqlens [nseq+1] int32.
With seg_src (int32 [nseq], packing.seg_src) the tensors stay in sample-major order and the packed
stream is virtual: segment m's rows are read / written at seg_src[m] + offset (the gather and the
scatter folded into the kernels' TMA coordinates).
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from . import _lib
from .errors import ConfigError

MASK_BIDIR, MASK_CAUSAL, MASK_PREFIX = 0, 1, 2


def _args(q, k, v, o, lse, cu_seqlens, mask_mode, prefix_len, softmax_scale, q_scale=None, k_scale=None,
          seg_src=None, sm_budget=0):
    if q.dim() != 3 or k.dim() != 3 or v.dim() != 3:
        raise ConfigError("q, k, v must be [T, heads, d]")
    T, H, d = q.shape
    if k.shape[0] != T or v.shape != k.shape or k.shape[2] != d:
        raise ConfigError("k/v shape mismatch with q")
    if H % k.shape[1]:
        raise ConfigError("num_kv_heads must divide num_heads")
    if cu_seqlens.dtype != torch.int32:
        raise ConfigError("cu_seqlens must be int32")
    for t in (q, k, v, o, cu_seqlens):
        if not t.is_cuda or not t.is_contiguous():
            raise ConfigError("tensors must be contiguous CUDA tensors")
    fp8 = q_scale is not None or k_scale is not None
    qk_dtype = torch.uint8 if fp8 else torch.bfloat16
    if q.dtype != qk_dtype or k.dtype != qk_dtype:
        raise ConfigError(f"q and k must be {qk_dtype} (got {q.dtype}, {k.dtype})")
    if v.dtype != torch.bfloat16 or o.dtype != torch.bfloat16:
        raise ConfigError(f"v and o must be torch.bfloat16 (got {v.dtype}, {o.dtype})")
    if o.shape != q.shape:
        raise ConfigError("o must have q's shape")
    if lse.dtype != torch.float32 or tuple(lse.shape) != (H, T) or not lse.is_contiguous():
        raise ConfigError("lse must be a contiguous float32 [H, T] tensor")
    dev = q.device
    if mask_mode not in (MASK_BIDIR, MASK_CAUSAL, MASK_PREFIX):
        raise ConfigError(f"unknown mask_mode {mask_mode}")
    if mask_mode == MASK_PREFIX and prefix_len is None:
        raise ConfigError("prefix mask needs prefix_len")
    if prefix_len is not None and (prefix_len.dtype != torch.int32 or prefix_len.numel() != cu_seqlens.numel() - 1):
        raise ConfigError("prefix_len must be int32 [num_seqs]")
    if seg_src is not None and (seg_src.dtype != torch.int32 or seg_src.numel() != cu_seqlens.numel() - 1):
        raise ConfigError("seg_src must be int32 [num_seqs]")
    for name, t in (("k", k), ("v", v), ("o", o), ("lse", lse), ("cu_seqlens", cu_seqlens), ("prefix_len", prefix_len),
                    ("seg_src", seg_src), ("q_scale", q_scale), ("k_scale", k_scale)):
        if t is not None and (t.device != dev or not t.is_contiguous()):
            raise ConfigError(f"{name} must be a contiguous tensor on {dev}")
    for name, t in (("q_scale", q_scale), ("k_scale", k_scale)):
        if t is not None and t.dtype != torch.float32:
            raise ConfigError(f"{name} must be float32")
    scale = float(softmax_scale) if softmax_scale is not None else 1.0 / math.sqrt(d)
    a = _lib.AttnArgs(
        _lib.ptr(q).value, _lib.ptr(k).value, _lib.ptr(v).value, _lib.ptr(o).value, _lib.ptr(lse, _lib.f32p),
        _lib.ptr(cu_seqlens, _lib.i32p), _lib.ptr(prefix_len, _lib.i32p) if prefix_len is not None else None,
        cu_seqlens.numel() - 1, T, H, k.shape[1], d, int(mask_mode), scale,
        _lib.ptr(q_scale, _lib.f32p) if q_scale is not None else None,
        _lib.ptr(k_scale, _lib.f32p) if k_scale is not None else None,
        _lib.ptr(seg_src, _lib.i32p) if seg_src is not None else None, int(sm_budget or 0))
    return a


class BwdWorkspace:
    """Reusable device workspace (fwd: per-token visible spans + tile table; bwd: LSE/D windows, spans,
    tiles).  One workspace serves one stream at a time; pass your own to every call that is captured
    into a CUDA graph (the graph bakes in its pointer)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes, device):
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


class _PerStream:
    """Default workspaces keyed by (device, stream): calls on different streams never share one."""

    def __init__(self):
        self.ws = {}

    def get(self, nbytes, device, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(device)
        w = self.ws.setdefault((device, s.cuda_stream), BwdWorkspace())
        return w.get(nbytes, device)


_default_ws = _PerStream()
_default_fwd_ws = _PerStream()


def varlen_attn_fwd(q, k, v, cu_seqlens, *, mask_mode=MASK_BIDIR, prefix_len=None, softmax_scale=None, out=None,
                    lse=None, workspace: BwdWorkspace | None = None, seg_src=None, sm_budget=0, stream=None):
    """Block-diagonal attention forward. Returns (o [T,H,d] bf16, lse [H,T] fp32 natural-log)."""
    T, H, d = q.shape
    o = out if out is not None else torch.empty_like(q)
    lse = lse if lse is not None else torch.empty(H, T, dtype=torch.float32, device=q.device)
    a = _args(q, k, v, o, lse, cu_seqlens, mask_mode, prefix_len, softmax_scale, seg_src=seg_src, sm_budget=sm_budget)
    L = _lib.lib()
    nbytes = L.vlasim_varlen_attn_workspace_size(C.byref(a), 0)
    ws = workspace.get(nbytes, q.device) if workspace else _default_fwd_ws.get(nbytes, q.device, stream)
    _lib.check(L.vlasim_varlen_attn_fwd_cuda(C.byref(a), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)),
               "varlen_attn_fwd")
    return o, lse


def varlen_attn_bwd(dout, q, k, v, o, lse, cu_seqlens, *, mask_mode=MASK_BIDIR, prefix_len=None,
                    softmax_scale=None, dq=None, dk=None, dv=None, workspace: BwdWorkspace | None = None,
                    row_map=None, seg_src=None, sm_budget=0, stream=None):
    """Backward of varlen_attn_fwd. Returns (dq, dk, dv) bf16.  With row_map (int32 [T], e.g. the
    packer's gather index) gradient row t is written to row row_map[t] — the scatter back to sample
    order fused into the kernels."""
    dq = dq if dq is not None else torch.empty_like(q)
    dk = dk if dk is not None else torch.empty_like(k)
    dv = dv if dv is not None else torch.empty_like(v)
    if not dout.is_contiguous() or dout.shape != q.shape or dout.dtype != torch.bfloat16 or dout.device != q.device:
        raise ConfigError("dout must be a contiguous bf16 tensor with q's shape on q's device")
    for name, t, ref in (("dq", dq, q), ("dk", dk, k), ("dv", dv, v)):
        if t.shape != ref.shape or t.dtype != torch.bfloat16 or not t.is_contiguous() or t.device != q.device:
            raise ConfigError(f"{name} must be a contiguous bf16 tensor shaped like its input")
    a = _args(q, k, v, o, lse, cu_seqlens, mask_mode, prefix_len, softmax_scale, seg_src=seg_src, sm_budget=sm_budget)
    if row_map is not None and (row_map.dtype != torch.int32 or row_map.numel() != q.shape[0]
                                or row_map.device != q.device):
        raise ConfigError("row_map must be int32 [T]")
    g = _lib.AttnGrads(_lib.ptr(dout).value, _lib.ptr(dq).value, _lib.ptr(dk).value, _lib.ptr(dv).value,
                       _lib.ptr(row_map, _lib.i32p) if row_map is not None else None)
    L = _lib.lib()
    nbytes = L.vlasim_varlen_attn_workspace_size(C.byref(a), 1)
    ws = workspace.get(nbytes, q.device) if workspace else _default_ws.get(nbytes, q.device, stream)
    _lib.check(L.vlasim_varlen_attn_bwd_cuda(C.byref(a), C.byref(g), _lib.ptr(ws), ws.numel(),
                                             _lib.stream_ptr(stream)), "varlen_attn_bwd")
    return dq, dk, dv


def packed_attention(q, k, v, cu_seqlens, **kw):
    """Reference name: per-segment attention over the packed stream; returns o."""
    return varlen_attn_fwd(q, k, v, cu_seqlens, **kw)[0]


class VarlenAttention(torch.autograd.Function):
    """autograd wrapper: o = packed_attention(q, k, v, cu_seqlens) with the hand-written backward."""

    @staticmethod
    def forward(ctx, q, k, v, cu_seqlens, mask_mode=MASK_BIDIR, prefix_len=None, softmax_scale=None):
        o, lse = varlen_attn_fwd(q, k, v, cu_seqlens, mask_mode=mask_mode, prefix_len=prefix_len,
                                 softmax_scale=softmax_scale)
        ctx.save_for_backward(q, k, v, o, lse, cu_seqlens, prefix_len)
        ctx.mask_mode, ctx.softmax_scale = mask_mode, softmax_scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse, cu, prefix = ctx.saved_tensors
        dq, dk, dv = varlen_attn_bwd(do.contiguous(), q, k, v, o, lse, cu, mask_mode=ctx.mask_mode,
                                     prefix_len=prefix, softmax_scale=ctx.softmax_scale)
        return dq, dk, dv, None, None, None, None
