"""E4M3 per-block quantisation and the FP8 Q/K attention forward (config 4).

quant_block(x [T, heads, d] bf16) → (codes uint8 [T, heads, d], scales fp32 [heads, ⌈T/128⌉, ⌈d/128⌉]):
per head, 128-token × 128-d blocks; scale = amax/448 (1 for an all-zero block); codes = RNE(x/scale)
saturated to ±448.  GPU only (vlasim_fp8_quant_block_cuda).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .attention import _args, _default_fwd_ws, _default_ws
from .errors import ConfigError


def quant_block(x: torch.Tensor, stream=None, *, check_finite: bool = True, codes=None, scales=None, status=None):
    """check_finite (default): synchronise and raise ConfigError on a non-finite element.
    check_finite=False keeps the call asynchronous (the error stays on device in `status`, if given)."""
    if x.dtype != torch.bfloat16 or x.dim() != 3 or not x.is_cuda or not x.is_contiguous():
        raise ConfigError("quant_block expects a contiguous CUDA bf16 [T, heads, d] tensor")
    T, Hh, d = x.shape
    codes = codes if codes is not None else torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    scales = scales if scales is not None else torch.empty(Hh, (T + 127) // 128, (d + 127) // 128,
                                                           dtype=torch.float32, device=x.device)
    if status is None and check_finite:
        status = torch.empty(2, dtype=torch.int32, device=x.device)
    _lib.check(_lib.lib().vlasim_fp8_quant_block_cuda(
        _lib.ptr(x), T, Hh, d, _lib.ptr(codes), _lib.ptr(scales, _lib.f32p),
        _lib.ptr(status, _lib.i32p) if status is not None else None, 1 if check_finite else 0,
        _lib.stream_ptr(stream)), "fp8_quant_block")
    return codes, scales


def dequant_block(codes: torch.Tensor, scales: torch.Tensor, stream=None) -> torch.Tensor:
    T, Hh, d = codes.shape
    out = torch.empty(codes.shape, dtype=torch.float32, device=codes.device)
    _lib.check(_lib.lib().vlasim_fp8_dequant_block_cuda(_lib.ptr(codes), _lib.ptr(scales, _lib.f32p), T, Hh, d,
                                                        _lib.ptr(out, _lib.f32p), _lib.stream_ptr(stream)),
               "fp8_dequant_block")
    return out


def quant_error(x: torch.Tensor, codes: torch.Tensor, scales: torch.Tensor, stream=None) -> dict:
    """quant_error(original, qt) for a PerBlock(128,128) E4M3 quantisation of
    x [T, heads, d] bf16: {"max_rel": max relative error over elements quantised to E4M3 normals,
    "mse": mean squared error, "groups": {"max_rel", "mse"} per (head, token block, d block)}."""
    T, Hh, d = x.shape
    g = Hh * ((T + 127) // 128) * ((d + 127) // 128)
    gmax = torch.empty(g, dtype=torch.float32, device=x.device)
    gsse = torch.empty(g, dtype=torch.float64, device=x.device)
    gcnt = torch.empty(g, dtype=torch.int32, device=x.device)
    _lib.check(_lib.lib().vlasim_fp8_quant_error_cuda(_lib.ptr(x), _lib.ptr(codes), _lib.ptr(scales, _lib.f32p), T, Hh,
                                                      d, _lib.ptr(gmax, _lib.f32p), _lib.ptr(gsse), _lib.ptr(gcnt),
                                                      _lib.stream_ptr(stream)), "fp8_quant_error")
    shape = scales.shape
    return {"max_rel": float(gmax.max()), "mse": float(gsse.sum() / gcnt.sum()),
            "groups": {"max_rel": gmax.view(shape), "mse": (gsse / gcnt).view(shape)}}


def varlen_attn_fwd_fp8qk(q_codes, q_scale, k_codes, k_scale, v, cu_seqlens, *, mask_mode=0, prefix_len=None,
                          softmax_scale=None, out=None, lse=None, seg_src=None, stream=None):
    """Forward with E4M3 Q/K (tcgen05 kind::f8f6f4 for QKᵀ, block scales applied to S; P·V in bf16)."""
    T, H, d = q_codes.shape
    if q_codes.dtype != torch.uint8 or k_codes.dtype != torch.uint8:
        raise ConfigError("q_codes / k_codes must be uint8 E4M3 codes")
    o = out if out is not None else torch.empty(T, H, d, dtype=torch.bfloat16, device=v.device)
    lse = lse if lse is not None else torch.empty(H, T, dtype=torch.float32, device=v.device)
    a = _args(q_codes, k_codes, v, o, lse, cu_seqlens, mask_mode, prefix_len, softmax_scale, q_scale, k_scale,
              seg_src=seg_src)
    L = _lib.lib()
    ws = _default_fwd_ws.get(L.vlasim_varlen_attn_workspace_size(C.byref(a), 0), v.device, stream)
    _lib.check(L.vlasim_varlen_attn_fwd_fp8qk_cuda(C.byref(a), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)),
               "varlen_attn_fwd_fp8qk")
    return o, lse


def varlen_attn_bwd_fp8qk(dout, q_codes, q_scale, k_codes, k_scale, v, o, lse, cu_seqlens, *, mask_mode=0,
                          prefix_len=None, softmax_scale=None, dq=None, dk=None, dv=None, seg_src=None, row_map=None,
                          workspace=None, stream=None):
    """Backward of varlen_attn_fwd_fp8qk: (dq, dk, dv) bf16, the gradients with respect to the
    dequantised Q / K (straight-through for the quantiser) and V, from the FP8 forward's o / lse."""
    T, H, d = q_codes.shape
    dq = dq if dq is not None else torch.empty(T, H, d, dtype=torch.bfloat16, device=v.device)
    dk = dk if dk is not None else torch.empty(k_codes.shape, dtype=torch.bfloat16, device=v.device)
    dv = dv if dv is not None else torch.empty_like(v)
    if dout.shape != (T, H, d) or dout.dtype != torch.bfloat16 or not dout.is_contiguous():
        raise ConfigError("dout must be a contiguous bf16 tensor shaped like q")
    if row_map is not None and (row_map.dtype != torch.int32 or row_map.numel() != T):
        raise ConfigError("row_map must be int32 [T]")
    a = _args(q_codes, k_codes, v, o, lse, cu_seqlens, mask_mode, prefix_len, softmax_scale, q_scale, k_scale,
              seg_src=seg_src)
    g = _lib.AttnGrads(_lib.ptr(dout).value, _lib.ptr(dq).value, _lib.ptr(dk).value, _lib.ptr(dv).value,
                       _lib.ptr(row_map, _lib.i32p) if row_map is not None else None)
    L = _lib.lib()
    nbytes = L.vlasim_varlen_attn_workspace_size(C.byref(a), 2)
    ws = workspace.get(nbytes, v.device) if workspace else _default_ws.get(nbytes, v.device, stream)
    _lib.check(L.vlasim_varlen_attn_bwd_fp8qk_cuda(C.byref(a), C.byref(g), _lib.ptr(ws), ws.numel(),
                                                   _lib.stream_ptr(stream)), "varlen_attn_bwd_fp8qk")
    return dq, dk, dv
