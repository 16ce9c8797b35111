"""The reference's quantizer module (proj/CMakeLists.txt:18-21
src/quant/{fp8,tensor,quantize,compression}.cpp) on the GPU.

    quantize(x, granularity, axis)   -> QuantizedTensor
    dequantize(qt)                   -> fp32 tensor
    quant_error(x, qt)               -> QuantError
    block_partition(shape, block)    -> block extents
    compression_ratio(spec)          -> fraction of bytes saved

Granularity: "tensor" | "channel" (with `axis`) | "block" (128 × 128 over the last two dims).
Codes are the exact RNE E4M3 codes of the real quotient x·448/amax (vlasim_fp8_quantize_cuda);
the input is fp32 or bf16 on a CUDA device — the SPEC's "high-precision real" is held at fp32 on
the device (codes are bit-exact with the SPEC for fp32-representable values).  No CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import torch

from . import _lib
from .errors import ConfigError

GRANULARITIES = {"tensor": 0, "channel": 1, "block": 2}
_DTYPES = {torch.float32: 0, torch.bfloat16: 1}
SCALE_BYTES = 4  # scale storage


@dataclass(frozen=True)
class Fp8Format:
    """E4M3 (the E4M3 choice SPEC.md:624)."""
    exponent_bits: int = 4
    mantissa_bits: int = 3
    bias: int = 7
    max_normal: float = 448.0


E4M3 = Fp8Format()


@dataclass
class QuantizedTensor:
    """codes (uint8 E4M3 bytes, the input's shape), fp32 scales shaped by the
    granularity, the original shape and the granularity tag."""
    codes: torch.Tensor
    scales: torch.Tensor
    shape: Tuple[int, ...]
    granularity: str
    axis: int = 0
    fmt: Fp8Format = E4M3


@dataclass
class QuantError:
    """quant_error metrics: max relative error over elements in E4M3's normal
    range, mean squared error, and the per-group table (scales' shape)."""
    max_rel: float
    mse: float
    group_max_rel: torch.Tensor
    group_mse: torch.Tensor
    group_count: torch.Tensor


def _gran(granularity: str) -> int:
    if granularity not in GRANULARITIES:
        raise ConfigError(f"unknown granularity '{granularity}' (tensor | channel | block)")
    return GRANULARITIES[granularity]


def _shape_arr(shape):
    arr = (C.c_int64 * len(shape))(*[int(s) for s in shape])
    return C.cast(arr, _lib.i64p), arr


def scales_shape(shape: Sequence[int], granularity: str, axis: int = 0) -> Tuple[int, ...]:
    """PerTensor (1,); PerChannel (shape[axis],); PerBlock (*shape[:-2], ⌈rows/128⌉, ⌈cols/128⌉)."""
    g = _gran(granularity)
    if g == 0:
        return (1,)
    if g == 1:
        if not -len(shape) <= axis < len(shape):
            raise ConfigError("quantize: channel axis out of range")
        return (int(shape[axis]),)
    if len(shape) < 2:
        raise ConfigError("quantize: PerBlock needs a tensor of >= 2 dims")
    return tuple(int(s) for s in shape[:-2]) + ((int(shape[-2]) + 127) // 128, (int(shape[-1]) + 127) // 128)


def block_partition(shape: Sequence[int], block: Tuple[int, int] = (128, 128)) -> List[Tuple[int, int, int, int]]:
    """blocks (row0, rows, col0, cols) tiling the last two dims, edge blocks
    truncated; the union is exact and disjoint (the same tiles the PerBlock kernels use)."""
    if len(shape) < 2:
        raise ConfigError("block_partition: shape needs >= 2 dims")
    R, Cc = int(shape[-2]), int(shape[-1])
    br, bc = block
    if br < 1 or bc < 1:
        raise ConfigError("block_partition: block dims must be >= 1")
    return [(r0, min(br, R - r0), c0, min(bc, Cc - c0)) for r0 in range(0, R, br) for c0 in range(0, Cc, bc)]


def quantize(x: torch.Tensor, granularity: str = "block", axis: int = 0, *, check_finite: bool = True,
             out: QuantizedTensor | None = None, workspace: torch.Tensor | None = None, stream=None) -> QuantizedTensor:
    """SPEC.md:580-588 on the GPU.  Non-finite input → ConfigError naming the flat index (synchronising;
    check_finite=False keeps the call asynchronous and leaves codes unwritten on error).  `out` (a
    QuantizedTensor of this shape and granularity) and `workspace` are reused when given."""
    if not torch.is_tensor(x) or not x.is_cuda or x.dtype not in _DTYPES or not x.is_contiguous():
        raise ConfigError("quantize expects a contiguous CUDA fp32 or bf16 tensor")
    if x.dim() < 1 or x.dim() > 8 or x.numel() < 1:
        raise ConfigError("quantize: 1-8 dims, non-empty")
    g = _gran(granularity)
    sshape = scales_shape(tuple(x.shape), granularity, axis)
    shp, keep = _shape_arr(x.shape)
    L = _lib.lib()
    nws = max(1, L.vlasim_fp8_quantize_workspace_size(shp, x.dim(), g, axis))
    nws = (nws + 15) // 16 * 16  # the 8-byte status word sits after the aligned workspace
    ws = workspace if workspace is not None and workspace.numel() >= nws + 8 else \
        torch.empty(nws + 8, dtype=torch.uint8, device=x.device)
    if out is not None and tuple(out.codes.shape) == tuple(x.shape) and tuple(out.scales.shape) == sshape:
        codes, scales = out.codes, out.scales
    else:
        codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
        scales = torch.empty(sshape, dtype=torch.float32, device=x.device)
    status = ws[nws:nws + 8].view(torch.int32)
    _lib.check(L.vlasim_fp8_quantize_cuda(_lib.ptr(x), _DTYPES[x.dtype], shp, x.dim(), g, axis, _lib.ptr(codes),
                                          _lib.ptr(scales, _lib.f32p), _lib.ptr(status, _lib.i32p), _lib.ptr(ws),
                                          nws, 1 if check_finite else 0, _lib.stream_ptr(stream)), "quantize")
    del keep
    return QuantizedTensor(codes, scales, tuple(x.shape), granularity, axis % x.dim() if g == 1 else 0)


def dequantize(qt: QuantizedTensor, stream=None) -> torch.Tensor:
    """codes × group scale (fp32, one rounding), original shape."""
    g = _gran(qt.granularity)
    shp, keep = _shape_arr(qt.shape)
    out = torch.empty(qt.shape, dtype=torch.float32, device=qt.codes.device)
    _lib.check(_lib.lib().vlasim_fp8_dequantize_cuda(_lib.ptr(qt.codes), _lib.ptr(qt.scales, _lib.f32p), shp,
                                                     len(qt.shape), g, qt.axis, _lib.ptr(out, _lib.f32p),
                                                     _lib.stream_ptr(stream)), "dequantize")
    del keep
    return out


def quant_error(x: torch.Tensor, qt: QuantizedTensor, stream=None) -> QuantError:
    """SPEC.md:599-606, reduced per group in a fixed order (deterministic)."""
    if tuple(x.shape) != tuple(qt.shape):
        raise ConfigError("quant_error: shapes differ")
    if x.dtype not in _DTYPES or not x.is_cuda or not x.is_contiguous():
        raise ConfigError("quant_error expects a contiguous CUDA fp32 or bf16 tensor")
    g = _gran(qt.granularity)
    shp, keep = _shape_arr(qt.shape)
    L = _lib.lib()
    ng = L.vlasim_fp8_error_groups(shp, len(qt.shape), g, qt.axis)
    gmax = torch.empty(ng, dtype=torch.float32, device=x.device)
    gsse = torch.empty(ng, dtype=torch.float64, device=x.device)
    gcnt = torch.empty(ng, dtype=torch.int64, device=x.device)
    _lib.check(L.vlasim_fp8_quant_error_general_cuda(_lib.ptr(x), _DTYPES[x.dtype], _lib.ptr(qt.codes),
                                                     _lib.ptr(qt.scales, _lib.f32p), shp, len(qt.shape), g, qt.axis,
                                                     _lib.ptr(gmax, _lib.f32p), _lib.ptr(gsse),
                                                     _lib.ptr(gcnt, _lib.i64p), _lib.stream_ptr(stream)),
               "quant_error")
    del keep
    if g == 0:
        gmax, gsse, gcnt = gmax[:1], gsse[:1], gcnt[:1]
    shape = qt.scales.shape
    return QuantError(float(gmax.max()), float(gsse.sum() / gcnt.sum()), gmax.view(shape),
                      (gsse / gcnt).view(shape), gcnt.view(shape))


# ------------------------------------------------------------------ compression
@dataclass
class ModelComponent:
    name: str
    params: int
    quantize: bool
    granularity: str = "block"


@dataclass
class ModelSizeSpec:
    """components (name, parameter count, quantize?), bytes_hi (2), bytes_lo (1),
    scale element bytes (4).  `group_elems` is the elements per scale under each granularity
    (PerBlock 128·128; PerChannel / PerTensor: pass the layer shapes' values for an exact count —
    the default treats them as negligible, like the SPEC's amortised accounting)."""
    components: List[ModelComponent] = field(default_factory=list)
    bytes_hi: float = 2.0
    bytes_lo: float = 1.0
    scale_bytes: float = SCALE_BYTES
    group_elems: dict = field(default_factory=lambda: {"block": 128 * 128, "channel": float("inf"),
                                                       "tensor": float("inf")})


def compression_ratio(spec: ModelSizeSpec) -> float:
    """1 − (Σ unquantized·bytes_hi + Σ quantized·(bytes_lo + scale bytes per element)) / (Σ all·bytes_hi)
    (SPEC.md:608-615)."""
    if not spec.components:
        raise ConfigError("compression_ratio: empty spec")
    total = hi = lo = 0.0
    for c in spec.components:
        if c.params <= 0:
            raise ConfigError(f"compression_ratio: component '{c.name}' has {c.params} parameters")
        total += c.params
        if c.quantize:
            lo += c.params * (spec.bytes_lo + spec.scale_bytes / spec.group_elems[c.granularity])
        else:
            hi += c.params * spec.bytes_hi
    return 1.0 - (hi + lo) / (total * spec.bytes_hi)
