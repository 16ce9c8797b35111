"""Seeded synthetic inputs, identical on CPU (oracle) and GPU.

Lengths come from the reference's seeding API (rng.hpp, via the C-ABI host generator);
tensor values are counter-based: x[i] = (top8(splitmix64(seed ^ i)) − 128) / 128, exactly
representable in bf16, with seed = derive_seed(root, label, 0).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

MASK64 = (1 << 64) - 1

DIST_UNIFORM, DIST_GEOMETRIC, DIST_GR00T, DIST_PI05 = 0, 1, 2, 3


def splitmix64(x: int) -> int:
    """rng.hpp:9-14."""
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def derive_seed(root: int, label: str, index: int = 0) -> int:
    """rng.hpp:19-24."""
    h = (root ^ 0x8824A7155D1E9E31) & MASK64
    for ch in label.encode():
        h = splitmix64(h ^ ch)
    return splitmix64(h ^ splitmix64(index))


def gen_lengths(n: int, dist: int = DIST_UNIFORM, p1: float = 16, p2: float = 512, p3: float = 0,
                seed: int = 42, label: str = "lengths") -> np.ndarray:
    """Sample lengths from make_rng(seed, label, 0) (rng.hpp:28-49); see vlasim_gen_lengths."""
    out = np.empty(n, dtype=np.int32)
    rc = _lib.lib().vlasim_gen_lengths(C.c_uint64(seed), label.encode(), dist, n, p1, p2, p3,
                                       out.ctypes.data_as(_lib.i32p))
    _lib.check(rc, "gen_lengths")
    return out


def fill_bf16(t: torch.Tensor, label: str, root: int = 42, stream=None) -> torch.Tensor:
    """Fill a contiguous bf16 CUDA tensor with the counter-based synthetic values."""
    assert t.dtype == torch.bfloat16 and t.is_cuda and t.is_contiguous()
    rc = _lib.lib().vlasim_fill_synthetic_bf16(_lib.ptr(t), t.numel(), C.c_uint64(derive_seed(root, label)),
                                               _lib.stream_ptr(stream))
    _lib.check(rc, "fill_synthetic")
    return t


def values_np(count: int, label: str, root: int = 42, offset: int = 0) -> np.ndarray:
    """CPU twin of fill_bf16 (float32, exact): values of flat indices [offset, offset+count)."""
    seed = np.uint64(derive_seed(root, label))
    i = np.arange(offset, offset + count, dtype=np.uint64) ^ seed
    with np.errstate(over="ignore"):
        z = i + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(56)).astype(np.int32) - 128).astype(np.float32) / 128.0
