"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of the CPU restatement (oracle/vlasim_oracle.cpp) plus the numpy layout
restatement of the packed stream.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs may import this module; the product (paper_2603_11101_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)

_lib = None


def build(force: bool = False) -> None:
    if force or not LIB.exists():
        subprocess.run(["make", "-C", str(HERE), "liboracle.so", "rng_kat"], check=True, capture_output=True)
        if Path("/root/reference/proj/include").exists():
            subprocess.run(["make", "-C", str(HERE), "ref"], check=True, capture_output=True)


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(LIB))
        _lib.oracle_last_error.restype = C.c_char_p
        I, L, D, V = C.c_int, C.c_int64, C.c_double, C.c_void_p
        sigs = {
            "oracle_pack": [V, L, L, I, V, V, V, V],
            "oracle_cu_seqlens": [V, L, V],
            "oracle_padding_rate": [V, L, L, V],
            "oracle_dynamic_pad_length": [V, L, V],
            "oracle_attention_flops": [V, L, L, L, V],
            "oracle_prune_view": [V, V, L, L, C.c_char_p, C.c_char_p, V],
            "oracle_reference_attention": [V, V, V, L, L, V],
            "oracle_packed_attention": [V, V, V, L, L, V, L, I, V],
            "oracle_mha_fwd_f64": [V, V, V, V, V, V, L, V, L, L, L, L, I, D, I],
            "oracle_mha_fwd_f32": [V, V, V, V, V, V, L, V, L, L, L, L, I, D, I],
            "oracle_mha_bwd_f64": [V] * 9 + [L, V, L, L, L, L, I, D, I],
            "oracle_mha_bwd_f32": [V] * 9 + [L, V, L, L, L, L, I, D, I],
            "oracle_fp8_quant_block": [V, L, L, L, I, V, V],
            "oracle_fp8_quantize": [V, V, I, I, I, V, V],
            "oracle_e4m3_encode": [V, L, V],
            "oracle_e4m3_values": [V],
            "oracle_gen_lengths": [C.c_uint64, C.c_char_p, I, L, D, D, D, V],
        }
        for name, args in sigs.items():
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
    return _lib


class OracleConfigError(ValueError):
    pass


def _chk(rc):
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        if rc == 2:
            raise OracleConfigError(msg)
        raise RuntimeError(msg)


def _p(a, t):
    return a.ctypes.data_as(t)


# ------------------------------------------------------------------ packing
def pack(lengths, capacity: int, mode: int = 1):
    """mode 0 FFD naive scan, 1 FFD segment tree, 2 greedy arrival order.
    Returns (bin_of, slot, tok_off, num_bins) as int32 arrays."""
    L = np.ascontiguousarray(lengths, dtype=np.int64)
    n = L.size
    bin_of = np.empty(n, np.int32)
    slot = np.empty(n, np.int32)
    tok = np.empty(n, np.int32)
    nb = C.c_int32(0)
    _chk(lib().oracle_pack(_p(L, i64p), n, capacity, mode, _p(bin_of, i32p), _p(slot, i32p), _p(tok, i32p),
                           C.byref(nb)))
    return bin_of, slot, tok, nb.value


def layout(lengths, bin_of, slot, tok_off, num_bins):
    """Packed-stream layout restated in numpy from the bin assignment:
    bins in index order, members in insertion order."""
    L = np.asarray(lengths, np.int64)
    n = L.size
    bin_count = np.bincount(bin_of, minlength=num_bins).astype(np.int64)
    bin_fill = np.bincount(bin_of, weights=L, minlength=num_bins).astype(np.int64)
    bmo = np.concatenate([[0], np.cumsum(bin_count)])
    bto = np.concatenate([[0], np.cumsum(bin_fill)])
    m = bmo[bin_of] + slot
    member_ids = np.empty(n, np.int64)
    member_ids[m] = np.arange(n)
    cu = np.empty(n + 1, np.int64)
    cu[m] = bto[bin_of] + tok_off
    cu[n] = L.sum()
    cub = np.empty(n + num_bins, np.int64)
    cub[bmo[bin_of] + bin_of + slot + 1] = tok_off + L
    cub[bmo[:-1] + np.arange(num_bins)] = 0
    src_off = np.concatenate([[0], np.cumsum(L)[:-1]])
    return dict(bin_count=bin_count, bin_fill=bin_fill, bin_member_off=bmo, bin_token_off=bto,
                member_ids=member_ids, cu_seqlens=cu, cu_seqlens_bins=cub, src_off=src_off)


def token_ids(lengths, lay):
    L = np.asarray(lengths, np.int64)
    pos, seg, gat = [], [], []
    for m, i in enumerate(lay["member_ids"]):
        l = L[i]
        pos.append(np.arange(l))
        seg.append(np.full(l, m))
        gat.append(lay["src_off"][i] + np.arange(l))
    return np.concatenate(pos), np.concatenate(seg), np.concatenate(gat)


def cu_seqlens(member_lens):
    a = np.ascontiguousarray(member_lens, np.int64)
    out = np.empty(a.size + 1, np.int64)
    _chk(lib().oracle_cu_seqlens(_p(a, i64p), a.size, _p(out, i64p)))
    return out


def padding_rate(lengths, pad_to):
    a = np.ascontiguousarray(lengths, np.int64)
    r = C.c_double()
    _chk(lib().oracle_padding_rate(_p(a, i64p), a.size, pad_to, C.byref(r)))
    return r.value


def dynamic_pad_length(lengths):
    a = np.ascontiguousarray(lengths, np.int64)
    r = C.c_int64()
    _chk(lib().oracle_dynamic_pad_length(_p(a, i64p), a.size, C.byref(r)))
    return r.value


def attention_flops(lengths, d, pad_to=None):
    a = np.ascontiguousarray(lengths, np.int64)
    r = C.c_double()
    _chk(lib().oracle_attention_flops(_p(a, i64p), a.size, pad_to or 0, d, C.byref(r)))
    return r.value


def prune_view(views: dict, text: int, prune1=None, prune2=None):
    names = (C.c_char_p * len(views))(*[k.encode() for k in views])
    counts = np.array(list(views.values()), np.int64)
    r = C.c_int64()
    _chk(lib().oracle_prune_view(names, _p(counts, i64p), len(views), text,
                                 prune1.encode() if prune1 else None, prune2.encode() if prune2 else None,
                                 C.byref(r)))
    return r.value


# ------------------------------------------------------------------ attention
def reference_attention(q, k, v):
    q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
    out = np.empty_like(q)
    _chk(lib().oracle_reference_attention(_p(q, f64p), _p(k, f64p), _p(v, f64p), q.shape[0], q.shape[1],
                                          _p(out, f64p)))
    return out


def packed_attention(q, k, v, cu, masked=False):
    q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
    cu = np.ascontiguousarray(cu, np.int64)
    out = np.empty_like(q)
    _chk(lib().oracle_packed_attention(_p(q, f64p), _p(k, f64p), _p(v, f64p), q.shape[0], q.shape[1],
                                       _p(cu, i64p), cu.size, 1 if masked else 0, _p(out, f64p)))
    return out


def _mha_common(q, k, cu, prefix, dtype):
    T, H, d = q.shape
    Hkv = k.shape[1]
    cu32 = np.ascontiguousarray(cu, np.int32)
    pre = np.ascontiguousarray(prefix, np.int32) if prefix is not None else np.zeros(1, np.int32)
    return T, H, Hkv, d, cu32, pre


def mha_fwd(q, k, v, cu, *, mask=0, prefix=None, scale=None, dtype=np.float64, threads=None):
    """Multi-head varlen forward (fp64 checker / fp32 CPU baseline). Returns (o, lse [H,T])."""
    q, k, v = (np.ascontiguousarray(x, dtype) for x in (q, k, v))
    T, H, Hkv, d, cu32, pre = _mha_common(q, k, cu, prefix, dtype)
    scale = scale if scale is not None else 1.0 / np.sqrt(d)
    o = np.empty_like(q)
    lse = np.empty((H, T), dtype)
    fn = lib().oracle_mha_fwd_f64 if dtype == np.float64 else lib().oracle_mha_fwd_f32
    tp = f64p if dtype == np.float64 else f32p
    _chk(fn(_p(q, tp), _p(k, tp), _p(v, tp), _p(o, tp), _p(lse, tp), _p(cu32, i32p), cu32.size - 1,
            _p(pre, i32p), T, H, Hkv, d, mask, C.c_double(scale), threads or os.cpu_count()))
    return o, lse


def mha_bwd(q, k, v, o, do, cu, *, mask=0, prefix=None, scale=None, dtype=np.float64, threads=None):
    q, k, v, o, do = (np.ascontiguousarray(x, dtype) for x in (q, k, v, o, do))
    T, H, Hkv, d, cu32, pre = _mha_common(q, k, cu, prefix, dtype)
    scale = scale if scale is not None else 1.0 / np.sqrt(d)
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    fn = lib().oracle_mha_bwd_f64 if dtype == np.float64 else lib().oracle_mha_bwd_f32
    tp = f64p if dtype == np.float64 else f32p
    _chk(fn(_p(q, tp), _p(k, tp), _p(v, tp), _p(o, tp), _p(do, tp), _p(dq, tp), _p(dk, tp), _p(dv, tp),
            _p(cu32, i32p), cu32.size - 1, _p(pre, i32p), T, H, Hkv, d, mask, C.c_double(scale),
            threads or os.cpu_count()))
    return dq, dk, dv


# ------------------------------------------------------------------ E4M3
def e4m3_values():
    out = np.empty(127, np.float64)
    _chk(lib().oracle_e4m3_values(_p(out, f64p)))
    return out


def e4m3_encode(x):
    x = np.ascontiguousarray(x, np.float64)
    codes = np.empty(x.shape, np.uint8)
    _chk(lib().oracle_e4m3_encode(_p(x, f64p), x.size, _p(codes, u8p)))
    return codes


def fp8_quant_block(x, quotient_fp32=True):
    """x [T, heads, d] float32 → (codes uint8 [T,heads,d], scales [heads, ceil(T/128), ceil(d/128)])."""
    x = np.ascontiguousarray(x, np.float32)
    T, Hh, d = x.shape
    codes = np.empty(x.shape, np.uint8)
    scales = np.empty((Hh, (T + 127) // 128, (d + 127) // 128), np.float32)
    _chk(lib().oracle_fp8_quant_block(_p(x, f32p), T, Hh, d, 1 if quotient_fp32 else 0, _p(codes, u8p),
                                      _p(scales, f32p)))
    return codes, scales


GRAN = {"tensor": 0, "channel": 1, "block": 2}


def fp8_groups(shape, gran, axis=0):
    """Group count and flat index → group map of a granularity."""
    shape = tuple(int(s) for s in shape)
    n = int(np.prod(shape))
    i = np.arange(n, dtype=np.int64)
    if gran == "tensor":
        return 1, np.zeros(n, np.int64)
    if gran == "channel":
        axis = axis % len(shape)
        inner = int(np.prod(shape[axis + 1:])) if axis + 1 < len(shape) else 1
        return shape[axis], (i // inner) % shape[axis]
    rows, cols = shape[-2], shape[-1]
    nbr, nbc = (rows + 127) // 128, (cols + 127) // 128
    c, r, b = i % cols, (i // cols) % rows, i // (rows * cols)
    return (n // (rows * cols)) * nbr * nbc, (b * nbr + r // 128) * nbc + c // 128


def fp8_quantize(x, gran="block", axis=0):
    """SPEC quantize at any granularity: (codes uint8 like x, scales f32 [groups])."""
    x = np.ascontiguousarray(x, np.float32)
    shape = np.asarray(x.shape, np.int64)
    ngroups, _ = fp8_groups(x.shape, gran, axis)
    codes = np.empty(x.shape, np.uint8)
    scales = np.empty(ngroups, np.float32)
    _chk(lib().oracle_fp8_quantize(_p(x, f32p), _p(shape, i64p), x.ndim, GRAN[gran], axis, _p(codes, u8p),
                                   _p(scales, f32p)))
    return codes, scales


def e4m3_decode_table():
    vals = np.zeros(256, np.float32)
    for c in range(256):  # E4M3 decode: bias 7, subnormals, 0x7f/0xff NaN
        e, m = (c >> 3) & 0xF, c & 7
        v = (m / 8.0) * 2.0 ** -6 if e == 0 else ((1 + m / 8.0) * 2.0 ** (e - 7) if not (e == 15 and m == 7) else np.nan)
        vals[c] = -v if c & 0x80 else v
    return vals


def fp8_dequantize(codes, scales, gran="block", axis=0):
    """codes × group scale in fp32, original shape restored."""
    _, grp = fp8_groups(codes.shape, gran, axis)
    return (e4m3_decode_table()[codes.reshape(-1)] * np.asarray(scales, np.float32)[grp]).astype(np.float32).reshape(
        codes.shape)


def fp8_quant_error_general(x, codes, scales, gran="block", axis=0):
    """quant_error per group, the arithmetic of fp8_quant_error below:
    (group max_rel f32, group sse f64, group count, max_rel, mse)."""
    x = np.asarray(x, np.float32).reshape(-1)
    ngroups, grp = fp8_groups(codes.shape, gran, axis)
    sc = np.asarray(scales, np.float32)[grp]
    deq = (e4m3_decode_table()[codes.reshape(-1)] * sc).astype(np.float32)
    diff = (deq - x).astype(np.float32)
    normal = np.abs((x / sc).astype(np.float32)) >= np.float32(2.0 ** -6)
    rel = np.where(normal, np.abs(diff) / np.where(x != 0, np.abs(x), np.float32(1)), np.float32(0)).astype(np.float32)
    gmax = np.zeros(ngroups, np.float32)
    np.maximum.at(gmax, grp, rel)
    gsse = np.bincount(grp, weights=diff.astype(np.float64) ** 2, minlength=ngroups)
    gcnt = np.bincount(grp, minlength=ngroups)
    return gmax, gsse, gcnt, float(gmax.max()), float(gsse.sum() / gcnt.sum())


def fp8_quant_error(x, codes, scales):
    """quant_error(original, qt) restated for PerBlock(128,128) per head, with the
    arithmetic the GPU path pins: deq = fp32(value(code) · scale), diff = fp32(deq − x), relative
    error fp32(|diff| / |x|) over elements in E4M3's normal range (|fp32(x / scale)| >= 2^-6,
    SPEC.md:586); squared errors summed in fp64.
    Returns (group_max_rel [heads, ⌈T/128⌉, ⌈d/128⌉] f32, group_sse f64, group_count int, max_rel, mse)."""
    x = np.asarray(x, np.float32)
    codes = np.asarray(codes, np.uint8)
    T, Hh, d = x.shape
    nbt, nbd = (T + 127) // 128, (d + 127) // 128
    vals = np.zeros(256, np.float32)
    for c in range(256):  # E4M3 decode: bias 7, subnormals, 0x7f/0xff NaN
        e, m = (c >> 3) & 0xF, c & 7
        v = (m / 8.0) * 2.0 ** -6 if e == 0 else ((1 + m / 8.0) * 2.0 ** (e - 7) if not (e == 15 and m == 7) else np.nan)
        vals[c] = -v if c & 0x80 else v
    deq = vals[codes] * np.repeat(np.repeat(np.transpose(np.asarray(scales, np.float32), (1, 0, 2)), 128, 0)[:T],
                                  128, 2)[:, :, :d]  # fp32 · fp32
    diff = (deq - x).astype(np.float32)
    sc = np.repeat(np.repeat(np.transpose(np.asarray(scales, np.float32), (1, 0, 2)), 128, 0)[:T], 128, 2)[:, :, :d]
    normal = np.abs((x / sc).astype(np.float32)) >= np.float32(2.0 ** -6)
    rel = np.where(normal, np.abs(diff) / np.where(x != 0, np.abs(x), np.float32(1)), np.float32(0)).astype(np.float32)
    gmax = np.zeros((Hh, nbt, nbd), np.float32)
    gsse = np.zeros((Hh, nbt, nbd), np.float64)
    gcnt = np.zeros((Hh, nbt, nbd), np.int64)
    sq = diff.astype(np.float64) ** 2
    for h in range(Hh):
        for bt in range(nbt):
            for bd in range(nbd):
                sl = (slice(bt * 128, min(T, bt * 128 + 128)), h, slice(bd * 128, min(d, bd * 128 + 128)))
                gmax[h, bt, bd] = rel[sl].max() if rel[sl].size else 0.0
                gsse[h, bt, bd] = sq[sl].sum()
                gcnt[h, bt, bd] = sq[sl].size
    return gmax, gsse, gcnt, float(gmax.max()), float(gsse.sum() / gcnt.sum())


# ------------------------------------------------------------------ synthetic inputs (CPU arms)
def gen_lengths(n, dist=0, p1=16, p2=512, p3=0, seed=42, label="lengths"):
    """Sample lengths on the reference's rng.hpp (make_rng(seed, label, 0)), same as the bench inputs."""
    out = np.empty(n, np.int32)
    _chk(lib().oracle_gen_lengths(seed, label.encode(), dist, n, p1, p2, p3, _p(out, i32p)))
    return out


_M64 = (1 << 64) - 1


def _splitmix64(x):
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _derive_seed(root, label, index=0):
    h = (root ^ 0x8824A7155D1E9E31) & _M64
    for ch in label.encode():
        h = _splitmix64(h ^ ch)
    return _splitmix64(h ^ _splitmix64(index))


def synthetic_values(count, label, root=42, offset=0):
    """Counter-based bench values: x[i] = (top8(splitmix64(seed ^ i)) − 128) / 128 with
    seed = derive_seed(root, label, 0) (rng.hpp:9-24); float32, exactly bf16-representable."""
    seed = np.uint64(_derive_seed(root, label))
    i = np.arange(offset, offset + count, dtype=np.uint64) ^ seed
    with np.errstate(over="ignore"):
        z = i + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(56)).astype(np.int32) - 128).astype(np.float32) / 128.0
