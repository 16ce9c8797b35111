"""Packing API — Python mirror of the reference's `vlasim` packing entry points.

Reference interface (reconstructed; behaviour from SPEC.md:408-537):
    SampleLen / prune_view          SPEC.md:413-417, 483-491   (host logic)
    padding_rate                    SPEC.md:456-463            (host logic)
    attention_flops                 SPEC.md:465-472            (host logic)
    dynamic_pad_length              SPEC.md:474-481            (host logic)
    pack_ffd(lengths, capacity)     SPEC.md:437-445            → GPU packer (vlasim_pack_ffd_cuda)
    cu_seqlens(pack)                SPEC.md:447-454            → produced by the GPU packer
Hot-path calls go through the C-ABI only; there is no CPU packer in the product.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Sequence

import torch

from . import _lib
from .errors import ConfigError

# ---------------------------------------------------------------- host-side SPEC helpers


@dataclass
class SampleLen:
    """total_len = Σ view_lens + text_len, all >= 0, total >= 1."""
    id: int
    view_lens: Dict[str, int] = field(default_factory=dict)
    text_len: int = 0

    def __post_init__(self):
        if self.text_len < 0 or any(v < 0 for v in self.view_lens.values()):
            raise ConfigError(f"sample {self.id}: negative token count")
        if self.total_len < 1:
            raise ConfigError(f"sample {self.id} has no tokens")

    @property
    def total_len(self) -> int:
        return sum(self.view_lens.values()) + self.text_len


def prune_view(sample: SampleLen, view: str) -> SampleLen:
    """SPEC.md:483-491 (π0.5 view pruning): drop a view; unknown view → ConfigError."""
    if view not in sample.view_lens:
        raise ConfigError(f"prune_view: sample {sample.id} has no view {view!r}")
    views = {k: v for k, v in sample.view_lens.items() if k != view}
    return SampleLen(sample.id, views, sample.text_len)


def padding_rate(lengths: Sequence[int], pad_to: int) -> float:
    """1 − Σl / (count · pad_to), pad_to >= max(lengths)."""
    if len(lengths) == 0:
        raise ConfigError("padding_rate: empty batch")
    if pad_to < max(lengths):
        raise ConfigError("padding_rate: pad_to below the longest sample")
    return 1.0 - sum(lengths) / (len(lengths) * pad_to)


def dynamic_pad_length(lengths: Sequence[int]) -> int:
    """the batch maximum (π0.5 dynamic padding)."""
    if len(lengths) == 0:
        raise ConfigError("dynamic_pad_length: empty batch")
    return max(lengths)


def attention_flops(lengths: Sequence[int], head_dim: int, pad_to: int | None = None, c: float = 4.0) -> float:
    """fixed(pad_to) = count·c·pad_to²·d ; packed = c·Σl²·d (c = 4, one head, fwd)."""
    if pad_to is not None:
        if any(l > pad_to for l in lengths):
            raise ConfigError("attention_flops: length above pad_to")
        return len(lengths) * c * pad_to * pad_to * head_dim
    return c * sum(l * l for l in lengths) * head_dim


def visible_pairs(lengths: Sequence[int], mask_mode: int = 0, prefix: Sequence[int] | None = None) -> int:
    """Number of visible (query, key) pairs — the algorithmic work unit of the attention path.
    bidirectional l², causal l(l+1)/2, prefix P² + (l−P)·P + (l−P)(l−P+1)/2."""
    tot = 0
    for i, l in enumerate(lengths):
        if mask_mode == 0:
            tot += l * l
        elif mask_mode == 1:
            tot += l * (l + 1) // 2
        else:
            P = min(l, max(0, prefix[i]))
            tot += P * P + (l - P) * P + (l - P) * (l - P + 1) // 2
    return tot


# ---------------------------------------------------------------- GPU packer


@dataclass
class PackedSequence:
    """capacity, member ids + lengths (insertion order)."""
    capacity: int
    member_ids: List[int]
    member_lens: List[int]

    @property
    def fill(self) -> int:
        return sum(self.member_lens)


def cu_seqlens(pack: PackedSequence) -> List[int]:
    """SPEC.md:447-454 on a host PackedSequence: prefix sums with a leading 0."""
    if not pack.member_lens:
        raise ConfigError("cu_seqlens: empty pack")
    out = [0]
    for l in pack.member_lens:
        out.append(out[-1] + l)
    return out


_FIELDS = ("bin_of", "slot", "tok_off", "bin_count", "bin_fill", "bin_member_off", "bin_token_off", "member_ids",
           "cu_seqlens", "cu_seqlens_bins", "src_off", "num_bins", "total_tokens", "status")


class PackPlan:
    """Device-resident result of the GPU packer (all arrays sized for the worst case, n bins)."""

    def __init__(self, n: int, capacity: int, device="cuda"):
        self.n, self.capacity = int(n), int(capacity)
        i32 = dict(dtype=torch.int32, device=device)
        n = self.n
        self.bin_of = torch.empty(n, **i32)
        self.slot = torch.empty(n, **i32)
        self.tok_off = torch.empty(n, **i32)
        self.bin_count = torch.empty(n, **i32)
        self.bin_fill = torch.empty(n, **i32)
        self.bin_member_off = torch.empty(n + 1, **i32)
        self.bin_token_off = torch.empty(n + 1, **i32)
        self.member_ids = torch.empty(n, **i32)
        self.cu_seqlens = torch.empty(n + 1, **i32)
        self.cu_seqlens_bins = torch.empty(2 * n, **i32)
        self.src_off = torch.empty(n + 1, **i32)
        self.num_bins_t = torch.empty(1, **i32)
        self.total_tokens_t = torch.empty(1, dtype=torch.int64, device=device)
        self.status = torch.empty(2, **i32)
        self.workspace = torch.empty(_lib.lib().vlasim_pack_workspace_size(n, self.capacity), dtype=torch.uint8,
                                     device=device)
        self._struct = _lib.PackOut(*[_lib.ptr(t, _lib.i32p) for t in (
            self.bin_of, self.slot, self.tok_off, self.bin_count, self.bin_fill, self.bin_member_off,
            self.bin_token_off, self.member_ids, self.cu_seqlens, self.cu_seqlens_bins, self.src_off,
            self.num_bins_t)], _lib.ptr(self.total_tokens_t, _lib.i64p), _lib.ptr(self.status, _lib.i32p))

    @property
    def c_struct(self):
        return C.byref(self._struct)

    def num_bins(self) -> int:
        return int(self.num_bins_t.item())

    def total_tokens(self) -> int:
        return int(self.total_tokens_t.item())

    def to_host(self, lengths) -> List[PackedSequence]:
        """Materialise the bins as reference PackedSequence objects (host copy)."""
        nb = self.num_bins()
        mo = self.bin_member_off[: nb + 1].cpu().tolist()
        ids = self.member_ids.cpu().tolist()
        L = lengths.cpu().tolist() if torch.is_tensor(lengths) else list(lengths)
        return [PackedSequence(self.capacity, ids[mo[b]:mo[b + 1]], [L[i] for i in ids[mo[b]:mo[b + 1]]])
                for b in range(nb)]


def _as_dev_i32(lengths, device="cuda") -> torch.Tensor:
    if torch.is_tensor(lengths):
        t = lengths
    else:
        t = torch.tensor(list(lengths), dtype=torch.int64)
    if t.dtype != torch.int32:
        if t.numel() and (int(t.max()) > 2**31 - 1 or int(t.min()) < -2**31):
            raise ConfigError("lengths out of int32 range")
        t = t.to(torch.int32)
    return t.to(device).contiguous()


def pack_ffd(lengths, capacity: int, *, plan: PackPlan | None = None, sync_check: bool = True, stream=None,
             greedy: bool = False) -> PackPlan:
    """GPU first-fit-decreasing, order (len desc, id asc); bit-exact with the
    reference semantics.  Oversize / empty samples raise ConfigError naming the id
    when sync_check (default); otherwise the status stays on device in plan.status."""
    d_len = _as_dev_i32(lengths)
    n = d_len.numel()
    if n < 1:
        raise ConfigError("pack_ffd: need at least one sample")
    if plan is None or plan.n != n or plan.capacity != capacity:
        plan = PackPlan(n, capacity, device=d_len.device)
    plan.lengths = d_len
    fn = _lib.lib().vlasim_pack_greedy_cuda if greedy else _lib.lib().vlasim_pack_ffd_cuda
    rc = fn(_lib.ptr(d_len, _lib.i32p), n, int(capacity), plan.c_struct, _lib.ptr(plan.workspace),
            plan.workspace.numel(), 1 if sync_check else 0, _lib.stream_ptr(stream))
    _lib.check(rc, "pack_greedy" if greedy else "pack_ffd")
    return plan


def pack_greedy(lengths, capacity: int, *, plan: PackPlan | None = None, sync_check: bool = True,
                stream=None) -> PackPlan:
    """GPU streaming first-fit in arrival order (SPEC.md:519 greedy variant): sample i goes to the
    lowest-index bin with room >= len[i].  Same outputs and errors as pack_ffd."""
    return pack_ffd(lengths, capacity, plan=plan, sync_check=sync_check, stream=stream, greedy=True)


def token_ids(plan: PackPlan, total_tokens: int, stream=None):
    """Per packed token: (position in sample, segment index, gather index into the source layout)."""
    dev = plan.bin_of.device
    pos = torch.empty(total_tokens, dtype=torch.int32, device=dev)
    seg = torch.empty_like(pos)
    gat = torch.empty_like(pos)
    rc = _lib.lib().vlasim_pack_token_ids_cuda(_lib.ptr(plan.lengths, _lib.i32p), plan.c_struct, plan.n,
                                               int(total_tokens), _lib.ptr(pos, _lib.i32p),
                                               _lib.ptr(seg, _lib.i32p), _lib.ptr(gat, _lib.i32p),
                                               _lib.stream_ptr(stream))
    _lib.check(rc, "token_ids")
    return pos, seg, gat


def token_ids_into(plan: PackPlan, total_tokens: int, pos_ids=None, seg_ids=None, gather_idx=None, stream=None):
    """token_ids into caller-owned buffers (any may be None); no allocation on the hot path."""
    P = lambda t: _lib.ptr(t, _lib.i32p) if t is not None else None
    rc = _lib.lib().vlasim_pack_token_ids_cuda(_lib.ptr(plan.lengths, _lib.i32p), plan.c_struct, plan.n,
                                               int(total_tokens), P(pos_ids), P(seg_ids), P(gather_idx),
                                               _lib.stream_ptr(stream))
    _lib.check(rc, "token_ids")


def seg_src(plan: PackPlan, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Source row of every packed segment, src_off[member_ids[m]] (int32 [n]): the attention kernels'
    seg_src, which folds gather_rows / scatter_rows into their TMA coordinates."""
    if out is None:
        out = torch.empty(plan.n, dtype=torch.int32, device=plan.member_ids.device)
    rc = _lib.lib().vlasim_pack_seg_src_cuda(plan.c_struct, plan.n, _lib.ptr(out, _lib.i32p), _lib.stream_ptr(stream))
    _lib.check(rc, "pack_seg_src")
    return out


def gather_rows(src: torch.Tensor, plan: PackPlan, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Sample-major rows [Σl, ...] (sample i at src_off[i]) → packed stream order (16-byte vector copies)."""
    if out is None:
        out = torch.empty_like(src)
    row_bytes = src[0].numel() * src.element_size()
    rc = _lib.lib().vlasim_gather_rows_cuda(_lib.ptr(src), _lib.ptr(out), row_bytes,
                                            _lib.ptr(plan.lengths, _lib.i32p), plan.c_struct, plan.n,
                                            _lib.stream_ptr(stream))
    _lib.check(rc, "gather_rows")
    return out


def scatter_rows(packed: torch.Tensor, plan: PackPlan, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Inverse of gather_rows: packed stream order → sample-major rows."""
    if out is None:
        out = torch.empty_like(packed)
    row_bytes = packed[0].numel() * packed.element_size()
    rc = _lib.lib().vlasim_scatter_rows_cuda(_lib.ptr(packed), _lib.ptr(out), row_bytes,
                                             _lib.ptr(plan.lengths, _lib.i32p), plan.c_struct, plan.n,
                                             _lib.stream_ptr(stream))
    _lib.check(rc, "scatter_rows")
    return out
