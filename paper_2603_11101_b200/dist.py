"""Multi-GPU sharding of packs.

Packs are independent (block-diagonal attention never crosses a pack), so the
path shards by pack with no collective on the attention path.  The only collective is one
all-gather of the per-rank sample lengths (the pack metadata): every rank then runs the same GPU FFD
on the global lengths and the same deterministic LPT assignment, so all ranks agree on the shard
without further communication.

LPT (longest processing time first): bins sorted by cost Σ l² descending (ties: lower bin index),
each assigned to the rank with the smallest load so far (ties: lowest rank).
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from . import _lib


def bin_costs(bins_members: Sequence[Sequence[int]], lengths) -> np.ndarray:
    L = np.asarray(lengths, np.float64)
    return np.array([float(np.sum(L[list(m)] ** 2)) for m in bins_members])


def lpt(costs: Sequence[float], world: int) -> List[List[int]]:
    """Deterministic LPT over bin costs → bins per rank (each list in ascending bin order)."""
    order = sorted(range(len(costs)), key=lambda b: (-costs[b], b))
    load = [0.0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for b in order:
        r = min(range(world), key=lambda i: (load[i], i))
        out[r].append(b)
        load[r] += costs[b]
    return [sorted(x) for x in out]


def lpt_assign(plan, lengths, world: int) -> List[List[int]]:
    """LPT over the bins of a GPU PackPlan (host copy of the bin membership)."""
    bins = plan.to_host(lengths)
    return lpt(bin_costs([b.member_ids for b in bins], lengths), world)


def shard_plan(plan, lengths, assign, rank: int) -> dict:
    """Sample ids (ascending) and token count of `rank`'s share of the bins."""
    bins = plan.to_host(lengths)
    ids = sorted(i for b in assign[rank] for i in bins[b].member_ids)
    L = np.asarray(lengths)
    return {"sample_ids": np.array(ids, dtype=np.int64), "tokens": int(L[ids].sum()) if ids else 0,
            "bins": list(assign[rank])}


class ShardPlan:
    """Device-resident result of vlasim_shard_lpt_cuda: the LPT assignment and this rank's packed stream."""

    def __init__(self, n: int, world: int, device):
        import torch
        i32 = dict(dtype=torch.int32, device=device)
        self.n, self.world = n, world
        self.bin_rank = torch.empty(n, **i32)
        self.rank_load = torch.empty(world, dtype=torch.int64, device=device)
        self.local_ids = torch.empty(n, **i32)
        self.local_cu = torch.empty(n + 1, **i32)
        self.local_seg_src = torch.empty(n, **i32)
        self.local_src_off = torch.empty(n, **i32)
        self.local_nseg = torch.empty(1, **i32)
        self.local_tokens = torch.empty(1, dtype=torch.int64, device=device)
        self.status = torch.empty(2, **i32)
        self.scratch = torch.empty(max(1, _lib.lib().vlasim_shard_scratch_size(n)), dtype=torch.uint8, device=device)
        P = _lib.ptr
        self._struct = _lib.ShardOut(P(self.bin_rank, _lib.i32p), P(self.rank_load, _lib.i64p),
                                     P(self.local_ids, _lib.i32p), P(self.local_cu, _lib.i32p),
                                     P(self.local_seg_src, _lib.i32p), P(self.local_src_off, _lib.i32p),
                                     P(self.local_nseg, _lib.i32p), P(self.local_tokens, _lib.i64p),
                                     P(self.status, _lib.i32p), P(self.scratch, _lib.i32p))

    def nseg(self) -> int:
        return int(self.local_nseg.item())

    def tokens(self) -> int:
        return int(self.local_tokens.item())


def shard_lpt(plan, world: int, rank: int, *, out: ShardPlan | None = None, sync_check: bool = True, stream=None):
    """Device LPT over the bins of a GPU PackPlan (identical on every rank) + this rank's packed stream,
    stream-ordered with no host round trip (vlasim_shard_lpt_cuda)."""
    import ctypes as C
    if out is None or out.n != plan.n or out.world != world:
        out = ShardPlan(plan.n, world, plan.bin_of.device)
    rc = _lib.lib().vlasim_shard_lpt_cuda(_lib.ptr(plan.lengths, _lib.i32p), plan.c_struct, plan.n, int(world),
                                          int(rank), C.byref(out._struct), 1 if sync_check else 0,
                                          _lib.stream_ptr(stream))
    _lib.check(rc, "shard_lpt")
    return out


def balance(assign, costs) -> float:
    """max / mean load of an assignment (1.0 = perfect)."""
    loads = [sum(costs[b] for b in a) for a in assign]
    m = float(np.mean(loads))
    return max(loads) / m if m > 0 else 1.0


def allgather_lengths(local_lengths, group=None):
    """The path's single collective: all-gather of the per-rank length shards (int32) — NCCL on
    GPU tensors, gloo on CPU tensors (tests)."""
    import torch
    import torch.distributed as dist
    t = local_lengths if torch.is_tensor(local_lengths) else torch.as_tensor(np.asarray(local_lengths, np.int32))
    world = dist.get_world_size(group)
    out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t.contiguous(), group=group) if t.is_cuda else \
        dist.all_gather(list(out.chunk(world)), t.contiguous(), group=group)
    return out
