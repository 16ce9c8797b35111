"""DDP gradient synchronisation after the packed forward / backward (PAPER.md:93-100 step 4;
SPEC.md:258-282 allreduce_time / ddp_epoch_time).

The attention path itself has no collective (packs are independent); in a training step the step
after it is the all-reduce of the parameter gradients.  This module is that step on B200:

    GradientBuckets        one flat gradient buffer, parameters laid out in REVERSE registration
                           order (the order the backward produces them) and cut into buckets of
                           `bucket_bytes`; every parameter's .grad is a view into it
    BucketAllReducer       launches each bucket's all-reduce (NCCL over NVLink / NVSwitch) on a
                           dedicated comm stream as soon as the compute stream marks its last
                           parameter ready, so communication overlaps the rest of the backward;
                           finish() waits and averages
    allreduce_time         the SPEC's ring model 2(n−1)/n·B/bw + 2(n−1)·lat
    measure_allreduce      the same quantity measured (CUDA events on the comm stream, max over
                           ranks) and fit_alpha_beta, the least-squares (latency, bandwidth) fit
                           that replaces the formula's constants with measured ones
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigError


# ------------------------------------------------------------------ cost model
def allreduce_time(param_bytes: float, n: int, bandwidth: float, link_latency: float) -> float:
    """Ring all-reduce: 0 for n = 1, else 2·(n−1)/n · param_bytes/bandwidth + 2·(n−1)·link_latency."""
    if n < 1:
        raise ConfigError("allreduce_time: n must be >= 1")
    if bandwidth <= 0:
        raise ConfigError("allreduce_time: bandwidth must be positive")
    if n == 1:
        return 0.0
    return 2.0 * (n - 1) / n * param_bytes / bandwidth + 2.0 * (n - 1) * link_latency


def ddp_epoch_time(steps_per_epoch: int, train_latency: float, param_bytes: float, n: int, bandwidth: float,
                   link_latency: float) -> float:
    """epoch_time = steps_per_epoch × (train_latency(mbs) + allreduce_time(...))."""
    return steps_per_epoch * (train_latency + allreduce_time(param_bytes, n, bandwidth, link_latency))


def steps_per_epoch(dataset_size: int, mbs: int, dp: int) -> int:
    """gbs = mbs × dp; ceil(dataset / gbs)."""
    if mbs < 1 or dp < 1:
        raise ConfigError("steps_per_epoch: mbs and dp must be >= 1")
    gbs = mbs * dp
    return (dataset_size + gbs - 1) // gbs


def fit_alpha_beta(sizes_bytes: Sequence[float], times: Sequence[float], n: int) -> Tuple[float, float, float]:
    """Least-squares fit of measured all-reduce times to the ring model's form
    t = 2(n−1)·lat + (2(n−1)/n)·B / bw  →  (link_latency, bandwidth, max relative residual)."""
    if n < 2:
        raise ConfigError("fit_alpha_beta: needs n >= 2")
    B = np.asarray(sizes_bytes, np.float64)
    t = np.asarray(times, np.float64)
    if B.size < 2 or np.unique(B).size < 2:
        raise ConfigError("fit_alpha_beta: needs >= 2 distinct sizes (rank-deficient otherwise)")
    A = np.stack([np.full_like(B, 2.0 * (n - 1)), 2.0 * (n - 1) / n * B], axis=1)
    (lat, inv_bw), *_ = np.linalg.lstsq(A, t, rcond=None)
    pred = A @ np.array([lat, inv_bw])
    resid = float(np.max(np.abs(pred - t) / np.maximum(t, 1e-30)))
    return float(lat), float(1.0 / inv_bw) if inv_bw > 0 else float("inf"), resid


# ------------------------------------------------------------------ buckets
@dataclass
class Bucket:
    offset: int          # elements into the flat buffer
    numel: int
    params: List[int]    # parameter indices in the bucket


class GradientBuckets:
    """Flat gradient storage for parameters of the given element counts.  Parameters are placed in
    reverse order (the backward's production order) and grouped into buckets of <= bucket_bytes
    (a parameter larger than a bucket gets its own).  views()[i] is parameter i's gradient."""

    def __init__(self, numels: Sequence[int], bucket_bytes: int = 32 << 20, dtype=torch.float32, device="cuda"):
        if not numels or any(int(n) < 1 for n in numels):
            raise ConfigError("GradientBuckets: parameter sizes must be >= 1")
        if bucket_bytes < 1:
            raise ConfigError("GradientBuckets: bucket_bytes must be >= 1")
        self.numels = [int(n) for n in numels]
        esz = torch.empty((), dtype=dtype).element_size()
        cap = max(1, bucket_bytes // esz)
        self.offsets = [0] * len(self.numels)
        self.buckets: List[Bucket] = []
        off = 0
        cur: Optional[Bucket] = None
        for i in reversed(range(len(self.numels))):
            n = self.numels[i]
            if cur is None or (cur.numel + n > cap and cur.params):
                cur = Bucket(off, 0, [])
                self.buckets.append(cur)
            self.offsets[i] = off
            cur.numel += n
            cur.params.append(i)
            off += n
        self.total = off
        self.flat = torch.zeros(self.total, dtype=dtype, device=device)
        self.bucket_of = {}
        for b, bk in enumerate(self.buckets):
            for i in bk.params:
                self.bucket_of[i] = b

    def views(self) -> List[torch.Tensor]:
        return [self.flat[o:o + n] for o, n in zip(self.offsets, self.numels)]

    def bucket_view(self, b: int) -> torch.Tensor:
        bk = self.buckets[b]
        return self.flat[bk.offset:bk.offset + bk.numel]


class BucketAllReducer:
    """Overlapped, bucketed gradient all-reduce (sum, then ×1/world = average).

    mark_ready(i) is called (on the compute stream's order) when parameter i's gradient is final;
    the bucket that completes launches its all-reduce on the comm stream behind an event recorded on
    the compute stream, so the collective overlaps the remaining backward work.  finish() makes the
    compute stream wait for every bucket and returns the number of collectives launched."""

    def __init__(self, buckets: GradientBuckets, group=None, comm_stream=None):
        self.b = buckets
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        cuda = buckets.flat.is_cuda
        self.comm = comm_stream if comm_stream is not None else (torch.cuda.Stream(buckets.flat.device)
                                                                 if cuda else None)
        self.reset()

    def reset(self):
        self.pending = [len(bk.params) for bk in self.b.buckets]
        self.launched: List[Tuple[int, object]] = []

    def mark_ready(self, i: int):
        b = self.b.bucket_of[i]
        self.pending[b] -= 1
        if self.pending[b] < 0:
            raise ConfigError(f"parameter {i} marked ready twice")
        if self.pending[b] == 0:
            self._launch(b)

    def _launch(self, b: int):
        view = self.b.bucket_view(b)
        if self.world == 1:
            self.launched.append((b, None))
            return
        if self.comm is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(view.device))
            self.comm.wait_event(ev)
            with torch.cuda.stream(self.comm):
                view.mul_(1.0 / self.world)  # pre-divide: the sum is the average, no second pass
                work = dist.all_reduce(view, group=self.group, async_op=True)
        else:
            view.mul_(1.0 / self.world)
            work = dist.all_reduce(view, group=self.group, async_op=True)
        self.launched.append((b, work))

    def finish(self) -> int:
        if any(p > 0 for p in self.pending):
            missing = [i for b, bk in enumerate(self.b.buckets) if self.pending[b] > 0 for i in bk.params]
            raise ConfigError(f"finish() with gradients not marked ready: {missing[:8]}")
        for _, work in self.launched:
            if work is not None:
                work.wait()
        if self.comm is not None and self.world > 1:
            torch.cuda.current_stream(self.b.flat.device).wait_stream(self.comm)
        n = sum(1 for _, w in self.launched if w is not None)
        self.reset()
        return n


def measure_allreduce(sizes_bytes: Sequence[int], group=None, iters: int = 10, warmup: int = 3,
                      dtype=torch.bfloat16, device=None) -> List[float]:
    """All-reduce time per size (seconds): CUDA events on the stream the collective runs on, averaged
    over `iters`, max over ranks (a barrier on both sides)."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    esz = torch.empty((), dtype=dtype).element_size()
    out = []
    for sb in sizes_bytes:
        x = torch.ones(max(1, int(sb) // esz), dtype=dtype, device=device)
        for _ in range(warmup):
            dist.all_reduce(x, group=group)
        torch.cuda.synchronize()
        dist.barrier(group=group)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            dist.all_reduce(x, group=group)
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / 1e3 / iters], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        out.append(float(t.item()))
    return out
