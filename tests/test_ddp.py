"""DDP gradient synchronisation: the ring cost model's examples,
bucket layout, and the bucketed all-reduce averaging gradients on world_size 2 (gloo, CPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def test_allreduce_time_examples():
    from paper_2603_11101_b200 import ConfigError
    from paper_2603_11101_b200.ddp import allreduce_time, ddp_epoch_time, steps_per_epoch
    assert allreduce_time(1e9, 1, 1e11, 1e-5) == 0.0  # n = 1 → 0
    assert allreduce_time(1e9, 2, 1e11, 0.0) == pytest.approx(1e9 / 1e11)  # n = 2, lat 0 → B/bw
    assert allreduce_time(8e8, 8, 1e11, 1e-6) == pytest.approx(2 * 7 / 8 * 8e8 / 1e11 + 14e-6)
    with pytest.raises(ConfigError):
        allreduce_time(1e9, 4, 0.0, 1e-6)
    # zero comm cost → epoch time halves exactly when dp doubles
    a = ddp_epoch_time(steps_per_epoch(1 << 20, 128, 32), 0.5, 0, 32, 1e11, 0)
    b = ddp_epoch_time(steps_per_epoch(1 << 20, 128, 64), 0.5, 0, 64, 1e11, 0)
    assert a == 2 * b


def test_fit_alpha_beta_recovers_coefficients():
    from paper_2603_11101_b200 import ConfigError
    from paper_2603_11101_b200.ddp import allreduce_time, fit_alpha_beta
    sizes = [1 << 20, 4 << 20, 16 << 20, 64 << 20]
    t = [allreduce_time(s, 8, 3.5e11, 4e-6) for s in sizes]
    lat, bw, resid = fit_alpha_beta(sizes, t, 8)
    assert lat == pytest.approx(4e-6, rel=1e-9) and bw == pytest.approx(3.5e11, rel=1e-9) and resid < 1e-9
    with pytest.raises(ConfigError):
        fit_alpha_beta([1 << 20, 1 << 20], t[:2], 8)  # rank-deficient


def test_bucket_layout():
    from paper_2603_11101_b200.ddp import GradientBuckets
    gb = GradientBuckets([10, 300, 5, 700, 20], bucket_bytes=400 * 4, device="cpu")
    # reverse order: 20, 700 (own bucket: larger than the cap), 5, 300, 10
    assert [bk.params for bk in gb.buckets] == [[4], [3], [2, 1, 0]]
    assert gb.total == 1035
    v = gb.views()
    assert [x.numel() for x in v] == [10, 300, 5, 700, 20]
    v[3].fill_(2.0)
    assert gb.bucket_view(1).sum() == 1400


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_11101_b200.ddp import BucketAllReducer, GradientBuckets
        sizes = [17, 1000, 3, 4096, 250]
        gb = GradientBuckets(sizes, bucket_bytes=2048 * 4, device="cpu")
        red = BucketAllReducer(gb)
        g = torch.Generator().manual_seed(rank)
        for i in reversed(range(len(sizes))):  # the backward produces the last parameters first
            gb.views()[i].copy_(torch.randn(sizes[i], generator=g))
            red.mark_ready(i)
        n = red.finish()
        np.save(os.path.join(out_dir, f"g{rank}.npy"), gb.flat.numpy())
        with open(os.path.join(out_dir, f"n{rank}.txt"), "w") as f:
            f.write(str(n))
    finally:
        dist.destroy_process_group()


def test_bucketed_allreduce_averages_on_two_ranks(tmp_path):
    from paper_2603_11101_b200.ddp import GradientBuckets
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    sizes = [17, 1000, 3, 4096, 250]
    exp = np.zeros(sum(sizes), np.float32)
    for r in range(world):
        gb = GradientBuckets(sizes, bucket_bytes=2048 * 4, device="cpu")
        g = torch.Generator().manual_seed(r)
        for i in reversed(range(len(sizes))):
            gb.views()[i].copy_(torch.randn(sizes[i], generator=g))
        exp += gb.flat.numpy() / world
    for r in range(world):
        got = np.load(tmp_path / f"g{r}.npy")
        np.testing.assert_allclose(got, exp, rtol=1e-6, atol=1e-7)
        assert int((tmp_path / f"n{r}.txt").read_text()) == len(GradientBuckets(sizes, 2048 * 4, device="cpu").buckets)
