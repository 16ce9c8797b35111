"""Multi-rank sharding of packs on CPU: world_size 2 over gloo (127.0.0.1).
The path's single collective (all-gather of the per-rank length shards) must hand every rank the
same global lengths; the global FFD (oracle, CPU) and the deterministic LPT assignment must then be
identical on every rank, and the shards disjoint and complete."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2603_11101_b200.dist import allgather_lengths, balance, bin_costs, lpt
        rng = np.random.default_rng(1000 + rank)
        local = rng.integers(16, 513, 300 + 17 * rank).astype(np.int32)  # ragged shards
        counts = [None] * world
        dist.all_gather_object(counts, int(local.size))
        # equal-size all-gather (pad to the largest shard), as the bench does on GPU
        pad = max(counts)
        buf = np.zeros(pad, np.int32)
        buf[: local.size] = local
        g = allgather_lengths(torch.from_numpy(buf)).numpy().reshape(world, pad)
        L = np.concatenate([g[r, : counts[r]] for r in range(world)])
        bin_of, slot, tok, nb = orc.pack(L, 8192, 1)
        lay = orc.layout(L, bin_of, slot, tok, nb)
        mo = lay["bin_member_off"]
        members = [lay["member_ids"][mo[b]:mo[b + 1]].tolist() for b in range(nb)]
        costs = bin_costs(members, L)
        assign = lpt(costs, world)
        np.save(os.path.join(out_dir, f"r{rank}.npy"),
                np.array([L, np.array([nb]), np.array([balance(assign, costs)])], dtype=object), allow_pickle=True)
        with open(os.path.join(out_dir, f"a{rank}.txt"), "w") as f:
            f.write(repr(assign))
    finally:
        dist.destroy_process_group()


def test_allgather_ffd_lpt_identical_on_two_ranks(tmp_path, orc):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True) for r in range(world)]
    asg = [eval((tmp_path / f"a{r}.txt").read_text()) for r in range(world)]
    # every rank sees the same global lengths (rank-order concatenation of the shards)
    exp = np.concatenate([np.random.default_rng(1000 + r).integers(16, 513, 300 + 17 * r).astype(np.int32)
                          for r in range(world)])
    for r in range(world):
        assert np.array_equal(res[r][0], exp)
    # identical deterministic assignment; shards disjoint and complete over the bins
    assert asg[0] == asg[1]
    nb = int(res[0][1][0])
    flat = sorted(b for a in asg[0] for b in a)
    assert flat == list(range(nb))
    assert res[0][2][0] < 1.25  # LPT balance (max/mean load) on ~40 bins


def test_lpt_deterministic_ties_and_balance():
    from paper_2603_11101_b200.dist import balance, lpt
    assert lpt([5, 5, 5, 5], 2) == [[0, 2], [1, 3]]   # ties: lower bin index first, lowest rank
    assert lpt([9, 1, 1, 1], 2) == [[0], [1, 2, 3]]
    costs = np.random.default_rng(0).uniform(1, 100, 64)
    for w in (1, 2, 4, 8):
        a = lpt(costs, w)
        assert sorted(b for x in a for b in x) == list(range(64))
        assert balance(a, costs) < 1.1
