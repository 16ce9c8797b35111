"""GPU packer parity: bin assignment, member order, cu_seqlens, token ids and gather indices must be
bit-exact with the CPU oracle (north_star)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _check_plan(orc, L, cap, plan, mode=None):
    from paper_2603_11101_b200 import packing
    if mode is None:
        mode = 1 if len(L) > 3000 else 0  # FFD: segment tree / naive scan (same result)
    bin_of, slot, tok, nb = orc.pack(L, cap, mode)
    assert plan.num_bins() == nb
    n = len(L)
    assert np.array_equal(plan.bin_of.cpu().numpy(), bin_of)
    assert np.array_equal(plan.slot.cpu().numpy(), slot)
    assert np.array_equal(plan.tok_off.cpu().numpy(), tok)
    lay = orc.layout(L, bin_of, slot, tok, nb)
    assert np.array_equal(plan.bin_count[:nb].cpu().numpy(), lay["bin_count"])
    assert np.array_equal(plan.bin_fill[:nb].cpu().numpy(), lay["bin_fill"])
    assert np.array_equal(plan.bin_member_off[: nb + 1].cpu().numpy(), lay["bin_member_off"])
    assert np.array_equal(plan.bin_token_off[: nb + 1].cpu().numpy(), lay["bin_token_off"])
    assert np.array_equal(plan.member_ids.cpu().numpy(), lay["member_ids"])
    assert np.array_equal(plan.cu_seqlens.cpu().numpy(), lay["cu_seqlens"])
    assert np.array_equal(plan.cu_seqlens_bins[: n + nb].cpu().numpy(), lay["cu_seqlens_bins"])
    assert np.array_equal(plan.src_off[:n].cpu().numpy(), lay["src_off"])
    assert int(plan.src_off[n]) == int(np.sum(L))
    assert plan.total_tokens() == int(np.sum(L))
    return lay


def test_spec_examples(gpu, orc):
    from paper_2603_11101_b200 import packing
    p = packing.pack_ffd([6, 5, 4, 3, 2], 8)
    bins = p.to_host([6, 5, 4, 3, 2])
    assert [b.member_lens for b in bins] == [[6, 2], [5, 3], [4]]
    assert [packing.cu_seqlens(b) for b in bins] == [[0, 6, 8], [0, 5, 8], [0, 4]]
    assert packing.pack_ffd([5], 8).num_bins() == 1
    assert packing.pack_ffd([8, 8, 8], 8).num_bins() == 3


def test_config1_appendix_a(gpu, orc):
    from paper_2603_11101_b200 import packing
    from paper_2603_11101_b200.synthetic import gen_lengths
    L = gen_lengths(64, 0, 16, 512)
    p = packing.pack_ffd(L, 2048)
    _check_plan(orc, L, 2048, p)
    bins = p.to_host(L)
    assert bins[0].member_ids == [13, 52, 19, 48, 2]
    assert packing.cu_seqlens(bins[0]) == [0, 508, 988, 1455, 1914, 2034]


def test_oversize_and_empty_raise_config_error_naming_id(gpu):
    from paper_2603_11101_b200 import ConfigError, packing
    with pytest.raises(ConfigError, match="id 2"):
        packing.pack_ffd([3, 4, 9, 1], 8)
    with pytest.raises(ConfigError, match="id 1"):
        packing.pack_ffd([3, 0, 9], 16)
    with pytest.raises(ConfigError):
        packing.pack_ffd([3], 1 << 20)


@pytest.mark.parametrize("seed", range(6))
def test_random_instances(gpu, orc, seed):
    from paper_2603_11101_b200 import packing
    rng = np.random.default_rng(seed)
    for _ in range(40):
        n = int(rng.integers(1, 3000))
        cap = int(rng.choice([8, 64, 300, 2048, 8192, 16384]))
        hi = int(rng.choice([cap, max(1, cap // 4), max(1, cap // 50)]))
        L = rng.integers(1, hi + 1, n).astype(np.int32)
        _check_plan(orc, L, cap, packing.pack_ffd(L, cap))


def test_equal_lengths_and_edge_caps(gpu, orc):
    from paper_2603_11101_b200 import packing
    for L, cap in [([8] * 100, 8), ([1] * 5000, 7), ([4] * 33, 8), ([16384] * 3, 16384), ([1], 1),
                   ([65535] * 2 + [1] * 3, 65535), ([40000, 30000, 25000, 1, 2, 3] * 50, 65535)]:
        L = np.array(L, np.int32)
        _check_plan(orc, L, cap, packing.pack_ffd(L, cap))


@pytest.mark.parametrize("n,dist,cap", [(200_000, 1, 8192), (1_000_000, 1, 8192), (20_000, 0, 2048),
                                        (50_000, 2, 8192)])
def test_large(gpu, orc, n, dist, cap):
    from paper_2603_11101_b200 import packing
    from paper_2603_11101_b200.synthetic import gen_lengths
    L = gen_lengths(n, dist, *((0.02, 500) if dist == 1 else (16, 512)))
    _check_plan(orc, L, cap, packing.pack_ffd(L, cap))


def test_token_ids_and_gather_scatter(gpu, orc):
    from paper_2603_11101_b200 import packing
    from paper_2603_11101_b200.synthetic import gen_lengths
    L = gen_lengths(300, 0, 1, 700)
    plan = packing.pack_ffd(L, 2048)
    lay = _check_plan(orc, L, 2048, plan)
    T = int(L.sum())
    pos, seg, gat = packing.token_ids(plan, T)
    rpos, rseg, rgat = orc.token_ids(L, lay)
    assert np.array_equal(pos.cpu().numpy(), rpos)
    assert np.array_equal(seg.cpu().numpy(), rseg)
    assert np.array_equal(gat.cpu().numpy(), rgat)
    src = torch.randn(T, 4, 64, device="cuda").bfloat16()
    packed = packing.gather_rows(src, plan)
    assert torch.equal(packed, src[gat.long()])
    back = packing.scatter_rows(packed, plan)
    assert torch.equal(back, src)


# ---- greedy arrival-order first-fit: bit-exact with the oracle's mode 2
def test_greedy_spec_shape_and_errors(gpu, orc):
    from paper_2603_11101_b200 import ConfigError, packing
    L = [6, 5, 4, 3, 2]
    p = packing.pack_greedy(L, 8)
    assert [b.member_lens for b in p.to_host(L)] == [[6, 2], [5, 3], [4]]
    _check_plan(orc, np.array(L, np.int32), 8, p, mode=2)
    with pytest.raises(ConfigError, match="id 2"):
        packing.pack_greedy([3, 4, 9, 1], 8)


@pytest.mark.parametrize("seed", range(4))
def test_greedy_random_instances(gpu, orc, seed):
    from paper_2603_11101_b200 import packing
    rng = np.random.default_rng(100 + seed)
    for _ in range(25):
        n = int(rng.integers(1, 4000))
        cap = int(rng.choice([8, 64, 300, 2048, 8192, 16384]))
        hi = int(rng.choice([cap, max(1, cap // 4), max(1, cap // 50)]))
        L = rng.integers(1, hi + 1, n).astype(np.int32)
        _check_plan(orc, L, cap, packing.pack_greedy(L, cap), mode=2)


def test_greedy_config1_and_long_tail(gpu, orc):
    from paper_2603_11101_b200 import packing
    from paper_2603_11101_b200.synthetic import DIST_GEOMETRIC, gen_lengths
    L = np.asarray(gen_lengths(64, 0, 16, 512), np.int32)
    _check_plan(orc, L, 2048, packing.pack_greedy(L, 2048), mode=2)
    L = np.asarray(gen_lengths(200000, DIST_GEOMETRIC, 0.02, 500, label="lengths", seed=42), np.int32)
    _check_plan(orc, L, 8192, packing.pack_greedy(L, 8192), mode=2)


# ---- inputs beyond the shared-memory working sets (ADVICE r1 pack.cu:211):
# the reference packs any list of lengths in [1, capacity]; so must the GPU.
@pytest.mark.parametrize("case", ["5000_then_1", "many_open_bins", "u1000_6000", "5000_3000"])
def test_ffd_open_bin_spill(gpu, orc, case):
    from paper_2603_11101_b200 import packing
    rng = np.random.default_rng(7)
    if case == "5000_then_1":      # 20k bins stay open (room 3192 >= every later length 1)
        L = np.array([5000] * 20000 + [1] * 20000, np.int32)
    elif case == "many_open_bins":  # 60k bins with room 1 left, then a class of length 1
        L = np.array([8191] * 60000 + [1] * 70000, np.int32)
    elif case == "u1000_6000":
        L = rng.integers(1000, 6001, 100_000).astype(np.int32)
    else:
        L = np.array([5000] * 20000 + [3000] * 20000, np.int32)
    _check_plan(orc, L, 8192, packing.pack_ffd(L, 8192), mode=1)


@pytest.mark.parametrize("cap", [32768, 65535])
def test_large_capacity(gpu, orc, cap):
    """cap > 40959: histogram / rank counters in HBM; cap up to VLASIM_PACK_MAX_CAPACITY."""
    from paper_2603_11101_b200 import packing
    rng = np.random.default_rng(cap)
    for n, hi in [(500, cap), (20_000, cap // 8), (3000, cap)]:
        L = rng.integers(1, hi + 1, n).astype(np.int32)
        _check_plan(orc, L, cap, packing.pack_ffd(L, cap), mode=1)
        _check_plan(orc, L, cap, packing.pack_greedy(L, cap), mode=2)


@pytest.mark.parametrize("case", ["40k_full_bins", "alternating", "long_tail_100k"])
def test_greedy_deep_tree(gpu, orc, case):
    """More than 32768 bins: the greedy room tree's level 0 lives in HBM (up to 2^20 bins)."""
    from paper_2603_11101_b200 import packing
    rng = np.random.default_rng(11)
    if case == "40k_full_bins":
        L = np.array([8192] * 40000 + [1] * 100, np.int32)
    elif case == "alternating":      # 5000, 1, 5000, 1 ...: 40k bins, ones fill the earliest
        L = np.array([5000, 1] * 40000, np.int32)
    else:
        L = rng.integers(1, 8193, 100_000).astype(np.int32)
    _check_plan(orc, L, 8192, packing.pack_greedy(L, 8192), mode=2)


def test_unsynchronised_error_leaves_defined_empty_plan(gpu):
    """sync_check=False (the CUDA-graph path): a bad length leaves the status on the device and a
    defined, empty plan (cu_seqlens all 0, num_bins 0) that downstream kernels treat as no work."""
    from paper_2603_11101_b200 import packing
    good = packing.pack_ffd([5, 3, 7, 2], 8)
    assert good.num_bins() > 0
    bad = packing.pack_ffd([5, 3, 9, 2], 8, plan=good, sync_check=False)
    torch.cuda.synchronize()
    assert bad.status.cpu().tolist() == [2, 2]  # VLASIM_ECONFIG, offending id
    assert bad.num_bins() == 0
    assert int(bad.cu_seqlens.abs().sum()) == 0
