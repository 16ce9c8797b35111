"""Device LPT shard plan (vlasim_shard_lpt_cuda) against the host restatement
(dist.py:lpt), and the multi-rank union property: running every rank's shard of
the packs — its bins, its sample-major rows, its local cu_seqlens / seg_src — and putting the rows
back gives, bit for bit, the single-rank outputs and gradients.  The ranks are emulated one after
another on one GPU (no rank waits on another)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_device_lpt_matches_host(gpu, world):
    from paper_2603_11101_b200 import dist as vdist, packing, synthetic
    L = synthetic.gen_lengths(512 * max(world, 2), synthetic.DIST_UNIFORM, 16, 512, seed=7 + world)
    plan = packing.pack_ffd(L, 8192)
    nb = plan.num_bins()
    host = vdist.lpt_assign(plan, L, world)
    costs = vdist.bin_costs([b.member_ids for b in plan.to_host(L)], L)
    mo = plan.bin_member_off[: nb + 1].cpu().numpy()
    mids = plan.member_ids.cpu().numpy()
    seen = np.zeros(L.size, bool)
    for r in range(world):
        sp = vdist.shard_lpt(plan, world, r)
        br = sp.bin_rank[:nb].cpu().numpy()
        assert sorted(np.nonzero(br == r)[0].tolist()) == host[r]
        loads = sp.rank_load.cpu().numpy()
        assert np.array_equal(loads, [int(sum(costs[b] for b in host[q])) for q in range(world)])
        ids = np.concatenate([mids[mo[b]:mo[b + 1]] for b in host[r]]) if host[r] else np.zeros(0, int)
        nseg = sp.nseg()
        assert nseg == ids.size and np.array_equal(sp.local_ids[:nseg].cpu().numpy(), ids)
        cu = sp.local_cu.cpu().numpy()
        assert np.array_equal(cu[: nseg + 1], np.concatenate([[0], np.cumsum(L[ids])]))
        assert np.all(cu[nseg:] == sp.tokens()) and sp.tokens() == int(L[ids].sum())
        src = sp.local_src_off.cpu().numpy()
        mine = np.isin(np.arange(L.size), ids)
        assert np.all(src[~mine] == -1)
        order = np.sort(ids)
        assert np.array_equal(src[order], np.concatenate([[0], np.cumsum(L[order])[:-1]]))
        assert np.array_equal(sp.local_seg_src[:nseg].cpu().numpy(), src[ids])
        seen[ids] = True
    assert seen.all()


@pytest.mark.parametrize("cap,lo,hi,world", [(65535, 9000, 65535, 5), (65535, 9000, 65535, 16),
                                             (8192, 16, 8192, 16), (16384, 12000, 16384, 7)])
def test_device_lpt_wide_and_narrow_keys(gpu, cap, lo, hi, world):
    """Bin costs past 2^27 (the 64-bit LPT keys) and below (the rebased 32-bit keys), every world
    width of the argmin tree up to 16: same assignment and loads as the host LPT."""
    from paper_2603_11101_b200 import dist as vdist, packing, synthetic
    L = synthetic.gen_lengths(600, synthetic.DIST_UNIFORM, lo, hi, seed=cap + world)
    plan = packing.pack_ffd(L, cap)
    nb = plan.num_bins()
    host = vdist.lpt_assign(plan, L, world)
    costs = vdist.bin_costs([b.member_ids for b in plan.to_host(L)], L)
    sp = vdist.shard_lpt(plan, world, 0)
    br = sp.bin_rank[:nb].cpu().numpy()
    for r in range(world):
        assert sorted(np.nonzero(br == r)[0].tolist()) == host[r]
    assert np.array_equal(sp.rank_load.cpu().numpy()[:world], [int(sum(costs[b] for b in host[q])) for q in range(world)])


@pytest.mark.parametrize("world,mask", [(2, 0), (4, 0), (3, 2)])
def test_union_of_rank_shards_equals_single_rank(gpu, world, mask):
    from paper_2603_11101_b200 import attention, dist as vdist, packing, synthetic
    H, Hkv, d = (4, 4, 128) if mask == 0 else (8, 1, 256)
    n = 96 * world
    L = synthetic.gen_lengths(n, synthetic.DIST_UNIFORM, 16, 600, seed=11) if mask == 0 else \
        synthetic.gen_lengths(n, synthetic.DIST_PI05, 16, 200, 50, seed=11)
    plan = packing.pack_ffd(L, 4096)
    T = int(L.sum())
    g = torch.Generator(device="cuda").manual_seed(world)
    q, do = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(2))
    k, v = (torch.randn(T, Hkv, d, device="cuda", generator=g).bfloat16() for _ in range(2))
    src_off = np.concatenate([[0], np.cumsum(L)[:-1]])
    Lp = L[plan.member_ids[:n].cpu().numpy()]
    pre = torch.tensor(Lp - 50, dtype=torch.int32, device="cuda") if mask == 2 else None
    seg = packing.seg_src(plan)
    o, lse = attention.varlen_attn_fwd(q, k, v, plan.cu_seqlens, mask_mode=mask, prefix_len=pre, seg_src=seg)
    full = (o,) + attention.varlen_attn_bwd(do, q, k, v, o, lse, plan.cu_seqlens, mask_mode=mask, prefix_len=pre,
                                            seg_src=seg)
    got = [torch.full_like(x, float("nan")) for x in full]
    for r in range(world):
        sp = vdist.shard_lpt(plan, world, r)
        nseg = sp.nseg()
        ids = np.sort(sp.local_ids[:nseg].cpu().numpy())
        rows = torch.from_numpy(np.concatenate([src_off[i] + np.arange(L[i]) for i in ids])).cuda()
        ql, kl, vl, dol = (x[rows].contiguous() for x in (q, k, v, do))
        cu = sp.local_cu[: nseg + 1]
        lids = sp.local_ids[:nseg].cpu().numpy()
        pl = torch.tensor(L[lids] - 50, dtype=torch.int32, device="cuda") if mask == 2 else None
        ol, lsel = attention.varlen_attn_fwd(ql, kl, vl, cu, mask_mode=mask, prefix_len=pl,
                                             seg_src=sp.local_seg_src[:nseg])
        res = (ol,) + attention.varlen_attn_bwd(dol, ql, kl, vl, ol, lsel, cu, mask_mode=mask, prefix_len=pl,
                                                seg_src=sp.local_seg_src[:nseg])
        for dst, x in zip(got, res):
            dst[rows] = x
    torch.cuda.synchronize()
    for name, a_, b_ in zip(("o", "dq", "dk", "dv"), got, full):
        assert torch.equal(a_, b_), name
