"""π0.5 dynamic padding on the GPU: device dynamic_pad_length, pad/unpad of token
rows, and the varlen kernels run directly on padded storage — bit-identical to the same attention on
the unpadded sample-major tensors, and within tolerance of the fp64 oracle."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_dynamic_pad_length_examples(gpu):
    from paper_2603_11101_b200 import ConfigError, padding
    dp = padding.dynamic_pad([37, 120, 85])
    assert dp.pad_to == 120
    assert dp.cu_seqlens.cpu().tolist() == [0, 37, 157, 242]
    assert dp.seg_src.cpu().tolist() == [0, 120, 240]
    assert padding.dynamic_pad([64] * 9).padding_rate() == 0.0
    with pytest.raises(ConfigError, match="id 1"):
        padding.dynamic_pad([5, 0, 3])
    with pytest.raises(ConfigError):
        padding.dynamic_pad([])


def test_random_batches_save_vs_fixed_cap(gpu):  # token slots saved vs a fixed cap of 200
    from paper_2603_11101_b200 import padding
    rng = np.random.default_rng(0)
    saved = 0
    recount = 0
    for _ in range(20):
        L = rng.integers(1, 201, int(rng.integers(1, 40)))
        dp = padding.dynamic_pad(L)
        assert dp.pad_to == L.max()
        saved += (200 - dp.pad_to) * len(L)
        recount += sum(200 - L.max() for _ in L)
    assert saved == recount


def test_pad_unpad_roundtrip(gpu):
    from paper_2603_11101_b200 import padding
    L = [5, 130, 1, 77]
    dp = padding.dynamic_pad(L)
    x = torch.randn(sum(L), 4, 64, device="cuda").bfloat16()
    xp = padding.pad_rows(x, dp)
    assert xp.shape == (4 * 130, 4, 64)
    off = 0
    for i, l in enumerate(L):
        assert torch.equal(xp[i * 130:i * 130 + l], x[off:off + l])
        assert not xp[i * 130 + l:(i + 1) * 130].any()
        off += l
    assert torch.equal(padding.unpad_rows(xp, dp), x)


@pytest.mark.parametrize("mask,H,Hkv,d", [(0, 4, 4, 128), (1, 4, 2, 64), (2, 8, 1, 256)])
def test_padded_attention_matches_unpadded_and_oracle(gpu, orc, mask, H, Hkv, d):
    from paper_2603_11101_b200 import attention, padding
    rng = np.random.default_rng(mask)
    L = rng.integers(1, 400, 9).tolist()
    dp = padding.dynamic_pad(L)
    T = sum(L)
    g = torch.Generator(device="cuda").manual_seed(mask)
    q, do = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(2))
    k, v = (torch.randn(T, Hkv, d, device="cuda", generator=g).bfloat16() for _ in range(2))
    prefix = torch.tensor([max(1, l // 2) for l in L], dtype=torch.int32, device="cuda") if mask == 2 else None
    kw = dict(mask_mode=mask, prefix_len=prefix)
    cu = dp.cu_seqlens
    o, lse = attention.varlen_attn_fwd(q, k, v, cu, **kw)
    dq, dk, dv = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, **kw)
    qp, kp, vp, dop = (padding.pad_rows(t, dp) for t in (q, k, v, do))
    op, lsep = padding.padded_attention_fwd(qp, kp, vp, dp, **kw)
    dqp, dkp, dvp = padding.padded_attention_bwd(dop, qp, kp, vp, op, lsep, dp, **kw)
    torch.cuda.synchronize()
    for a, b in ((o, op), (dq, dqp), (dk, dkp), (dv, dvp)):
        assert torch.equal(padding.unpad_rows(b, dp), a)
    for i, l in enumerate(L):  # pad rows untouched (zero)
        for t in (op, dqp, dkp, dvp):
            assert not t[i * dp.pad_to + l:(i + 1) * dp.pad_to].any()
    f = lambda t: t.float().cpu().numpy()
    pre = prefix.cpu().numpy() if prefix is not None else None
    ro, _ = orc.mha_fwd(f(q), f(k), f(v), cu.cpu().numpy(), mask=mask, prefix=pre)
    err = np.abs(f(o) - ro).max() / max(1.0, np.abs(ro).max())
    assert err < 2e-2
