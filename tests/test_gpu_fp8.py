"""FP8 E4M3 path (config 4): per-block quantisation bit-exact with the oracle's fp32-quotient
restatement, and the FP8 Q/K attention forward within the north_star
FP8 tolerance (6e-2 of the fp64 reference on the original bf16 inputs)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,H,d,scale", [(300, 3, 128, 1.0), (128, 2, 128, 1000.0), (77, 1, 64, 1e-3),
                                          (513, 2, 256, 3.0), (200, 2, 100, 1.0), (130, 2, 192, 5.0)])
def test_quant_block_bit_exact(gpu, orc, T, H, d, scale):
    from paper_2603_11101_b200 import fp8
    g = torch.Generator(device="cuda").manual_seed(T + H)
    x = (torch.randn(T, H, d, device="cuda", generator=g) * scale).bfloat16()
    if H > 1:
        x[:, 0, :] = 0  # an all-zero head → scale 1, codes 0
    codes, scales = fp8.quant_block(x)
    rc, rs = orc.fp8_quant_block(x.float().cpu().numpy(), quotient_fp32=True)
    assert np.array_equal(scales.cpu().numpy(), rs)
    assert np.array_equal(codes.cpu().numpy(), rc)
    deq = fp8.dequant_block(codes, scales).cpu().numpy()
    vals = orc.e4m3_values()
    c = rc.astype(np.int64)
    ref = vals[c & 0x7F] * np.where(c & 0x80, -1.0, 1.0)
    sc = rs[np.arange(H)[None, :, None], (np.arange(T) // 128)[:, None, None], (np.arange(d) // 128)[None, None, :]]
    assert np.array_equal(deq, (ref * sc).astype(np.float32))


def test_quant_matches_high_precision_quotient_almost_everywhere(gpu, orc):
    """fp32 quotient vs the SPEC's real-valued quotient: codes differ only at rare rounding ties."""
    from paper_2603_11101_b200 import fp8
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(1024, 4, 128, device="cuda", generator=g).bfloat16()
    codes, _ = fp8.quant_block(x)
    rc, _ = orc.fp8_quant_block(x.float().cpu().numpy(), quotient_fp32=False)
    diff = np.count_nonzero(codes.cpu().numpy() != rc)
    assert diff <= 1e-3 * rc.size


@pytest.mark.parametrize("L,H,Hkv,mask", [([100, 28, 300, 5, 1, 130], 2, 2, 0), ([600, 40, 260], 4, 2, 2),
                                          ([513, 77, 1000, 3], 2, 1, 1)])
def test_fp8qk_attention_within_tolerance(gpu, orc, L, H, Hkv, mask):
    from paper_2603_11101_b200 import attention, fp8
    g = torch.Generator(device="cuda").manual_seed(sum(L))
    T, d = sum(L), 128
    q = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
    k = torch.randn(T, Hkv, d, device="cuda", generator=g).bfloat16()
    v = torch.randn(T, Hkv, d, device="cuda", generator=g).bfloat16()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(L)]), dtype=torch.int32, device="cuda")
    prefix = torch.tensor([l // 3 for l in L], dtype=torch.int32, device="cuda") if mask == 2 else None
    qc, qs = fp8.quant_block(q)
    kc, ks = fp8.quant_block(k)
    o8, _ = fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu, mask_mode=mask, prefix_len=prefix)
    o16, _ = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix)
    torch.cuda.synchronize()
    pre = None if prefix is None else prefix.cpu().numpy()
    ro, _ = orc.mha_fwd(q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy(),
                        cu.cpu().numpy(), mask=mask, prefix=pre)
    err8 = np.max(np.abs(o8.float().cpu().numpy() - ro)) / max(1.0, np.max(np.abs(ro)))
    err16 = np.max(np.abs(o16.float().cpu().numpy() - ro)) / max(1.0, np.max(np.abs(ro)))
    assert err8 < 6e-2, err8
    assert err16 < 2e-2, err16


# ---- quant_error
@pytest.mark.parametrize("shape", [(300, 3, 128), (128, 2, 256), (77, 1, 64), (1, 1, 1)])
def test_quant_error_matches_oracle(gpu, orc, shape):
    from paper_2603_11101_b200 import fp8
    torch.manual_seed(sum(shape))
    x = (torch.randn(*shape, device="cuda") * torch.logspace(-3, 2, shape[0], device="cuda")[:, None, None]).bfloat16()
    codes, scales = fp8.quant_block(x)
    m = fp8.quant_error(x, codes, scales)
    gmax, gsse, gcnt, mx, mse = orc.fp8_quant_error(x.float().cpu().numpy(), codes.cpu().numpy(), scales.cpu().numpy())
    assert np.array_equal(m["groups"]["max_rel"].cpu().numpy(), gmax)  # fp32, same roundings
    np.testing.assert_allclose(m["groups"]["mse"].cpu().numpy(), gsse / gcnt, rtol=1e-12, atol=0)
    assert m["max_rel"] == mx
    np.testing.assert_allclose(m["mse"], mse, rtol=1e-12)
    assert m["max_rel"] <= 2.0 ** -4  # normal-range relative error <= 2^-4


def test_quant_error_known_answers(gpu):
    from paper_2603_11101_b200 import fp8
    z = torch.zeros(130, 2, 64, dtype=torch.bfloat16, device="cuda")
    m = fp8.quant_error(z, *fp8.quant_block(z))  # zero tensor: exact roundtrip
    assert m["max_rel"] == 0.0 and m["mse"] == 0.0
    e = torch.tensor([-448.0, 0.0, 448.0], device="cuda").bfloat16().view(3, 1, 1)  # representable at scale 1
    m = fp8.quant_error(e, *fp8.quant_block(e))
    assert m["max_rel"] == 0.0 and m["mse"] == 0.0
    c = torch.full((256, 1, 128), 3.0, dtype=torch.bfloat16, device="cuda")  # all-equal tensor
    m = fp8.quant_error(c, *fp8.quant_block(c))
    assert m["max_rel"] <= 2.0 ** -23  # zero up to the fp32 rounding of scale = amax / 448


def test_quant_block_quotient_stress(gpu, orc):
    """The block quantiser's reciprocal + one-correction quotient against the oracle's correctly
    rounded fp32 division: 64 blocks, each with its own amax (hence scale) and 16383 other
    elements drawn uniformly over the bf16 bit patterns below it (every exponent range)."""
    from paper_2603_11101_b200 import fp8
    g = torch.Generator(device="cpu").manual_seed(7)
    nblk = 64
    amax_bits = torch.randint(0x3000, 0x4f00, (nblk,), generator=g, dtype=torch.int32)  # ~5e-10 .. 2e9
    x = torch.empty(nblk * 128, 1, 128, dtype=torch.bfloat16)
    for b in range(nblk):
        top = int(amax_bits[b])
        bits = torch.randint(0, top, (128 * 128,), generator=g, dtype=torch.int32)
        sign = torch.randint(0, 2, (128 * 128,), generator=g, dtype=torch.int32) << 15
        bits = bits | sign
        bits[0] = top  # the block's amax
        x[128 * b:128 * (b + 1), 0, :] = bits.to(torch.int16).view(torch.bfloat16).view(128, 128)
    xc = x.cuda()
    codes, scales = fp8.quant_block(xc)
    rc, rs = orc.fp8_quant_block(x.float().numpy(), quotient_fp32=True)
    assert np.array_equal(scales.cpu().numpy(), rs)
    assert np.array_equal(codes.cpu().numpy(), rc)
