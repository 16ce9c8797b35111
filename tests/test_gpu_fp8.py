"""FP8 E4M3 path (config 4): per-block quantisation bit-exact with the oracle's exact restatement of
the SPEC (the RNE code of the REAL quotient x·448/amax; non-finite input →
ConfigError), and the FP8 Q/K attention forward / backward within the north_star FP8
tolerance (6e-2 of the fp64 reference on the original bf16 inputs)."""
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
    rc, rs = orc.fp8_quant_block(x.float().cpu().numpy(), quotient_fp32=False)
    assert np.array_equal(scales.cpu().numpy(), rs)
    assert np.array_equal(codes.cpu().numpy(), rc)
    deq = fp8.dequant_block(codes, scales).cpu().numpy()
    vals = orc.e4m3_values()
    c = rc.astype(np.int64)
    ref = vals[c & 0x7F] * np.where(c & 0x80, -1.0, 1.0)
    sc = rs[np.arange(H)[None, :, None], (np.arange(T) // 128)[:, None, None], (np.arange(d) // 128)[None, None, :]]
    assert np.array_equal(deq, (ref * sc).astype(np.float32))


def test_quant_matches_real_quotient_everywhere(gpu, orc):
    """Random normal blocks at several magnitudes: every code byte equals the SPEC's (exact quotient)."""
    from paper_2603_11101_b200 import fp8
    g = torch.Generator(device="cuda").manual_seed(5)
    x = (torch.randn(4096, 4, 128, device="cuda", generator=g) *
         torch.logspace(-4, 4, 4096, device="cuda")[:, None, None]).bfloat16()
    codes, _ = fp8.quant_block(x)
    rc, _ = orc.fp8_quant_block(x.float().cpu().numpy(), quotient_fp32=False)
    assert np.array_equal(codes.cpu().numpy(), rc)


def _tie_block(amax, rng):
    """A 128×128 block whose amax is `amax` and whose other elements sit exactly on E4M3 midpoints of
    the real quotient x·448/amax (x = m·amax/448 when that is a bf16), or one bf16 ulp either side."""
    vals = []
    for E in range(-9, 9):
        for k in (17, 19, 21, 23, 25, 27, 29, 31):  # midpoints 2^(E-4)·k of the binade [2^E, 2^(E+1))
            x = np.float64(k) * 2.0 ** (E - 4) * amax / 448.0
            xb = torch.tensor([x], dtype=torch.float64).bfloat16()
            if float(xb) == x and 0 < x < amax:
                b = xb.view(torch.int16)
                vals += [xb, (b + 1).view(torch.bfloat16), (b - 1).view(torch.bfloat16)]
    v = torch.cat(vals).float().numpy() if vals else np.zeros(1, np.float32)
    blk = rng.choice(v, size=128 * 128) * rng.choice([-1.0, 1.0], size=128 * 128)
    blk[0] = amax
    return blk.astype(np.float32).reshape(128, 128)


def test_quant_exact_ties_and_neighbours(gpu, orc):
    """Exact ties of the real quotient (decided to the even code) and their bf16 neighbours, for block
    maxima whose scale amax/448 is not exact in fp32: the fp32 quotient alone gets some of these wrong."""
    from paper_2603_11101_b200 import fp8
    rng = np.random.default_rng(1)
    # the two bf16 mantissas whose fp32 scale RN(amax / 448) moves some exact ties off their midpoint
    amaxes = [1.78125, 1.9375, 1.78125 * 2 ** 10, 1.9375 * 2 ** -12, 1.78125 * 2 ** -30, 1.9375 * 2 ** 40, 5.0, 3.0]
    x = np.concatenate([_tie_block(a, rng) for a in amaxes], 0)[:, None, :]
    xt = torch.from_numpy(x).bfloat16()
    assert torch.equal(xt.float(), torch.from_numpy(x))  # exactly representable
    codes, scales = fp8.quant_block(xt.cuda())
    rc, rs = orc.fp8_quant_block(x, quotient_fp32=False)
    assert np.array_equal(scales.cpu().numpy(), rs)
    assert np.array_equal(codes.cpu().numpy(), rc)
    rc32, _ = orc.fp8_quant_block(x, quotient_fp32=True)
    assert np.count_nonzero(rc32 != rc) > 0  # the case the exact decision exists for


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), float("-inf")])
def test_quant_non_finite_is_config_error(gpu, bad):
    """non-finite input → error (ConfigError naming the element)."""
    from paper_2603_11101_b200 import fp8
    from paper_2603_11101_b200.errors import ConfigError
    x = torch.randn(300, 2, 128, device="cuda").bfloat16()
    x[257, 1, 77] = bad
    with pytest.raises(ConfigError, match=str((257 * 2 + 1) * 128 + 77)):
        fp8.quant_block(x)
    y = torch.randn(100, 1, 100, device="cuda").bfloat16()  # scalar (unaligned-d) kernel
    y[5, 0, 3] = bad
    with pytest.raises(ConfigError, match="non-finite"):
        fp8.quant_block(y)
    status = torch.zeros(2, dtype=torch.int32, device="cuda")
    fp8.quant_block(x, check_finite=False, status=status)  # asynchronous: the error stays on device
    assert status.tolist() == [2, (257 * 2 + 1) * 128 + 77]


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
    o8, lse8 = fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu, mask_mode=mask, prefix_len=prefix)
    o16, _ = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix)
    torch.cuda.synchronize()
    pre = None if prefix is None else prefix.cpu().numpy()
    ro, _ = orc.mha_fwd(q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy(),
                        cu.cpu().numpy(), mask=mask, prefix=pre)
    err8 = np.max(np.abs(o8.float().cpu().numpy() - ro)) / max(1.0, np.max(np.abs(ro)))
    err16 = np.max(np.abs(o16.float().cpu().numpy() - ro)) / max(1.0, np.max(np.abs(ro)))
    assert err8 < 6e-2, err8
    assert err16 < 2e-2, err16
    # FP8 backward (gradients of the FP8 forward) within the FP8 tolerance of the fp64 reference
    do = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
    dq8, dk8, dv8 = fp8.varlen_attn_bwd_fp8qk(do, qc, qs, kc, ks, v, o8, lse8, cu, mask_mode=mask, prefix_len=prefix)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    rdq, rdk, rdv = orc.mha_bwd(f(q), f(k), f(v), ro, f(do), cu.cpu().numpy(), mask=mask, prefix=pre)
    for name, x, r in (("dq", dq8, rdq), ("dk", dk8, rdk), ("dv", dv8, rdv)):
        e = np.max(np.abs(f(x) - r)) / max(1.0, np.max(np.abs(r)))
        assert e < 6e-2, (name, e)


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
    """The block quantiser (reciprocal + one-correction quotient, then the exact midpoint decision)
    against the oracle's exact real quotient: 64 blocks, each with its own amax (hence scale) and 16383 other
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
    rc, rs = orc.fp8_quant_block(x.float().numpy(), quotient_fp32=False)
    assert np.array_equal(scales.cpu().numpy(), rs)
    assert np.array_equal(codes.cpu().numpy(), rc)
