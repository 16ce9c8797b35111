"""General E4M3 quantizer on the GPU vs the oracle: codes and scales bit-exact at
every granularity, fp32 and bf16 inputs, odd shapes; dequantize bit-exact; quant_error per group
(max_rel bit-exact, MSE to fp64 rounding) and bit-identical run to run."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = [((300, 260), "tensor", 0), ((300, 260), "channel", 0), ((300, 260), "channel", 1),
         ((300, 260), "block", 0), ((3, 129, 257), "block", 0), ((5, 7, 11), "channel", 1),
         ((4, 6, 130, 33), "block", 0), ((1000,), "tensor", 0), ((1000,), "channel", 0),
         ((2, 3000, 64), "channel", -1), ((257, 4100), "channel", 1), ((1, 1), "block", 0),
         # one case per kernel route: PerTensor with a scalar tail, fused PerChannel (vector and
         # scalar), generic PerChannel (middle axis / a group above 16 K elements), a column slab split
         ((7, 333), "tensor", 0), ((2, 9000), "channel", 0), ((3, 5001), "channel", 0),
         ((3, 40, 6000), "channel", 1), ((2, 20000), "channel", 0), ((5000, 12), "channel", 1)]


def _inputs(shape, seed, kind):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(shape).astype(np.float32)
    if kind == 1:  # heterogeneous magnitudes + exact midpoints (values k/128 · 2^e hit E4M3 ties)
        x *= rng.choice([1e-4, 1.0, 37.0, 3000.0], shape).astype(np.float32)
    elif kind == 2:
        x = (rng.integers(-128, 128, shape) / 128.0).astype(np.float32)
    return x


@pytest.mark.parametrize("shape,g,axis", CASES)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_quantize_bit_exact(gpu, orc, shape, g, axis, dtype):
    from paper_2603_11101_b200 import quant
    for kind in range(3):
        x = _inputs(shape, hash((shape, kind)) & 0xFFFF, kind)
        xt = torch.from_numpy(x).cuda()
        if dtype == "bf16":
            xt = xt.bfloat16()
            x = xt.float().cpu().numpy()
        qt = quant.quantize(xt, g, axis)
        codes, scales = orc.fp8_quantize(x, g, axis)
        assert tuple(qt.scales.shape) == quant.scales_shape(shape, g, axis)
        assert np.array_equal(qt.scales.cpu().numpy().reshape(-1), scales)
        assert np.array_equal(qt.codes.cpu().numpy(), codes), f"{shape} {g} {axis} kind {kind}"
        deq = quant.dequantize(qt)
        assert np.array_equal(deq.cpu().numpy(), orc.fp8_dequantize(codes, scales, g, axis))
        err = quant.quant_error(xt, qt)
        gmax, gsse, gcnt, mx, mse = orc.fp8_quant_error_general(x, codes, scales, g, axis)
        assert np.array_equal(err.group_max_rel.cpu().numpy().reshape(-1), gmax)
        assert np.array_equal(err.group_count.cpu().numpy().reshape(-1), gcnt)
        assert err.mse == pytest.approx(mse, rel=1e-12, abs=1e-300)
        err2 = quant.quant_error(xt, qt)
        assert torch.equal(err.group_mse, err2.group_mse)  # fixed-order reductions


def test_large_tensor_and_determinism(gpu, orc):
    from paper_2603_11101_b200 import quant
    x = torch.randn(2048, 4096, device="cuda") * torch.logspace(-3, 3, 4096, device="cuda")
    xn = x.cpu().numpy()
    for g, axis in (("tensor", 0), ("channel", 0), ("channel", 1), ("block", 0)):
        qt = quant.quantize(x, g, axis)
        codes, scales = orc.fp8_quantize(xn, g, axis)
        assert np.array_equal(qt.codes.cpu().numpy(), codes)
        assert np.array_equal(qt.scales.cpu().numpy().reshape(-1), scales)
        a, b = quant.quant_error(x, qt), quant.quant_error(x, qt)
        assert a.mse == b.mse and a.max_rel == b.max_rel


def test_non_finite_raises_naming_index(gpu):
    from paper_2603_11101_b200 import ConfigError, quant
    x = torch.ones(64, 300, device="cuda")
    x[17, 5] = float("nan")
    with pytest.raises(ConfigError, match=str(17 * 300 + 5)):
        quant.quantize(x, "block")
    x[17, 5] = float("inf")
    with pytest.raises(ConfigError):
        quant.quantize(x, "channel", 1)


def test_bad_arguments(gpu):
    from paper_2603_11101_b200 import ConfigError, quant
    with pytest.raises(ConfigError):
        quant.quantize(torch.ones(10, device="cuda"), "block")  # PerBlock needs >= 2 dims
    with pytest.raises(ConfigError):
        quant.quantize(torch.ones(4, 4, device="cuda"), "channel", 2)
    with pytest.raises(ConfigError):
        quant.quantize(torch.ones(4, 4, device="cuda", dtype=torch.float16), "tensor")


def test_unaligned_input_view(gpu, orc):
    """An input that starts off a 16-byte boundary (a contiguous view into a larger buffer) takes the
    scalar-load path and gives the same codes."""
    from paper_2603_11101_b200 import quant
    buf = torch.randn(1 + 300 * 260, device="cuda")
    x = buf[1:].view(300, 260)
    assert x.data_ptr() % 16 != 0
    for g, ax in (("tensor", 0), ("channel", 0), ("channel", 1), ("block", 0)):
        qt = quant.quantize(x, g, ax)
        codes, scales = orc.fp8_quantize(x.cpu().numpy(), g, ax)
        assert np.array_equal(qt.codes.cpu().numpy(), codes)


@pytest.mark.parametrize("shape,g,axis", [((300, 260), "tensor", 0), ((300, 260), "channel", 0),
                                          ((300, 260), "channel", 1), ((300, 260), "block", 0),
                                          ((3, 40, 6000), "channel", 1)])
def test_extreme_magnitudes(gpu, orc, shape, g, axis):
    """Group maxima from fp32 subnormals to 1e38 (the degenerate-maximum fp64 path and the
    subnormal-range midpoint test), small elements in wide-range groups, and exact E4M3 midpoints."""
    from paper_2603_11101_b200 import quant
    rng = np.random.default_rng(7)
    x = rng.standard_normal(shape).astype(np.float32)
    mag = rng.choice(np.array([1e-40, 1e-38, 1e-31, 1e-3, 1.0, 1e31, 3e37], np.float32), shape[:-1] + (1,))
    x = (x * mag).astype(np.float32)
    x.reshape(-1)[::17] *= np.float32(1e-6)  # tiny elements inside large groups
    mid = (rng.integers(-512, 512, shape) / 1024.0).astype(np.float32)  # subnormal-range midpoints
    x.reshape(-1)[::5] = mid.reshape(-1)[::5]
    qt = quant.quantize(torch.from_numpy(x).cuda(), g, axis)
    codes, scales = orc.fp8_quantize(x, g, axis)
    assert np.array_equal(qt.scales.cpu().numpy().reshape(-1), scales)
    assert np.array_equal(qt.codes.cpu().numpy(), codes)
