"""Quantizer oracle pinned to the SPEC's examples, plus the host-side pieces of the
product's quantizer module (block_partition, compression_ratio) — CPU only."""
import json
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    return oracle


def test_zero_tensor(orc):
    x = np.zeros((3, 130, 200), np.float32)
    for g in ("tensor", "channel", "block"):
        codes, scales = orc.fp8_quantize(x, g, 1)
        assert not codes.any() and np.all(scales == 1)
        assert np.array_equal(orc.fp8_dequantize(codes, scales, g, 1), x)


def test_per_tensor_exact_roundtrip(orc):
    x = np.array([-448.0, 0.0, 448.0], np.float32)
    codes, scales = orc.fp8_quantize(x, "tensor")
    assert scales.tolist() == [1.0]
    assert np.array_equal(orc.fp8_dequantize(codes, scales, "tensor"), x)


@pytest.mark.parametrize("g", ["tensor", "channel", "block"])
def test_random_normal_error_bound_and_idempotence(orc, g):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((300, 260)).astype(np.float32)
    codes, scales = orc.fp8_quantize(x, g, 0)
    gmax, _, _, mx, _ = orc.fp8_quant_error_general(x, codes, scales, g, 0)
    assert mx <= 2.0 ** -4
    deq = orc.fp8_dequantize(codes, scales, g, 0)
    codes2, scales2 = orc.fp8_quantize(deq, g, 0)  # quantize∘dequantize∘quantize = quantize
    assert np.array_equal(codes2, codes) and np.array_equal(scales2, scales)


def test_block_larger_than_tensor_equals_per_tensor(orc):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((100, 90)).astype(np.float32)
    cb, sb = orc.fp8_quantize(x, "block")
    ct, st = orc.fp8_quantize(x, "tensor")
    assert np.array_equal(cb, ct) and np.array_equal(sb, st)


def test_per_channel_isolates_magnitudes(orc):
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, 512)).astype(np.float32)
    x[0] *= 1000.0
    cc, sc = orc.fp8_quantize(x, "channel", 0)
    ct, st = orc.fp8_quantize(x, "tensor")
    gc = orc.fp8_quant_error_general(x, cc, sc, "channel", 0)
    small = x[1:]
    cs, ss = orc.fp8_quantize(small, "tensor")
    alone = orc.fp8_quant_error_general(small, cs, ss, "tensor")
    assert gc[0][1] == alone[0][0]  # channel 1's error is unchanged by channel 0
    # per-tensor: channel 1 degrades (its small values fall into E4M3's subnormal range at the shared
    # scale): mean relative error 0.036 vs 0.022
    rel = lambda d: float(np.mean(np.abs(d[1] - x[1]) / np.abs(x[1])))
    assert rel(orc.fp8_dequantize(ct, st, "tensor")) > 1.3 * rel(orc.fp8_dequantize(cc, sc, "channel", 0))


def test_refinement_lowers_mse_and_equal_tensor_is_exact(orc):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((256, 256)).astype(np.float32)
    x[:128, :128] *= 300.0
    ct, st = orc.fp8_quantize(x, "tensor")
    cb, sb = orc.fp8_quantize(x, "block")
    assert orc.fp8_quant_error_general(x, cb, sb, "block")[4] <= orc.fp8_quant_error_general(x, ct, st, "tensor")[4]
    e = np.full((40, 50), 3.3, np.float32)
    for g in ("tensor", "channel", "block"):
        c, s = orc.fp8_quantize(e, g, 0)
        assert orc.fp8_quant_error_general(e, c, s, g, 0)[3] == 0.0
        assert orc.fp8_quant_error_general(e, c, s, g, 0)[4] == 0.0


def test_non_finite_is_config_error(orc):
    x = np.ones((4, 4), np.float32)
    x[2, 3] = np.inf
    with pytest.raises(orc.OracleConfigError):
        orc.fp8_quantize(x, "block")


def test_codes_are_exhaustive_nearest(orc):  # SPEC.md:616 invariant, on random scaled values
    rng = np.random.default_rng(4)
    x = (rng.standard_normal(4000) * rng.choice([1e-3, 1.0, 50.0], 4000)).astype(np.float32)
    codes, scales = orc.fp8_quantize(x, "tensor")
    vals = orc.e4m3_values()
    q = np.abs(x.astype(np.float64)) * 448.0 / np.abs(x).astype(np.float64).max()
    got = orc.e4m3_decode_table()[codes & 0x7F].astype(np.float64)
    best = np.abs(vals[None, :] - q[:, None]).min(1)
    assert np.all(np.abs(got - q) <= best + 1e-12)


def test_block_partition_examples():
    from paper_2603_11101_b200.quant import block_partition
    assert len(block_partition((256, 256))) == 4
    b = block_partition((200, 300))
    assert sorted({r for _, r, _, _ in b}) == [72, 128] and sorted({c for _, _, _, c in b}) == [44, 128]
    assert len(b) == 6
    rng = np.random.default_rng(5)
    for _ in range(50):
        R, Cc = (int(v) for v in rng.integers(1, 700, 2))
        assert sum(r * c for _, r, _, c in block_partition((R, Cc))) == R * Cc


def test_compression_ratio():
    from paper_2603_11101_b200.quant import ModelComponent, ModelSizeSpec, compression_ratio
    everything = ModelSizeSpec([ModelComponent("a", 10**9, True), ModelComponent("b", 10**8, True)], scale_bytes=0)
    assert compression_ratio(everything) == pytest.approx(0.5)
    nothing = ModelSizeSpec([ModelComponent("a", 10**9, False)])
    assert compression_ratio(nothing) == 0.0
    # Qwen2.5-VL-3B: ViT and embeddings high precision, the LM's linear weights FP8
    # PerBlock; counts from tests/golden/make_qwen25vl_params.py
    p = json.loads((GOLDEN / "qwen25vl_3b_params.json").read_text())
    assert p["total"] == 3754622976
    spec = ModelSizeSpec([ModelComponent("vision", p["vision"], False),
                          ModelComponent("embeddings", p["embeddings"], False),
                          ModelComponent("lm_1d", p["lm_1d"], False),
                          ModelComponent("lm_linear", p["lm_linear"], True, "block")])
    assert abs(compression_ratio(spec) - 0.366) <= 0.01
