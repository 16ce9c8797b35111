"""Varlen attention parity on the GPU against the fp64 CPU oracle (north_star tolerance: outputs and
gradients within max-abs 2e-2 for bf16, measured relative to max(1, max|ref|))."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2


def _inputs(L, H, Hkv, d, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    T = int(sum(L))
    q = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
    k = torch.randn(T, Hkv, d, device="cuda", generator=g).bfloat16()
    v = torch.randn(T, Hkv, d, device="cuda", generator=g).bfloat16()
    do = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(L)]), dtype=torch.int32, device="cuda")
    return q, k, v, do, cu


def _err(x, ref):
    x = x.float().cpu().numpy().astype(np.float64)
    return np.max(np.abs(x - ref)) / max(1.0, np.max(np.abs(ref)))


CASES = [
    # (lengths, H, Hkv, d, mask)
    ([100, 28, 300, 5, 1, 130], 2, 2, 128, 0),
    ([128, 128, 256], 2, 1, 128, 0),
    ([513, 77, 1000, 3], 2, 2, 128, 0),
    ([100, 28, 300, 5, 1, 130], 2, 2, 128, 1),
    ([600, 40, 260], 4, 2, 128, 2),
    ([100, 28, 300, 5, 1, 130], 2, 2, 64, 0),
    ([700, 20, 129], 4, 4, 64, 1),
    ([300, 50, 17], 4, 1, 256, 2),
    ([1, 1, 1, 2, 3], 1, 1, 128, 0),
    ([700, 33, 260], 8, 1, 256, 2),   # config-3 shape: H=8, Hkv=1 (MQA), prefix-LM
    ([100, 28, 300, 5, 1, 130], 2, 2, 256, 0),
    ([513, 77, 129], 4, 2, 256, 1),
    # segment-aligned tiles: partial tiles of every 64/32/16/8/tail row combination, neighbours
    # that a clipped store must not touch
    ([127, 1, 255, 9, 135, 64, 72, 200, 7, 385, 128, 120], 2, 2, 128, 0),
    ([127, 1, 255, 9, 135, 64, 72, 200, 7, 385, 128, 120], 2, 1, 64, 1),
    ([127, 1, 255, 9, 135, 64, 72, 200, 7, 385], 2, 1, 256, 2),
    # token counts whose last k_bwd_pre block covers < 32 lanes of work (warp-uniform shuffles)
    ([385], 1, 1, 64, 1),
    ([129], 1, 1, 64, 0),
    ([256, 1], 1, 1, 128, 0),
    # > 1024 segments: the tile builder's chunked stable sort
    (list(np.random.default_rng(5).integers(1, 41, 1500)), 1, 1, 64, 0),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_fwd_matches_oracle(gpu, orc, case):
    from paper_2603_11101_b200 import attention
    L, H, Hkv, d, mask = CASES[case]
    q, k, v, do, cu = _inputs(L, H, Hkv, d, case)
    prefix = torch.tensor([max(0, l // 3) for l in L], dtype=torch.int32, device="cuda") if mask == 2 else None
    o, lse = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix)
    torch.cuda.synchronize()
    ro, rlse = orc.mha_fwd(q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy(),
                           cu.cpu().numpy(), mask=mask, prefix=None if prefix is None else prefix.cpu().numpy())
    assert _err(o, ro) < TOL_BF16
    assert np.max(np.abs(lse.cpu().numpy() - rlse)) < 1e-2


@pytest.mark.parametrize("case", range(len(CASES)))
def test_bwd_matches_oracle(gpu, orc, case):
    from paper_2603_11101_b200 import attention
    L, H, Hkv, d, mask = CASES[case]
    q, k, v, do, cu = _inputs(L, H, Hkv, d, 100 + case)
    prefix = torch.tensor([max(0, l // 3) for l in L], dtype=torch.int32, device="cuda") if mask == 2 else None
    o, lse = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix)
    dq, dk, dv = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, mask_mode=mask, prefix_len=prefix)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    pre = None if prefix is None else prefix.cpu().numpy()
    ro, _ = orc.mha_fwd(f(q), f(k), f(v), cu.cpu().numpy(), mask=mask, prefix=pre)
    rdq, rdk, rdv = orc.mha_bwd(f(q), f(k), f(v), ro, f(do), cu.cpu().numpy(), mask=mask, prefix=pre)
    assert _err(dv, rdv) < TOL_BF16, "dv"
    assert _err(dk, rdk) < TOL_BF16, "dk"
    assert _err(dq, rdq) < TOL_BF16, "dq"


def test_segment_isolation_on_gpu(gpu):
    """perturbing segment j leaves every other segment's output bit-identical."""
    from paper_2603_11101_b200 import attention
    L = [200, 77, 300]
    q, k, v, do, cu = _inputs(L, 2, 2, 128, 7)
    o1, _ = attention.varlen_attn_fwd(q, k, v, cu)
    q2, k2, v2 = q.clone(), k.clone(), v.clone()
    q2[200:277] += 1
    k2[200:277] -= 1
    v2[200:277] *= 2
    o2, _ = attention.varlen_attn_fwd(q2, k2, v2, cu)
    assert torch.equal(o1[:200], o2[:200]) and torch.equal(o1[277:], o2[277:])


@pytest.mark.parametrize("d", [128, 256])
def test_bwd_row_map_fuses_scatter(gpu, d):
    """row_map[t] redirects gradient row t (the packer's gather index → sample order)."""
    from paper_2603_11101_b200 import attention
    L = [300, 45, 129, 2]
    q, k, v, do, cu = _inputs(L, 2, 1, d, 11)
    T = q.shape[0]
    o, lse = attention.varlen_attn_fwd(q, k, v, cu)
    dq, dk, dv = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu)
    perm = torch.randperm(T, device="cuda").int()
    dq2, dk2, dv2 = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, row_map=perm)
    torch.cuda.synchronize()
    pl = perm.long()
    # every gradient row is produced by exactly one CTA with a fixed reduction order (no atomics):
    # the redirected rows are bit-identical
    assert torch.equal(dv2[pl], dv) and torch.equal(dk2[pl], dk) and torch.equal(dq2[pl], dq)


SHARP = [  # (case index into CASES, Q/K multiplier): very sharp softmax — the running max grows by
    # more than the lazy-rescale threshold (2^8) inside a row, and the bf16 rounded-up row max matters
    (0, 8.0), (0, 16.0), (3, 16.0), (4, 8.0), (7, 16.0), (9, 8.0), (12, 16.0), (13, 8.0), (14, 16.0), (6, 16.0)]


@pytest.mark.parametrize("case", range(len(SHARP)))
def test_sharp_softmax_fwd_bwd(gpu, orc, case):
    from paper_2603_11101_b200 import attention
    ci, mult = SHARP[case]
    L, H, Hkv, d, mask = CASES[ci]
    q, k, v, do, cu = _inputs(L, H, Hkv, d, 200 + case)
    q, k = (q.float() * mult).bfloat16(), (k.float() * mult).bfloat16()
    prefix = torch.tensor([max(0, l // 3) for l in L], dtype=torch.int32, device="cuda") if mask == 2 else None
    o, lse = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix)
    dq, dk, dv = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, mask_mode=mask, prefix_len=prefix)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    pre = None if prefix is None else prefix.cpu().numpy()
    ro, rlse = orc.mha_fwd(f(q), f(k), f(v), cu.cpu().numpy(), mask=mask, prefix=pre)
    rdq, rdk, rdv = orc.mha_bwd(f(q), f(k), f(v), ro, f(do), cu.cpu().numpy(), mask=mask, prefix=pre)
    assert _err(o, ro) < TOL_BF16, "o"
    assert np.max(np.abs(lse.cpu().numpy() - rlse)) / max(1.0, np.max(np.abs(rlse))) < 1e-3, "lse"
    assert _err(dv, rdv) < TOL_BF16, "dv"
    if mult <= 8:
        assert _err(dk, rdk) < TOL_BF16, "dk"
        assert _err(dq, rdq) < TOL_BF16, "dq"
    else:
        # ×16: dQ / dK = scale · dS · K (Q) with |K|, |Q| ~ 16 amplify the bf16 rounding of the stored O
        # inside D = rowsum(dO ∘ O) (≈ √d · 2^-9 per row) to ~3e-2 — a property of bf16 O, not of the
        # kernels.  Checked against the oracle given the same (bf16) O the kernels differentiate.
        gdq, gdk, _ = orc.mha_bwd(f(q), f(k), f(v), f(o), f(do), cu.cpu().numpy(), mask=mask, prefix=pre)
        assert _err(dk, gdk) < TOL_BF16, "dk"
        assert _err(dq, gdq) < TOL_BF16, "dq"


@pytest.mark.parametrize("d", [64, 128, 256])
def test_bwd_workspace_garbage_is_harmless(gpu, orc, d):
    """The backward must not read workspace cells it did not write: a workspace
    pre-filled with NaN and -inf gives the same, finite gradients as a zeroed one."""
    from paper_2603_11101_b200 import attention
    L = [300, 45, 129, 2, 77]
    q, k, v, do, cu = _inputs(L, 3, 1, d, 31)
    o, lse = attention.varlen_attn_fwd(q, k, v, cu)
    res = []
    for fill in (0.0, float("nan"), float("-inf")):
        ws = attention.BwdWorkspace()
        ws.buf = torch.full((4 << 20,), fill, dtype=torch.float32, device="cuda").view(torch.uint8)  # 16 MB
        res.append(attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, workspace=ws))
    torch.cuda.synchronize()
    for g in res[0]:
        assert torch.isfinite(g.float()).all()
    for other in res[1:]:
        assert all(torch.equal(x, y) for x, y in zip(res[0], other))


def test_api_rejects_wrong_dtypes_and_devices(gpu):
    from paper_2603_11101_b200 import attention
    from paper_2603_11101_b200.errors import ConfigError
    q, k, v, do, cu = _inputs([10, 20], 2, 2, 64, 1)
    with pytest.raises(ConfigError):
        attention.varlen_attn_fwd(q.half(), k, v, cu)
    with pytest.raises(ConfigError):
        attention.varlen_attn_fwd(q.float(), k, v, cu)
    with pytest.raises(ConfigError):
        attention.varlen_attn_fwd(q, k, v, cu, mask_mode=2, prefix_len=torch.zeros(2, dtype=torch.int64, device="cuda"))
    with pytest.raises(ConfigError):
        attention.varlen_attn_fwd(q, k, v, cu, mask_mode=2, prefix_len=torch.zeros(2, dtype=torch.int32))
    o, lse = attention.varlen_attn_fwd(q, k, v, cu)
    with pytest.raises(ConfigError):
        attention.varlen_attn_bwd(do, q, k, v, o, lse.double(), cu)
    with pytest.raises(ConfigError):
        attention.varlen_attn_bwd(do.half(), q, k, v, o, lse, cu)
